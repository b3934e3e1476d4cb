// csflow-b200: route ns to the per-bucket launchers (csb_bucket.cu).
#include <atomic>

#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

static std::atomic<unsigned long long> g_launches{0};
void note_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

#define CSB_DECL(b)                                                                               \
  cudaError_t launch_residual_b##b(const Model*, int, const GridDev&, const BCDev&, const Mech&,   \
                                   const double*, double*, int, int, unsigned long long*,          \
                                   cudaStream_t, NormsOut, bool*, const unsigned long long*, int); \
  cudaError_t launch_padded_b##b(const Model*, int, const GridDev&, const BCDev&, const double*,   \
                                 double*, unsigned long long*, cudaStream_t);                      \
  cudaError_t launch_decode_b##b(const Model*, int, const GridDev&, const double*, double*,        \
                                 unsigned long long*, cudaStream_t);                               \
  cudaError_t launch_source_jacobian_b##b(const Model*, int, const GridDev&, const Mech&,          \
                                          const double*, double*, int, double*, const double*,     \
                                          unsigned long long*, cudaStream_t);                      \
  cudaError_t launch_production_b##b(const Model*, int, const GridDev&, const Mech&,               \
                                     const double*, double*, unsigned long long*, cudaStream_t);   \
  cudaError_t launch_time_step_b##b(const Model*, int, const GridDev&, const double*, const double*,\
                                    const double*, double*, double*, double*,                      \
                                    unsigned long long*, cudaStream_t);                            \
  cudaError_t launch_assemble_cell_b##b(const Model*, int, const GridDev&, const double*,          \
                                        const double*, double, double, OpDev&,                     \
                                        unsigned long long*, cudaStream_t);                        \
  cudaError_t launch_sweeps_generic_b##b(const Model*, int, const GridDev&, const OpDev&,          \
                                         const double*, double*, double*, cudaStream_t);           \
  cudaError_t launch_update_b##b(const Model*, int, const GridDev&, int, const double*,            \
                                 const double*, double*, unsigned long long*, cudaStream_t);       \
  cudaError_t launch_export_op_b##b(const Model*, int, const GridDev&, const OpDev&,               \
                                    const double*, int, double*, cudaStream_t);                    \
  cudaError_t launch_wave_step_b##b(const Model*, int, const GridDev&, const WaveBufs&,            \
                                    const double*, const double*, const double*, const double*,    \
                                    const double*, int, int, int, double, double*, double*,        \
                                    unsigned long long*, cudaStream_t, cudaEvent_t*);
CSB_BUCKET_LIST(CSB_DECL)
#undef CSB_DECL

#define CSB_ROUTE(NAME, ...)                                 \
  switch (bucket_of(ns)) {                                  \
    case 2: return NAME##_b2(__VA_ARGS__);                  \
    case 4: return NAME##_b4(__VA_ARGS__);                  \
    case 5: return NAME##_b5(__VA_ARGS__);                  \
    case 6: return NAME##_b6(__VA_ARGS__);                  \
    case 8: return NAME##_b8(__VA_ARGS__);                  \
    case 12: return NAME##_b12(__VA_ARGS__);                \
    case 16: return NAME##_b16(__VA_ARGS__);                \
    case 20: return NAME##_b20(__VA_ARGS__);                \
    case 24: return NAME##_b24(__VA_ARGS__);                \
    case 32: return NAME##_b32(__VA_ARGS__);                \
    case 40: return NAME##_b40(__VA_ARGS__);                \
    case 48: return NAME##_b48(__VA_ARGS__);                \
    default: return NAME##_b64(__VA_ARGS__);                \
  }

cudaError_t launch_residual(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                            const Mech& mech, const double* q, double* R, int first_order, int mode,
                            unsigned long long* flags, cudaStream_t st, NormsOut nrm, bool* fused,
                            const unsigned long long* guard, int guard_bit) {
  note_launches(1);
  if (fused) *fused = false;
  CSB_ROUTE(launch_residual, mp, ns, g, bc, mech, q, R, first_order, mode, flags, st, nrm, fused, guard,
            guard_bit)
}
cudaError_t launch_padded(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                          const double* q, double* P, unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_padded, mp, ns, g, bc, q, P, flags, st)
}
cudaError_t launch_decode(const Model* mp, int ns, const GridDev& g, const double* q, double* out,
                          unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_decode, mp, ns, g, q, out, flags, st)
}
cudaError_t launch_source_jacobian(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                                   const double* q, double* dom, int dom_full, double* lamS,
                                   const double* dom_in, unsigned long long* flags,
                                   cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_source_jacobian, mp, ns, g, mech, q, dom, dom_full, lamS, dom_in, flags, st)
}
cudaError_t launch_production(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                              const double* q, double* om, unsigned long long* flags,
                              cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_production, mp, ns, g, mech, q, om, flags, st)
}
cudaError_t launch_time_step(const Model* mp, int ns, const GridDev& g, const double* q, const double* cfl,
                             const double* lamS, double* dtau, double* lam_inv, double* lam_vis,
                             unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_time_step, mp, ns, g, q, cfl, lamS, dtau, lam_inv, lam_vis, flags, st)
}
cudaError_t launch_assemble_cell(const Model* mp, int ns, const GridDev& g, const double* q,
                                 const double* dtau, double theta, double dt, OpDev& op,
                                 unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_assemble_cell, mp, ns, g, q, dtau, theta, dt, op, flags, st)
}
cudaError_t launch_sweeps_generic(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                                  const double* rhs, double* dq, double* dq_star, cudaStream_t st) {
  // (counted by launch_sweeps, which replays these launches as one graph)
  CSB_ROUTE(launch_sweeps_generic, mdl, ns, g, op, rhs, dq, dq_star, st)
}
cudaError_t launch_update(const Model* mp, int ns, const GridDev& g, int scheme, const double* q,
                          const double* dq, double* qn, unsigned long long* flags,
                          cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_update, mp, ns, g, scheme, q, dq, qn, flags, st)
}
cudaError_t launch_export_op(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                             const double* q, int what, double* dst, cudaStream_t st) {
  note_launches(1);
  CSB_ROUTE(launch_export_op, mdl, ns, g, op, q, what, dst, st)
}

cudaError_t launch_wave_step(const Model* mp, int ns, const GridDev& g, const WaveBufs& wb,
                             const double* q, const double* R, const double* cfl, const double* lamS,
                             const double* domd, int dom_stride, int per_species, int scheme,
                             double sp_scale, double* qn, double* dq_std,
                             unsigned long long* flags, cudaStream_t st, cudaEvent_t* ev) {
  note_launches(4);
  CSB_ROUTE(launch_wave_step, mp, ns, g, wb, q, R, cfl, lamS, domd, dom_stride, per_species, scheme,
            sp_scale, qn, dq_std, flags, st, ev)
}

}  // namespace csb
