// csflow-b200: internal launcher declarations shared by the .cu files.
#pragma once

#include <algorithm>
#include <utility>

#include "csb_common.cuh"

namespace csb {

// per-cell operator state written by the assembly, read by the sweeps
enum StIdx : int {
  ST_RHO = 0, ST_U0 = 1, ST_U1 = 2, ST_U2 = 3, ST_H = 4, ST_BETA = 5, ST_EK = 6,
  ST_C = 7, ST_NF = 8, ST_NSP = 9, ST_NU = 10, ST_T = 11, NST = 12
};

enum Scheme : int { SCH_CI = 0, SCH_CS1 = 1, SCH_CS2 = 2 };

struct OpDev {
  int mode;            // Scheme
  double sp_scale;     // 0.5 symmetrized, 1.0 paper (implicit.py:385)
  int chem;            // chemistry contributes to the diagonal
  int dsp_per_species; // d_sp stored per species (chemistry) or once per cell
  double* st;          // [NST][N]
  double* Y;           // [ns][N] decoded mass fractions (CI sweeps: w, b species rows)
  double* d;           // [N] d_flow (CS) or d_scal (CI)
  double* dsp;         // [ns or 1][N] CS species diagonal
  double* dinv_sp;     // [ns or 1][N] 1/d_sp
  double* lam[3];      // face radii (CS flow / CI unified), face-shaped SoA
  double* lamsp[3];    // CS species face radii
  double* dom;         // [ns*ns][N] dOmega (full) or [ns][N] diagonal only (CS)
  int dom_full;
  double* lamS;        // [N] source spectral radius
  double* dinv;        // [ns*ns][N] CI species block inverse
  int neg_rhs;         // sweeps use rhs = -input (the residual R)
};

// Strip-skewed 2-D layout of the wavefront path (csb_wave.cuh): cell (i, j)
// at ((j>>5)*T + i + (j&31))*32 + (j&31).
constexpr int TQ = 16;  // T is a multiple of TQ; wavefront slot lengths divide TQ
constexpr int HPAD = 32;  // zero rows either side of a strip's hand-off rows

struct Skew {
  int ni, nj, nstrip, T;
  long long Np;  // plane stride (padded)
};

// Sweep records of the wavefront path, one set per subsystem, all step-major
// (plane layouts in csb_wave.cuh).  NSB = species bucket of the model.
struct WaveBufs {
  Skew sk;
  double* ff;     // flow forward group (30 planes)
  double* fb;     // flow backward group (30 planes, incl. dq*)
  double* fw;     // flow dq (5 planes)
  double* sf;     // species forward group (nsI + NSB + 2 planes)
  double* sb;     // species backward group (nsI + 2 + NSB planes, incl. dq*)
  double* sw;     // species dq (NSB planes)
  double* hand;   // strip hand-off rows [2 sweeps][flow nstrip*(T+2*HPAD)*5 | species ..*NSB]
  int* prog;      // [2]: flow and species CTA tickets
  int nsI;        // species-diagonal planes of the current layout (0 = unset)
  // records -> forward sweep overlap: the records kernel publishes epoch in
  // rdy[strip][records tile] once a tile is stored; the forward sweep runs
  // concurrently on the high-priority stream s2 and its TMA producer waits
  // for the tiles of each ring slot (csb_wave.cuh)
  int* rdy;       // [nstrip][T] (tiles of >= 1 step)
  int* nonplanar; // == epoch when the step is not planar (csb_wave.cuh k_hand_reset)
  int* epoch;     // device: this step's tag, bumped on the device at the start of every
                  // wavefront step (graph replays see a fresh tag each time)
  cudaStream_t s2;
  cudaEvent_t e1, e2;
  int serial;     // no records / forward-sweep overlap (graph capture: single stream)
  // coupled operator with chemistry on the wavefront: the scalar diagonal d
  // written by the records kernel ([N]) and the species block inverses
  // inv(d I - V dOmega) ([ns * ns][N]) scattered into the CF / CB records
  double* ci_d;
  double* ci_dinv;
};

cudaError_t launch_wave_step(const Model* mp, int ns, const GridDev& g, const WaveBufs& wb,
                             const double* q, const double* R, const double* cfl, const double* lamS,
                             const double* domd, int dom_stride, int per_species, int scheme,
                             double sp_scale, double* qn, double* dq_std,
                             unsigned long long* flags, cudaStream_t st,
                             cudaEvent_t* ev = nullptr);

// residual_norms fused into the residual kernel (driver.py:85-90): per-tile
// partial sums + a last-block reduction in fixed order (deterministic).
struct NormsOut {
  double* partial;         // [3][cap]
  int cap;                 // tiles the partial buffer can hold
  unsigned int* counter;   // zero between launches (reset by the last block)
  double* out;             // [3] flow, species, density (null: no norms)
};

// launch_residual returns with *fused = true when the norms were computed
// in the same launch (nrm.out set and the tile count fits nrm.cap).
// mode: RES_GENERAL, RES_K2D (nk == 1 fast path) or RES_K2D_PLANAR (K2D with
// w == 0 everywhere: raises EB_NONPLANAR otherwise).  guard: run only when
// bit guard_bit of *guard is set (device-side fallback behind a faster mode).
enum ResidualMode : int { RES_GENERAL = 0, RES_K2D = 1, RES_K2D_PLANAR = 2 };
cudaError_t launch_residual(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                            const Mech& mech, const double* q, double* R, int first_order, int mode,
                            unsigned long long* flags, cudaStream_t st,
                            NormsOut nrm = NormsOut{nullptr, 0, nullptr, nullptr},
                            bool* fused = nullptr, const unsigned long long* guard = nullptr,
                            int guard_bit = 6 /* EB_KSKIP */);
cudaError_t launch_padded(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                          const double* q, double* P, unsigned long long* flags, cudaStream_t st);

cudaError_t launch_decode(const Model* mp, int ns, const GridDev& g, const double* q, double* out,
                          unsigned long long* flags, cudaStream_t st);
cudaError_t launch_source_jacobian(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                                   const double* q, double* dom, int dom_full, double* lamS,
                                   const double* dom_in, unsigned long long* flags, cudaStream_t st);
cudaError_t launch_production(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                              const double* q, double* om, unsigned long long* flags,
                              cudaStream_t st);
cudaError_t launch_time_step(const Model* mp, int ns, const GridDev& g, const double* q, const double* cfl,
                             const double* lamS, double* dtau, double* lam_inv, double* lam_vis,
                             unsigned long long* flags, cudaStream_t st);
cudaError_t launch_assemble(const Model* mp, int ns, const GridDev& g, const double* q,
                            const double* dtau, double theta, double dt, OpDev& op,
                            unsigned long long* flags, cudaStream_t st);
cudaError_t launch_block_inverse(int n, long long N, const double* dom, const double* d,
                                 const double* V, double* dinv, unsigned long long* flags,
                                 cudaStream_t st);
cudaError_t launch_fp64_peak(int iters, double* out, cudaStream_t st);
cudaError_t launch_assemble_cell(const Model* mp, int ns, const GridDev& g, const double* q,
                                 const double* dtau, double theta, double dt, OpDev& op,
                                 unsigned long long* flags, cudaStream_t st);
cudaError_t launch_sweeps_generic(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                                  const double* rhs, double* dq, double* dq_star, cudaStream_t st);
cudaError_t launch_sweeps(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                          const double* rhs, double* dq, double* dq_star, unsigned long long* flags,
                          cudaStream_t st);
cudaError_t launch_update(const Model* mp, int ns, const GridDev& g, int scheme, const double* q,
                          const double* dq, double* qn, unsigned long long* flags, cudaStream_t st);
cudaError_t launch_norms(int ns, long long N, const double* R, double* partial, double* out,
                         cudaStream_t st);
cudaError_t launch_correct(int mode, long long rows, int ns, const double* rs, const double* drs,
                           const double* drho, double* out, unsigned long long* flags,
                           cudaStream_t st);
cudaError_t launch_transpose(long long N, int nv, const double* src, double* dst, int to_soa,
                             cudaStream_t st);
cudaError_t launch_dual_rhs(long long N, int nv, const double* R, const double* qm,
                            const double* qn, const double* qnm1, const double* vol, double theta,
                            double dt, double* out, cudaStream_t st);
cudaError_t launch_sumsq(long long n, const double* x, double* partial, double* out,
                         cudaStream_t st);
cudaError_t launch_export_op(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                             const double* q, int what, double* dst, cudaStream_t st);
cudaError_t launch_dtau_arrays(long long N, const double* li, const double* lv, const double* lS,
                               double lS_scalar, double cfl, const double* J, double* dtau,
                               unsigned long long* flags, cudaStream_t st);
cudaError_t launch_check_2d(const GridDev& g, int* ok, cudaStream_t st);
cudaError_t launch_face_metrics2d(const GridDev& g, double* fm0, double* fm1, cudaStream_t st);
cudaError_t launch_set_double(double* dst, double v, cudaStream_t st);
void note_launches(unsigned long long n);
unsigned long long launch_count();

}  // namespace csb
