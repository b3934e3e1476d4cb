// csflow-b200: sweep dispatch (reference lusgs.py:250-274).
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

cudaError_t launch_sweeps(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                          const double* rhs, double* dq, double* dq_star, unsigned long long* flags,
                          cudaStream_t st) {
  (void)flags;
  return launch_sweeps_generic(mdl, ns, g, op, rhs, dq, dq_star, st);
}

}  // namespace csb
