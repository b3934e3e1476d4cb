// csflow-b200: species closure + admissibility gate (reference driver.py:216-229,
// 250; implicit.py:113-141), residual norms (driver.py:85-90), layout helpers
// and operator export for the drop-in ImplicitOperator view.
#pragma once
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// The species closure of one cell; returns false if _check_corrected (CS) or
// the last-species test (CI) fails.  q, dq, qn strided by N.
template <int NSB>
CSB_DEV bool closure(int scheme, int ns, const double* q, const double* dq, double* qn,
                     long long N) {
#pragma unroll
  for (int m = 0; m < 5; ++m) qn[m * N] = q[m * N] + dq[m * N];
  if (scheme == SCH_CI) {
    double tail = 0.0;
    double last = 0.0;
#pragma unroll
    for (int s = 0; s < NSB; ++s) {
      if (s < ns) {
        const double v = q[(5 + s) * N] + dq[(5 + s) * N];
        if (s < ns - 1) {
          qn[(5 + s) * N] = v;
          tail += v;
        }
      }
    }
    last = qn[0] - tail;
    qn[(4 + ns) * N] = last;
    return !(last < -1e-10 * qn[0]);
  }
  double rs[NSB], drs[NSB];
  double tot = 0.0, dsum = 0.0;
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      rs[s] = q[(5 + s) * N];
      drs[s] = dq[(5 + s) * N];
      tot += rs[s];
      dsum += drs[s];
    }
  }
  double out[NSB];
  if (scheme == SCH_CS1) {
    const double defect = dq[0] - dsum;  // d_rho - sum d_rho_s
#pragma unroll
    for (int s = 0; s < NSB; ++s)
      if (s < ns) out[s] = rs[s] + drs[s] + (rs[s] / tot) * defect;
  } else {
    const double rnew = tot + dq[0];
    double rawsum = 0.0;
    double raw[NSB];
#pragma unroll
    for (int s = 0; s < NSB; ++s)
      if (s < ns) {
        raw[s] = rs[s] + drs[s];
        rawsum += raw[s];
      }
#pragma unroll
    for (int s = 0; s < NSB; ++s)
      if (s < ns) out[s] = rnew * raw[s] / rawsum;
  }
  double osum = 0.0;
#pragma unroll
  for (int s = 0; s < NSB; ++s)
    if (s < ns) {
      qn[(5 + s) * N] = out[s];
      osum += out[s];
    }
  bool ok = !(osum <= 0.0);
#pragma unroll
  for (int s = 0; s < NSB; ++s)
    if (s < ns && out[s] < -EPS_NEG * osum) ok = false;
  return ok;
}

template <int NSB>
__global__ void k_update(const Model* __restrict__ mp, long long N, int scheme,
                         const double* __restrict__ q, const double* __restrict__ dq,
                         double* __restrict__ qn, unsigned long long* flags) {
  const Model& m = *mp;
  // per-thread tallies, reduced per warp at the end (random states fail the
  // gate in most cells: one atomic per warp, not per cell)
  unsigned long long bad_count = 0, first1 = ~0ull, first2 = ~0ull;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    const bool ok1 = closure<NSB>(scheme, m.ns, q + c, dq + c, qn + c, N);
    Cell<NSB> cs;
    const bool ok2 = decode<NSB>(m, qn + c, N, cs);  // admissibility gate (driver.py:250)
    if (!ok1 && first1 == ~0ull) first1 = (unsigned long long)c;
    if (!ok2 && first2 == ~0ull) first2 = (unsigned long long)c;
    if (!(ok1 && ok2)) ++bad_count;
  }
  for (int o = 16; o > 0; o >>= 1) {
    bad_count += __shfl_xor_sync(0xffffffffu, bad_count, o);
    first1 = min(first1, __shfl_xor_sync(0xffffffffu, first1, o));
    first2 = min(first2, __shfl_xor_sync(0xffffffffu, first2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad_count) atomicAdd(flags + FLAG_GATE_COUNT, bad_count);
    if (first1 != ~0ull) raise_flag(flags, EB_GATE, (long long)first1);
    if (first2 != ~0ull) raise_flag(flags, EB_GATE_DECODE, (long long)first2);
  }
}

// Operator export (reference ImplicitOperator fields, implicit.py:59-81, 385-395)
// what: 0 w [nv][N], 1 b [nv][N], 2 sp_lower [3][N], 3 sp_upper [3][N]
template <int NSB>
__global__ void k_export(const Model* __restrict__ mp, GridDev g, OpDev op,
                         const double* __restrict__ q, int what, double* __restrict__ dst) {
  const Model& m = *mp;
  const int ns = m.ns;
  const long long N = g.N;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    if (what == 4) {  // vdom = dOmega * V (implicit.py:356)
      const double V = __ldg(g.vol + c);
      for (int e = 0; e < ns * ns; ++e) dst[(long long)e * N + c] = op.dom[(long long)e * N + c] * V;
    } else if (what <= 1) {
      Cell<NSB> cs;
      decode<NSB>(m, q + c, N, cs);
      if (what == 0) {
        dst[c] = cs.rho;
        for (int x = 0; x < 3; ++x) dst[(1 + x) * N + c] = cs.rho * cs.u[x];
        dst[4 * N + c] = cs.rho * cs.h;
        for (int s = 0; s < ns; ++s) dst[(5 + s) * N + c] = cs.rho * cs.Y[s];
      } else {
        const double beta = cs.gamma - 1.0;
        dst[c] = beta * cs.Ek;
        for (int x = 0; x < 3; ++x) dst[(1 + x) * N + c] = -beta * cs.u[x];
        dst[4 * N + c] = beta;
        for (int s = 0; s < ns; ++s) {
          const double hs = m.bs[s] + m.cp[s] * cs.T;
          const double es = hs - m.Rs[s] * cs.T;
          dst[(5 + s) * N + c] = m.Rs[s] * cs.T - beta * es;
        }
      }
    } else {
      const int k = c % g.nk, j = (c / g.nk) % g.nj, i = c / ((long long)g.nk * g.nj);
      const double u[3] = {op.st[ST_U0 * N + c], op.st[ST_U1 * N + c], op.st[ST_U2 * N + c]};
      for (int d = 0; d < 3; ++d) {
        int f3[3] = {i, j, k};
        if (what == 2) f3[d] += 1;
        const long long f = face_index(g, d, f3[0], f3[1], f3[2]);
        double S[3];
        load_S(g, d, f, S);
        const double U = u[0] * S[0] + u[1] * S[1] + u[2] * S[2];
        const double ls = op.lamsp[d][f];
        dst[d * N + c] = what == 2 ? op.sp_scale * (U + ls) : op.sp_scale * (U - ls);
      }
    }
  }
}

cudaError_t CSB_BK(launch_update)(const Model* mp, int ns, const GridDev& g, int scheme, const double* q,
                          const double* dq, double* qn, unsigned long long* flags,
                          cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_update<NSB><<<grid_for(g.N, 256), 256, 0, st>>>(mp, g.N, scheme, q, dq, qn, flags);
  });
  return cudaGetLastError();
}

cudaError_t CSB_BK(launch_export_op)(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                             const double* q, int what, double* dst, cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_export<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mdl, g, op, q, what, dst);
  });
  return cudaGetLastError();
}

}  // namespace csb
