// csflow-b200: LU-SGS forward/backward sweeps (reference lusgs.py:24-274).
//
// Generic path: one launch per hyperplane h = i + j + k.  Every cell of a
// hyperplane depends only on cells of hyperplane h - 1 (forward) or h + 1
// (backward), so the result equals the reference's lexicographic order as
// long as each cell accumulates its neighbours in the same i, j, k order
// (lusgs.py:3-6).  The 2-D production path (nk == 1) is the pipelined
// wavefront kernel in csb_wavefront.cu.
#pragma once
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// acc[0..n) += 0.5*(A(nb, S) + sgn*lam*I) x in rank-2 form (below); the
// reference materialises the block (lusgs.py:24-59); w, b of the neighbour rebuilt
// from its stored state.  Returns U = u_nb . S.
template <int NV>
CSB_DEV double acc_block(int n, const OpDev& op, long long N, long long nb, const double S[3],
                         double lam, double sgn, const double* x, double* acc, int ns,
                         const Model* mdl_for_species) {
  const double* st = op.st;
  const double rho = st[ST_RHO * N + nb];
  const double u0 = st[ST_U0 * N + nb], u1 = st[ST_U1 * N + nb], u2 = st[ST_U2 * N + nb];
  const double h = st[ST_H * N + nb], beta = st[ST_BETA * N + nb], Ek = st[ST_EK * N + nb];
  const double U = u0 * S[0] + u1 * S[1] + u2 * S[2];
  const double a0 = -0.5 * U / rho, a1 = 0.5 * S[0] / rho, a2 = 0.5 * S[1] / rho,
               a3 = 0.5 * S[2] / rho;
  double w[NV], b[NV];
  w[0] = rho;
  w[1] = rho * u0;
  w[2] = rho * u1;
  w[3] = rho * u2;
  w[4] = rho * h;
  b[0] = beta * Ek;
  b[1] = -beta * u0;
  b[2] = -beta * u1;
  b[3] = -beta * u2;
  b[4] = beta;
  if (n > 5) {
    const double T = st[ST_T * N + nb];
#pragma unroll
    for (int s = 0; s < NV - 5; ++s) {
      if (s < ns) {
        w[5 + s] = rho * op.Y[(long long)s * N + nb];
        const double Rs = mdl_for_species->Rs[s];
        const double hs = mdl_for_species->bs[s] + mdl_for_species->cp[s] * T;
        const double es = hs - Rs * T;
        b[5 + s] = Rs * T - beta * es;
      }
    }
  }
  const double dv = 0.5 * (U + sgn * lam);
  // rank-2 form of the half block (as the wavefront chains apply it):
  // A x = w (a . x) + v (b . x) / 2 + dv x with a = (-U, S) / (2 rho),
  // v = (0, S, U, 0..) -- O(nv) per neighbour instead of the O(nv^2)
  // materialised block (lusgs.py:24-59; the same products, reassociated)
  const double ax = ((a0 * x[0] + a1 * x[1]) + a2 * x[2]) + a3 * x[3];
  double bx = 0.0;
#pragma unroll
  for (int c = 0; c < NV; ++c)
    if (c < n) bx += b[c] * x[c];
  bx *= 0.5;
#pragma unroll
  for (int r = 0; r < NV; ++r) {
    if (r >= n) break;
    const double v = (r >= 1 && r <= 3) ? S[r - 1] : (r == 4 ? U : 0.0);
    acc[r] += (w[r] * ax + v * bx) + dv * x[r];
  }
  return U;
}

template <int NSB, bool CI>
__global__ void k_plane(const Model* __restrict__ mdl, GridDev g, OpDev op,
                        const double* __restrict__ rhs, double* __restrict__ dq, int h,
                        int forward) {
  constexpr int NV = CI ? 5 + NSB : 5;  // CI: NSB is the bucket bound
  const int ns = mdl->ns;
  const int nv = 5 + ns;
  const long long N = g.N;
  // enumerate (i, j) of the plane, k = h - i - j
  const int jlo = 0;
  const long long npairs = (long long)g.ni * g.nj;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < npairs;
       t += (long long)gridDim.x * blockDim.x) {
    int i, j;
    if (g.nk == 1) {
      // dense enumeration of the 2-D diagonal
      const int ilo = max(0, h - (g.nj - 1)), ihi = min(h, g.ni - 1);
      if (t > ihi - ilo) break;
      i = ilo + (int)t;
      j = h - i;
    } else {
      i = (int)(t / g.nj);
      j = (int)(t % g.nj) + jlo;
    }
    const int k = h - i - j;
    if (k < 0 || k >= g.nk || j < 0 || j >= g.nj) continue;
    const long long c = cell_index(g, i, j, k);
    const int idx[3] = {i, j, k};
    const int nd[3] = {g.ni, g.nj, g.nk};
    const long long stride[3] = {(long long)g.nj * g.nk, g.nk, 1};
    double acc[NV];
    double accs[NSB];
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      if (m < (CI ? nv : 5)) acc[m] = forward ? (op.neg_rhs ? -rhs[m * N + c] : rhs[m * N + c]) : 0.0;
    }
    if (!CI) {
#pragma unroll
      for (int s = 0; s < NSB; ++s)
        if (s < ns)
          accs[s] = forward ? (op.neg_rhs ? -rhs[(5 + s) * N + c] : rhs[(5 + s) * N + c]) : 0.0;
    }
    for (int d = 0; d < 3; ++d) {
      const bool has = forward ? idx[d] > 0 : idx[d] < nd[d] - 1;
      if (!has) continue;
      const long long nb = forward ? c - stride[d] : c + stride[d];
      int fi[3] = {i, j, k};
      if (!forward) fi[d] += 1;
      const long long f = face_index(g, d, fi[0], fi[1], fi[2]);
      double S[3];
      load_S(g, d, f, S);
      const double lam = op.lam[d][f];
      double x[NV];
#pragma unroll
      for (int m = 0; m < NV; ++m)
        if (m < (CI ? nv : 5)) x[m] = dq[m * N + nb];
      const double U = acc_block<NV>(CI ? nv : 5, op, N, nb, S, lam, forward ? 1.0 : -1.0, x, acc,
                                     ns, mdl);
      if (!CI) {
        const double ls = op.lamsp[d][f];
        const double cf = forward ? op.sp_scale * (U + ls) : op.sp_scale * (U - ls);
#pragma unroll
        for (int s = 0; s < NSB; ++s)
          if (s < ns) accs[s] += cf * dq[(5 + s) * N + nb];
      }
    }
    const double dd = op.d[c];
    if (CI) {
      if (op.chem) {
#pragma unroll
        for (int m = 0; m < 5; ++m) {
          const double v = acc[m] / dd;
          dq[m * N + c] = forward ? v : dq[m * N + c] - v;
        }
        for (int r = 0; r < ns; ++r) {
          double t2 = 0.0;
#pragma unroll
          for (int cc = 0; cc < NSB; ++cc)
            if (cc < ns) t2 += op.dinv[((long long)r * ns + cc) * N + c] * acc[5 + cc];
          dq[(5 + r) * N + c] = forward ? t2 : dq[(5 + r) * N + c] - t2;
        }
      } else {
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          if (m < nv) {
            const double v = acc[m] / dd;
            dq[m * N + c] = forward ? v : dq[m * N + c] - v;
          }
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const double v = acc[m] / dd;
        dq[m * N + c] = forward ? v : dq[m * N + c] - v;
      }
#pragma unroll
      for (int s = 0; s < NSB; ++s) {
        if (s < ns) {
          const double di = op.dsp_per_species ? op.dinv_sp[(long long)s * N + c] : op.dinv_sp[c];
          const double v = accs[s] * di;
          dq[(5 + s) * N + c] = forward ? v : dq[(5 + s) * N + c] - v;
        }
      }
    }
  }
}

cudaError_t CSB_BK(launch_sweeps_generic)(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                                  const double* rhs, double* dq, double* dq_star, cudaStream_t st) {
  if (!(g.ni > 0 && g.nj > 0 && g.nk > 0)) return cudaSuccess;
  const int nplanes = (g.ni - 1) + (g.nj - 1) + (g.nk - 1) + 1;
  const long long npairs = g.nk == 1 ? std::min(g.ni, g.nj) : (long long)g.ni * g.nj;
  const int bs = 128;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((npairs + bs - 1) / bs, 148 * 8));
  const int nv = 5 + ns;
  cudaError_t e = cudaSuccess;
  CSB_NS_DISPATCH(ns, {
    for (int pass = 0; pass < 2; ++pass) {
      const int fwd = pass == 0;
      for (int t = 0; t < nplanes; ++t) {
        const int h = fwd ? t : nplanes - 1 - t;
        if (op.mode == SCH_CI)
          k_plane<NSB, true><<<blocks, bs, 0, st>>>(mdl, g, op, rhs, dq, h, fwd);
        else
          k_plane<NSB, false><<<blocks, bs, 0, st>>>(mdl, g, op, rhs, dq, h, fwd);
      }
      if (fwd && dq_star)
        cudaMemcpyAsync(dq_star, dq, sizeof(double) * nv * g.N, cudaMemcpyDeviceToDevice, st);
    }
    e = cudaGetLastError();
  });
  return e;
}

}  // namespace csb
