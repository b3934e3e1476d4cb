// csflow-b200: norms, standalone corrections, layout transpose
// (reference driver.py:85-90, implicit.py:113-135).
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// correct_increment_cs1 / correct_normalize_cs2 on plain (rows, ns) arrays
// (implicit.py:113-135); mode 1 = CS1, 2 = CS2.  Row-major AoS like the
// reference's (..., ns) arrays; drho has one value per row.
__global__ void k_correct(int mode, long long rows, int ns, const double* rs, const double* drs,
                          const double* drho, double* out, unsigned long long* flags) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    const double* a = rs + r * ns;
    const double* b = drs + r * ns;
    double* o = out + r * ns;
    double tot = 0.0, ds = 0.0;
    for (int s = 0; s < ns; ++s) {
      tot += a[s];
      ds += b[s];
    }
    if (mode == 1) {
      const double defect = drho[r] - ds;
      for (int s = 0; s < ns; ++s) o[s] = a[s] + b[s] + (a[s] / tot) * defect;
    } else {
      const double rnew = tot + drho[r];
      double rawsum = 0.0;
      for (int s = 0; s < ns; ++s) rawsum += a[s] + b[s];
      for (int s = 0; s < ns; ++s) o[s] = rnew * (a[s] + b[s]) / rawsum;
    }
    double osum = 0.0;
    for (int s = 0; s < ns; ++s) osum += o[s];
    bool ok = !(osum <= 0.0);
    for (int s = 0; s < ns; ++s)
      if (o[s] < -EPS_NEG * osum) ok = false;
    if (!ok) raise_flag(flags, EB_GATE, r);
  }
}

// residual_norms partial sums: flow = sum R[0..4]^2, species = sum (sum_s R_s)^2,
// density = sum R0^2.  Deterministic two-pass reduction.
constexpr int NORM_BS = 256;
__global__ void k_norms_partial(int ns, long long N, const double* __restrict__ R, double* partial) {
  __shared__ double sh[3][NORM_BS / 32];
  double a = 0.0, b = 0.0, d = 0.0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    const double r0 = R[c];
    double f = r0 * r0;
#pragma unroll
    for (int m = 1; m < 5; ++m) {
      const double v = R[m * N + c];
      f += v * v;
    }
    double s = 0.0;
    for (int k = 0; k < ns; ++k) s += R[(5 + k) * N + c];
    a += f;
    b += s * s;
    d += r0 * r0;
  }
  double v3[3] = {a, b, d};
  for (int k = 0; k < 3; ++k) {
    double v = v3[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[k][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int w = 0; w < NORM_BS / 32; ++w) v += sh[threadIdx.x][w];
    partial[threadIdx.x * gridDim.x + blockIdx.x] = v;
  }
}

__global__ void k_norms_final(int nblocks, const double* partial, double* out) {
  const int k = threadIdx.x;
  if (k < 3) {
    double v = 0.0;
    for (int i = 0; i < nblocks; ++i) v += partial[k * nblocks + i];
    out[k] = sqrt(v);
  }
}

// Dual-time right-hand side (implicit.py:47-56):
//   rhs = -R - V [(1 + theta)(Q^m - Q^n) - theta (Q^n - Q^{n-1})] / dt
// in numpy's operation order (no FMA contraction), SoA (nv, N).
__global__ void k_dual_rhs(long long N, int nv, const double* __restrict__ R,
                           const double* __restrict__ qm, const double* __restrict__ qn,
                           const double* __restrict__ qnm1, const double* __restrict__ vol,
                           double theta, double dt, double* __restrict__ out) {
  const long long total = N * nv;
  const double a = __dadd_rn(1.0, theta);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long c = e % N;
    const double src = __dsub_rn(__dmul_rn(a, __dsub_rn(qm[e], qn[e])),
                                 __dmul_rn(theta, __dsub_rn(qn[e], qnm1[e])));
    out[e] = __dsub_rn(-R[e], __ddiv_rn(__dmul_rn(vol[c], src), dt));
  }
}

// Sum of squares of n values, deterministic two-level reduction (fixed
// block count and order): the inner-residual norm of the dual-time loop.
__global__ void k_sumsq_partial(long long n, const double* __restrict__ x, double* partial) {
  __shared__ double sh[NORM_BS / 32];
  double v = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    v += x[e] * x[e];
  const double t = block_sum<NORM_BS>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void k_sumsq_final(int nblocks, const double* partial, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double v = 0.0;
    for (int i = 0; i < nblocks; ++i) v += partial[i];
    out[0] = v;
  }
}

// AoS (N, nv) <-> SoA (nv, N), tiled through shared memory: a CTA moves
// TT cells, reading and writing contiguous runs on both sides (the naive
// element-wise form read ~13x the data at config 4: 2.1 ms for 1.07 GB).
__global__ void __launch_bounds__(256) k_transpose(long long N, int nv, const double* __restrict__ src,
                                                   double* __restrict__ dst, int to_soa, int TT) {
  extern __shared__ double tile[];  // [TT][nv + 1] (odd pitch: no bank conflicts)
  const int pitch = nv + 1;
  for (long long c0 = (long long)blockIdx.x * TT; c0 < N; c0 += (long long)gridDim.x * TT) {
    const int n = (int)min((long long)TT, N - c0);
    if (to_soa) {
      const double* s = src + c0 * nv;  // n * nv contiguous doubles
      for (int e = threadIdx.x; e < n * nv; e += blockDim.x) tile[(e / nv) * pitch + e % nv] = s[e];
      __syncthreads();
      for (int e = threadIdx.x; e < n * nv; e += blockDim.x) {
        const int m = e / n, c = e % n;
        dst[(long long)m * N + c0 + c] = tile[c * pitch + m];
      }
    } else {
      for (int e = threadIdx.x; e < n * nv; e += blockDim.x) {
        const int m = e / n, c = e % n;
        tile[c * pitch + m] = src[(long long)m * N + c0 + c];
      }
      __syncthreads();
      double* d = dst + c0 * nv;
      for (int e = threadIdx.x; e < n * nv; e += blockDim.x) d[e] = tile[(e / nv) * pitch + e % nv];
    }
    __syncthreads();
  }
}

cudaError_t launch_correct(int mode, long long rows, int ns, const double* rs, const double* drs,
                           const double* drho, double* out, unsigned long long* flags,
                           cudaStream_t st) {
  note_launches(1);
  k_correct<<<grid_for(rows, 128), 128, 0, st>>>(mode, rows, ns, rs, drs, drho, out, flags);
  return cudaGetLastError();
}

cudaError_t launch_norms(int ns, long long N, const double* R, double* partial, double* out,
                         cudaStream_t st) {
  const int nb = 296;
  note_launches(2);
  k_norms_partial<<<nb, NORM_BS, 0, st>>>(ns, N, R, partial);
  k_norms_final<<<1, 32, 0, st>>>(nb, partial, out);
  return cudaGetLastError();
}

__global__ void k_set_double(double* dst, double v) { *dst = v; }

cudaError_t launch_set_double(double* dst, double v, cudaStream_t st) {
  note_launches(1);
  k_set_double<<<1, 1, 0, st>>>(dst, v);
  return cudaGetLastError();
}

cudaError_t launch_dual_rhs(long long N, int nv, const double* R, const double* qm,
                            const double* qn, const double* qnm1, const double* vol, double theta,
                            double dt, double* out, cudaStream_t st) {
  note_launches(1);
  k_dual_rhs<<<grid_for(N * nv, 256), 256, 0, st>>>(N, nv, R, qm, qn, qnm1, vol, theta, dt, out);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(long long n, const double* x, double* partial, double* out,
                         cudaStream_t st) {
  const int nb = 296;
  note_launches(2);
  k_sumsq_partial<<<nb, NORM_BS, 0, st>>>(n, x, partial);
  k_sumsq_final<<<1, 32, 0, st>>>(nb, partial, out);
  return cudaGetLastError();
}

cudaError_t launch_transpose(long long N, int nv, const double* src, double* dst, int to_soa,
                             cudaStream_t st) {
  note_launches(1);
  // TT cells per tile: 128, fewer for very wide rows (<= 200 KB of tile)
  const int TT = (int)std::max<long long>(1, std::min<long long>(128, (200LL * 1024) / ((nv + 1) * 8LL)));
  const size_t smem = (size_t)TT * (nv + 1) * sizeof(double);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_transpose, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const long long tiles = (N + TT - 1) / TT;
  k_transpose<<<(int)std::min<long long>(std::max<long long>(tiles, 1), 148LL * 16), 256, smem, st>>>(
      N, nv, src, dst, to_soa, TT);
  return cudaGetLastError();
}

}  // namespace csb
