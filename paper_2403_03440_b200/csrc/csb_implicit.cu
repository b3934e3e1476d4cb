// csflow-b200: non-templated assembly kernels (reference implicit.py:176-197,
// 362-368) and the bucket-independent launchers.
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

__global__ void k_dtau_arrays(long long N, const double* li, const double* lv, const double* lS,
                              double lS_scalar, double cfl, const double* J, double* dtau,
                              unsigned long long* flags) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    const double si = (li[3 * c] + li[3 * c + 1]) + li[3 * c + 2];
    const double sv = (lv[3 * c] + lv[3 * c + 1]) + lv[3 * c + 2];
    const double den = J[c] * (si + sv) + (lS ? lS[c] : lS_scalar);
    if (!(den > 0.0)) raise_flag(flags, EB_ZERO_WAVE, c);
    dtau[c] = cfl / den;
  }
}

// ------------------------------------------------------------- assembly (faces)
// _face_radius (implicit.py:176-197): max over the two cells at the face metric
__global__ void k_assemble_face(GridDev g, OpDev op, int d) {
  const long long NF = g.NF[d];
  const long long N = g.N;
  const int fx = g.ni + (d == 0), fy = g.nj + (d == 1), fz = g.nk + (d == 2);
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < NF;
       f += (long long)gridDim.x * blockDim.x) {
    const int k = f % fz, j = (f / fz) % fy, i = f / ((long long)fz * fy);
    (void)fx;
    double S[3];
    load_S(g, d, f, S);
    const double a2 = (S[0] * S[0] + S[1] * S[1]) + S[2] * S[2];
    const double ar = sqrt(a2);
    const int pos = d == 0 ? i : (d == 1 ? j : k);
    const int nd = d == 0 ? g.ni : (d == 1 ? g.nj : g.nk);
    double lf[2], ls[2];
    int nc = 0;
    for (int side = 0; side < 2; ++side) {
      int cc[3] = {i, j, k};
      if (side == 0) {
        if (pos == 0) continue;
        cc[d] -= 1;
      } else if (pos == nd) {
        continue;
      }
      const long long c = cell_index(g, cc[0], cc[1], cc[2]);
      const double* st = op.st;
      const double U = fabs(st[ST_U0 * N + c] * S[0] + st[ST_U1 * N + c] * S[1] +
                            st[ST_U2 * N + c] * S[2]);
      const double V = __ldg(g.vol + c);
      const double nuf = op.mode == SCH_CI ? st[ST_NU * N + c] : st[ST_NF * N + c];
      lf[nc] = (U + st[ST_C * N + c] * ar) + 2.0 * nuf * a2 / V;
      ls[nc] = U + 2.0 * st[ST_NSP * N + c] * a2 / V;
      ++nc;
    }
    op.lam[d][f] = nc == 2 ? npmax(lf[0], lf[1]) : lf[0];
    if (op.mode != SCH_CI) op.lamsp[d][f] = nc == 2 ? npmax(ls[0], ls[1]) : ls[0];
  }
}

// ------------------------------------------------- CI species block inverse
// dinv = inv(d I - V dOmega) (implicit.py:362-368), one warp per cell,
// augmented Gauss-Jordan with partial pivoting in shared memory.
__global__ void k_block_inverse(int ns, GridDev g, OpDev op, unsigned long long* flags) {
  extern __shared__ double sh[];
  const int wpb = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = 2 * ns + 1;
  double* A = sh + (long long)w * ns * ld;
  const long long N = g.N;
  for (long long c = (long long)blockIdx.x * wpb + w; c < N; c += (long long)gridDim.x * wpb) {
    const double V = __ldg(g.vol + c);
    const double d = op.d[c];
    for (int e = lane; e < ns * ns; e += 32) {
      const int r = e / ns, cc = e % ns;
      const double vd = op.dom[((long long)r * ns + cc) * N + c] * V;
      A[r * ld + cc] = (r == cc ? d : 0.0) - vd;
      A[r * ld + ns + cc] = r == cc ? 1.0 : 0.0;
    }
    __syncwarp();
    bool singular = false;
    for (int k = 0; k < ns; ++k) {
      double best = -1.0;
      int bi = k;
      for (int r = k + lane; r < ns; r += 32) {
        const double v = fabs(A[r * ld + k]);
        if (v > best) {
          best = v;
          bi = r;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      best = __shfl_sync(0xffffffffu, best, 0);
      bi = __shfl_sync(0xffffffffu, bi, 0);
      if (!(best > 0.0) || !isfinite(best)) singular = true;
      if (bi != k) {
        for (int cc = lane; cc < 2 * ns; cc += 32) {
          const double t = A[k * ld + cc];
          A[k * ld + cc] = A[bi * ld + cc];
          A[bi * ld + cc] = t;
        }
      }
      __syncwarp();
      const double piv = A[k * ld + k];
      __syncwarp();
      for (int cc = lane; cc < 2 * ns; cc += 32) A[k * ld + cc] = A[k * ld + cc] / piv;
      __syncwarp();
      for (int r = lane; r < ns; r += 32) {
        if (r == k) continue;
        const double f = A[r * ld + k];
        if (f != 0.0)
          for (int cc = 0; cc < 2 * ns; ++cc) A[r * ld + cc] -= f * A[k * ld + cc];
      }
      __syncwarp();
    }
    if (singular && lane == 0) raise_flag(flags, EB_BLOCK, c);
    for (int e = lane; e < ns * ns; e += 32) {
      const int r = e / ns, cc = e % ns;
      op.dinv[((long long)r * ns + cc) * N + c] = A[r * ld + ns + cc];
    }
    __syncwarp();
  }
}

// 2-D fast-path geometric precondition: i/j faces have zero
// z-component, k faces are pure z and identical on both k planes.
__global__ void k_check_2d(GridDev g, int* ok) {
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < g.N;
       f += (long long)gridDim.x * blockDim.x) {
    const double* Sk = g.S[2];
    const long long nf = g.NF[2];
    // k faces of cell f: indices 2f and 2f+1 when nk == 1
    const double a0 = Sk[2 * f], a1 = Sk[nf + 2 * f], a2 = Sk[2 * nf + 2 * f];
    const double b0 = Sk[2 * f + 1], b1 = Sk[nf + 2 * f + 1], b2 = Sk[2 * nf + 2 * f + 1];
    if (a0 != 0.0 || a1 != 0.0 || b0 != 0.0 || b1 != 0.0 || a2 != b2) atomicExch(ok, 0);
  }
  for (int d = 0; d < 2; ++d) {
    const double* S = g.S[d];
    const long long nf = g.NF[d];
    for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nf;
         f += (long long)gridDim.x * blockDim.x)
      if (S[2 * nf + f] != 0.0) atomicExch(ok, 0);
  }
}


cudaError_t launch_dtau_arrays(long long N, const double* li, const double* lv, const double* lS,
                               double lS_scalar, double cfl, const double* J, double* dtau,
                               unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  k_dtau_arrays<<<grid_for(N, 256), 256, 0, st>>>(N, li, lv, lS, lS_scalar, cfl, J, dtau, flags);
  return cudaGetLastError();
}

cudaError_t launch_assemble(const Model* mp, int ns, const GridDev& g, const double* q,
                            const double* dtau, double theta, double dt, OpDev& op,
                            unsigned long long* flags, cudaStream_t st) {
  cudaError_t e = launch_assemble_cell(mp, ns, g, q, dtau, theta, dt, op, flags, st);
  if (e != cudaSuccess) return e;
  note_launches(3);
  for (int d = 0; d < 3; ++d) k_assemble_face<<<grid_for(g.NF[d], 256), 256, 0, st>>>(g, op, d);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (op.mode == SCH_CI && op.chem) {
    const int wpb = 4;
    const size_t smem = (size_t)wpb * ns * (2 * ns + 1) * sizeof(double);
    cudaFuncSetAttribute(k_block_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int blocks = (int)std::min<long long>((g.N + wpb - 1) / wpb, 148LL * 64);
    note_launches(1);
    k_block_inverse<<<blocks, 32 * wpb, smem, st>>>(ns, g, op, flags);
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t launch_check_2d(const GridDev& g, int* ok, cudaStream_t st) {
  k_check_2d<<<grid_for(g.N, 256), 256, 0, st>>>(g, ok);
  return cudaGetLastError();
}

// Static 2-D viscous face metrics (spatial.py:236-248): xn = S / Vf and the
// face-averaged tangential Sc * J, once per grid.
template <int D>
__global__ void k_face_metrics2d(GridDev g, double* fm) {
  const int fx = g.ni + (D == 0), fy = g.nj + (D == 1);
  const long long nf = g.NF[D];
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < (long long)fx * fy;
       f += (long long)gridDim.x * blockDim.x) {
    const int gi = (int)(f / fy), gj = (int)(f % fy);
    double S[3], xn[3], xt[3];
    const long long fidx = face_index(g, D, gi, gj, 0);
    load_S(g, D, fidx, S);
    bool hasm, hasp;
    long long cm, cp;
    face_metric2d<D>(g, gi, gj, S, xn, xt, hasm, hasp, cm, cp);
    for (int x = 0; x < 3; ++x) {
      fm[x * nf + fidx] = xn[x];
      fm[(3 + x) * nf + fidx] = xt[x];
    }
  }
}

cudaError_t launch_face_metrics2d(const GridDev& g, double* fm0, double* fm1, cudaStream_t st) {
  note_launches(2);
  k_face_metrics2d<0><<<grid_for(g.NF[0], 256), 256, 0, st>>>(g, fm0);
  k_face_metrics2d<1><<<grid_for(g.NF[1], 256), 256, 0, st>>>(g, fm1);
  return cudaGetLastError();
}

// Static cell metrics (cell_metric): Sc_d, |Sc_d|^2, |Sc_d| for d = 0..2 and 1/V.
__global__ void k_cell_metrics(GridDev g, double* cm) {
  g.cm = nullptr;  // compute from the face vectors
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(c % g.nk), j = (int)((c / g.nk) % g.nj), i = (int)(c / ((long long)g.nk * g.nj));
    for (int d = 0; d < 3; ++d) {
      double Sc[3], a2, sq;
      cell_metric(g, c, i, j, k, d, Sc, a2, sq);
      for (int x = 0; x < 3; ++x) cm[(5 * d + x) * g.N + c] = Sc[x];
      cm[(5 * d + 3) * g.N + c] = a2;
      cm[(5 * d + 4) * g.N + c] = sq;
    }
    cm[15 * g.N + c] = 1.0 / g.vol[c];
  }
}

cudaError_t launch_cell_metrics(const GridDev& g, double* cm, cudaStream_t st) {
  note_launches(1);
  k_cell_metrics<<<grid_for(g.N, 256), 256, 0, st>>>(g, cm);
  return cudaGetLastError();
}

}  // namespace csb
