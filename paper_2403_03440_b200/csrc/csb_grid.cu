// csflow-b200: setup-time kernels that run on the device instead of host numpy
// (SURVEY §8(f) rows 2 and 4):
//   * node fill of the reference's grid generators from their 1-D axes
//     (grid.py:102-111 generate_box, 139-162 generate_cylinder_ogrid);
//   * metric terms from nodes (grid.py:51-99 compute_metrics): half cross
//     product of the face diagonals, face centroids, divergence-theorem
//     volumes, degenerate-cell check;
//   * primitive construction / encoding of given states (mixture.py:310-351
//     make_primitive, prim_to_cons);
//   * the wall heat flux and the stagnation-point monitor (driver.py:132-205).
//
// The metric and node kernels round every operation exactly as numpy does
// (no FMA contraction: __dmul_rn / __dadd_rn / __dsub_rn in numpy's
// evaluation order), so device metrics are bit-identical to the reference's
// and a march on them follows the reference's CFL trajectory.
#include "../../include/csflow_b200.h"
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// ------------------------------------------------------------------ nodes
// mode 0 (box): node(i,j,k) = (a[i], b[j], c[k]);
// mode 1 (cylinder): node(i,j,k) = (b[j] * a[i], b[j] * s[i], c[k]) with
// a = cos(theta), s = sin(theta), b = r (grid.py:157-160 broadcasting products).
__global__ void k_fill_nodes(int mode, int n0, int n1, int n2, const double* __restrict__ a,
                             const double* __restrict__ s, const double* __restrict__ b,
                             const double* __restrict__ c, double* __restrict__ nodes) {
  const long long total = (long long)n0 * n1 * n2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % n2);
    const long long ij = e / n2;
    const int j = (int)(ij % n1), i = (int)(ij / n1);
    double x, y;
    if (mode == 0) {
      x = a[i];
      y = b[j];
    } else {
      x = __dmul_rn(b[j], a[i]);
      y = __dmul_rn(b[j], s[i]);
    }
    nodes[e * 3 + 0] = x;
    nodes[e * 3 + 1] = y;
    nodes[e * 3 + 2] = c[k];
  }
}

// ---------------------------------------------------------------- metrics
// Face vectors of direction D (grid.py:51-70).  With (A, B) the two
// tangential axes ((1,2), (2,0), (0,1))[D], the corners of face (i,j,k) are
// p00, pa0 (+A), pab (+A+B), p0b (+B); S = 0.5 * cross(pa0 - p0b, pab - p00)
// (numpy.cross: c0 = a1*b2 - a2*b1, ...), centroid = 0.25*(p00 + pa0 + pab + p0b).
// Writes S (SoA over faces) and sc = S . centroid (the volume terms).
template <int D>
__global__ void k_face_vectors(int ni, int nj, int nk, const double* __restrict__ nodes,
                               double* __restrict__ S, double* __restrict__ sc) {
  constexpr int A = D == 0 ? 1 : D == 1 ? 2 : 0;
  constexpr int B = D == 0 ? 2 : D == 1 ? 0 : 1;
  const int f0 = ni + (D == 0), f1 = nj + (D == 1), f2 = nk + (D == 2);
  const long long NF = (long long)f0 * f1 * f2;
  const long long s1 = nk + 1, s0 = (long long)(nj + 1) * (nk + 1);  // node strides
  for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < NF;
       f += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(f % f2);
    const long long ij = f / f2;
    const int j = (int)(ij % f1), i = (int)(ij / f1);
    const long long base = (long long)i * s0 + (long long)j * s1 + k;
    const long long st[3] = {s0, s1, 1};
    const double* p00 = nodes + 3 * base;
    const double* pa0 = nodes + 3 * (base + st[A]);
    const double* pab = nodes + 3 * (base + st[A] + st[B]);
    const double* p0b = nodes + 3 * (base + st[B]);
    double u[3], v[3], cen[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      u[x] = __dsub_rn(pa0[x], p0b[x]);  // d2
      v[x] = __dsub_rn(pab[x], p00[x]);  // d1
      cen[x] = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(p00[x], pa0[x]), pab[x]), p0b[x]));
    }
    double cr[3];
    cr[0] = __dsub_rn(__dmul_rn(u[1], v[2]), __dmul_rn(u[2], v[1]));
    cr[1] = __dsub_rn(__dmul_rn(u[2], v[0]), __dmul_rn(u[0], v[2]));
    cr[2] = __dsub_rn(__dmul_rn(u[0], v[1]), __dmul_rn(u[1], v[0]));
    double Sx[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      Sx[x] = __dmul_rn(0.5, cr[x]);
      S[x * NF + f] = Sx[x];
    }
    // einsum("...c,...c->...") over 3 components sums (x0 + x2) + x1
    // (numpy 2.3's inner loop; checked bit for bit against the reference's
    // metrics of a warped 3-D grid)
    sc[f] = __dadd_rn(__dadd_rn(__dmul_rn(Sx[0], cen[0]), __dmul_rn(Sx[2], cen[2])),
                      __dmul_rn(Sx[1], cen[1]));
  }
}

// V = (sc_i+ - sc_i- + sc_j+ - sc_j- + sc_k+ - sc_k-) / 3 (grid.py:81-91), in
// Python's left-to-right order; degenerate (V <= 1e-30 or non-finite) cells
// set bad[0] and the smallest such cell index in bad[1].
__global__ void k_volumes(int ni, int nj, int nk, const double* __restrict__ sci,
                          const double* __restrict__ scj, const double* __restrict__ sck,
                          double* __restrict__ vol, unsigned long long* bad) {
  const long long N = (long long)ni * nj * nk;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
       c += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(c % nk);
    const long long ij = c / nk;
    const int j = (int)(ij % nj), i = (int)(ij / nj);
    const long long fi = ((long long)i * nj + j) * nk + k;
    const long long fj = ((long long)i * (nj + 1) + j) * nk + k;
    const long long fk = ((long long)i * nj + j) * (nk + 1) + k;
    double v = __dsub_rn(sci[fi + (long long)nj * nk], sci[fi]);
    v = __dadd_rn(v, scj[fj + nk]);
    v = __dsub_rn(v, scj[fj]);
    v = __dadd_rn(v, sck[fk + 1]);
    v = __dsub_rn(v, sck[fk]);
    v = __ddiv_rn(v, 3.0);
    vol[c] = v;
    if (!(v > 1e-30) || !isfinite(v)) {
      atomicOr(bad, 1ull);
      atomicMin(bad + 1, (unsigned long long)c);
    }
  }
}

// ------------------------------------------------------------ primitives
// make_primitive (mixture.py:326-351) for n states: two of (rho, p, T) are
// given (the missing pointer is null) plus u (n x 3 AoS) and Y (n x ns AoS,
// used as given, not renormalised).  out: the csb_cons_to_prim layout
// [rho, u0, u1, u2, p, T, c, gamma, h, Ek, R, cp, Y_0..Y_ns-1] x n (SoA);
// q (optional): the conservative vector (prim_to_cons, mixture.py:310-323),
// SoA (5 + ns) x n.  Non-positive rho, p or T raises EB_DECODE.
__global__ void k_primitive(const Model* __restrict__ mp, long long n, const double* __restrict__ rho_in,
                            const double* __restrict__ u_in, const double* __restrict__ p_in,
                            const double* __restrict__ T_in, const double* __restrict__ Y_in,
                            double* __restrict__ out, double* __restrict__ q,
                            unsigned long long* flags) {
  const Model& m = *mp;
  const int ns = m.ns;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const double* Y = Y_in + c * ns;
    double R = 0.0, cp = 0.0, yb = 0.0;
    for (int s = 0; s < ns; ++s) {  // Y @ R_s etc.: sequential dot products
      R = __dadd_rn(R, __dmul_rn(Y[s], m.Rs[s]));
      cp = __dadd_rn(cp, __dmul_rn(Y[s], m.cp[s]));
      yb = __dadd_rn(yb, __dmul_rn(Y[s], m.bs[s]));
    }
    double rho, p, T;
    if (!rho_in) {
      p = p_in[c];
      T = T_in[c];
      rho = __ddiv_rn(p, __dmul_rn(R, T));
    } else if (!T_in) {
      rho = rho_in[c];
      p = p_in[c];
      T = __ddiv_rn(p, __dmul_rn(rho, R));
    } else {
      rho = rho_in[c];
      T = T_in[c];
      p = p_in ? p_in[c] : __dmul_rn(__dmul_rn(rho, R), T);
    }
    const double u0 = u_in[3 * c], u1 = u_in[3 * c + 1], u2 = u_in[3 * c + 2];
    const double Ek = __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(u0, u0), __dmul_rn(u1, u1)),
                                               __dmul_rn(u2, u2)));
    const double cv = __dsub_rn(cp, R);
    const double gamma = __ddiv_rn(cp, cv);
    if (!(rho > 0.0) || !(T > 0.0) || !(p > 0.0)) raise_flag(flags, EB_DECODE, c);
    if (out) {
      double v[12] = {rho, u0, u1, u2, p, T, sqrt(__dmul_rn(__dmul_rn(gamma, R), T)), gamma,
                      __dadd_rn(__dadd_rn(yb, __dmul_rn(cp, T)), Ek), Ek, R, cp};
#pragma unroll
      for (int x = 0; x < 12; ++x) out[x * n + c] = v[x];
      for (int s = 0; s < ns; ++s) out[(12 + s) * n + c] = Y[s];
    }
    if (q) {
      // e_t = Y.b + (Y.cp) T - (Y.R) T + Ek
      const double et = __dadd_rn(__dsub_rn(__dadd_rn(yb, __dmul_rn(cp, T)), __dmul_rn(R, T)), Ek);
      q[c] = rho;
      q[n + c] = __dmul_rn(rho, u0);
      q[2 * n + c] = __dmul_rn(rho, u1);
      q[3 * n + c] = __dmul_rn(rho, u2);
      q[4 * n + c] = __dmul_rn(rho, et);
      for (int s = 0; s < ns; ++s) q[(5 + s) * n + c] = __dmul_rn(rho, Y[s]);
    }
  }
}

// ------------------------------------------------------- wall heat flux
// One wall face (axis, side).  slab: the three node planes nearest the wall
// along `axis` (plane 0 = the wall), AoS (3, m1 + 1, m2 + 1, 3) over the two
// remaining axes in increasing order.  For each wall cell (t1, t2):
//   nhat = S_wall / |S_wall| (flipped on the max side), fc = face centroid,
//   c1, c2 = centroids (node averages) of the first two cells,
//   d1, d2 = |(c - fc) . nhat|,
//   dT/dn = ((T1 - Tw) d2^2 - (T2 - Tw) d1^2) / (d1 d2 (d2 - d1)),
//   rho_w = p1 / (R(Y1) Tw), k_w = mu(Tw, Y1) cp(Y1) / Pr,  qw = k_w dT/dn
// (driver.py:132-184), with T, p, Y the decoded cell states
// (fields.py:39-46).  Writes qw and p1 per wall cell, (m1, m2) C order.
template <int NSB>
__global__ void k_wall_flux(const Model* __restrict__ mp, GridDev g, int axis, int side, double Tw,
                            const double* __restrict__ q, const double* __restrict__ slab,
                            double* __restrict__ qw, double* __restrict__ pw,
                            unsigned long long* flags) {
  const Model& m = *mp;
  const int dims[3] = {g.ni, g.nj, g.nk};
  const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;
  const int m1 = dims[a1], m2 = dims[a2];
  const long long nw = (long long)m1 * m2;
  const int n = dims[axis];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nw;
       e += (long long)gridDim.x * blockDim.x) {
    const int t1 = (int)(e / m2), t2 = (int)(e % m2);
    auto node = [&](int plane, int x1, int x2, int comp) {
      return slab[(((long long)plane * (m1 + 1) + x1) * (m2 + 1) + x2) * 3 + comp];
    };
    // wall face vector and unit normal (into the fluid)
    int fidx[3];
    fidx[axis] = side ? n : 0;
    fidx[a1] = t1;
    fidx[a2] = t2;
    double S[3];
    load_S(g, axis, face_index(g, axis, fidx[0], fidx[1], fidx[2]), S);
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(S[0], S[0]), __dmul_rn(S[1], S[1])),
                                      __dmul_rn(S[2], S[2])));
    double nh[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) nh[x] = side ? -__ddiv_rn(S[x], nrm) : __ddiv_rn(S[x], nrm);
    // centroids in numpy's summation order (driver.py:147-149, 161-163): the
    // wall distances are differences of O(1) positions that agree to ~1e-5
    // relative on stretched wall grids, so every rounding is reproduced
    // (slab plane of cell layer l, normal node offset o: side 0 l + o,
    // side 1 l + 1 - o)
    double fc[3], cc[2][3];
    const int offs[8][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1},
                            {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      fc[x] = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(node(0, t1, t2, x), node(0, t1 + 1, t2, x)),
                                                  node(0, t1, t2 + 1, x)),
                                        node(0, t1 + 1, t2 + 1, x)));
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        double acc = 0.0;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int on = offs[v][axis], o1 = offs[v][a1], o2 = offs[v][a2];
          const double nv = node(side ? l + 1 - on : l + on, t1 + o1, t2 + o2, x);
          acc = v == 0 ? nv : __dadd_rn(acc, nv);
        }
        cc[l][x] = __dmul_rn(0.125, acc);
      }
    }
    double dist[2];
#pragma unroll
    for (int l = 0; l < 2; ++l) {  // |einsum(c - fc, nhat)|: (x0 + x2) + x1
      const double e0 = __dmul_rn(__dsub_rn(cc[l][0], fc[0]), nh[0]);
      const double e1 = __dmul_rn(__dsub_rn(cc[l][1], fc[1]), nh[1]);
      const double e2 = __dmul_rn(__dsub_rn(cc[l][2], fc[2]), nh[2]);
      dist[l] = fabs(__dadd_rn(__dadd_rn(e0, e2), e1));
    }
    // first two cells off the wall
    int ci[3];
    ci[a1] = t1;
    ci[a2] = t2;
    ci[axis] = side ? n - 1 : 0;
    const long long c1 = cell_index(g, ci[0], ci[1], ci[2]);
    ci[axis] = side ? n - 2 : 1;
    const long long c2 = cell_index(g, ci[0], ci[1], ci[2]);
    Cell<NSB> P1, P2;
    bool ok = decode<NSB>(m, q + c1, g.N, P1);
    ok = decode<NSB>(m, q + c2, g.N, P2) && ok;
    if (!ok) raise_flag(flags, EB_DECODE, c1);
    const double d1 = dist[0], d2 = dist[1];
    const double dTdn = __ddiv_rn(__dsub_rn(__dmul_rn(P1.T - Tw, __dmul_rn(d2, d2)),
                                            __dmul_rn(P2.T - Tw, __dmul_rn(d1, d1))),
                                  __dmul_rn(__dmul_rn(d1, d2), __dsub_rn(d2, d1)));
    double mu, kc, D;
    transport<NSB>(m, Tw, P1.Y, P1.p / (P1.R * Tw), mu, kc, D);
    qw[e] = kc * dTdn;
    pw[e] = P1.p;
  }
}

// numpy.argmax of key (first maximum; a NaN is the maximum, first NaN wins)
// and val at that index: out = [key_max, val_at, index].  One CTA.
__global__ void k_argmax_pick(long long n, const double* __restrict__ key,
                              const double* __restrict__ val, double* __restrict__ out) {
  __shared__ double bk[32];
  __shared__ long long bi[32];
  double best = -INFINITY;
  long long idx = -1;
  auto better = [](double a, long long ia, double b, long long ib) {
    // is (a, ia) before (b, ib) in numpy argmax order?
    if (ib < 0) return ia >= 0;
    if (ia < 0) return false;
    const bool na = a != a, nb = b != b;
    if (na || nb) return na && (!nb || ia < ib);
    return a > b || (a == b && ia < ib);
  };
  for (long long e = threadIdx.x; e < n; e += blockDim.x) {
    const double k = key[e];
    if (better(k, e, best, idx)) {
      best = k;
      idx = e;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const long long oi = __shfl_down_sync(0xffffffffu, idx, o);
    if (better(ob, oi, best, idx)) {
      best = ob;
      idx = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    bk[w] = best;
    bi[w] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (better(bk[i], bi[i], best, idx)) {
        best = bk[i];
        idx = bi[i];
      }
    out[0] = best;
    out[1] = idx >= 0 ? val[idx] : NAN;
    out[2] = (double)idx;
  }
}

}  // namespace csb

using namespace csb;

cudaError_t csb_launch_fill_nodes(int mode, int n0, int n1, int n2, const double* a, const double* s,
                                  const double* b, const double* c, double* nodes, cudaStream_t st) {
  note_launches(1);
  k_fill_nodes<<<grid_for((long long)n0 * n1 * n2, 256), 256, 0, st>>>(mode, n0, n1, n2, a, s, b, c,
                                                                      nodes);
  return cudaGetLastError();
}

cudaError_t csb_launch_metrics(int ni, int nj, int nk, const double* nodes, double* Si, double* Sj,
                               double* Sk, double* vol, double* scratch,
                               unsigned long long* bad, cudaStream_t st) {
  const long long NF0 = (long long)(ni + 1) * nj * nk, NF1 = (long long)ni * (nj + 1) * nk,
                  NF2 = (long long)ni * nj * (nk + 1);
  double* sc0 = scratch;
  double* sc1 = sc0 + NF0;
  double* sc2 = sc1 + NF1;
  note_launches(4);
  k_face_vectors<0><<<grid_for(NF0, 256), 256, 0, st>>>(ni, nj, nk, nodes, Si, sc0);
  k_face_vectors<1><<<grid_for(NF1, 256), 256, 0, st>>>(ni, nj, nk, nodes, Sj, sc1);
  k_face_vectors<2><<<grid_for(NF2, 256), 256, 0, st>>>(ni, nj, nk, nodes, Sk, sc2);
  k_volumes<<<grid_for((long long)ni * nj * nk, 256), 256, 0, st>>>(ni, nj, nk, sc0, sc1, sc2, vol,
                                                                     bad);
  return cudaGetLastError();
}

cudaError_t csb_launch_primitive(const Model* mp, long long n, const double* rho, const double* u,
                                 const double* p, const double* T, const double* Y, double* out,
                                 double* q, unsigned long long* flags, cudaStream_t st) {
  note_launches(1);
  k_primitive<<<grid_for(n, 128), 128, 0, st>>>(mp, n, rho, u, p, T, Y, out, q, flags);
  return cudaGetLastError();
}

cudaError_t csb_launch_wall_flux(const Model* mp, int ns, const GridDev& g, int axis, int side,
                                 double Tw, const double* q, const double* slab, double* qw,
                                 double* pw, unsigned long long* flags, cudaStream_t st) {
  const int dims[3] = {g.ni, g.nj, g.nk};
  const long long nw = (long long)dims[axis == 0 ? 1 : 0] * dims[axis == 2 ? 1 : 2];
  note_launches(1);
  const int nb = grid_for(nw, 128);
  if (ns <= 8)
    k_wall_flux<8><<<nb, 128, 0, st>>>(mp, g, axis, side, Tw, q, slab, qw, pw, flags);
  else if (ns <= 16)
    k_wall_flux<16><<<nb, 128, 0, st>>>(mp, g, axis, side, Tw, q, slab, qw, pw, flags);
  else if (ns <= 32)
    k_wall_flux<32><<<nb, 128, 0, st>>>(mp, g, axis, side, Tw, q, slab, qw, pw, flags);
  else
    k_wall_flux<64><<<nb, 128, 0, st>>>(mp, g, axis, side, Tw, q, slab, qw, pw, flags);
  return cudaGetLastError();
}

cudaError_t csb_launch_argmax_pick(long long n, const double* key, const double* val, double* out,
                                   cudaStream_t st) {
  note_launches(1);
  k_argmax_pick<<<1, 1024, 0, st>>>(n, key, val, out);
  return cudaGetLastError();
}
