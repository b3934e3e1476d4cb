// csflow-b200: 2-D (nk == 1) production path of the implicit step.
//
//   k_records2d  : fused local time step + CS operator assembly (reference
//                  implicit.py:33-44, 144-197, 329-403), written as "sweep
//                  records" in the strip-skewed, step-major layout below;
//   k_wave2d<F/B>: the LU-SGS forward / backward sweep (lusgs.py:150-247) as
//                  a pipelined wavefront over 32-row strips;
//   k_epilogue2d : species closure CS1/CS2 + admissibility gate
//                  (driver.py:216-229, 250; implicit.py:113-141).
//
// Strip-skewed, step-major layout.  Rows j are grouped in strips of 32
// (s = j >> 5, r = j & 31).  At wavefront step t of strip s, row r processes
// column i = t - r.  A record group with NG planes stores plane p of cell
// (i, j) at ((s*T + t)*NG + p)*32 + r with t = i + r (T = ni + 31 rounded up
// to a multiple of WK).  WK consecutive steps of one strip are therefore one
// contiguous block of WK*NG*32 doubles: the sweep streams each group with a
// single TMA bulk copy per WK steps into an mbarrier ring.  The backward sweep
// visits the same physical steps in reverse (backward slot t holds the same
// cells), so it streams the same blocks in reverse order.
//
// Record groups: C (both sweeps) = invd, invs[nsI], w[5], b[5], u, v, hr;
// F (forward) = rhs[nv], upper-i face (Sx, Sy, lam, lamsp), upper-j face;
// B (backward) = lower-i face, lower-j face; Q = dq* (forward output,
// backward input); W = dq (backward output).
//
// One CTA per strip (dynamic ticket => deadlock-free ordering):
//   warp 0: flow chain (5 components, rank-2 half-block products),
//   warp 1: species chain (ns scalar chains),
//   warp 2: producer (TMA bulk copies + the upstream strip's hand-off values,
//           polled from L2),
//   warp 3: publisher (this strip's hand-off row to L2 + progress flag).
// Row r hands its j-direction contribution to row r+1 (r-1 backward) with a
// warp shuffle; strip boundaries go through L2.
#pragma once

#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

constexpr int WK = 4;          // wavefront steps per ring slot
constexpr int HRING = 64;      // hand-off ring (columns)

struct RecMap {
  int nv, nsI;
  // group C
  CSB_DEV int invd() const { return 0; }
  CSB_DEV int invs() const { return 1; }
  CSB_DEV int w() const { return 1 + nsI; }
  CSB_DEV int b() const { return w() + 5; }
  CSB_DEV int uv() const { return w() + 10; }
  CSB_DEV int hr() const { return w() + 12; }
  CSB_DEV int nc() const { return w() + 13; }
  // group F: rhs[nv], fi[4], fj[4]; group B: fi[4], fj[4]
  CSB_DEV int nf() const { return nv + 8; }
};

// ---------------------------------------------------------------- PTX helpers
CSB_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
CSB_DEV void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
CSB_DEV void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
CSB_DEV void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
CSB_DEV void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
CSB_DEV void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
CSB_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
CSB_DEV int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CSB_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
CSB_DEV void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CSB_DEV int ld_volatile_s(const int* p) { return *(volatile const int*)p; }

// step-major group address of (strip s, step t, plane p, row r)
CSB_DEV long long gaddr(const Skew& k, int NG, int s, int t, int p, int r) {
  return (((long long)s * k.T + t) * NG + p) * 32 + r;
}

// ============================================================== records
// Tile = one strip (32 rows) x C columns.  Phase A: per cell (tile + 1-cell
// halo) decode + transport (face quantities); interior cells also get dtau,
// the diagonals and the Jacobian ingredients.  Phase B: face radii (max of
// the two adjacent cells at the face metric).  Phase C: skewed stores.
template <int NSB>
__global__ void __launch_bounds__(256) k_records2d(const Model* __restrict__ mp, GridDev g, Skew sk,
                                                   const double* __restrict__ q,
                                                   const double* __restrict__ R, double cfl,
                                                   const double* __restrict__ lamS,
                                                   const double* __restrict__ domd, int dom_stride,
                                                   int per_species, double* __restrict__ recC,
                                                   double* __restrict__ recF,
                                                   double* __restrict__ recB, int C,
                                                   unsigned long long* flags) {
  extern __shared__ double sm[];
  const Model& m = *mp;
  const int ns = m.ns, nv = 5 + ns, nsI = per_species ? ns : 1;
  RecMap rm{nv, nsI};
  const int NC = rm.nc(), NF = rm.nf();
  const int ncb = (g.ni + C - 1) / C;
  const int s = blockIdx.x / ncb, ib = blockIdx.x % ncb;
  const int i0 = ib * C, j0 = s * 32;
  const int HX = C + 2, HY = 34, NH = HX * HY;
  const int CT = C * 32;
  double* A = sm;            // [7][NH]: u, v, w, c, nf, nsp, V
  double* BC = sm + 7 * NH;  // [NC][CT] | [NF][CT] | [8][CT]
  double* BF = BC + (long long)NC * CT;
  double* BB = BF + (long long)NF * CT;
  const long long N = g.N;
  // ---------------- phase A: halo-extended per-cell quantities
  for (int l = threadIdx.x; l < NH; l += blockDim.x) {
    const int hx = l / HY, hy = l % HY;
    const int i = i0 - 1 + hx, j = j0 - 1 + hy;
    if (i < 0 || i >= g.ni || j < 0 || j >= g.nj) continue;
    const long long c = (long long)i * g.nj + j;
    Cell<NSB> cs;
    const bool ok = decode<NSB>(m, q + c, N, cs);
    double mu, kc, D, nf, nsp, nu;
    transport<NSB>(m, cs.T, cs.Y, cs.rho, mu, kc, D);
    diffusivities(mu, kc, D, cs.rho, cs.cp - cs.R, nf, nsp, nu);
    const double V = __ldg(g.vol + c);
    A[0 * NH + l] = cs.u[0];
    A[1 * NH + l] = cs.u[1];
    A[2 * NH + l] = cs.u[2];
    A[3 * NH + l] = cs.c;
    A[4 * NH + l] = nf;
    A[5 * NH + l] = nsp;
    A[6 * NH + l] = V;
    const bool inner = hx >= 1 && hx <= C && hy >= 1 && hy <= 32;
    if (!inner) continue;
    if (!ok) raise_flag(flags, EB_DECODE, c);
    const int e = (hx - 1) * 32 + (hy - 1);  // tile-local cell (column-major by i)
    // cell radii at the cell-averaged metric, dtau (implicit.py:152-163, 33-44)
    double li[3], lv[3], rf = 0.0, rsp = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      int hi[3] = {i, j, 0};
      hi[d] += 1;
      double a[3], b[3];
      load_S(g, d, face_index(g, d, i, j, 0), a);
      load_S(g, d, face_index(g, d, hi[0], hi[1], hi[2]), b);
      double Sc[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) Sc[x] = 0.5 * (a[x] + b[x]);
      const double a2 = (Sc[0] * Sc[0] + Sc[1] * Sc[1]) + Sc[2] * Sc[2];
      const double U = fabs(cs.u[0] * Sc[0] + cs.u[1] * Sc[1] + cs.u[2] * Sc[2]);
      const double sq = sqrt(a2);
      li[d] = U + cs.c * sq;
      lv[d] = nu * a2 / V;
      const double lf = (U + cs.c * sq) + 2.0 * nf * a2 / V;
      const double ls = U + 2.0 * nsp * a2 / V;
      rf = d == 0 ? lf : rf + lf;
      rsp = d == 0 ? ls : rsp + ls;
    }
    const double J = 1.0 / V;
    const double den = J * (((li[0] + li[1]) + li[2]) + ((lv[0] + lv[1]) + lv[2])) +
                       (lamS ? lamS[c] : 0.0);
    if (!(den > 0.0)) raise_flag(flags, EB_ZERO_WAVE, c);
    const double dtau = cfl / den;
    const double base = V / dtau;
    const double dflow = base + rf;
    bool bad = !(fabs(dflow) >= 1e-300) || !isfinite(dflow);
    BC[rm.invd() * CT + e] = 1.0 / dflow;
    const double dsp0 = base + rsp;
    if (per_species) {
      for (int sp = 0; sp < ns; ++sp) {
        const double v = dsp0 - domd[(long long)sp * dom_stride * N + c] * V;
        bad |= !(fabs(v) >= 1e-300) || !isfinite(v);
        BC[(rm.invs() + sp) * CT + e] = 1.0 / v;
      }
    } else {
      bad |= !(fabs(dsp0) >= 1e-300) || !isfinite(dsp0);
      BC[rm.invs() * CT + e] = 1.0 / dsp0;
    }
    if (bad) raise_flag(flags, EB_SINGULAR, c);
    for (int k = 0; k < nv; ++k) BF[k * CT + e] = -R[(long long)k * N + c];
    const double beta = cs.gamma - 1.0;
    const int pw = rm.w(), pb = rm.b();
    BC[(pw + 0) * CT + e] = cs.rho;
    BC[(pw + 1) * CT + e] = cs.rho * cs.u[0];
    BC[(pw + 2) * CT + e] = cs.rho * cs.u[1];
    BC[(pw + 3) * CT + e] = cs.rho * cs.u[2];
    BC[(pw + 4) * CT + e] = cs.rho * cs.h;
    BC[(pb + 0) * CT + e] = beta * cs.Ek;
    BC[(pb + 1) * CT + e] = -beta * cs.u[0];
    BC[(pb + 2) * CT + e] = -beta * cs.u[1];
    BC[(pb + 3) * CT + e] = -beta * cs.u[2];
    BC[(pb + 4) * CT + e] = beta;
    BC[(rm.uv() + 0) * CT + e] = cs.u[0];
    BC[(rm.uv() + 1) * CT + e] = cs.u[1];
    BC[rm.hr() * CT + e] = 0.5 / cs.rho;
  }
  __syncthreads();
  // ---------------- phase B: face radii of the 4 faces of every tile cell
  for (int e = threadIdx.x; e < CT; e += blockDim.x) {
    const int ii = e / 32, jj = e % 32;
    const int i = i0 + ii, j = j0 + jj;
    if (i >= g.ni || j >= g.nj) continue;
    const int hc = (ii + 1) * HY + (jj + 1);
    // faces: 0 upper-i (i+1), 1 upper-j (j+1), 2 lower-i (i), 3 lower-j (j)
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int d = f & 1;
      const bool upper = f < 2;
      int fi = i, fj = j;
      if (upper) {
        if (d == 0) fi += 1;
        else fj += 1;
      }
      double S[3];
      load_S(g, d, face_index(g, d, fi, fj, 0), S);
      const double a2 = (S[0] * S[0] + S[1] * S[1]) + S[2] * S[2];
      const double ar = sqrt(a2);
      const int nb = upper ? (d == 0 ? hc + HY : hc + 1) : (d == 0 ? hc - HY : hc - 1);
      const bool nb_in = upper ? (d == 0 ? i + 1 < g.ni : j + 1 < g.nj) : (d == 0 ? i > 0 : j > 0);
      const int lo = upper ? hc : nb, hi = upper ? nb : hc;  // lower/upper cell of the face
      auto lam = [&](int h, bool sp) {
        const double U = fabs(A[0 * NH + h] * S[0] + A[1 * NH + h] * S[1] + A[2 * NH + h] * S[2]);
        if (sp) return U + 2.0 * A[5 * NH + h] * a2 / A[6 * NH + h];
        return (U + A[3 * NH + h] * ar) + 2.0 * A[4 * NH + h] * a2 / A[6 * NH + h];
      };
      double lf, ls;
      if (nb_in) {
        lf = npmax(lam(lo, false), lam(hi, false));
        ls = npmax(lam(lo, true), lam(hi, true));
      } else {
        lf = lam(hc, false);
        ls = lam(hc, true);
      }
      double* dst = upper ? BF + (long long)(nv + 4 * d) * CT : BB + (long long)(4 * d) * CT;
      dst[0 * CT + e] = S[0];
      dst[1 * CT + e] = S[1];
      dst[2 * CT + e] = lf;
      dst[3 * CT + e] = ls;
    }
  }
  __syncthreads();
  // ---------------- phase C: skewed step-major stores
  // tile steps tt in [0, C + 31): element (tt, r) <-> cell (i0 + tt - r, j0 + r)
  const int nt = C + 31;
  for (int e = threadIdx.x; e < nt * 32; e += blockDim.x) {
    const int tt = e / 32, r = e % 32;
    const int ii = tt - r;
    if (ii < 0 || ii >= C) continue;
    const int i = i0 + ii, j = j0 + r;
    // cells outside the grid are padding slots: zeroed once at workspace
    // setup and never written (i >= ni would also step past the strip)
    if (i >= g.ni || j >= g.nj) continue;
    const int t = i + r;
    const int el = ii * 32 + r;
    for (int p = 0; p < NC; ++p) recC[gaddr(sk, NC, s, t, p, r)] = BC[p * CT + el];
    for (int p = 0; p < NF; ++p) recF[gaddr(sk, NF, s, t, p, r)] = BF[p * CT + el];
    for (int p = 0; p < 8; ++p) recB[gaddr(sk, 8, s, t, p, r)] = BB[p * CT + el];
  }
}

// ============================================================== wavefront
struct WaveArgs {
  Skew sk;
  int ni, nj, ns, nv, nsI, nslots, D;
  const double* recC;
  const double* recX;  // forward: F group; backward: Q (dq*)
  const double* recB;  // backward faces
  double* out;         // forward: dq* (Q); backward: dq (W), step-major [nv]
  double* hand;        // [nstrip][ni][nv]
  int* prog;           // [nstrip]
  int* ticket;
  double sp_scale;
};

template <int NSB, bool BWD>
__global__ void __launch_bounds__(128, 1) k_wave2d(WaveArgs a) {
  extern __shared__ __align__(128) double wsm[];
  __shared__ unsigned long long full_bar[8], empty_bar[8];
  __shared__ int s_strip, done_cnt[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = a.nv, ns = a.ns, D = a.D;
  RecMap rm{nv, a.nsI};
  const int NC = rm.nc();
  const int NX = BWD ? nv : rm.nf();  // planes of the X group (rhs+faces | dq*)
  const int NB = BWD ? 8 : 0;
  const long long slotC = (long long)WK * NC * 32, slotX = (long long)WK * NX * 32,
                  slotB = (long long)WK * NB * 32;
  double* ringC = wsm;                // [D][WK][NC][32]
  double* ringX = ringC + D * slotC;  // [D][WK][NX][32]
  double* ringB = ringX + D * slotX;  // [D][WK][8][32] (backward)
  double* hin = ringB + D * slotB;    // [D][WK][nv]
  double* hout = hin + D * WK * nv;   // [HRING][nv]
  if (threadIdx.x == 0) {
    const int tk = atomicAdd(a.ticket, 1);
    s_strip = BWD ? a.sk.nstrip - 1 - tk : tk;
    for (int b = 0; b < D; ++b) {
      mbar_init(&full_bar[b], 32);
      mbar_init(&empty_bar[b], 2);
    }
    done_cnt[0] = done_cnt[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int s = s_strip;
  const int j0 = s * 32;
  const int rt = min(31, a.nj - 1 - j0);  // highest valid row of this strip
  const int nslots = a.nslots;
  const int T = a.sk.T;
  const int up = BWD ? s + 1 : s - 1;
  const bool has_up = BWD ? (s + 1 < a.sk.nstrip) : (s > 0);
  const bool has_down = BWD ? (s > 0) : (s + 1 < a.sk.nstrip);

  if (warp == 2) {
    // ---------------------------------------------------- producer
    for (int ks = 0; ks < nslots; ++ks) {
      const int k = BWD ? nslots - 1 - ks : ks;
      const int buf = ks % D;
      if (ks >= D) mbar_wait(&empty_bar[buf], ((ks / D) - 1) & 1);
      if (lane == 0) {
        // bulk copies first: they do not depend on the upstream strip
        const unsigned bC = (unsigned)(slotC * 8), bX = (unsigned)(slotX * 8),
                       bB = (unsigned)(slotB * 8);
        mbar_expect_tx(&full_bar[buf], bC + bX + bB);
        const long long st = (long long)s * T + (long long)k * WK;
        bulk_g2s(ringC + buf * slotC, a.recC + st * NC * 32, bC, &full_bar[buf]);
        bulk_g2s(ringX + buf * slotX, a.recX + st * NX * 32, bX, &full_bar[buf]);
        if (BWD) bulk_g2s(ringB + buf * slotB, a.recB + st * 8 * 32, bB, &full_bar[buf]);
      }
      // upstream hand-off for this slot's WK steps (first row's columns)
      double* hb = hin + buf * WK * nv;
      if (has_up) {
        int need;
        if (!BWD) need = min(k * WK + WK - 1, a.ni - 1) + 1;  // first row 0: col = t
        else need = a.ni - max(k * WK - rt, 0);               // first row rt: col = t - rt
        need = max(0, min(need, a.ni));
        while (ld_relaxed(a.prog + up) < need) __nanosleep(20);
        (void)ld_acquire(a.prog + up);
        for (int e = lane; e < WK * nv; e += 32) {
          const int kk = e / nv, c = e % nv;
          const int t = k * WK + kk;
          const int col = BWD ? t - rt : t;
          double v = 0.0;
          if (col >= 0 && col < a.ni) v = __ldcg(a.hand + ((long long)up * a.ni + col) * nv + c);
          hb[kk * nv + c] = v;
        }
      } else {
        for (int e = lane; e < WK * nv; e += 32) hb[e] = 0.0;
      }
      __syncwarp();
      mbar_arrive(&full_bar[buf]);  // all 32 lanes, after their hand-off writes
    }
    return;
  }

  if (warp == 3) {
    // ---------------------------------------------------- publisher
    if (!has_down) return;
    int next = 0;
    while (next < a.ni) {
      const int d0 = ld_volatile_s(&done_cnt[0]), d1 = ld_volatile_s(&done_cnt[1]);
      __threadfence_block();
      const int dn = min(d0, d1);
      int cnt;
      if (!BWD) cnt = dn * WK - rt;          // cols < cnt done (top row rt: t = col + rt)
      else cnt = a.ni - (nslots - dn) * WK;  // bottom row 0: cols >= (nslots-dn)*WK done
      cnt = max(0, min(cnt, a.ni));
      if (cnt > next) {
        for (int e = lane; e < (cnt - next) * nv; e += 32) {
          const int co = next + e / nv, c = e % nv;
          const int col = BWD ? a.ni - 1 - co : co;
          a.hand[((long long)s * a.ni + col) * nv + c] = hout[(col % HRING) * nv + c];
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(a.prog + s, cnt);
        next = cnt;
      } else {
        __nanosleep(20);
      }
    }
    return;
  }

  // -------------------------------------------------------- chains
  const unsigned FULL = 0xffffffffu;
  const double sgn = BWD ? -1.0 : 1.0;
  const bool first = BWD ? (lane == rt) : (lane == 0);  // receives the upstream hand-off
  const bool last = BWD ? (lane == 0) : (lane == rt);   // sends the downstream hand-off
  const bool row_ok = j0 + lane < a.nj;
  auto real = [&](int t) { return row_ok && t - lane >= 0 && t - lane < a.ni; };
  // plane pointers inside a slot: C group, X group (rhs|dq*), faces (F tail | B)
  auto slot_ptrs = [&](int buf, int kk, const double*& pc, const double*& px, const double*& pfc) {
    pc = ringC + buf * slotC + (long long)kk * NC * 32 + lane;
    px = ringX + buf * slotX + (long long)kk * NX * 32 + lane;
    pfc = BWD ? ringB + buf * slotB + (long long)kk * 8 * 32 + lane : px + (long long)nv * 32;
  };
  if (warp == 0) {
    // ------------------------------ flow chain: 5 components per row
    double oi[5] = {0, 0, 0, 0, 0}, oj[5] = {0, 0, 0, 0, 0};
    for (int ks = 0; ks < nslots; ++ks) {
      const int k = BWD ? nslots - 1 - ks : ks;
      const int buf = ks % D;
      mbar_wait(&full_bar[buf], (ks / D) & 1);
      const double* hb = hin + buf * WK * nv;
#pragma unroll
      for (int mstep = 0; mstep < WK; ++mstep) {
        const int kk = BWD ? WK - 1 - mstep : mstep;
        const int t = k * WK + kk;
        const double *pc, *px, *pf;
        slot_ptrs(buf, kk, pc, px, pf);
        double ij[5];
#pragma unroll
        for (int c = 0; c < 5; ++c)
          ij[c] = BWD ? __shfl_down_sync(FULL, oj[c], 1) : __shfl_up_sync(FULL, oj[c], 1);
        if (first) {
#pragma unroll
          for (int c = 0; c < 5; ++c) ij[c] = hb[kk * nv + c];
        }
        const double invd = pc[rm.invd() * 32];
        double dq[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          if (BWD) dq[c] = px[c * 32] - (oi[c] + ij[c]) * invd;
          else dq[c] = ((px[c * 32] + oi[c]) + ij[c]) * invd;
          if (!real(t)) dq[c] = 0.0;  // padding cells carry exactly nothing
        }
        if (t < T) {
#pragma unroll
          for (int c = 0; c < 5; ++c) a.out[gaddr(a.sk, nv, s, t, c, lane)] = dq[c];
        }
        // outgoing half-block products through the two faces (rank-2 form)
        const int pw = rm.w(), pb = rm.b();
        const double w0 = pc[pw * 32], w1 = pc[(pw + 1) * 32], w2 = pc[(pw + 2) * 32],
                     w3 = pc[(pw + 3) * 32], w4 = pc[(pw + 4) * 32];
        const double sb = pc[pb * 32] * dq[0] + pc[(pb + 1) * 32] * dq[1] +
                          pc[(pb + 2) * 32] * dq[2] + pc[(pb + 3) * 32] * dq[3] +
                          pc[(pb + 4) * 32] * dq[4];
        const double u = pc[rm.uv() * 32], v = pc[(rm.uv() + 1) * 32], hr = pc[rm.hr() * 32];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          const double Sx = pf[(4 * f) * 32], Sy = pf[(4 * f + 1) * 32], lam = pf[(4 * f + 2) * 32];
          const double U = u * Sx + v * Sy;
          const double sa = (-U * hr) * dq[0] + (Sx * hr) * dq[1] + (Sy * hr) * dq[2];
          const double sig = 0.5 * (U + sgn * lam);
          double* o = f == 0 ? oi : oj;
          o[0] = w0 * sa + sig * dq[0];
          o[1] = w1 * sa + (0.5 * Sx) * sb + sig * dq[1];
          o[2] = w2 * sa + (0.5 * Sy) * sb + sig * dq[2];
          o[3] = w3 * sa + sig * dq[3];
          o[4] = w4 * sa + (0.5 * U) * sb + sig * dq[4];
        }
        const int col = t - lane;
        if (last && col >= 0 && col < a.ni) {
#pragma unroll
          for (int c = 0; c < 5; ++c) hout[(col % HRING) * nv + c] = oj[c];
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_bar[buf]);
        __threadfence_block();
        *(volatile int*)&done_cnt[0] = ks + 1;
      }
    }
  } else if (warp == 1) {
    // ------------------------------ species chain: ns scalar chains per row
    double oi[NSB], oj[NSB];
#pragma unroll
    for (int c = 0; c < NSB; ++c) oi[c] = oj[c] = 0.0;
    const int per = a.nsI > 1;
    for (int ks = 0; ks < nslots; ++ks) {
      const int k = BWD ? nslots - 1 - ks : ks;
      const int buf = ks % D;
      mbar_wait(&full_bar[buf], (ks / D) & 1);
      const double* hb = hin + buf * WK * nv;
#pragma unroll
      for (int mstep = 0; mstep < WK; ++mstep) {
        const int kk = BWD ? WK - 1 - mstep : mstep;
        const int t = k * WK + kk;
        const double *pc, *px, *pf;
        slot_ptrs(buf, kk, pc, px, pf);
        const double u = pc[rm.uv() * 32], v = pc[(rm.uv() + 1) * 32];
        const double U1 = u * pf[0] + v * pf[32];
        const double U2 = u * pf[4 * 32] + v * pf[5 * 32];
        const double c1 = a.sp_scale * (U1 + sgn * pf[3 * 32]);
        const double c2 = a.sp_scale * (U2 + sgn * pf[7 * 32]);
        const int col = t - lane;
        const bool rl = real(t);
        const double inv0 = pc[rm.invs() * 32];
#pragma unroll
        for (int c = 0; c < NSB; ++c) {
          if (c < ns) {
            double ijc = BWD ? __shfl_down_sync(FULL, oj[c], 1) : __shfl_up_sync(FULL, oj[c], 1);
            if (first) ijc = hb[kk * nv + 5 + c];
            const double inv = per ? pc[(rm.invs() + c) * 32] : inv0;
            double dq;
            if (BWD) dq = px[(5 + c) * 32] - (oi[c] + ijc) * inv;
            else dq = ((px[(5 + c) * 32] + oi[c]) + ijc) * inv;
            if (!rl) dq = 0.0;
            if (t < T) a.out[gaddr(a.sk, nv, s, t, 5 + c, lane)] = dq;
            oi[c] = c1 * dq;
            oj[c] = c2 * dq;
            if (last && col >= 0 && col < a.ni) hout[(col % HRING) * nv + 5 + c] = oj[c];
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_bar[buf]);
        __threadfence_block();
        *(volatile int*)&done_cnt[1] = ks + 1;
      }
    }
  }
}

// ============================================================== epilogue
template <int NSB>
__global__ void __launch_bounds__(256) k_epilogue2d(const Model* __restrict__ mp, GridDev g, Skew sk,
                                                    int scheme, const double* __restrict__ q,
                                                    const double* __restrict__ dqw,
                                                    double* __restrict__ qn,
                                                    double* __restrict__ dq_std, int C,
                                                    unsigned long long* flags) {
  extern __shared__ double es[];
  const Model& m = *mp;
  const int ns = m.ns, nv = 5 + ns;
  const int ncb = (g.ni + C - 1) / C;
  const int s = blockIdx.x / ncb, ib = blockIdx.x % ncb;
  const int i0 = ib * C, j0 = s * 32;
  const int CT = C * 32;
  const long long N = g.N;
  // phase A: skewed dq -> smem (tile-local column-major)
  const int nt = C + 31;
  for (int e = threadIdx.x; e < nt * 32; e += blockDim.x) {
    const int tt = e / 32, r = e % 32;
    const int ii = tt - r;
    if (ii < 0 || ii >= C || i0 + ii >= g.ni || j0 + r >= g.nj) continue;
    const int t = i0 + ii + r;
    for (int c = 0; c < nv; ++c) es[c * CT + ii * 32 + r] = dqw[gaddr(sk, nv, s, t, c, r)];
  }
  __syncthreads();
  // phase B: closure + gate in standard order (coalesced over j)
  unsigned long long bad_count = 0, first1 = ~0ull, first2 = ~0ull;
  for (int e = threadIdx.x; e < CT; e += blockDim.x) {
    const int ii = e / 32, r = e % 32;
    const int i = i0 + ii, j = j0 + r;
    if (i >= g.ni || j >= g.nj) continue;
    const long long c = (long long)i * g.nj + j;
    double d[5 + NSB];
#pragma unroll
    for (int k = 0; k < 5 + NSB; ++k)
      if (k < nv) d[k] = es[k * CT + e];
    if (dq_std)
      for (int k = 0; k < nv; ++k) dq_std[(long long)k * N + c] = d[k];
    const double* qc = q + c;
    double* qo = qn + c;
#pragma unroll
    for (int k = 0; k < 5; ++k) qo[k * N] = qc[k * N] + d[k];
    bool ok1 = true;
    if (scheme == SCH_CI) {
      double tail = 0.0;
      for (int sp = 0; sp < ns - 1; ++sp) {
        const double v = qc[(5 + sp) * N] + d[5 + sp];
        qo[(5 + sp) * N] = v;
        tail += v;
      }
      const double lastv = qo[0] - tail;
      qo[(4 + ns) * N] = lastv;
      ok1 = !(lastv < -1e-10 * qo[0]);
    } else {
      double rs[NSB], tot = 0.0, dsum = 0.0;
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns) {
          rs[sp] = qc[(5 + sp) * N];
          tot += rs[sp];
          dsum += d[5 + sp];
        }
      double out[NSB], osum = 0.0;
      if (scheme == SCH_CS1) {
        const double defect = d[0] - dsum;
#pragma unroll
        for (int sp = 0; sp < NSB; ++sp)
          if (sp < ns) out[sp] = rs[sp] + d[5 + sp] + (rs[sp] / tot) * defect;
      } else {
        const double rnew = tot + d[0];
        double rawsum = 0.0;
#pragma unroll
        for (int sp = 0; sp < NSB; ++sp)
          if (sp < ns) rawsum += rs[sp] + d[5 + sp];
#pragma unroll
        for (int sp = 0; sp < NSB; ++sp)
          if (sp < ns) out[sp] = rnew * (rs[sp] + d[5 + sp]) / rawsum;
      }
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns) {
          qo[(5 + sp) * N] = out[sp];
          osum += out[sp];
        }
      ok1 = !(osum <= 0.0);
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns && out[sp] < -EPS_NEG * osum) ok1 = false;
    }
    Cell<NSB> cs;
    const bool ok2 = decode<NSB>(m, qn + c, N, cs);
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

// ============================================================== launcher
inline size_t wave_smem(int D, int NC, int NX, int NB, int nv) {
  return ((size_t)D * WK * 32 * (NC + NX + NB) + (size_t)D * WK * nv + (size_t)HRING * nv) *
         sizeof(double);
}

inline int wave_ring_depth(int NC, int nv) {
  const int NX = nv + 8;  // forward is the larger of the two layouts
  for (int D = 6; D >= 2; --D)
    if (wave_smem(D, NC, NX, 0, nv) <= 215 * 1024 && wave_smem(D, NC, nv, 8, nv) <= 215 * 1024)
      return D;
  return 0;
}

cudaError_t CSB_BK(launch_wave_step)(const Model* mp, int ns, const GridDev& g, const WaveBufs& wb,
                                     const double* q, const double* R, double cfl,
                                     const double* lamS, const double* domd, int dom_stride,
                                     int per_species, int scheme, double sp_scale, double* qn,
                                     double* dq_std, unsigned long long* flags, cudaStream_t st,
                                     cudaEvent_t* ev) {
  CSB_NS_DISPATCH(ns, {
    const int nv = 5 + ns, nsI = per_species ? ns : 1;
    const Skew& sk = wb.sk;
    const int NC = 14 + nsI, NF = nv + 8;
    const int D = wave_ring_depth(NC, nv);
    if (D == 0) return cudaErrorInvalidConfiguration;
    // records
    int C = 8;
    auto rsm_of = [&](int c) {
      return ((size_t)(NC + NF + 8) * c * 32 + 7 * (size_t)(c + 2) * 34) * sizeof(double);
    };
    while (C > 1 && rsm_of(C) > 200 * 1024) C /= 2;
    const size_t rsm = rsm_of(C);
    cudaFuncSetAttribute(k_records2d<NSB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
    const int ncb = (g.ni + C - 1) / C;
    if (ev) cudaEventRecord(ev[0], st);
    k_records2d<NSB><<<sk.nstrip * ncb, 256, rsm, st>>>(mp, g, sk, q, R, cfl, lamS, domd,
                                                        dom_stride, per_species, wb.recC, wb.recF,
                                                        wb.recB, C, flags);
    if (ev) cudaEventRecord(ev[1], st);
    // sweeps
    WaveArgs wa;
    wa.sk = sk;
    wa.ni = g.ni;
    wa.nj = g.nj;
    wa.ns = ns;
    wa.nv = nv;
    wa.nsI = nsI;
    wa.nslots = sk.T / WK;
    wa.D = D;
    wa.recC = wb.recC;
    wa.hand = wb.hand;
    wa.prog = wb.prog;
    wa.ticket = wb.prog + sk.nstrip;
    wa.sp_scale = sp_scale;
    const size_t fsm = wave_smem(D, NC, NF, 0, nv), bsm = wave_smem(D, NC, nv, 8, nv);
    cudaFuncSetAttribute(k_wave2d<NSB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
    cudaFuncSetAttribute(k_wave2d<NSB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    cudaMemsetAsync(wb.prog, 0, sizeof(int) * (sk.nstrip + 1), st);
    wa.recX = wb.recF;
    wa.recB = nullptr;
    wa.out = wb.dqs;
    k_wave2d<NSB, false><<<sk.nstrip, 128, fsm, st>>>(wa);
    if (ev) cudaEventRecord(ev[2], st);
    cudaMemsetAsync(wb.prog, 0, sizeof(int) * (sk.nstrip + 1), st);
    wa.recX = wb.dqs;
    wa.recB = wb.recB;
    wa.out = wb.dqw;
    k_wave2d<NSB, true><<<sk.nstrip, 128, bsm, st>>>(wa);
    if (ev) cudaEventRecord(ev[3], st);
    // epilogue
    const int CE = 8;
    const size_t esm = (size_t)nv * CE * 32 * sizeof(double);
    cudaFuncSetAttribute(k_epilogue2d<NSB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm);
    k_epilogue2d<NSB><<<sk.nstrip * ((g.ni + CE - 1) / CE), 256, esm, st>>>(
        mp, g, sk, scheme, q, wb.dqw, qn, dq_std, CE, flags);
    if (ev) cudaEventRecord(ev[4], st);
  });
  return cudaGetLastError();
}

}  // namespace csb
