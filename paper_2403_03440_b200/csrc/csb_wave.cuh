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
// to a multiple of 16).  A run of WK consecutive steps of one strip is one
// contiguous block, so each sweep streams ONE TMA bulk copy per ring slot
// (measured on B200: a CTA's bulk copies complete at ~one request per ~830
// cycles whatever their size up to 64 KiB, scripts/tma_probe.cu).  Slots
// outside the grid (t - r outside [0, ni), rows beyond nj) are padding: their
// records are zero (set once at workspace setup, never written), so padding
// cells carry exactly zero through the chains.
//
// The split (CS) operator decouples the flow and species subsystems inside
// the sweeps (implicit.py:329-403), so every strip runs two independent CTAs:
//   flow    : FF (forward, 30 planes)  invd, w[5], b[5], rhs[5], and per upper
//             face (i, j) a[3] = (-U hr, Sx hr, Sy hr), e[3] = (Sx, Sy, U)/2,
//             sig = (U + lam)/2;
//             FB (backward, 30 planes) invd, w, b, per lower face a, e,
//             sig = (U - lam)/2, dq*[5] (written by the forward chain);
//             FW (5 planes) dq;
//   species : SF (nsI + NSB + 2) invs[nsI], rhs[NSB], c_i, c_j with
//             c = sp_scale (U + lam_sp) at the upper faces;
//             SB (nsI + 2 + NSB) invs, c_i, c_j at the lower faces
//             (sp_scale (U - lam_sp)), dq*[NSB]; SW (NSB planes) dq.
// The half-block products through a face are then (rank-2 form of
// implicit.py:350-380)  sa = a . dq[0:3],  sb = b . dq,
//   o = w sa + e sb + sig dq  (e acting on components 1, 2, 4).
// Each CTA: warp 0 chain (one lane per row; the j-direction contribution goes
// to the next row by warp shuffle), warp 1 producer (TMA ring + the upstream
// strip's hand-off row polled from L2), warp 2 publisher.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

constexpr int HRING = 128;  // hand-off ring (steps)
#ifndef CSB_CHAIN_UNROLL
#define CSB_CHAIN_UNROLL 8
#endif
constexpr int CHAIN_UNROLL = CSB_CHAIN_UNROLL;  // steps of a ring slot unrolled in the chains
// signalling NaN marking a hand-off word not yet written (see the chains)
constexpr unsigned long long HAND_SENTINEL = 0x7FF4DEADBEEF0001ull;
constexpr int NFF = 30, NFB = 30, FB_DQ = 25;
#ifndef CSB_WKF
#define CSB_WKF 8
#endif
#ifndef CSB_DMAX
#define CSB_DMAX 4
#endif
constexpr int WKF = CSB_WKF;  // flow slot: 8 steps x 30 planes = 60 KiB (measured: 4 is slower)

// Coupled (CI, frozen chemistry) records, NV = 5 + NSB components:
//   CF (forward)  invd, hr2, w[NV], b[NV], rhs[NV], upper faces (e[3], sig) x 2
//   CB (backward) invd, hr2, w[NV], b[NV], lower faces (e[3], sig) x 2, dq*[NV]
template <int NSB>
constexpr int ci_planes() { return 3 * (5 + NSB) + 10; }
#ifndef CSB_CI_SLOT_KB
#define CSB_CI_SLOT_KB 100  // measured: 512^2 CI 0.842 -> 0.817 ms against 64 KB (8-step slots at ns = 5)
#endif
// With chemistry (CHEM) the coupled records also carry the species block
// inverse dinv[NSB][NSB] (row-major) after those planes, in CF and CB.
template <int NSB, bool CHEM>
constexpr int ci_ng() { return ci_planes<NSB>() + (CHEM ? NSB * NSB : 0); }
template <int NSB, bool CHEM = false>
constexpr int ci_wk() {
  // (the larger slots only for the register chain: the smem-resident chain
  // above CI_MAXNSB also needs its state next to the ring)
  const int kb = NSB <= 16 ? CSB_CI_SLOT_KB : 64;
  int w = 8;
  while (w > 1 && w * ci_ng<NSB, CHEM>() * 256 > kb * 1024) w /= 2;
  return w;
}
constexpr int CI_MAXNSB = 16;  // register-resident CI chain up to here; smem-resident above

// Species slot length (steps) for the record layout with nsI diagonal planes
// (PER: nsI = NSB, chemistry; else 1): a slot holds <= CSB_SP_SLOT_KB and a
// 2-deep ring plus the hand-off ring (HRING + WK rows of NSB words) fits the
// 210 KiB budget of wave_depth, so every bucket has a valid launch shape
// (checked by static_assert below for every bucket and both layouts).
#ifndef CSB_SP_SLOT_KB
#define CSB_SP_SLOT_KB 100  // measured: 100 KB slots (8 steps up to ns = 24, 2-deep ring) beat 64 KB (4-step slots) by 7-8% at ns = 16-40
#endif
constexpr int WAVE_SMEM_BUDGET = 210 * 1024;
template <int NSB, bool PER>
constexpr int wave_wks() {
  constexpr int NG = (PER ? NSB : 1) + NSB + 2;
  int w = 8;  // also the hand-off granularity (a slot starts when its columns are in)
  while (w > 1 && (w * NG * 256 > CSB_SP_SLOT_KB * 1024 ||
                   2 * w * NG * 256 + (HRING + w) * NSB * 8 > WAVE_SMEM_BUDGET))
    w /= 2;
  return w;
}
template <int NSB, bool PER>
constexpr bool wave_species_fits() {
  constexpr int w = wave_wks<NSB, PER>(), NG = (PER ? NSB : 1) + NSB + 2;
  return 2 * w * NG * 256 + (HRING + w) * NSB * 8 <= WAVE_SMEM_BUDGET && TQ % w == 0 &&
         HRING % w == 0;
}
#define CSB_CHECK_WKS(b) \
  static_assert(wave_species_fits<b, true>() && wave_species_fits<b, false>(), "species ring");
CSB_BUCKET_LIST(CSB_CHECK_WKS)
#undef CSB_CHECK_WKS

// ---------------------------------------------------------------- PTX helpers
CSB_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
CSB_DEV void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
CSB_DEV void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
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
CSB_DEV unsigned long long l2_evict_first() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
CSB_DEV unsigned long long l2_evict_last() {
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Hand-off words (sentinel reset, chain stores, receiver polls) carry an
// L2 evict-last hint and the sweeps' record streams an evict-first one: the
// hand-off buffer (73 MB at config 4) then stays in L2 while the records
// stream through it.  Without the hints the streams evicted the hand-off
// lines, every poll became an HBM round trip under full load, and the
// receiver (one poll in flight) set the pace of every strip with an upstream
// strip (config 4: species strips 119 -> ~250 ns per step once ~25 strips ran;
// sweeps 1.42 + 1.50 -> 1.23 + 1.25 ms).
CSB_DEV void st_hand(double* p, double v) {
#ifndef CSB_HAND_NORMAL
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(l2_evict_last())
               : "memory");
#else
  *p = v;
#endif
}
CSB_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
#ifndef CSB_TMA_NORMAL
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(l2_evict_first())
      : "memory");
#else
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
#endif
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
// 8-byte asynchronous global -> shared copies (records staging, epilogue gather)
CSB_DEV void cp_async8(double* dst_smem, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src)
               : "memory");
}
CSB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
CSB_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}

// step-major group address of (strip s, step t, plane p, row r)
CSB_DEV long long gaddr(const Skew& k, int NG, int s, int t, int p, int r) {
  return (((long long)s * k.T + t) * NG + p) * 32 + r;
}

static __global__ void k_epoch_bump(int* e) { *e += 1; }

// ============================================================== hand-off reset
// Both sweeps' strip hand-off rows: signalling-NaN sentinel in the data rows,
// zero in the HPAD pad rows (one thread per row).
static __global__ void k_hand_reset(double* __restrict__ hand, int nstrip, int T, int nhf, int nhs,
                                    long long N, const double* __restrict__ q3,
                                    const double* __restrict__ R3, int* flag, const int* epoch_p) {
  const int epoch = *epoch_p;
  // planarity of the step (chain_flow PL): epoch stored when any cell has a
  // nonzero (or non-finite) z-momentum q3 or z-momentum residual R3
  {
    bool bad = false;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N;
         c += (long long)gridDim.x * blockDim.x)
      bad |= !(q3[c] == 0.0) || !(R3[c] == 0.0);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = epoch;
  }
  const int rows = T + 2 * HPAD;
  const long long nrow = 2LL * 2 * nstrip * rows;  // [sweep][role][strip][row]
  const double sent = __longlong_as_double((long long)HAND_SENTINEL);
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < nrow;
       l += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(l % rows);
    const long long sr = l / rows;                 // [sweep][role][strip]
    const int strip = (int)(sr % nstrip);
    const int role = (int)((sr / nstrip) % 2);
    const int sweep = (int)(sr / (2LL * nstrip));
    const long long per_sweep = (long long)nstrip * rows * (nhf + nhs);
    const int nh = role ? nhs : nhf;
    double* p = hand + sweep * per_sweep + (role ? (long long)nstrip * rows * nhf : 0) +
                ((long long)strip * rows + r) * nh;
    const double v = (r < HPAD || r >= rows - HPAD) ? 0.0 : sent;
    for (int c = 0; c < nh; ++c) st_hand(p + c, v);
  }
}

// records tile (strip s, step block ib) stored: publish the launch epoch
CSB_DEV void publish_tile(const WaveBufs& wb, int s, int ib) {
  if (!wb.rdy) return;  // serial order: no concurrent forward sweep reads the flags
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(wb.rdy + (long long)s * wb.sk.T + ib),
                 "r"(*wb.epoch)
                 : "memory");
  }
}

// ============================================================== records
// Tile = one strip (32 rows) x C wavefront steps, i.e. a parallelogram in
// (i, j): element (tt, r) is cell (i = t0 + tt - r, j = j0 + r).  In these
// skew coordinates the face neighbours of (tt, r) are (tt +- 1, r) in i and
// (tt +- 1, r +- 1) in j, so a 1-element halo in tt and r covers them.  A warp
// handles one step (32 rows), so every record store is one contiguous 256-byte
// row of the step-major layout; the strided q/R loads hit L1 (the four cells
// of a 32-byte sector are (tt..tt+3, r..r+3), all in the same tile).
// Phase A: per cell of tile + halo decode + transport (face quantities);
// interior cells also get dtau, the diagonals, the Jacobian ingredients and
// -R.  Phase B: per interior cell, face radii (max of the two adjacent cells
// at the face metric), face coefficients, and all record stores.
template <int NSB, bool CI>
// (measured: 4 CTAs/SM for small species counts; above, 3 CTAs/SM with 80
// registers removes the spills: ns = 11 records 493 -> 400 us at 1024^2)
__global__ void __launch_bounds__(256, NSB <= 8 ? 4 : 3) k_records2d(const Model* __restrict__ mp, GridDev g, Skew sk,
                                                   const double* __restrict__ q,
                                                   const double* __restrict__ R, const double* __restrict__ cfl_p,
                                                   const double* __restrict__ lamS,
                                                   const double* __restrict__ domd, int dom_stride,
                                                   int per_species, double sp_scale, WaveBufs wb,
                                                   int C, unsigned long long* flags) {
  extern __shared__ double sm[];
  const Model& m = *mp;
  const int ns = m.ns, nsI = per_species ? NSB : 1;  // species-diagonal planes
  const int NSF = nsI + NSB + 2;  // = SB group planes
  const int ncb = sk.T / C;
  // tiles in step-block-major order: the concurrently running forward sweep
  // consumes every strip's first columns first
  const int s = blockIdx.x % sk.nstrip, ib = blockIdx.x / sk.nstrip;
  const int t0 = ib * C, j0 = s * 32;
  const int HX = C + 2, HY = 34, NH = HX * HY;
  const int CT = C * 32;
  constexpr int NV = 5 + NSB;
  // cell planes: CS invd w b rhs | invs rhs_s;  CI invd hr2 w[NV] b[NV] rhs[NV]
  const int NCP = CI ? 2 + 3 * NV : 16 + nsI + NSB;
  double* A = sm;                              // [12][NH]: u, v, w, c, nf, nsp, V, hr,
                                               //   lower-i face Sx Sy, lower-j face Sx Sy
  double* TC = sm + 12 * NH;                   // [NCP][CT]
  const long long N = g.N;
  // ---------------- phase A: halo-extended per-cell quantities.  Enumerated
  // column by column (fixed i, consecutive j) so that the loads of a warp are
  // contiguous runs of up to C + 2 cells: i' = tt - r in [-33, C + 1],
  // r in [max(-1, -1 - i'), min(32, C - i')].
  const int CW = C + 2;
  for (int l = threadIdx.x; l < (C + 35) * CW; l += blockDim.x) {
    const int ip = -33 + l / CW;
    const int r = max(-1, -1 - ip) + l % CW;
    if (r > min(32, C - ip)) continue;
    const int tt = ip + r;
    const int hl = (tt + 1) * HY + (r + 1);
    const int i = t0 + ip, j = j0 + r;
    if (i < 0 || j < 0 || i > g.ni || j > g.nj) continue;
    // lower faces of (i, j) (these include the upper boundary faces i = ni, j = nj)
    if (j < g.nj) {
      const long long f = face_index(g, 0, i, j, 0);
      A[8 * NH + hl] = __ldg(g.S[0] + f);
      A[9 * NH + hl] = __ldg(g.S[0] + g.NF[0] + f);
    }
    if (i < g.ni) {
      const long long f = face_index(g, 1, i, j, 0);
      A[10 * NH + hl] = __ldg(g.S[1] + f);
      A[11 * NH + hl] = __ldg(g.S[1] + g.NF[1] + f);
    }
    if (i >= g.ni || j >= g.nj) continue;
    const long long c = (long long)i * g.nj + j;
    Cell<NSB> cs;
    const bool ok = decode<NSB>(m, q + c, N, cs);
    double mu, kc, D, nf, nsp, nu;
    transport<NSB>(m, cs.T, cs.Y, cs.rho, mu, kc, D);
    diffusivities(mu, kc, D, cs.rho, cs.cp - cs.R, nf, nsp, nu);
    const double V = __ldg(g.vol + c);
    A[0 * NH + hl] = cs.u[0];
    A[1 * NH + hl] = cs.u[1];
    A[2 * NH + hl] = cs.u[2];
    A[3 * NH + hl] = cs.c;
    A[4 * NH + hl] = nf;
    A[5 * NH + hl] = nsp;
    A[6 * NH + hl] = inv_volume(g, c);  // 1 / V (face radii multiply)
    A[7 * NH + hl] = 0.5 / cs.rho;
    const bool inner = tt >= 0 && tt < C && r >= 0 && r < 32;
    if (!inner) continue;
    if (!ok) raise_flag(flags, EB_DECODE, c);
    const int e = tt * 32 + r;  // tile element (tt, r)
    // cell radii at the cell-averaged metric, dtau (implicit.py:152-163, 33-44)
    double li[3], lv[3], rf = 0.0, rsp = 0.0;
    const double iV = inv_volume(g, c);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double Sc[3], a2, sq;
      cell_metric(g, c, i, j, 0, d, Sc, a2, sq);
      const double U = fabs(cs.u[0] * Sc[0] + cs.u[1] * Sc[1] + cs.u[2] * Sc[2]);
      li[d] = U + cs.c * sq;
      lv[d] = nu * a2 * iV;
      const double lf = (U + cs.c * sq) + 2.0 * nf * a2 * iV;
      const double ls = U + 2.0 * nsp * a2 * iV;
      rf = d == 0 ? lf : rf + lf;
      rsp = d == 0 ? ls : rsp + ls;
    }
    const double J = iV;
    const double den = J * (((li[0] + li[1]) + li[2]) + ((lv[0] + lv[1]) + lv[2])) +
                       (lamS ? lamS[c] : 0.0);
    if (!(den > 0.0)) raise_flag(flags, EB_ZERO_WAVE, c);
    const double dtau = *cfl_p / den;
    const double base = V / dtau;
    if constexpr (CI) {
      // CI: one scalar diagonal with the unified radius (implicit.py:362-373)
      double rci = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double Sc[3], a2, sq;
        cell_metric(g, c, i, j, 0, d, Sc, a2, sq);
        const double U = fabs(cs.u[0] * Sc[0] + cs.u[1] * Sc[1] + cs.u[2] * Sc[2]);
        const double lu = (U + cs.c * sq) + 2.0 * nu * a2 * iV;
        rci = d == 0 ? lu : rci + lu;
      }
      const double dci = base + rci;
      if (!(fabs(dci) >= 1e-300) || !isfinite(dci)) raise_flag(flags, EB_SINGULAR, c);
      if (per_species && wb.ci_d) wb.ci_d[c] = dci;  // chemistry: the block inverse needs d
      const double beta = cs.gamma - 1.0;
      TC[0 * CT + e] = 1.0 / dci;
      TC[1 * CT + e] = 1.0 / cs.rho;
      double* tw = TC + 2 * CT;
      double* tb = TC + (2 + NV) * CT;
      double* tr = TC + (2 + 2 * NV) * CT;
      tw[0 * CT + e] = cs.rho;
      tw[1 * CT + e] = cs.rho * cs.u[0];
      tw[2 * CT + e] = cs.rho * cs.u[1];
      tw[3 * CT + e] = cs.rho * cs.u[2];
      tw[4 * CT + e] = cs.rho * cs.h;
      tb[0 * CT + e] = beta * cs.Ek;
      tb[1 * CT + e] = -beta * cs.u[0];
      tb[2 * CT + e] = -beta * cs.u[1];
      tb[3 * CT + e] = -beta * cs.u[2];
      tb[4 * CT + e] = beta;
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp) {
        // _w_column / _grad_p_row species entries (implicit.py:59-81)
        const bool real = sp < ns;
        const double RsT = real ? m.Rs[sp] * cs.T : 0.0;
        const double hs = real ? m.bs[sp] + m.cp[sp] * cs.T : 0.0;
        tw[(5 + sp) * CT + e] = real ? cs.rho * cs.Y[sp] : 0.0;
        tb[(5 + sp) * CT + e] = real ? RsT - beta * (hs - RsT) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < NV; ++k)
        tr[k * CT + e] = k < 5 + ns ? -R[(long long)k * N + c] : 0.0;
      continue;
    }
    const double dflow = base + rf;
    bool bad = !(fabs(dflow) >= 1e-300) || !isfinite(dflow);
    const double dsp0 = base + rsp;
    double* ts = TC + 16 * CT;
    if (per_species) {
      for (int sp = 0; sp < ns; ++sp) {
        const double v = dsp0 - domd[(long long)sp * dom_stride * N + c] * V;
        bad |= !(fabs(v) >= 1e-300) || !isfinite(v);
        ts[sp * CT + e] = 1.0 / v;
      }
      for (int sp = ns; sp < NSB; ++sp) ts[sp * CT + e] = 0.0;  // padding species
    } else {
      bad |= !(fabs(dsp0) >= 1e-300) || !isfinite(dsp0);
      ts[0 * CT + e] = 1.0 / dsp0;
    }
    if (bad) raise_flag(flags, EB_SINGULAR, c);
#pragma unroll
    for (int k = 0; k < NSB; ++k)
      ts[(nsI + k) * CT + e] = k < ns ? -R[(long long)(5 + k) * N + c] : 0.0;
    for (int k = 0; k < 5; ++k) TC[(11 + k) * CT + e] = -R[(long long)k * N + c];
    const double beta = cs.gamma - 1.0;
    TC[0 * CT + e] = 1.0 / dflow;
    TC[1 * CT + e] = cs.rho;
    TC[2 * CT + e] = cs.rho * cs.u[0];
    TC[3 * CT + e] = cs.rho * cs.u[1];
    TC[4 * CT + e] = cs.rho * cs.u[2];
    TC[5 * CT + e] = cs.rho * cs.h;
    TC[6 * CT + e] = beta * cs.Ek;
    TC[7 * CT + e] = -beta * cs.u[0];
    TC[8 * CT + e] = -beta * cs.u[1];
    TC[9 * CT + e] = -beta * cs.u[2];
    TC[10 * CT + e] = beta;
  }
  __syncthreads();
  // ---------------- phase B: faces + all record stores, one cell per thread
  for (int e = threadIdx.x; e < CT; e += blockDim.x) {
    const int tt = e / 32, r = e % 32;
    const int t = t0 + tt;
    const int i = t - r, j = j0 + r;
    // cells outside the grid are padding slots: zeroed once at workspace
    // setup, never written
    if (i < 0 || i >= g.ni || j >= g.nj) continue;
    const int hc = (tt + 1) * HY + (r + 1);
    const double u = A[0 * NH + hc], v = A[1 * NH + hc], hr = A[7 * NH + hc];
    if constexpr (CI) {
      const int NG = per_species ? ci_ng<NSB, true>() : ci_ng<NSB, false>();
      double* cf = wb.ff + gaddr(sk, NG, s, t, 0, r);
      double* cb = wb.fb + gaddr(sk, NG, s, t, 0, r);
      for (int p = 0; p < 2 + 2 * NV; ++p) {
        const double xv = TC[p * CT + e];
        cf[p * 32] = xv;
        cb[p * 32] = xv;
      }
      for (int p = 2 + 2 * NV; p < 2 + 3 * NV; ++p) cf[p * 32] = TC[p * CT + e];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const int d = f & 1;
        const bool upper = f < 2;
        const int hf = upper ? (d == 0 ? hc + HY : hc + HY + 1) : hc;
        double S[3];
        S[0] = A[(8 + 2 * d) * NH + hf];
        S[1] = A[(9 + 2 * d) * NH + hf];
        S[2] = 0.0;
        const double a2 = (S[0] * S[0] + S[1] * S[1]) + S[2] * S[2];
        const double ar = sqrt(a2);
        const int nb = upper ? (d == 0 ? hc + HY : hc + HY + 1) : (d == 0 ? hc - HY : hc - HY - 1);
        const bool nb_in = upper ? (d == 0 ? i + 1 < g.ni : j + 1 < g.nj) : (d == 0 ? i > 0 : j > 0);
        const int lo = upper ? hc : nb, hi = upper ? nb : hc;
        // unified face radius (implicit.py:176-197 with nu = max(nu_flow, nu_sp))
        auto lam = [&](int h) {
          const double Uh = fabs(A[0 * NH + h] * S[0] + A[1 * NH + h] * S[1] + A[2 * NH + h] * S[2]);
          const double nuh = npmax(A[4 * NH + h], A[5 * NH + h]);
          return (Uh + A[3 * NH + h] * ar) + 2.0 * nuh * a2 * A[6 * NH + h];
        };
        const double lu = nb_in ? npmax(lam(lo), lam(hi)) : lam(hc);
        const double U = u * S[0] + v * S[1];
        double* fd = upper ? cf + (2 + 3 * NV + 4 * d) * 32 : cb + (2 + 2 * NV + 4 * d) * 32;
        fd[0 * 32] = 0.5 * S[0];
        fd[1 * 32] = 0.5 * S[1];
        fd[2 * 32] = 0.5 * U;
        fd[3 * 32] = 0.5 * (U + (upper ? lu : -lu));
      }
      continue;
    }
    double* ff = wb.ff + gaddr(sk, NFF, s, t, 0, r);
    double* fb = wb.fb + gaddr(sk, NFB, s, t, 0, r);
    double* sf = wb.sf + gaddr(sk, NSF, s, t, 0, r);
    double* sb = wb.sb + gaddr(sk, NSF, s, t, 0, r);
    for (int p = 0; p < 11; ++p) {
      const double x = TC[p * CT + e];
      ff[p * 32] = x;
      fb[p * 32] = x;
    }
    for (int p = 11; p < 16; ++p) ff[p * 32] = TC[p * CT + e];
    for (int p = 0; p < nsI; ++p) {
      const double x = TC[(16 + p) * CT + e];
      sf[p * 32] = x;
      sb[p * 32] = x;
    }
#pragma unroll
    for (int p = 0; p < NSB; ++p) sf[(nsI + p) * 32] = TC[(16 + nsI + p) * CT + e];
    // faces: 0 upper-i (i+1), 1 upper-j (j+1), 2 lower-i (i), 3 lower-j (j)
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int d = f & 1;
      const bool upper = f < 2;
      // face metric from the halo: upper-i = lower-i face of (tt+1, r),
      // upper-j = lower-j face of (tt+1, r+1); S_z = 0 on i/j faces of a
      // 2-D grid (csb_implicit.cu k_check_2d)
      const int hf = upper ? (d == 0 ? hc + HY : hc + HY + 1) : hc;
      double S[3];
      S[0] = A[(8 + 2 * d) * NH + hf];
      S[1] = A[(9 + 2 * d) * NH + hf];
      S[2] = 0.0;
      const double a2 = (S[0] * S[0] + S[1] * S[1]) + S[2] * S[2];
      const double ar = sqrt(a2);
      // neighbour across the face, in skew coordinates
      const int nb = upper ? (d == 0 ? hc + HY : hc + HY + 1) : (d == 0 ? hc - HY : hc - HY - 1);
      const bool nb_in = upper ? (d == 0 ? i + 1 < g.ni : j + 1 < g.nj) : (d == 0 ? i > 0 : j > 0);
      const int lo = upper ? hc : nb, hi = upper ? nb : hc;  // lower/upper cell of the face
      auto lam = [&](int h, bool sp) {
        const double U = fabs(A[0 * NH + h] * S[0] + A[1 * NH + h] * S[1] + A[2 * NH + h] * S[2]);
        if (sp) return U + 2.0 * A[5 * NH + h] * a2 * A[6 * NH + h];
        return (U + A[3 * NH + h] * ar) + 2.0 * A[4 * NH + h] * a2 * A[6 * NH + h];
      };
      double lf, ls;
      if (nb_in) {
        lf = npmax(lam(lo, false), lam(hi, false));
        ls = npmax(lam(lo, true), lam(hi, true));
      } else {
        lf = lam(hc, false);
        ls = lam(hc, true);
      }
      const double sgn_lf = upper ? lf : -lf, sgn_ls = upper ? ls : -ls;
      const double U = u * S[0] + v * S[1];
      double* fd = upper ? ff + (16 + 7 * d) * 32 : fb + (11 + 7 * d) * 32;
      fd[0 * 32] = -U * hr;
      fd[1 * 32] = S[0] * hr;
      fd[2 * 32] = S[1] * hr;
      fd[3 * 32] = 0.5 * S[0];
      fd[4 * 32] = 0.5 * S[1];
      fd[5 * 32] = 0.5 * U;
      fd[6 * 32] = 0.5 * (U + sgn_lf);
      const double csp = sp_scale * (U + sgn_ls);
      if (upper) sf[(nsI + NSB + d) * 32] = csp;
      else sb[(nsI + d) * 32] = csp;
    }
  }
  publish_tile(wb, s, ib);
}

// ============================================================== records, sliding window
// The CS records of the serial launch order (no concurrent forward sweep).
// A persistent CTA walks along one strip in blocks of C wavefront steps and
// keeps the per-cell quantities of the last C + 2 steps in shared-memory rings
// indexed by step, so every cell is decoded once per strip it touches (34 / 32
// of the cells) instead of once per tile halo ((C + 2) x 34 / (C x 32) = 1.6
// at the 4-step tiles of k_records2d), and the natural-layout loads come in
// runs of C consecutive rows of one grid column (k_records2d: runs of C + 2 on
// a 4-step tile; measured at config 4: 10.8 GB through L2 for 2.7 GB of
// input).
//   phase A (item = cell of steps t0 + 1 .. t0 + C, rows -1 .. 32): decode +
//     transport into the A ring (what the face radii of the neighbours need);
//     the pass-through inputs of the cell itself (-R, V, S_k, lam_S, dOmega
//     diagonal) and the face vectors go to shared memory by cp.async.
//   phase B (warp = step t0 .. t0 + C - 1, lane = row): local time step,
//     diagonals, the four faces, and all record stores (256-byte rows).
// Work unit = (chunk of L steps, strip), chunks outermost, so the strips of a
// chunk run side by side (their halo rows hit L2).
#ifndef CSB_REC_QFIRST
#define CSB_REC_QFIRST 1  // measured at config 4: records 2.51 -> 2.28 ms (ns = 40: 1.34 -> 1.55, so up to 16 species)
#endif
#ifndef CSB_REC_RB
#define CSB_REC_RB 8  // pass-through loads in flight per batch
#endif
template <int C>
constexpr int rec_s_threads() { return (34 * C + 31) / 32 * 32; }
constexpr int REC_S_NA = 11;  // A ring planes: u v w c nf nsp 1/V | lower-i Sx Sy, lower-j Sx Sy
// T ring planes (cell itself): rho h beta hr V Sz | -R source [5 + NSB] | lamS |
// CS with chemistry: dOmega diag [NSB];  CI: T, rho Y [NSB]
template <int NSB>
constexpr int rec_s_ntp(bool per_species, bool ci = false) {
  return 6 + 5 + NSB + 1 + (ci ? 1 + NSB : (per_species ? NSB : 0));
}
template <int NSB, int C>
constexpr size_t rec_s_smem(bool per_species, bool ci = false) {
  return ((size_t)REC_S_NA * (C + 2) * 34 + (size_t)rec_s_ntp<NSB>(per_species, ci) * (C + 1) * 32) *
         sizeof(double);
}

template <int NSB, int C, bool CI>
__global__ void __launch_bounds__(rec_s_threads<C>(), C >= 16 ? 1 : (C >= 8 ? 2 : 4))
    k_records2d_s(const Model* __restrict__ mp, GridDev g, Skew sk, const double* __restrict__ q,
                  const double* __restrict__ R, const double* __restrict__ cfl_p,
                  const double* __restrict__ lamS, const double* __restrict__ domd, int dom_stride,
                  int per_species, double sp_scale, WaveBufs wb, int L, unsigned long long* flags) {
  extern __shared__ double sm[];
  const Model& m = *mp;
  const int ns = m.ns, nv = 5 + ns;
  const int nsI = per_species ? NSB : 1;
  const int NSF = nsI + NSB + 2;
  constexpr int RA = C + 2, RT = C + 1, HY = 34;
  constexpr int SA = RA * HY, ST = RT * 32;  // plane strides of the rings
  double* A = sm;
  double* TP = sm + REC_S_NA * SA;
  constexpr int T_RHS = 6, T_LAMS = 6 + 5 + NSB, T_DOM = T_LAMS + 1;
  constexpr int T_TEMP = T_LAMS + 1, T_RY = T_TEMP + 1;  // CI
  constexpr int NV = 5 + NSB;
  const long long N = g.N;
  const double cfl = *cfl_p;
  const int nchunk = (sk.T + L - 1) / L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto slot_a = [](int step) { return (step + 1) % RA; };  // step >= -1
  auto slot_t = [](int step) { return step % RT; };

  for (int unit = blockIdx.x; unit < nchunk * sk.nstrip; unit += gridDim.x) {
    const int s = unit % sk.nstrip, tb = (unit / sk.nstrip) * L, te = min(tb + L, sk.T);
    const int j0 = s * 32;
    // ---------------- phase A: n steps from tf
    auto phase_a = [&](int tf, int n, int tin) {  // T ring (cell itself) from step tin on
      const int l = threadIdx.x;
      if (l >= 34 * C) return;
      const int rr = l % 34, tt = (l / 34 + rr) % C;  // a run of C lanes shares one grid column
      if (tt >= n) return;
      const int step = tf + tt, r = rr - 1;
      const int i = step - r, j = j0 + r;
      if (i < 0 || j < 0 || i > g.ni || j > g.nj) return;
      double* a = A + slot_a(step) * HY + rr;
      if (j < g.nj) {  // lower-i face (includes the boundary face i = ni)
        const long long f = face_index(g, 0, i, j, 0);
        a[7 * SA] = __ldg(g.S[0] + f);
        a[8 * SA] = __ldg(g.S[0] + g.NF[0] + f);
      }
      if (i < g.ni) {  // lower-j face (includes j = nj)
        const long long f = face_index(g, 1, i, j, 0);
        a[9 * SA] = __ldg(g.S[1] + f);
        a[10 * SA] = __ldg(g.S[1] + g.NF[1] + f);
      }
      if (i >= g.ni || j >= g.nj) return;
      const long long c = (long long)i * g.nj + j;
      const bool inner = r >= 0 && r < 32 && step >= tin;
      double* tp = TP + slot_t(inner ? step : 0) * 32 + (inner ? r : 0);
      constexpr bool QF = CSB_REC_QFIRST && NSB <= 16;
#if CSB_REC_QFIRST
      // the decode's loads first: in flight while the pass-through inputs
      // are copied
      double qv[QF ? 5 + NSB : 1];
      if constexpr (QF) {
#pragma unroll
        for (int k = 0; k < 5 + NSB; ++k) qv[k] = k < nv ? __ldg(q + c + (long long)k * N) : 0.0;
      }
#endif
      if (inner) {
        // (plain loads: a warp's 8-byte cp.async requests reach L2 one sector
        // per lane, measured 291 M L2 read sectors for 157 M requested)
        tp[5 * ST] = __ldg(g.S[2] + 2 * g.NF[2] + 2 * c);  // k-face z component (nk == 1)
#pragma unroll
        for (int k0 = 0; k0 < 5 + NSB; k0 += CSB_REC_RB) {
          double rv[CSB_REC_RB];
#pragma unroll
          for (int k = 0; k < CSB_REC_RB; ++k)
            rv[k] = k0 + k < nv ? __ldg(R + (long long)(k0 + k) * N + c) : 0.0;
#pragma unroll
          for (int k = 0; k < CSB_REC_RB; ++k)
            if (k0 + k < 5 + NSB) tp[(T_RHS + k0 + k) * ST] = rv[k];
        }
        if (lamS) tp[T_LAMS * ST] = lamS[c];
        if (!CI && per_species)
          for (int sp = 0; sp < ns; ++sp)
            tp[(T_DOM + sp) * ST] = domd[(long long)sp * dom_stride * N + c];
      }
      Cell<NSB> cs;
#if CSB_REC_QFIRST
      const bool ok = QF ? decode_from<NSB>(m, [&](int kq) { return qv[QF ? kq : 0]; }, cs)
                         : decode_from<NSB>(m, [&](int kq) { return __ldg(q + c + kq * N); }, cs);
#else
      const bool ok = decode_from<NSB>(m, [&](int kq) { return __ldg(q + c + kq * N); }, cs);
#endif
      double mu, kc, D, nf, nsp, nu;
      transport<NSB>(m, cs.T, cs.Y, cs.rho, mu, kc, D);
      diffusivities(mu, kc, D, cs.rho, cs.cp - cs.R, nf, nsp, nu);
      a[0 * SA] = cs.u[0];
      a[1 * SA] = cs.u[1];
      a[2 * SA] = cs.u[2];
      a[3 * SA] = cs.c;
      a[4 * SA] = nf;
      a[5 * SA] = nsp;
      const double V = __ldg(g.vol + c);
      a[6 * SA] = 1.0 / V;
      if (inner) {
        if (!ok) raise_flag(flags, EB_DECODE, c);
        tp[4 * ST] = V;
        tp[0 * ST] = cs.rho;
        tp[1 * ST] = cs.h;
        tp[2 * ST] = cs.gamma - 1.0;
        tp[3 * ST] = CI ? 1.0 / cs.rho : 0.5 / cs.rho;
        if constexpr (CI) {
          tp[T_TEMP * ST] = cs.T;
#pragma unroll
          for (int sp = 0; sp < NSB; ++sp) tp[(T_RY + sp) * ST] = sp < ns ? cs.rho * cs.Y[sp] : 0.0;
        }
      }
    };
    // ---------------- phase B: step t0 + warp, row = lane
    auto phase_b = [&](int t0) {
      if (warp >= C) return;
      const int t = t0 + warp, r = lane;
      const int i = t - r, j = j0 + r;
      // cells outside the grid are padding slots: zeroed once at workspace
      // setup, never written
      if (i < 0 || i >= g.ni || j >= g.nj) return;
      const long long c = (long long)i * g.nj + j;
      const int hc = slot_a(t) * HY + r + 1;
      const int up = slot_a(t + 1) * HY + r + 1;  // (i + 1, j); (i, j + 1) at up + 1
      const int lo = slot_a(t - 1) * HY + r + 1;  // (i - 1, j); (i, j - 1) at lo - 1
      const double* tp = TP + slot_t(t) * 32 + r;
      const double u = A[0 * SA + hc], v = A[1 * SA + hc], w = A[2 * SA + hc], cc = A[3 * SA + hc];
      const double nf = A[4 * SA + hc], nsp = A[5 * SA + hc], iV = A[6 * SA + hc];
      const double rho = tp[0 * ST], h = tp[1 * ST], beta = tp[2 * ST], hr = tp[3 * ST];
      const double V = tp[4 * ST], Sz = tp[5 * ST];
      const double nu = npmax(nf, nsp);
      // cell radii at the cell-averaged metric, dtau (implicit.py:152-163, 33-44)
      double li[3], lv[3], rf = 0.0, rsp = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double U, a2, sq;
        if (d < 2) {
          const int hu = d == 0 ? up : up + 1;
          const double s0 = 0.5 * (A[(7 + 2 * d) * SA + hc] + A[(7 + 2 * d) * SA + hu]);
          const double s1 = 0.5 * (A[(8 + 2 * d) * SA + hc] + A[(8 + 2 * d) * SA + hu]);
          U = fabs(u * s0 + v * s1);
          a2 = s0 * s0 + s1 * s1;
          sq = sqrt(a2);
        } else {
          U = fabs(w * Sz);
          a2 = Sz * Sz;
          sq = fabs(Sz);
        }
        li[d] = U + cc * sq;
        lv[d] = nu * a2 * iV;
        const double lf = (U + cc * sq) + 2.0 * nf * a2 * iV;
        const double ls = U + 2.0 * nsp * a2 * iV;
        rf = d == 0 ? lf : rf + lf;
        rsp = d == 0 ? ls : rsp + ls;
      }
      const double den = iV * (((li[0] + li[1]) + li[2]) + ((lv[0] + lv[1]) + lv[2])) +
                         (lamS ? tp[T_LAMS * ST] : 0.0);
      if (!(den > 0.0)) raise_flag(flags, EB_ZERO_WAVE, c);
      const double dtau = cfl / den;
      const double base = V / dtau;
      if constexpr (CI) {
        // one scalar diagonal with the unified radius (implicit.py:362-373)
        double rci = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          // (U + c |Sc|) + 2 nu a2 / V from the terms formed above
          rci = d == 0 ? li[d] + 2.0 * lv[d] : rci + (li[d] + 2.0 * lv[d]);
        }
        const double dci = base + rci;
        if (!(fabs(dci) >= 1e-300) || !isfinite(dci)) raise_flag(flags, EB_SINGULAR, c);
        if (per_species && wb.ci_d) wb.ci_d[c] = dci;  // chemistry: the block inverse needs d
        const int NGc = per_species ? ci_ng<NSB, true>() : ci_ng<NSB, false>();
        double* cf = wb.ff + gaddr(sk, NGc, s, t, 0, r);
        double* cb = wb.fb + gaddr(sk, NGc, s, t, 0, r);
        const double Ek = 0.5 * ((u * u + v * v) + w * w);
        const double Tc = tp[T_TEMP * ST];
        auto both = [&](int p, double x) {
          __stcs(&cf[p * 32], x);
          __stcs(&cb[p * 32], x);
        };
        both(0, 1.0 / dci);
        both(1, hr);  // 1 / rho
        both(2, rho);
        both(3, rho * u);
        both(4, rho * v);
        both(5, rho * w);
        both(6, rho * h);
        both(2 + NV + 0, beta * Ek);
        both(2 + NV + 1, -beta * u);
        both(2 + NV + 2, -beta * v);
        both(2 + NV + 3, -beta * w);
        both(2 + NV + 4, beta);
#pragma unroll
        for (int sp = 0; sp < NSB; ++sp) {
          // _w_column / _grad_p_row species entries (implicit.py:59-81)
          const bool real = sp < ns;
          const double RsT = real ? m.Rs[sp] * Tc : 0.0;
          const double hs = real ? m.bs[sp] + m.cp[sp] * Tc : 0.0;
          both(2 + 5 + sp, tp[(T_RY + sp) * ST]);
          both(2 + NV + 5 + sp, real ? RsT - beta * (hs - RsT) : 0.0);
        }
#pragma unroll
        for (int k = 0; k < NV; ++k)
          __stcs(&cf[(2 + 2 * NV + k) * 32], k < nv ? -tp[(T_RHS + k) * ST] : 0.0);
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int d = f & 1;
          const bool upper = f < 2;
          const int nb = upper ? (d == 0 ? up : up + 1) : (d == 0 ? lo : lo - 1);
          const int hf = upper ? nb : hc;
          const double S0 = A[(7 + 2 * d) * SA + hf], S1 = A[(8 + 2 * d) * SA + hf];
          const double a2 = S0 * S0 + S1 * S1;
          const double ar = sqrt(a2);
          const bool nb_in = upper ? (d == 0 ? i + 1 < g.ni : j + 1 < g.nj) : (d == 0 ? i > 0 : j > 0);
          // unified face radius (implicit.py:176-197 with nu = max(nu_flow, nu_sp))
          auto lam = [&](int hh) {
            const double Uh = fabs(A[0 * SA + hh] * S0 + A[1 * SA + hh] * S1);
            const double nuh = npmax(A[4 * SA + hh], A[5 * SA + hh]);
            return (Uh + A[3 * SA + hh] * ar) + 2.0 * nuh * a2 * A[6 * SA + hh];
          };
          double lu = lam(hc);
          if (nb_in) lu = npmax(lu, lam(nb));
          const double U = u * S0 + v * S1;
          double* fd = upper ? cf + (2 + 3 * NV + 4 * d) * 32 : cb + (2 + 2 * NV + 4 * d) * 32;
          __stcs(&fd[0 * 32], 0.5 * S0);
          __stcs(&fd[1 * 32], 0.5 * S1);
          __stcs(&fd[2 * 32], 0.5 * U);
          __stcs(&fd[3 * 32], 0.5 * (U + (upper ? lu : -lu)));
        }
        return;
      }
      const double dflow = base + rf;
      bool bad = !(fabs(dflow) >= 1e-300) || !isfinite(dflow);
      const double dsp0 = base + rsp;
      double* ff = wb.ff + gaddr(sk, NFF, s, t, 0, r);
      double* fb = wb.fb + gaddr(sk, NFB, s, t, 0, r);
      double* sf = wb.sf + gaddr(sk, NSF, s, t, 0, r);
      double* sb = wb.sb + gaddr(sk, NSF, s, t, 0, r);
      if (per_species) {
        for (int sp = 0; sp < ns; ++sp) {
          const double x = dsp0 - tp[(T_DOM + sp) * ST] * V;
          bad |= !(fabs(x) >= 1e-300) || !isfinite(x);
          const double ix = 1.0 / x;
          __stcs(&sf[sp * 32], ix);
          __stcs(&sb[sp * 32], ix);
        }
        for (int sp = ns; sp < NSB; ++sp) {  // padding species
          __stcs(&sf[sp * 32], 0.0);
          __stcs(&sb[sp * 32], 0.0);
        }
      } else {
        bad |= !(fabs(dsp0) >= 1e-300) || !isfinite(dsp0);
        const double ix = 1.0 / dsp0;
        __stcs(&sf[0], ix);
        __stcs(&sb[0], ix);
      }
      if (bad) raise_flag(flags, EB_SINGULAR, c);
#pragma unroll
      for (int k = 0; k < NSB; ++k) __stcs(&sf[(nsI + k) * 32], k < ns ? -tp[(T_RHS + 5 + k) * ST] : 0.0);
      {
        const double Ek = 0.5 * ((u * u + v * v) + w * w);
        double cell[11];
        cell[0] = 1.0 / dflow;
        cell[1] = rho;
        cell[2] = rho * u;
        cell[3] = rho * v;
        cell[4] = rho * w;
        cell[5] = rho * h;
        cell[6] = beta * Ek;
        cell[7] = -beta * u;
        cell[8] = -beta * v;
        cell[9] = -beta * w;
        cell[10] = beta;
#pragma unroll
        for (int p = 0; p < 11; ++p) {
          __stcs(&ff[p * 32], cell[p]);
          __stcs(&fb[p * 32], cell[p]);
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) __stcs(&ff[(11 + k) * 32], -tp[(T_RHS + k) * ST]);
      }
      // faces: 0 upper-i (i+1), 1 upper-j (j+1), 2 lower-i (i), 3 lower-j (j)
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const int d = f & 1;
        const bool upper = f < 2;
        // face metric: upper-i = lower-i face of (i + 1, j), upper-j = lower-j
        // face of (i, j + 1); S_z = 0 on i/j faces of a 2-D grid (k_check_2d)
        const int nb = upper ? (d == 0 ? up : up + 1) : (d == 0 ? lo : lo - 1);
        const int hf = upper ? nb : hc;
        const double S0 = A[(7 + 2 * d) * SA + hf], S1 = A[(8 + 2 * d) * SA + hf];
        const double a2 = S0 * S0 + S1 * S1;
        const double ar = sqrt(a2);
        const bool nb_in = upper ? (d == 0 ? i + 1 < g.ni : j + 1 < g.nj) : (d == 0 ? i > 0 : j > 0);
        auto lam = [&](int hh, bool sp) {
          const double U = fabs(A[0 * SA + hh] * S0 + A[1 * SA + hh] * S1);
          if (sp) return U + 2.0 * A[5 * SA + hh] * a2 * A[6 * SA + hh];
          return (U + A[3 * SA + hh] * ar) + 2.0 * A[4 * SA + hh] * a2 * A[6 * SA + hh];
        };
        double lf = lam(hc, false), ls = lam(hc, true);
        if (nb_in) {
          lf = npmax(lf, lam(nb, false));
          ls = npmax(ls, lam(nb, true));
        }
        const double sgn_lf = upper ? lf : -lf, sgn_ls = upper ? ls : -ls;
        const double U = u * S0 + v * S1;
        double* fd = upper ? ff + (16 + 7 * d) * 32 : fb + (11 + 7 * d) * 32;
        __stcs(&fd[0 * 32], -U * hr);
        __stcs(&fd[1 * 32], S0 * hr);
        __stcs(&fd[2 * 32], S1 * hr);
        __stcs(&fd[3 * 32], 0.5 * S0);
        __stcs(&fd[4 * 32], 0.5 * S1);
        __stcs(&fd[5 * 32], 0.5 * U);
        __stcs(&fd[6 * 32], 0.5 * (U + sgn_lf));
        const double csp = sp_scale * (U + sgn_ls);
        if (upper) __stcs(&sf[(nsI + NSB + d) * 32], csp);
        else __stcs(&sb[(nsI + d) * 32], csp);
      }
    };
    __syncthreads();  // the previous unit's phase B is done with the rings
    phase_a(tb - 1, 2, tb);
    for (int t0 = tb; t0 < te; t0 += C) {
      phase_a(t0 + 1, C, tb);
      __syncthreads();
      phase_b(t0);
      __syncthreads();
    }
  }
}

// Coupled operator with chemistry: the species block inverses dinv[r][c]
// (natural layout [ns * ns][N], csb_batched_inverse) into the dinv planes of
// the CF and CB records; one warp per (strip, step) row, so every store is a
// 256-byte row of the step-major layout.  Padding rows / columns (>= ns)
// keep their zeros.
template <int NSB>
__global__ void k_dinv2d(GridDev g, Skew sk, int ns, const double* __restrict__ dinv, WaveBufs wb) {
  constexpr int NG = ci_ng<NSB, true>(), PD = ci_planes<NSB>();
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)sk.nstrip * sk.T;
  for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w < rows;
       w += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int s = (int)(w / sk.T), t = (int)(w % sk.T);
    const int i = t - lane, j = s * 32 + lane;
    if (i < 0 || i >= g.ni || j >= g.nj) continue;
    const long long c = (long long)i * g.nj + j;
    double* cf = wb.ff + gaddr(sk, NG, s, t, PD, lane);
    double* cb = wb.fb + gaddr(sk, NG, s, t, PD, lane);
    for (int r = 0; r < ns; ++r)
      for (int cc = 0; cc < ns; ++cc) {
        const double v = dinv[((long long)r * ns + cc) * g.N + c];
        cf[(r * NSB + cc) * 32] = v;
        cb[(r * NSB + cc) * 32] = v;
      }
  }
}

// ============================================================== wavefront
struct WaveRole {
  const double* in;  // streamed group
  int ng;            // its planes per step
  int D;             // ring depth
  double* out;       // chain output group
  double* out2;      // CI backward: species components (SW); out gets the flow part (FW)
  int ngo, po;       // its planes per step, first output plane
  double* hand;      // [nstrip][ni][nh] hand-off rows (sentinel-initialised)
  int* ticket;
};

struct WaveArgs {
  Skew sk;
  int ni, nj, nsI;
  int only;          // -1: both roles (production); 0/1: one role (timing probe)
  int ci;            // coupled operator: one CI chain per strip (role[0])
  int poll_ns;       // receiver back-off between empty polls
  int fake_recv;     // probe: strips without upstream still get a receiver arrival per slot
  const int* rdy;    // forward sweep overlapped with the records kernel: tile flags (or null)
  const int* nonplanar;  // == epoch: some cell has z-momentum or its residual != 0 (or null)
  const int* epoch;  // the step's tag (device)
  int rC;            // records tile length (steps)
  unsigned long long* dbg;  // timing probe: [CTA][4] globaltimer stamps (or null)
  WaveRole role[2];  // 0 flow, 1 species
};

// ------------------------------------------------------------------ chains
// Hand-off between strips, in "sequence" space q (the order in which a strip
// produces / consumes its boundary columns): forward q = col, backward
// q = ni - 1 - col.  The last row of a strip stores its outgoing j-face
// products for column q straight into the L2 hand-off buffer
// hand[strip][q][nh]; the buffer is reset to a signalling-NaN sentinel before
// the sweep, and since every hand-off value is the result of a floating-point
// operation (which never yields a signalling NaN), a word != sentinel is
// final.  The receiver warp of the next strip polls the columns a ring slot
// needs, copies them into the smem ring hin[HRING][nh] and then arrives on the
// slot's full barrier, next to the producer's TMA transaction: the chain's
// only synchronisation is the per-slot mbarrier wait (measured: a per-4-step
// availability check inside the chain cost ~9% per step).

struct ChainCtx {
  const WaveArgs* a;
  int s, nslots, D, rt;
  bool has_up, has_down, first, last;
  bool recv;            // first row of a strip with an upstream strip
  bool send;            // last row of a strip with a downstream strip
  double mul;           // 0 on the first row (takes the hand-off), 1 elsewhere
  const double* ring;
  const double* hin;
  double* hand_out;     // this strip's row of the hand-off buffer, at its step 0
  unsigned long long* full_bar;
  unsigned long long* empty_bar;
  unsigned long long* pd;  // timing probe (CSB_PROBES): this CTA's stamp row, or null
};

// timing probe helpers (CSB_PROBES builds only): per-slot progress stamps and
// the total time a chain waits for its ring slots
CSB_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef CSB_PROBES
#define CSB_PROBE_WAIT(bar, ph)                                       \
  {                                                                   \
    const unsigned long long tw0 = x.pd ? gtime() : 0ull;             \
    mbar_wait(bar, ph);                                               \
    if (x.pd) {                                                       \
      const unsigned long long tw1 = gtime();                         \
      pwait += tw1 - tw0;                                             \
      if ((threadIdx.x & 31) == 0 && ks % 32 == 0 && ks / 32 < 56) x.pd[4 + ks / 32] = tw1; \
    }                                                                 \
  }
#define CSB_PROBE_DECL unsigned long long pwait = 0ull;
#define CSB_PROBE_END(slot_) \
  if (x.pd && (threadIdx.x & 31) == 0) x.pd[slot_] = pwait;
#else
#define CSB_PROBE_WAIT(bar, ph) mbar_wait(bar, ph);
#define CSB_PROBE_DECL
#define CSB_PROBE_END(slot_)
#endif

// predicated store without a branch (a branch would end the scheduling region
// of the unrolled step loop)
CSB_DEV void st_pred_cg_f64(double* p, double v, bool pred) {
#ifndef CSB_HAND_NORMAL
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.cg.L2::cache_hint.f64 [%0], %1, %3;\n}" ::"l"(p),
      "d"(v), "r"((int)pred), "l"(l2_evict_last()));
#else
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.global.cg.f64 [%0], %1;\n}" ::"l"(p),
               "d"(v), "r"((int)pred));
#endif
}
// hand-off poll load (L2, bypassing L1)
CSB_DEV unsigned long long ld_hand(const long long* p) {
#ifndef CSB_HAND_NORMAL
  unsigned long long v;
  asm volatile("ld.global.cg.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(l2_evict_last()));
  return v;
#else
  return (unsigned long long)__ldcg(p);
#endif
}

// flow chain: 5 coupled components per row (rank-2 half blocks)
// Lane shuffles of the chains as volatile asm: volatile asm statements keep
// their order, so the hand-off stores of step m (st_pred_cg_f64, also
// volatile) stay ahead of the shuffles of step m + 1 instead of being sunk to
// the end of the unrolled slot (measured in SASS: ~5 steps late, which adds
// directly to the strip-to-strip lag).  No memory clobber: the records loads
// and dq stores still schedule freely around them.
template <bool DOWN>
CSB_DEV double shfl1_f64(double v) {
  double r;
  if constexpr (DOWN) {
    asm volatile(
        "{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %1;\n"
        "shfl.sync.down.b32 lo, lo, 1, 0x1f, 0xffffffff;\n"
        "shfl.sync.down.b32 hi, hi, 1, 0x1f, 0xffffffff;\nmov.b64 %0, {lo, hi};\n}"
        : "=d"(r)
        : "d"(v));
  } else {
    asm volatile(
        "{\n.reg .b32 lo, hi;\nmov.b64 {lo, hi}, %1;\n"
        "shfl.sync.up.b32 lo, lo, 1, 0x0, 0xffffffff;\n"
        "shfl.sync.up.b32 hi, hi, 1, 0x0, 0xffffffff;\nmov.b64 %0, {lo, hi};\n}"
        : "=d"(r)
        : "d"(v));
  }
  return r;
}

// PL (planar): every cell has z-momentum 0 and z-momentum residual 0 this
// step (checked by k_hand_reset), so the component-3 records (w3, b3, rhs3) are zero
// and dq3, oi3, oj3 stay exactly zero: the chain skips component 3 (8 fewer
// FP64 operations, a shuffle and 4 shared-memory loads per step).
template <bool BWD, bool PL>
CSB_DEV void chain_flow(const ChainCtx& x, const WaveRole& ro) {
  constexpr int WK = WKF, NG = 30;
  constexpr int FQ = BWD ? 11 : 16;                         // first face plane
  constexpr int NGO = BWD ? 5 : NFB, PO = BWD ? 0 : FB_DQ;  // output: FW | FB dq* planes
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const WaveArgs& a = *x.a;
  const long long slot = (long long)WK * NG * 32;
  double oi[5] = {0, 0, 0, 0, 0}, oj[5] = {0, 0, 0, 0, 0};
  int buf = 0, phase = 0;
  CSB_PROBE_DECL
  for (int ks = 0; ks < x.nslots; ++ks) {
    const int k = BWD ? x.nslots - 1 - ks : ks;
    CSB_PROBE_WAIT(&x.full_bar[buf], phase)
    const double* base = x.ring + buf * slot + lane;
    double* ob = ro.out + (((long long)x.s * a.sk.T + (long long)k * WK) * NGO + PO) * 32 + lane;
    const double* hb = x.recv ? x.hin + ((k * WK) % HRING) * 5 : x.hin + HRING * 5;
    double* ho = x.hand_out + (long long)k * WK * 5;
#pragma unroll (CHAIN_UNROLL)
    for (int m = 0; m < WK; ++m) {
      const int kk = BWD ? WK - 1 - m : m;
      const double* p = base + kk * NG * 32;
      // the first row takes the upstream hand-off instead of the shuffled
      // value: ij = sh * mul + hv with mul = 0 and hv the hand-off there,
      // mul = 1 and hv = +0 (the zero block of hin) elsewhere
      const double* hv = hb + kk * 5;
      double ij[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        if (PL && c == 3) {
          ij[c] = 0.0;
          continue;
        }
        const double sh = shfl1_f64<BWD>(oj[c]);
        ij[c] = fma(sh, x.mul, hv[c]);
      }
      const double invd = p[0];
      double dq[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        if (PL && c == 3) {
          dq[c] = 0.0;
          if (BWD) ob[(kk * NGO + c) * 32] = 0.0;  // the epilogue reads dq3
          continue;
        }
        if (BWD) dq[c] = p[(FB_DQ + c) * 32] - (oi[c] + ij[c]) * invd;
        else dq[c] = ((p[(11 + c) * 32] + oi[c]) + ij[c]) * invd;
        ob[(kk * NGO + c) * 32] = dq[c];
      }
      const double w0 = p[1 * 32], w1 = p[2 * 32], w2 = p[3 * 32], w3 = PL ? 0.0 : p[4 * 32],
                   w4 = p[5 * 32];
      // balanced sums: short dependency chains behind dq
      const double sb = PL ? ((p[6 * 32] * dq[0] + p[7 * 32] * dq[1]) + p[8 * 32] * dq[2]) +
                                 p[10 * 32] * dq[4]
                           : ((p[6 * 32] * dq[0] + p[7 * 32] * dq[1]) +
                              (p[8 * 32] * dq[2] + p[9 * 32] * dq[3])) +
                                 p[10 * 32] * dq[4];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* pf = p + (FQ + 7 * f) * 32;
        const double sa = pf[0] * dq[0] + (pf[32] * dq[1] + pf[64] * dq[2]);
        const double sig = pf[6 * 32];
        double* o = f == 0 ? oi : oj;
        o[0] = w0 * sa + sig * dq[0];
        o[1] = w1 * sa + pf[3 * 32] * sb + sig * dq[1];
        o[2] = w2 * sa + pf[4 * 32] * sb + sig * dq[2];
        o[3] = PL ? 0.0 : w3 * sa + sig * dq[3];
        o[4] = w4 * sa + pf[5 * 32] * sb + sig * dq[4];
      }
#pragma unroll
      for (int c = 0; c < 5; ++c)
        if (!(PL && c == 3)) st_pred_cg_f64(ho + kk * 5 + c, oj[c], x.send);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&x.empty_bar[buf]);
    if (++buf == x.D) {
      buf = 0;
      phase ^= 1;
    }
  }
  CSB_PROBE_END(2)
}

// species chains: NSB independent scalar chains per row (padding species carry
// zero records, so they stay exactly zero).  PER: one diagonal per species
// (chemistry) instead of one shared diagonal.  Large species counts split
// over sp_warps<NSB>() chain warps of SG = NSB / sp_warps species each (all
// in registers; measured: one warp with NSB = 48 register chains spills, and
// an smem-resident state is MIO-bound).  All chain warps read the same ring.
template <int NSB>
constexpr int sp_warps() {
  // fewest warps with <= 8 register chains each (NSB divisible): the species
  // chain then issues no more per step than the flow chain
  int w = 1;
  while (NSB / w > 8 || NSB % w != 0) ++w;
  return w;
}

template <int NSB, bool BWD, bool PER>
CSB_DEV void chain_species(const ChainCtx& x, const WaveRole& ro, int grp) {
  constexpr int WK = wave_wks<NSB, PER>();
  constexpr int SG = NSB / sp_warps<NSB>();   // species of this warp
  constexpr int NI = PER ? NSB : 1, NG = NI + NSB + 2;
  constexpr int PC = BWD ? NI : NI + NSB;   // c_i, c_j planes
  constexpr int PV = BWD ? NI + 2 : NI;     // dq* (backward) | rhs (forward) planes
  constexpr int NGO = BWD ? NSB : NG, PO = BWD ? 0 : NI + 2;  // output: SW | SB dq* planes
  static_assert(NSB % sp_warps<NSB>() == 0, "species groups");
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int c0 = grp * SG;
  const WaveArgs& a = *x.a;
  const long long slot = (long long)WK * NG * 32;
  double oi[SG], oj[SG];
#pragma unroll
  for (int c = 0; c < SG; ++c) oi[c] = oj[c] = 0.0;
  int buf = 0, phase = 0;
  CSB_PROBE_DECL
  for (int ks = 0; ks < x.nslots; ++ks) {
    const int k = BWD ? x.nslots - 1 - ks : ks;
    if (grp == 0) {
      CSB_PROBE_WAIT(&x.full_bar[buf], phase)
    } else {
      mbar_wait(&x.full_bar[buf], phase);
    }
    const double* base = x.ring + buf * slot + lane;
    double* ob = ro.out + (((long long)x.s * a.sk.T + (long long)k * WK) * NGO + PO + c0) * 32 + lane;
    const double* hb = (x.recv ? x.hin + ((k * WK) % HRING) * NSB : x.hin + HRING * NSB) + c0;
    double* ho = x.hand_out + (long long)k * WK * NSB + c0;
#pragma unroll (CHAIN_UNROLL)
    for (int m = 0; m < WK; ++m) {
      const int kk = BWD ? WK - 1 - m : m;
      const double* p = base + kk * NG * 32;
      const double* hv = hb + kk * NSB;
      double ij[SG];
#pragma unroll
      for (int c = 0; c < SG; ++c) {
        const double sh = shfl1_f64<BWD>(oj[c]);
        ij[c] = fma(sh, x.mul, hv[c]);
      }
      const double ci = p[PC * 32], cj = p[(PC + 1) * 32];
      const double* pi = p + (PER ? c0 : 0) * 32;
      const double* pv = p + (PV + c0) * 32;
#pragma unroll
      for (int c = 0; c < SG; ++c) {
        const double inv = pi[(PER ? c : 0) * 32];
        const double v = pv[c * 32];
        const double dq = BWD ? v - (oi[c] + ij[c]) * inv : ((v + oi[c]) + ij[c]) * inv;
        ob[(kk * NGO + c) * 32] = dq;
        oi[c] = ci * dq;
        oj[c] = cj * dq;
      }
#pragma unroll
      for (int c = 0; c < SG; ++c) st_pred_cg_f64(ho + kk * NSB + c, oj[c], x.send);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&x.empty_bar[buf]);
    if (++buf == x.D) {
      buf = 0;
      phase ^= 1;
    }
  }
  if (grp == 0) { CSB_PROBE_END(2) }
}

// coupled (CI, frozen chemistry) chain: NV = 5 + NSB components per row with
// the full rank-2 half blocks of lusgs.py:24-59 and the scalar diagonal
// (lusgs.py:62-147); padding species carry zero records.
template <int NSB, bool BWD, bool CHEM>
CSB_DEV void chain_ci(const ChainCtx& x, const WaveRole& ro) {
  constexpr int NV = 5 + NSB, NG = ci_ng<NSB, CHEM>(), WK = ci_wk<NSB, CHEM>();
  constexpr int PD = ci_planes<NSB>();  // CHEM: first dinv plane
  constexpr int PV = BWD ? 2 + 2 * NV + 8 : 2 + 2 * NV;  // dq* (backward) | rhs (forward)
  constexpr int FQ = BWD ? 2 + 2 * NV : 2 + 3 * NV;      // first face plane
  constexpr int NGO = BWD ? 5 : NG, PO = BWD ? 0 : 2 + 2 * NV + 8;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const WaveArgs& a = *x.a;
  const long long slot = (long long)WK * NG * 32;
  double oi[NV], oj[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) oi[c] = oj[c] = 0.0;
  int buf = 0, phase = 0;
  for (int ks = 0; ks < x.nslots; ++ks) {
    const int k = BWD ? x.nslots - 1 - ks : ks;
    mbar_wait(&x.full_bar[buf], phase);
    const double* base = x.ring + buf * slot + lane;
    const long long st0 = (long long)x.s * a.sk.T + (long long)k * WK;
    double* ob = ro.out + (st0 * NGO + PO) * 32 + lane;
    double* ob2 = BWD ? ro.out2 + st0 * NSB * 32 + lane : nullptr;
    const double* hb = x.recv ? x.hin + ((k * WK) % HRING) * NV : x.hin + HRING * NV;
    double* ho = x.hand_out + (long long)k * WK * NV;
#pragma unroll
    for (int m = 0; m < WK; ++m) {
      const int kk = BWD ? WK - 1 - m : m;
      const double* p = base + kk * NG * 32;
      const double* hv = hb + kk * NV;
      double ij[NV];
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        const double sh = shfl1_f64<BWD>(oj[c]);
        ij[c] = fma(sh, x.mul, hv[c]);
      }
      const double invd = p[0], hr2 = p[32];
      double dq[NV];
      if constexpr (!CHEM) {
#pragma unroll
        for (int c = 0; c < NV; ++c) {
          const double v = p[(PV + c) * 32];
          if (BWD) dq[c] = v - (oi[c] + ij[c]) * invd;
          else dq[c] = ((v + oi[c]) + ij[c]) * invd;
        }
      } else {
        // chemistry (lusgs.py:92-100, 136-144): flow rows / d, species rows
        // dinv acc[5:] with dinv = inv(d I - V dOmega) from the records
        double acc[NV];
#pragma unroll
        for (int c = 0; c < NV; ++c)
          acc[c] = BWD ? oi[c] + ij[c] : (p[(PV + c) * 32] + oi[c]) + ij[c];
#pragma unroll
        for (int c = 0; c < 5; ++c) dq[c] = BWD ? p[(PV + c) * 32] - acc[c] * invd : acc[c] * invd;
#pragma unroll
        for (int r = 0; r < NSB; ++r) {
          double t = 0.0;
#pragma unroll
          for (int c = 0; c < NSB; ++c) t = fma(p[(PD + r * NSB + c) * 32], acc[5 + c], t);
          dq[5 + r] = BWD ? p[(PV + 5 + r) * 32] - t : t;
        }
      }
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        if (!BWD) ob[(kk * NGO + c) * 32] = dq[c];
        else if (c < 5) ob[(kk * 5 + c) * 32] = dq[c];
        else ob2[(kk * NSB + c - 5) * 32] = dq[c];
      }
      // b . dq over all NV components, two interleaved partial sums
      double sb0 = p[(2 + NV) * 32] * dq[0], sb1 = p[(3 + NV) * 32] * dq[1];
#pragma unroll
      for (int c = 2; c < NV; c += 2) {
        sb0 = fma(p[(2 + NV + c) * 32], dq[c], sb0);
        if (c + 1 < NV) sb1 = fma(p[(3 + NV + c) * 32], dq[c + 1], sb1);
      }
      const double sb = sb0 + sb1;
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* pf = p + (FQ + 4 * f) * 32;
        const double e0 = pf[0], e1 = pf[32], e2 = pf[64], sig = pf[96];
        // a = (-U hr, Sx hr, Sy hr) = hr2 (-e2, e0, e1)
        const double sa = hr2 * ((e0 * dq[1] + e1 * dq[2]) - e2 * dq[0]);
        double* o = f == 0 ? oi : oj;
#pragma unroll
        for (int c = 0; c < NV; ++c) {
          const double wc = p[(2 + c) * 32];
          const double ec = c == 1 ? e0 : c == 2 ? e1 : c == 4 ? e2 : 0.0;
          o[c] = (c == 1 || c == 2 || c == 4) ? wc * sa + ec * sb + sig * dq[c]
                                              : wc * sa + sig * dq[c];
        }
      }
#pragma unroll
      for (int c = 0; c < NV; ++c) st_pred_cg_f64(ho + kk * NV + c, oj[c], x.send);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&x.empty_bar[buf]);
    if (++buf == x.D) {
      buf = 0;
      phase ^= 1;
    }
  }
}

// coupled chain for large species counts (NSB > CI_MAXNSB): the same
// arithmetic as chain_ci with the per-row state in shared memory -- oi, the
// double-buffered oj (read by the neighbouring row instead of a shuffle) and
// dq -- laid out [component][lane].
template <int NSB, bool BWD>
CSB_DEV void chain_ci_big(const ChainCtx& x, const WaveRole& ro, double* st) {
  constexpr int NV = 5 + NSB, NG = ci_planes<NSB>(), WK = ci_wk<NSB>();
  constexpr int PV = BWD ? 2 + 2 * NV + 8 : 2 + 2 * NV;
  constexpr int FQ = BWD ? 2 + 2 * NV : 2 + 3 * NV;
  constexpr int NGO = BWD ? 5 : NG, PO = BWD ? 0 : 2 + 2 * NV + 8;
  const int lane = threadIdx.x & 31;
  const int nbr = BWD ? min(lane + 1, 31) : max(lane - 1, 0);  // j-neighbour row's lane
  const WaveArgs& a = *x.a;
  const long long slot = (long long)WK * NG * 32;
  double* soi = st;                 // [NV][32]
  double* soj = st + NV * 32;       // [2][NV][32]
  double* sdq = st + 3 * NV * 32;   // [NV][32]
  for (int c = 0; c < NV; ++c) soi[c * 32 + lane] = soj[c * 32 + lane] = soj[(NV + c) * 32 + lane] = 0.0;
  __syncwarp();
  int cur = 0;
  int buf = 0, phase = 0;
  for (int ks = 0; ks < x.nslots; ++ks) {
    const int k = BWD ? x.nslots - 1 - ks : ks;
    mbar_wait(&x.full_bar[buf], phase);
    const double* base = x.ring + buf * slot + lane;
    const long long st0 = (long long)x.s * a.sk.T + (long long)k * WK;
    double* ob = ro.out + (st0 * NGO + PO) * 32 + lane;
    double* ob2 = BWD ? ro.out2 + st0 * NSB * 32 + lane : nullptr;
    const double* hb = x.recv ? x.hin + ((k * WK) % HRING) * NV : x.hin + HRING * NV;
    double* ho = x.hand_out + (long long)k * WK * NV;
    for (int m = 0; m < WK; ++m) {
      const int kk = BWD ? WK - 1 - m : m;
      const double* p = base + kk * NG * 32;
      const double* hv = hb + kk * NV;
      const double* ojp = soj + cur * NV * 32;      // previous step's products
      double* ojn = soj + (cur ^ 1) * NV * 32;      // this step's
      const double invd = p[0], hr2 = p[32];
      double sb0 = 0.0, sb1 = 0.0, dq0 = 0.0, dq1 = 0.0, dq2 = 0.0;
      for (int c = 0; c < NV; ++c) {
        const double ij = fma(ojp[c * 32 + nbr], x.mul, hv[c]);
        const double oic = soi[c * 32 + lane];
        const double v = p[(PV + c) * 32];
        const double dq = BWD ? v - (oic + ij) * invd : ((v + oic) + ij) * invd;
        sdq[c * 32 + lane] = dq;
        if (!BWD) ob[(kk * NGO + c) * 32] = dq;
        else if (c < 5) ob[(kk * 5 + c) * 32] = dq;
        else ob2[(kk * NSB + c - 5) * 32] = dq;
        if (c & 1) sb1 = fma(p[(2 + NV + c) * 32], dq, sb1);
        else sb0 = fma(p[(2 + NV + c) * 32], dq, sb0);
        if (c == 0) dq0 = dq;
        if (c == 1) dq1 = dq;
        if (c == 2) dq2 = dq;
      }
      const double sb = sb0 + sb1;
      double sa[2], e[2][3], sig[2];
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double* pf = p + (FQ + 4 * f) * 32;
        e[f][0] = pf[0];
        e[f][1] = pf[32];
        e[f][2] = pf[64];
        sig[f] = pf[96];
        sa[f] = hr2 * ((e[f][0] * dq1 + e[f][1] * dq2) - e[f][2] * dq0);
      }
      for (int c = 0; c < NV; ++c) {
        const double dq = sdq[c * 32 + lane];
        const double wc = p[(2 + c) * 32];
        const bool ev = c == 1 || c == 2 || c == 4;
        const int ei = c == 1 ? 0 : c == 2 ? 1 : 2;
        const double oi = ev ? wc * sa[0] + e[0][ei] * sb + sig[0] * dq : wc * sa[0] + sig[0] * dq;
        const double oj = ev ? wc * sa[1] + e[1][ei] * sb + sig[1] * dq : wc * sa[1] + sig[1] * dq;
        soi[c * 32 + lane] = oi;
        ojn[c * 32 + lane] = oj;
        st_pred_cg_f64(ho + kk * NV + c, oj, x.send);
      }
      __syncwarp();
      cur ^= 1;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&x.empty_bar[buf]);
    if (++buf == x.D) {
      buf = 0;
      phase ^= 1;
    }
  }
}

// threads per wavefront CTA: chain warps (up to sp_warps<NSB>()) + producer +
// receiver
template <int NSB>
constexpr int wave_threads() { return 32 * (sp_warps<NSB>() + 2); }

template <int NSB, bool BWD, bool PER>
__global__ void __launch_bounds__(wave_threads<NSB>(), 1) k_wave2d(WaveArgs a) {
  extern __shared__ __align__(128) double wsm[];
  __shared__ unsigned long long full_bar[8], empty_bar[8];
  __shared__ int s_strip;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((a.only == 2 || a.only == 3) && (blockIdx.x & 1) != a.only - 2) return;  // probe: idle partner
  if (a.only == 4 && (blockIdx.x & 1)) return;  // probe: one idle CTA between working ones
  // role: 0 flow, 1 species.  Block pairs share a role: the two SMs of a TPC
  // run the same code (measured: a flow and a species CTA side by side on a
  // TPC slow the flow chain by ~14%)
  const int kind = a.ci ? 2
                   : (a.only == 0 || a.only == 1) ? a.only
                   : a.only == 5                  ? (blockIdx.x & 1)
                                                  : ((blockIdx.x >> 1) & 1);
  const WaveRole ro = kind == 1 ? a.role[1] : a.role[0];
  const int WK = kind == 2 ? (PER ? ci_wk<NSB, true>() : ci_wk<NSB, false>())
                 : kind ? wave_wks<NSB, PER>() : WKF;
  const int nh = kind == 2 ? 5 + NSB : kind ? NSB : 5;
  const int nchain = kind == 1 ? sp_warps<NSB>() : 1;  // chain warps of this role
  const int D = ro.D, NG = ro.ng;
  const long long slot = (long long)WK * NG * 32;
  double* ring = wsm;                     // [D][WK][NG][32]
  double* hin = ring + D * slot;          // [HRING + WK][nh], rows >= HRING zero
  if (threadIdx.x == 0) {
    const int tk = atomicAdd(ro.ticket, 1);
    s_strip = tk >= a.sk.nstrip ? -1 : (BWD ? a.sk.nstrip - 1 - tk : tk);
  }
  __syncthreads();
  if (s_strip < 0) return;  // surplus CTA of the role-pair layout
  ChainCtx x;
  x.a = &a;
  x.s = s_strip;
  x.D = D;
  x.rt = min(31, a.nj - 1 - x.s * 32);  // highest valid row of this strip
  const int T = a.sk.T;
  x.nslots = T / WK;
  x.has_up = BWD ? (x.s + 1 < a.sk.nstrip) : (x.s > 0);
  x.has_down = BWD ? (x.s > 0) : (x.s + 1 < a.sk.nstrip);
  x.first = BWD ? (lane == x.rt) : (lane == 0);  // receives the upstream hand-off
  x.last = BWD ? (lane == 0) : (lane == x.rt);   // sends the downstream hand-off
  x.mul = x.first ? 0.0 : 1.0;
  x.recv = x.first && x.has_up;
  x.send = x.last && x.has_down;
  x.ring = ring;
  x.hin = hin;
  // hand-off rows are indexed by the producing strip's step, with HPAD
  // zero rows on both sides (steps whose partner column lies outside the grid)
  x.hand_out = ro.hand + ((long long)x.s * (T + 2 * HPAD) + HPAD) * nh;
  x.full_bar = full_bar;
  x.empty_bar = empty_bar;
  x.pd = a.dbg ? a.dbg + 64 * (2 * s_strip + kind) : nullptr;
  if (threadIdx.x == 0) {
    for (int b = 0; b < D; ++b) {
      mbar_init(&full_bar[b], (x.has_up || a.fake_recv) ? 2 : 1);  // TMA producer (+ hand-off receiver)
      mbar_init(&empty_bar[b], nchain);  // every chain warp releases the slot
    }
    for (int c = 0; c < WK * nh; ++c) hin[HRING * nh + c] = 0.0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int s = x.s;
  const int up = BWD ? s + 1 : s - 1;

  if (warp == nchain) {
    // ---------------------------------------------------- producer (TMA)
    if (lane == 0) {
      const int ep = a.rdy ? *a.epoch : 0;
      int buf = 0, phase = 0;
#ifdef CSB_PROBES
      unsigned long long pw = 0ull;
#endif
      for (int ks = 0; ks < x.nslots; ++ks) {
        const int k = BWD ? x.nslots - 1 - ks : ks;
#ifdef CSB_PROBES
        const unsigned long long tw0 = x.pd ? gtime() : 0ull;
        if (ks >= D) mbar_wait(&empty_bar[buf], phase ^ 1);
        if (x.pd) pw += gtime() - tw0;
#else
        if (ks >= D) mbar_wait(&empty_bar[buf], phase ^ 1);
#endif
        if (a.rdy) {
          // records tiles of this slot's steps stored (records kernel running
          // concurrently): acquire their flags, then order the bulk copy
          // (async proxy) after the acquire
          const int* f = a.rdy + (long long)s * T;
          for (int b = (k * WK) / a.rC; b <= (k * WK + WK - 1) / a.rC; ++b)
            while (ld_acquire(f + b) != ep) __nanosleep(64);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const unsigned bytes = (unsigned)(slot * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full_bar[buf])),
                     "r"(bytes)
                     : "memory");
        bulk_g2s(ring + buf * slot, ro.in + ((long long)s * T + (long long)k * WK) * NG * 32, bytes,
                 &full_bar[buf]);
        if (++buf == D) {
          buf = 0;
          phase ^= 1;
        }
      }
#ifdef CSB_PROBES
      if (x.pd) x.pd[60] = pw;
#endif
    }
    return;
  }

  if (warp == nchain + 1) {
    // ---------------------------------------------------- hand-off receiver
    // For each ring slot: the upstream columns its steps need (one per lane,
    // at most WK <= 32), polled until complete, copied into hin, then one
    // arrival on the slot's full barrier (release: the chain's wait acquires).
    if (!x.has_up) {
      if (a.fake_recv) {  // probe: arrive per slot without any data
        int buf = 0, phase = 0;
        for (int ks = 0; ks < x.nslots; ++ks) {
          if (ks >= D) mbar_wait(&empty_bar[buf], phase ^ 1);
          if (lane == 0) mbar_arrive(&full_bar[buf]);
          if (++buf == D) {
            buf = 0;
            phase ^= 1;
          }
        }
      }
      return;
    }
    // upstream row u of the hand-off buffer holds what the upstream strip's
    // sending row produced at its step u; our receiving row needs, at our step
    // t, the upstream step t + 31 (forward: upstream row 31 -> our row 0) or
    // t - 31 (backward: upstream row 0 -> our row 31).  A slot needs WK rows
    // of nh words: the words are spread over the lanes (up to 8 per lane),
    // all loaded at once, and the slot is released when none is the sentinel.
    const double* src = ro.hand + ((long long)up * (T + 2 * HPAD) + HPAD) * nh;
    const int nw = WK * nh;  // words per slot (<= 256)
    // planar step: the flow chains neither send nor read hand-off word 3
    const bool skip3 = BWD && kind == 0 && a.nonplanar && ld_relaxed(a.nonplanar) != *a.epoch;
    // Windows of Q consecutive slots (Q x WK >= 8 steps, <= 512 words): the
    // window's hand-off rows are contiguous both in the L2 buffer and in the
    // hin ring, so one poll round trip covers all of them.  (Measured: with one
    // 4-step slot per poll the receiver, not the chain, set the pace of the
    // ns = 20 species sweep: 311 vs 120 ns per step on 2 strips.)
    // (Q x WK must divide HRING and TQ so a window never wraps the hin ring:
    // Q is rounded down to a power of two; WK is one already)
    int Q = max(1, min(WK >= 8 ? 1 : 8 / WK, 512 / nw));
    while (Q & (Q - 1)) Q &= Q - 1;
#ifdef CSB_PROBES
    unsigned long long rpoll = 0ull;
#endif
    if (Q == 1) {
    // one slot per poll (slots of >= 8 steps)
    int buf = 0, phase = 0;
    for (int ks = 0; ks < x.nslots; ++ks) {
      const int k = BWD ? x.nslots - 1 - ks : ks;
      if (ks >= D) mbar_wait(&empty_bar[buf], phase ^ 1);  // slot free: hin rows too
#ifdef CSB_RECV_LAG
      {  // probe: poll only once the chain has released slot ks - D + LAG
        const int j = ks - D + CSB_RECV_LAG;
        if (j >= 0 && CSB_RECV_LAG > 0) mbar_wait(&empty_bar[j % D], (j / D) & 1);
      }
#endif
      const long long u0 = (long long)k * WK + (BWD ? -31 : 31);  // upstream step of kk = 0
      const long long* sw = reinterpret_cast<const long long*>(src) + u0 * nh;
      double* dst = hin + ((k * WK) % HRING) * nh;
      unsigned long long w[8];
      unsigned have = 0u;  // bit r: word lane + 32 r loaded and final
      const int cnt = nw > lane ? (nw - lane + 31) / 32 : 0;
      const unsigned need = (1u << cnt) - 1u;
#ifdef CSB_PROBES
      const unsigned long long tp0 = x.pd ? gtime() : 0ull;
#endif
      while (true) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int e = lane + 32 * r;
          if (e < nw && !(have >> r & 1u)) {
            if (skip3 && e % nh == 3) {
              w[r] = 0ull;
              have |= 1u << r;
            } else {
              w[r] = ld_hand(sw + e);
              if (w[r] != HAND_SENTINEL) have |= 1u << r;
            }
          }
        }
        if (__all_sync(0xffffffffu, (have & need) == need)) break;
        __nanosleep(a.poll_ns);
      }
#ifdef CSB_PROBES
      if (x.pd) rpoll += gtime() - tp0;
#endif
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int e = lane + 32 * r;
        if (e < nw) dst[e] = __longlong_as_double((long long)w[r]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[buf]);
      if (++buf == D) {
        buf = 0;
        phase ^= 1;
      }
    }
    } else {
    int buf = 0, phase = 0;
    for (int ks0 = 0; ks0 < x.nslots; ks0 += Q) {
      const int nq = min(Q, x.nslots - ks0);
      const int nwq = nq * nw;
      // poll only once the chain has released the window's first slot (the
      // receiver stays within D slots of the chain: no L2 polling far ahead)
      if (ks0 >= D) mbar_wait(&empty_bar[buf], phase ^ 1);
      // lowest step index of the window (forward: slot ks0; backward: the
      // window's last slot in consumption order)
      const int kmin = BWD ? x.nslots - ks0 - nq : ks0;
      const long long u0 = (long long)kmin * WK + (BWD ? -31 : 31);  // upstream step of its row 0
      const long long* sw = reinterpret_cast<const long long*>(src) + u0 * nh;
      double* dst = hin + ((kmin * WK) % HRING) * nh;
      unsigned long long w[16];
      unsigned have = 0u;  // bit r: word lane + 32 r loaded and final
      const int cnt = nwq > lane ? (nwq - lane + 31) / 32 : 0;
      const unsigned need = cnt >= 32 ? 0xffffffffu : (1u << cnt) - 1u;
      while (true) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (32 * r >= nwq) break;
          const int e = lane + 32 * r;
          if (e < nwq && !(have >> r & 1u)) {
            if (skip3 && e % nh == 3) {
              w[r] = 0ull;
              have |= 1u << r;
            } else {
              w[r] = ld_hand(sw + e);
              if (w[r] != HAND_SENTINEL) have |= 1u << r;
            }
          }
        }
        if (__all_sync(0xffffffffu, (have & need) == need)) break;
        __nanosleep(a.poll_ns);
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (32 * r >= nwq) break;
        const int e = lane + 32 * r;
        if (e < nwq) dst[e] = __longlong_as_double((long long)w[r]);
      }
      __syncwarp();
      for (int j = 0; j < nq; ++j) {
        if (j > 0 && ks0 + j >= D) mbar_wait(&empty_bar[buf], phase ^ 1);  // slot's phase is free
        if (lane == 0) mbar_arrive(&full_bar[buf]);
        if (++buf == D) {
          buf = 0;
          phase ^= 1;
        }
      }
    }
    }
#ifdef CSB_PROBES
    if (x.pd && lane == 0) x.pd[3] = rpoll;
#endif
    return;
  }

  // -------------------------------------------------------- chain warps
  if (warp >= nchain) return;  // surplus warps of a role with fewer chains
  unsigned long long t0 = 0;
  if (a.dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (kind == 0) {
    // planarity of this step: k_hand_reset stores the launch epoch on
    // any nonzero z-momentum or z-momentum residual
    // (backward sweep only -- measured: the planar forward chain is faster on
    // one strip, 147 -> 130 ns per step, but its multi-strip pipeline is
    // slower, 512^2 199 -> 216 us; the planar backward sweep gains 207 -> 200)
    if (BWD && a.nonplanar && ld_relaxed(a.nonplanar) != *a.epoch) chain_flow<BWD, true>(x, ro);
    else chain_flow<BWD, false>(x, ro);
  } else if (kind == 1) {
    chain_species<NSB, BWD, PER>(x, ro, warp);
  } else {
    if constexpr (!PER) {
      if constexpr (NSB <= CI_MAXNSB) chain_ci<NSB, BWD, false>(x, ro);
      else chain_ci_big<NSB, BWD>(x, ro, hin + (HRING + WK) * nh);
    } else {  // coupled operator with chemistry (register chain only)
      if constexpr (NSB <= CI_MAXNSB) chain_ci<NSB, BWD, true>(x, ro);
    }
  }
  if (a.dbg && lane == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned long long* d = a.dbg + 64 * (2 * s + kind);
    d[0] = t0;
    d[1] = t1;
  }
}

// ============================================================== epilogue
// Tile = one strip (32 rows j) x CI columns i, CI = warps per CTA: a rectangle
// in (i, j), so every q / q_new access of a warp is one aligned 256-byte row
// (warp = column, lane = row).  The step-major dq rows of the tile (steps
// i0 .. i0 + CI + 30; each row is shared with the neighbouring column tiles)
// are gathered into shared memory by 8-byte cp.async, row by row (a warp
// reads the contiguous lanes of one step that fall into the tile), into
// element (plane k, column ii, row r) at (k * CI + ii) * 32 + r.  The grid is
// persistent and the tiles are double-buffered: the gather of the next tile
// is in flight while this one is closed and gated.

#ifndef CSB_EPI_PTR
#define CSB_EPI_PTR 1  // q / q_new through running pointers: config 4 epilogue 0.82 -> 0.76 ms
#endif
struct GateAcc {
  unsigned long long bad_count = 0, first1 = ~0ull, first2 = ~0ull;
};

// Closure + gate of one cell, register form: all q loads first (memory-level
// parallelism), the closure in place in those registers (dq is read from
// shared memory where it is used: 5 + NSB live doubles instead of three such
// arrays), the gate decodes the new state from registers (no read-back of
// q_new).  dd: the cell's dq planes, stride DS.
template <int NSB>
CSB_DEV void epilogue_cell(const Model& m, int scheme, const double* __restrict__ qc,
                           double* __restrict__ qo, const double* dd, int DS, long long N,
                           long long c, double* __restrict__ dq_std, GateAcc& ga) {
  const int ns = m.ns, nv = 5 + ns;
  if (dq_std) {
#pragma unroll
    for (int k = 0; k < 5 + NSB; ++k)
      if (k < nv) dq_std[(long long)k * N + c] = dd[k * DS];
  }
  double o[5 + NSB];  // q, then q_new in place
#if CSB_EPI_PTR
  {
    const double* qp = qc;  // running pointer: one 64-bit add per component
#pragma unroll
    for (int k = 0; k < 5 + NSB; ++k, qp += N) o[k] = k < nv ? *qp : 0.0;
  }
#else
#pragma unroll
  for (int k = 0; k < 5 + NSB; ++k) o[k] = k < nv ? qc[k * N] : 0.0;
#endif
  const double d0 = dd[0];
  bool ok1 = true;
  if (scheme == SCH_CI) {
    o[0] = o[0] + d0;
    double tail = 0.0;
#pragma unroll
    for (int sp = 0; sp < NSB; ++sp)
      if (sp < ns - 1) {
        o[5 + sp] = o[5 + sp] + dd[(5 + sp) * DS];
        tail += o[5 + sp];
      }
    const double lastv = o[0] - tail;
    // bitwise select (a guarded store here becomes one dynamically indexed
    // store, which moves o[] to local memory)
#pragma unroll
    for (int sp = 0; sp < NSB; ++sp) {
      const unsigned long long msk = 0ull - (unsigned long long)(sp == ns - 1);
      o[5 + sp] = __longlong_as_double((long long)(((unsigned long long)__double_as_longlong(o[5 + sp]) & ~msk) |
                                                   ((unsigned long long)__double_as_longlong(lastv) & msk)));
    }
    ok1 = !(lastv < -1e-10 * o[0]);
  } else {
    double tot = 0.0, dsum = 0.0;
#pragma unroll
    for (int sp = 0; sp < NSB; ++sp)
      if (sp < ns) {
        tot += o[5 + sp];
        dsum += dd[(5 + sp) * DS];
      }
    double osum = 0.0;
    if (scheme == SCH_CS1) {
      // (rho_s / sum rho_s) defect as rho_s (defect / sum rho_s): one division
      // per cell instead of one per species (1-2 ulp of the correction term)
      const double dfr = (d0 - dsum) / tot;
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns) o[5 + sp] = o[5 + sp] + dd[(5 + sp) * DS] + o[5 + sp] * dfr;
    } else {
      const double rnew = tot + d0;
      double rawsum = 0.0;
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns) {
          o[5 + sp] = o[5 + sp] + dd[(5 + sp) * DS];
          rawsum += o[5 + sp];
        }
      const double rsc = rnew / rawsum;
#pragma unroll
      for (int sp = 0; sp < NSB; ++sp)
        if (sp < ns) o[5 + sp] = o[5 + sp] * rsc;
    }
    o[0] = o[0] + d0;
#pragma unroll
    for (int sp = 0; sp < NSB; ++sp)
      if (sp < ns) osum += o[5 + sp];
    ok1 = !(osum <= 0.0);
#pragma unroll
    for (int sp = 0; sp < NSB; ++sp)
      if (sp < ns && o[5 + sp] < -EPS_NEG * osum) ok1 = false;
  }
#pragma unroll
  for (int k = 1; k < 5; ++k) o[k] = o[k] + dd[k * DS];
#if CSB_EPI_PTR
  {
    double* qp = qo;
#pragma unroll
    for (int k = 0; k < 5 + NSB; ++k, qp += N)
      if (k < nv) *qp = o[k];
  }
#else
#pragma unroll
  for (int k = 0; k < 5 + NSB; ++k)
    if (k < nv) qo[k * N] = o[k];
#endif
  Cell<NSB> cs;
  const bool ok2 = decode_from<NSB>(m, [&](int k) { return o[k]; }, cs);
  if (!ok1 && ga.first1 == ~0ull) ga.first1 = (unsigned long long)c;
  if (!ok2 && ga.first2 == ~0ull) ga.first2 = (unsigned long long)c;
  if (!(ok1 && ok2)) ++ga.bad_count;
}

// Large species counts (NSB > 24): the same closure + gate with the species
// streamed instead of held in three register arrays of 5 + NSB doubles (which
// capped the kernel at 2 CTAs per SM with spills): every species pass
// recomputes o_s from q (L1) and dq (shared memory) with pinned rounding
// (__d*_rn), so every pass sees the value that was stored.
// dfr = (drho - sum drho_s) / sum rho_s, rsc = (sum rho_s + drho) / sum(rho_s + drho_s)
CSB_DEV double closure_species(int scheme, double qs, double ds, double dfr, double rsc) {
  if (scheme == SCH_CS1)  // rho_s + drho_s + rho_s (drho - sum drho_s) / sum rho_s
    return __dadd_rn(__dadd_rn(qs, ds), __dmul_rn(qs, dfr));
  if (scheme == SCH_CS2)  // (rho_s + drho_s)(sum rho_s + drho) / sum(rho_s + drho_s)
    return __dmul_rn(__dadd_rn(qs, ds), rsc);
  return __dadd_rn(qs, ds);  // CI (the last species is reconstructed)
}

CSB_DEV void epilogue_cell_streamed(const Model& m, int scheme, const double* __restrict__ qc,
                                    double* __restrict__ qo, const double* dd, int DS, long long N,
                                    long long c, double* __restrict__ dq_std, GateAcc& ga) {
  const int ns = m.ns, nv = 5 + ns;
  if (dq_std)
    for (int k = 0; k < nv; ++k) dq_std[(long long)k * N + c] = dd[k * DS];
  double o[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    o[k] = qc[k * N] + dd[k * DS];
    qo[k * N] = o[k];
  }
  // pass 1: species sums
  double tot = 0.0, dsum = 0.0, rawsum = 0.0, tail = 0.0;
  for (int sp = 0; sp < ns; ++sp) {
    const double qs = qc[(5 + sp) * N], ds = dd[(5 + sp) * DS];
    tot += qs;
    dsum += ds;
    rawsum += qs + ds;
    if (sp < ns - 1) tail += __dadd_rn(qs, ds);
  }
  const double dfr = (dd[0] - dsum) / tot, rsc = (tot + dd[0]) / rawsum;
  const double lastv = o[0] - tail;
  auto o_s = [&](int sp) {
    if (scheme == SCH_CI && sp == ns - 1) return lastv;
    return closure_species(scheme, qc[(5 + sp) * N], dd[(5 + sp) * DS], dfr, rsc);
  };
  // pass 2: store
  double osum = 0.0;
  for (int sp = 0; sp < ns; ++sp) {
    const double v = o_s(sp);
    qo[(5 + sp) * N] = v;
    osum += v;
  }
  bool ok1 = scheme == SCH_CI ? !(lastv < -1e-10 * o[0]) : !(osum <= 0.0);
  // pass 3: gate (CS) and the clipped mass fractions of the decode
  const double rho = o[0];
  bool ok2 = (rho > 0.0) && finite(rho);
  const double ir = 1.0 / rho;
  double ysum = 0.0;
  for (int sp = 0; sp < ns; ++sp) {
    const double v = o_s(sp);
    if (scheme != SCH_CI && v < -EPS_NEG * osum) ok1 = false;
    double y = v * ir;
    if (y < -EPS_NEG) ok2 = false;
    if (y < 0.0) y = 0.0;
    ysum += y;
  }
  // pass 4: renormalised mixture sums and temperature (decode_from)
  const double isum = 1.0 / ysum;
  double R = 0.0, cp = 0.0, yb = 0.0;
  for (int sp = 0; sp < ns; ++sp) {
    double y = o_s(sp) * ir;
    if (y < 0.0) y = 0.0;
    y = y * isum;
    R += y * m.Rs[sp];
    cp += y * m.cp[sp];
    yb += y * m.bs[sp];
  }
  const double u0 = o[1] * ir, u1 = o[2] * ir, u2 = o[3] * ir;
  const double Ek = 0.5 * ((u0 * u0 + u1 * u1) + u2 * u2);
  const double T = ((o[4] * ir - Ek) - yb) * (1.0 / (cp - R));
  if (!(T > 0.0) || !finite(T)) ok2 = false;
  if (!ok1 && ga.first1 == ~0ull) ga.first1 = (unsigned long long)c;
  if (!ok2 && ga.first2 == ~0ull) ga.first2 = (unsigned long long)c;
  if (!(ok1 && ok2)) ++ga.bad_count;
}

#ifndef CSB_EPI_MINB
#define CSB_EPI_MINB 4
#endif
template <int NSB>
constexpr int epilogue_minb() {
#ifdef CSB_EPI_MINB_REG
  return NSB > 24 ? CSB_EPI_MINB : CSB_EPI_MINB_REG;
#else
  // measured (config 4 / 512^2 ns = 5): 2 CTAs per SM 0.875 / 0.027 ms, 3-4 CTAs
  // (80 / 64 registers, spills) 0.947 / 0.035 ms
  return NSB > 24 ? CSB_EPI_MINB : 2;
#endif
}

template <int NSB>
__global__ void __launch_bounds__(256, epilogue_minb<NSB>())
    k_epilogue2d(const Model* __restrict__ mp, GridDev g, Skew sk, int scheme,
                 const double* __restrict__ q, const double* __restrict__ fw,
                 const double* __restrict__ sw, double* __restrict__ qn,
                 double* __restrict__ dq_std, int nbuf, unsigned long long* flags) {
  extern __shared__ double es[];
  const Model& m = *mp;
  const int ns = m.ns, nv = 5 + ns;
  const int CI = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int DS = CI * 32;            // plane stride inside a tile
  const int tile_doubles = nv * DS;  // one buffer
  const int ncol = (g.ni + CI - 1) / CI;
  const long long ntiles = (long long)ncol * sk.nstrip;
  const long long N = g.N;
  // tile -> (column block, strip), strips fastest: concurrently running CTAs
  // cover whole rows of q
  auto gather = [&](long long tile, double* buf) {
    const int s = (int)(tile % sk.nstrip), i0 = (int)(tile / sk.nstrip) * CI;
    const bool row_in = s * 32 + lane < g.nj;
    for (int rr = warp; rr < CI + 31; rr += CI) {
      const int ii = rr - lane;
      if (ii < 0 || ii >= CI || i0 + ii >= g.ni || !row_in) continue;
      const int t = i0 + rr;
      double* dst = buf + ii * 32 + lane;
      const double* f = fw + gaddr(sk, 5, s, t, 0, lane);
      const double* sp = sw + gaddr(sk, NSB, s, t, 0, lane);
#pragma unroll
      for (int k = 0; k < 5; ++k) cp_async8(dst + k * DS, f + k * 32);
      for (int k = 0; k < ns; ++k) cp_async8(dst + (5 + k) * DS, sp + k * 32);
    }
  };
  GateAcc ga;
  long long tile = blockIdx.x;
  int cur = 0;
  if (tile < ntiles) gather(tile, es);
  cp_async_commit();
  for (; tile < ntiles; tile += gridDim.x) {
    const long long next = tile + gridDim.x;
    if (nbuf > 1) {
      if (next < ntiles) gather(next, es + (cur ^ 1) * tile_doubles);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    {
      const int s = (int)(tile % sk.nstrip), i = (int)(tile / sk.nstrip) * CI + warp;
      const int j = s * 32 + lane;
      if (i < g.ni && j < g.nj) {
        const long long c = (long long)i * g.nj + j;
        const double* dd = es + cur * tile_doubles + warp * 32 + lane;
        if constexpr (NSB > 24) epilogue_cell_streamed(m, scheme, q + c, qn + c, dd, DS, N, c, dq_std, ga);
        else epilogue_cell<NSB>(m, scheme, q + c, qn + c, dd, DS, N, c, dq_std, ga);
      }
    }
    __syncthreads();
    if (nbuf > 1) {
      cur ^= 1;
    } else {
      if (next < ntiles) gather(next, es);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
  for (int o = 16; o > 0; o >>= 1) {
    ga.bad_count += __shfl_xor_sync(0xffffffffu, ga.bad_count, o);
    ga.first1 = min(ga.first1, __shfl_xor_sync(0xffffffffu, ga.first1, o));
    ga.first2 = min(ga.first2, __shfl_xor_sync(0xffffffffu, ga.first2, o));
  }
  if (lane == 0) {
    if (ga.bad_count) atomicAdd(flags + FLAG_GATE_COUNT, ga.bad_count);
    if (ga.first1 != ~0ull) raise_flag(flags, EB_GATE, (long long)ga.first1);
    if (ga.first2 != ~0ull) raise_flag(flags, EB_GATE_DECODE, (long long)ga.first2);
  }
}

// ============================================================== launcher
inline size_t wave_role_smem(int D, int WK, int NG, int nh) {
  return ((size_t)D * WK * NG * 32 + (size_t)(HRING + WK) * nh) * sizeof(double);
}
// deepest ring (2..4) that fits the shared-memory budget, 0 if none
inline int wave_depth(int WK, int NG, int nh) {
  for (int D = CSB_DMAX; D >= 2; --D)
    if (wave_role_smem(D, WK, NG, nh) <= WAVE_SMEM_BUDGET) return D;
  return 0;
}

// One implicit step on the 2-D wavefront path.  Stream order: hand-off reset,
// records, forward sweep, backward sweep, epilogue -- except that (outside
// the per-stage timing probe, ev == nullptr) the forward sweep runs on the
// high-priority side stream wb.s2 CONCURRENTLY with the records kernel (when
// the sweeps use at most 48 SMs): the
// sweep's 2 x nstrip CTAs take their SMs first, the records tiles fill the
// remaining ones in step-block-major order, and each sweep ring slot waits
// only for its own records tiles (WaveBufs::rdy).  CSB_NO_OVERLAP=1 restores
// the serial order.
cudaError_t CSB_BK(launch_wave_step)(const Model* mp, int ns, const GridDev& g, const WaveBufs& wb,
                                     const double* q, const double* R, const double* cfl,
                                     const double* lamS, const double* domd, int dom_stride,
                                     int per_species, int scheme, double sp_scale, double* qn,
                                     double* dq_std, unsigned long long* flags, cudaStream_t st,
                                     cudaEvent_t* ev) {
  CSB_NS_DISPATCH(ns, {
    const Skew& sk = wb.sk;
    const bool ci = scheme == SCH_CI;
    // coupled operator with chemistry: register chain + dinv records only
    const bool ci_chem = ci && per_species;
    if (ci_chem && (NSB > CI_MAXNSB || !wb.ci_d || !wb.ci_dinv)) return cudaErrorInvalidConfiguration;
    constexpr int NV = 5 + NSB;
    const int nsI = per_species ? NSB : 1;
    const int NSF = nsI + NSB + 2;
    const int WKS = per_species ? wave_wks<NSB, true>() : wave_wks<NSB, false>();
    const int NGC = ci_chem ? ci_ng<NSB, true>() : ci_ng<NSB, false>();
    const int WKC = ci_chem ? ci_wk<NSB, true>() : ci_wk<NSB, false>();
    // large NSB (CI): + the smem-resident chain state (4 x NV x 32 doubles)
    const size_t ci_extra = NSB > CI_MAXNSB ? (size_t)4 * NV * 32 * sizeof(double) : 0;
    int Df = 0, Ds = 0, Dc = 0;
    if (ci) {
      for (int D = 4; D >= 2 && !Dc; --D)
        if (wave_role_smem(D, WKC, NGC, NV) + ci_extra <= WAVE_SMEM_BUDGET) Dc = D;
      if (!Dc) return cudaErrorInvalidConfiguration;
    } else {
      Df = wave_depth(WKF, NFF, 5);
      for (int D = CSB_DMAX; D >= 2 && !Ds; --D)
        if (wave_role_smem(D, WKS, NSF, NSB) <= WAVE_SMEM_BUDGET) Ds = D;
      if (!Df || !Ds) return cudaErrorInvalidConfiguration;
    }
    // ---------------- records tile length C (steps) and shared memory
    int C = 4;  // measured: 4 steps per tile with 4 CTAs/SM beats 8 (1 CTA/SM less)
    if (const char* ev_c = probe_env("CSB_REC_C")) C = atoi(ev_c);  // tuning probe
    auto rsm_of = [&](int c) {
      const int ncp = ci ? 2 + 3 * NV : 16 + nsI + NSB;
      return ((size_t)ncp * c * 32 + 12 * (size_t)(c + 2) * 34) * sizeof(double);
    };
    if (C < 1 || sk.T % C) C = 4;  // a tile length must divide T (T is a multiple of TQ = 16)
    while (C > 1 && rsm_of(C) > 200 * 1024) C /= 2;
    const size_t rsm = rsm_of(C);
    auto krec = ci ? k_records2d<NSB, true> : k_records2d<NSB, false>;
    cudaFuncSetAttribute(krec, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm);
    const int nrec = sk.nstrip * (sk.T / C);
    // serial order (CS and CI): the sliding-window kernel with the longest blocks whose
    // rings fit (measured at config 4, ns = 11: 16-step blocks at 1 CTA/SM
    // 2.48 ms with 4.6 GB of DRAM reads, 8-step blocks at 2 CTAs/SM 2.60 ms
    // with 7.7 GB, 4-step blocks 3.33 ms; tile kernel 3.16 ms), else the tile
    // kernel.  CSB_REC_S = 0 | 4 | 8 | 16 picks one (all parity-tested).
    int CS_ = 0;
    auto ssm_of = [&](int c) -> size_t {
      const bool ps = per_species != 0;
      return c == 16  ? rec_s_smem<NSB, 16>(ps, ci)
             : c == 8 ? rec_s_smem<NSB, 8>(ps, ci)
                      : rec_s_smem<NSB, 4>(ps, ci);
    };
    {
      const size_t cap = 224 * 1024;  // (227 KB per CTA on sm_100)
      // (1024^2: ns = 5 0.249 ms with 8-step blocks at 2 CTAs/SM, 0.271 with 16; ns = 11 0.35 /
      // 0.36; ns = 40 1.34 with 8-step blocks at 1 CTA/SM; tile kernel 0.263 / 0.39 / 1.43)
      CS_ = NSB > 8 && ssm_of(16) <= cap ? 16 : (ssm_of(8) <= cap ? 8 : (ssm_of(4) <= cap ? 4 : 0));
      if (const char* ev_s = getenv("CSB_REC_S")) {
        const int c = atoi(ev_s);
        if (c == 0 || ((c == 4 || c == 8 || c == 16) && ssm_of(c) <= cap)) CS_ = c;
      }
    }
    auto launch_records_s = [&](cudaStream_t s) {
      const int Cs = CS_;
      const size_t ssm = ssm_of(Cs);
      auto ks = ci ? (Cs == 16  ? k_records2d_s<NSB, 16, true>
                      : Cs == 8 ? k_records2d_s<NSB, 8, true>
                                : k_records2d_s<NSB, 4, true>)
                   : (Cs == 16  ? k_records2d_s<NSB, 16, false>
                      : Cs == 8 ? k_records2d_s<NSB, 8, false>
                                : k_records2d_s<NSB, 4, false>);
      const int nt = Cs == 16 ? rec_s_threads<16>() : Cs == 8 ? rec_s_threads<8>() : rec_s_threads<4>();
      cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks, nt, ssm) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      const int G = per_sm * device_sms();
      // chunk count: fewest scheduling rounds x (chunk length + the 2-step prologue)
      int best_nc = 1;
      long long best_cost = -1;
      const int max_nc = sk.T / Cs;
      for (int nc = 1; nc <= max_nc; ++nc) {
        const int Lc = ((sk.T + nc - 1) / nc + Cs - 1) / Cs * Cs;
        if ((long long)Lc * (nc - 1) >= sk.T) continue;  // fewer chunks already cover T
        const long long rounds = ((long long)nc * sk.nstrip + G - 1) / G;
        const long long cost = rounds * (Lc + 2);
        if (best_cost < 0 || cost < best_cost) {
          best_cost = cost;
          best_nc = nc;
        }
      }
      const int Lc = ((sk.T + best_nc - 1) / best_nc + Cs - 1) / Cs * Cs;
      const int nunit = ((sk.T + Lc - 1) / Lc) * sk.nstrip;
      WaveBufs wr = wb;
      wr.rdy = nullptr;
      ks<<<std::min(nunit, G), nt, ssm, s>>>(mp, g, sk, q, R, cfl, lamS, domd, dom_stride,
                                             per_species, sp_scale, wr, Lc, flags);
    };
    auto launch_records = [&](cudaStream_t s, bool publish) {
      WaveBufs wr = wb;
      if (!publish) wr.rdy = nullptr;  // (no per-tile fence when nothing consumes the flags)
      if (!publish && CS_) launch_records_s(s);
      else
      krec<<<nrec, 256, rsm, s>>>(mp, g, sk, q, R, cfl, lamS, domd, dom_stride, per_species,
                                  sp_scale, wr, C, flags);
      if (ci_chem) {
        // dinv = inv(d I - V dOmega) per cell (implicit.py:362-368), into the records
        launch_block_inverse(ns, g.N, domd, wb.ci_d, g.vol, wb.ci_dinv, flags, s);
        note_launches(1);
        k_dinv2d<NSB><<<grid_for((long long)sk.nstrip * sk.T * 32, 256), 256, 0, s>>>(
            g, sk, ns, wb.ci_dinv, wb);
      }
    };
    // ---------------- one sweep
    int only = -1;
    if (const char* ev_o = probe_env("CSB_WAVE_ONLY")) only = atoi(ev_o);  // timing probe
    const long long hrows = (long long)sk.T + 2 * HPAD;
    auto launch_pass = [&](bool bwd, cudaStream_t s, const int* rdy) -> cudaError_t {
      WaveArgs wa{};
      wa.sk = sk;
      wa.ni = g.ni;
      wa.nj = g.nj;
      wa.nsI = ci ? 1 : nsI;
      wa.ci = ci ? 1 : 0;
      wa.only = ci ? -1 : only;
      wa.poll_ns = 16;
      if (const char* ev_p = probe_env("CSB_POLL_NS")) wa.poll_ns = atoi(ev_p);  // tuning probe
      wa.fake_recv = probe_env("CSB_FAKE_RECV") ? 1 : 0;                         // timing probe
      wa.rdy = rdy;
      wa.nonplanar = probe_env("CSB_NO_PLANAR") ? nullptr : wb.nonplanar;  // (tuning probe)
      wa.epoch = wb.epoch;
      wa.rC = C;
      wa.dbg = nullptr;
      static unsigned long long* dbg = nullptr;
      if (probe_env("CSB_WAVE_DBG")) {
        if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 64 * 2 * 4096);
        cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 64 * 2 * sk.nstrip, s);
        wa.dbg = dbg;
      }
      size_t smem;
      int nblk;
      if (ci) {
        WaveRole& rc = wa.role[0];
        rc.in = bwd ? wb.fb : wb.ff;
        rc.ng = NGC;
        rc.D = Dc;
        rc.out = bwd ? wb.fw : wb.fb;
        rc.out2 = bwd ? wb.sw : nullptr;
        rc.ngo = bwd ? 5 : NGC;
        rc.po = bwd ? 0 : 2 + 2 * NV + 8;
        rc.hand = wb.hand + (bwd ? (long long)sk.nstrip * hrows * NV : 0);
        rc.ticket = wb.prog;
        wa.role[1] = rc;
        smem = wave_role_smem(Dc, WKC, NGC, NV) + ci_extra;
        nblk = sk.nstrip;
      } else {
        WaveRole& rf = wa.role[0];
        WaveRole& rs = wa.role[1];
        rf.in = bwd ? wb.fb : wb.ff;
        rf.ng = bwd ? NFB : NFF;
        rf.D = Df;
        rf.out = bwd ? wb.fw : wb.fb;
        rf.out2 = nullptr;
        rf.ngo = bwd ? 5 : NFB;
        rf.po = bwd ? 0 : FB_DQ;
        const long long hsz = (long long)sk.nstrip * hrows * (5 + NSB);  // one sweep
        rf.hand = wb.hand + (bwd ? hsz : 0);
        rf.ticket = wb.prog;
        rs.in = bwd ? wb.sb : wb.sf;
        rs.ng = NSF;
        rs.D = Ds;
        rs.out = bwd ? wb.sw : wb.sb;
        rs.out2 = nullptr;
        rs.ngo = bwd ? NSB : NSF;
        rs.po = bwd ? 0 : nsI + 2;
        rs.hand = wb.hand + (bwd ? hsz : 0) + (long long)sk.nstrip * hrows * 5;
        rs.ticket = wb.prog + 1;
        smem = std::max(wave_role_smem(Df, WKF, NFF, 5), wave_role_smem(Ds, WKS, NSF, NSB));
        nblk = only == 0 || only == 1 ? sk.nstrip
               : only == 4            ? 4 * sk.nstrip
                                      : (2 * sk.nstrip + 3) / 4 * 4;
      }
      auto kfn = bwd ? (per_species ? k_wave2d<NSB, true, true> : k_wave2d<NSB, true, false>)
                     : (per_species ? k_wave2d<NSB, false, true> : k_wave2d<NSB, false, false>);
      cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaMemsetAsync(wb.prog, 0, sizeof(int) * 2, s);
      kfn<<<nblk, wave_threads<NSB>(), smem, s>>>(wa);
      if (wa.dbg) {
        std::vector<unsigned long long> h(64 * 2 * sk.nstrip);
        cudaMemcpyAsync(h.data(), wa.dbg, h.size() * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        unsigned long long tmin = ~0ull;
        for (int e = 0; e < 2 * sk.nstrip; ++e)
          if (h[64 * e]) tmin = std::min(tmin, h[64 * e]);
        for (int e = 0; e < 2 * sk.nstrip; ++e)
          if (h[64 * e]) {
            const unsigned long long* d = &h[64 * e];
            fprintf(stderr,
                    "wave%s strip %d kind %d: start %.2f end %.2f chain_wait %.2f recv_poll %.2f "
                    "prod_wait %.2f stamps",
                    bwd ? "B" : "F", e / 2, e % 2, (d[0] - tmin) * 1e-3, (d[1] - tmin) * 1e-3,
                    d[2] * 1e-3, d[3] * 1e-3, d[60] * 1e-3);
            for (int q = 4; q < 60 && d[q]; ++q) fprintf(stderr, " %.1f", (d[q] - tmin) * 1e-3);
            fprintf(stderr, "\n");
          }
      }
      return cudaGetLastError();
    };
    // ---------------- the step
    note_launches(2);
    k_epoch_bump<<<1, 1, 0, st>>>(wb.epoch);  // fresh tag for this step (graph replays too)
    k_hand_reset<<<grid_for(std::max(4LL * sk.nstrip * hrows, g.N), 256), 256, 0, st>>>(
        wb.hand, sk.nstrip, sk.T, ci ? NV : 5, ci ? 0 : NSB, g.N, q + 3 * g.N, R + 3 * g.N,
        wb.nonplanar, wb.epoch);
    // measured: the overlap pays while the sweeps hold a small share of the
    // SMs (512^2: 32 of 148 SMs, 0.649 -> 0.587 ms per iteration); at 1024^2
    // (64 SMs) the concurrent records tiles slow the chains more than they hide
    // (2.23 -> 2.35 ms at ns = 11)
    // The sweep CTAs (one per SM: ~200 KB of shared memory each) spin on the
    // records tiles, so the records kernel must keep SMs of its own: the
    // overlap is used while the sweeps hold at most a third of the device
    // (48 of 148 SMs on B200), forced overlap only while 8 SMs stay free.
    // (the threshold counts 2 CTAs per strip for CI too, as measured)
    const int sms = device_sms();
    const int nsweep = ci ? sk.nstrip : 2 * sk.nstrip;
    const bool overlap = !ev && wb.s2 && !wb.serial && !ci_chem && only == -1 &&
                         (2 * sk.nstrip <= sms * 48 / 148 ||
                          (getenv("CSB_FORCE_OVERLAP") && nsweep <= sms - 8)) &&
                         !getenv("CSB_NO_OVERLAP");
    cudaError_t e;
    if (overlap) {
      // the records kernel is submitted FIRST: the sweep only ever waits for
      // a kernel that is already running or queued ahead of it, so the step
      // cannot deadlock even where kernels are serialised (ncu replay,
      // CUDA_LAUNCH_BLOCKING) -- it then simply runs in the serial order
      cudaEventRecord(wb.e1, st);
      launch_records(st, true);
      cudaStreamWaitEvent(wb.s2, wb.e1, 0);
      e = launch_pass(false, wb.s2, wb.rdy);
      if (e != cudaSuccess) return e;
      cudaEventRecord(wb.e2, wb.s2);
      cudaStreamWaitEvent(st, wb.e2, 0);
    } else {
      if (ev) cudaEventRecord(ev[0], st);
      launch_records(st, false);
      if (ev) cudaEventRecord(ev[1], st);
      e = launch_pass(false, st, nullptr);
      if (e != cudaSuccess) return e;
      if (ev) cudaEventRecord(ev[2], st);
    }
    e = launch_pass(true, st, nullptr);
    if (e != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[3], st);
    // ---------------- epilogue (persistent grid over strip x column tiles)
    {
      // warps per CTA = columns per tile: 8 with two tile buffers while they
      // stay within ~100 KB (2 CTAs per SM), one buffer above (ns > 19),
      // fewer columns as the last resort (ns > 45)
      int CE = 8, nbuf = 2;
      auto esm_of = [&](int ce, int nb) { return (size_t)nb * (5 + ns) * ce * 32 * sizeof(double); };
      // (measured at 1024^2: ns = 20 one buffer 0.182 vs two 0.199 ms; ns = 5 / 11 equal)
      if (esm_of(CE, 2) > 96 * 1024) nbuf = 1;
      while (CE > 2 && esm_of(CE, nbuf) > 100 * 1024) CE /= 2;
      const size_t esm = esm_of(CE, nbuf);
      auto kepi = k_epilogue2d<NSB>;
      cudaFuncSetAttribute(kepi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esm);
      static int per_sm = 0;  // (per bucket instantiation; CE and esm depend on ns only)
      static int per_sm_ns = -1;
      if (per_sm_ns != ns) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kepi, CE * 32, esm);
        per_sm_ns = ns;
      }
      const long long ntile = (long long)sk.nstrip * ((g.ni + CE - 1) / CE);
      const int nblk = (int)std::min<long long>(ntile, (long long)sms * std::max(per_sm, 1));
      kepi<<<nblk, CE * 32, esm, st>>>(mp, g, sk, scheme, q, wb.fw, wb.sw, qn, dq_std, nbuf, flags);
    }
    if (ev) cudaEventRecord(ev[4], st);
  });
  return cudaGetLastError();
}

}  // namespace csb
