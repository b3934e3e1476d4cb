// csflow-b200: explicit residual R (V dQ/dt = -R), reference spatial.py:207-274.
//
// One CTA owns a TI x TJ x TK tile of cells.  It stages the decoded
// primitives of the tile plus a 2-cell halo in shared memory (SoA, one
// plane per component), evaluating boundary ghosts on the fly with the
// reference's face-by-face fill order (boundary.py:53-114, see ghost_value),
// then computes each face flux of the tile exactly once per direction
// (MUSCL-minmod + Rusanov + central viscous, spatial.py:217-256) into a
// shared flux buffer and differences it into R in direction order 0, 1, 2.
//
// K2D: nk == 1 with a k-boundary pair whose k-face fluxes and k tangential
// differences cancel bit-exactly (outflow/outflow, periodic/periodic, or
// symmetry/symmetry with w == 0).  The k layers are then neither
// staged nor evaluated.  Any cell with w != 0 under symmetry raises
// EB_KSKIP so the host can recompute with the general path.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// ----------------------------------------------------------------------------
// ghost evaluation
// ----------------------------------------------------------------------------

// last fill op (index a*4 + side*2 + g-1, the reference's loop order) with
// index < t that writes padded cell p; -1 if none.
CSB_DEV int last_op(const int p[3], const int n[3], int t) {
  int best = -1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int side, g;
    if (p[a] < NG) {
      side = 0;
      g = NG - p[a];
    } else if (p[a] >= n[a] + NG) {
      side = 1;
      g = p[a] - (n[a] + NG) + 1;
    } else {
      continue;
    }
    const int o = a * 4 + side * 2 + (g - 1);
    if (o < t && o > best) best = o;
  }
  return best;
}

// Value of padded cell (pi, pj, pk) after the full ghost fill, as the
// composition of the per-face formulas applied to one interior source cell
// (or the freestream, or NaN for a ghost the reference never fills).
// out[0..nc) in padded layout [rho, u, v, w, p, Y.., T].
template <int NSB>
CSB_DEV void padded_value(const Model& m, const GridDev& g, const BCDev& bc,
                          const double* __restrict__ q, int pi, int pj, int pk, double* out,
                          unsigned long long* flags) {
  const int ns = m.ns;
  const int nc = 6 + ns;
  int p[3] = {pi, pj, pk};
  const int n[3] = {g.ni, g.nj, g.nk};
  int op_list[12];
  int op_pos[12][3];
  int nops = 0;
  int t = 12;
  int base_kind = 0;  // 0 interior decode, 1 NaN, 2 farfield of face base_face
  int base_face = 0;
  while (true) {
    const int o = last_op(p, n, t);
    if (o < 0) break;
    const int a = o >> 2, side = (o >> 1) & 1, gg = (o & 1) + 1;
    const int face = a * 2 + side;
    const int kind = bc.kind[face];
    if (kind == BC_FARFIELD) {
      base_kind = 2;
      base_face = face;
      break;
    }
    if (kind == BC_WALL || kind == BC_SYMMETRY) {
      op_list[nops] = o;
      op_pos[nops][0] = p[0];
      op_pos[nops][1] = p[1];
      op_pos[nops][2] = p[2];
      ++nops;
    }
    int src;
    if (kind == BC_OUTFLOW) src = side == 0 ? NG : n[a] + NG - 1;
    else if (kind == BC_PERIODIC) src = side == 0 ? NG + n[a] - gg : NG + gg - 1;
    else src = side == 0 ? NG + gg - 1 : NG + n[a] - gg;
    p[a] = src;
    t = o;
  }
  if (base_kind == 0) {
    const bool interior = p[0] >= NG && p[0] < n[0] + NG && p[1] >= NG && p[1] < n[1] + NG &&
                          p[2] >= NG && p[2] < n[2] + NG;
    if (!interior) base_kind = 1;
  }
  if (base_kind == 1) {
    for (int c = 0; c < nc; ++c) out[c] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  if (base_kind == 2) {
    const double* fs = bc.fs + (long long)base_face * nc;
    for (int c = 0; c < nc; ++c) out[c] = __ldg(fs + c);
  } else {
    const long long cell = cell_index(g, p[0] - NG, p[1] - NG, p[2] - NG);
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + cell, g.N, cs)) raise_flag(flags, EB_DECODE, cell);
    out[0] = cs.rho;
    out[1] = cs.u[0];
    out[2] = cs.u[1];
    out[3] = cs.u[2];
    out[4] = cs.p;
#pragma unroll
    for (int s = 0; s < NSB; ++s)
      if (s < ns) out[5 + s] = cs.Y[s];
    out[5 + ns] = cs.T;
  }
  // apply the recorded transforms innermost first
  for (int r = nops - 1; r >= 0; --r) {
    const int o = op_list[r];
    const int a = o >> 2, side = (o >> 1) & 1;
    const int face = a * 2 + side;
    if (bc.kind[face] == BC_WALL) {
      const double Tw = bc.Tw[face];
      out[1] = -out[1];
      out[2] = -out[2];
      out[3] = -out[3];
      const double Tg = npmax(2.0 * Tw - out[5 + ns], 0.1 * Tw);
      double R = 0.0;
      for (int s = 0; s < ns; ++s) R += out[5 + s] * m.Rs[s];
      out[5 + ns] = Tg;
      out[0] = out[4] / (R * Tg);
    } else {  // symmetry
      double nh[3];
      if (bc.axis[face] >= 0) {
        nh[0] = nh[1] = nh[2] = 0.0;
        nh[bc.axis[face]] = 1.0;
      } else {
        int t3[3];
        for (int x = 0; x < 3; ++x) {
          int v = op_pos[r][x] - NG;
          v = v < 0 ? 0 : (v > n[x] - 1 ? n[x] - 1 : v);
          t3[x] = v;
        }
        t3[a] = side == 0 ? 0 : n[a];
        double S[3];
        load_S(g, a, face_index(g, a, t3[0], t3[1], t3[2]), S);
        const double nrm = sqrt((S[0] * S[0] + S[1] * S[1]) + S[2] * S[2]);
        nh[0] = S[0] / nrm;
        nh[1] = S[1] / nrm;
        nh[2] = S[2] / nrm;
      }
      const double un = (out[1] * nh[0] + out[2] * nh[1]) + out[3] * nh[2];
      const double tu = 2.0 * un;
      out[1] = out[1] - tu * nh[0];
      out[2] = out[2] - tu * nh[1];
      out[3] = out[3] - tu * nh[2];
    }
  }
}

// ----------------------------------------------------------------------------
// face flux
// ----------------------------------------------------------------------------

struct FaceGeom {
  double S[3];
  double xn[3];      // S / Vf
  double xt[2][3];   // face-averaged Sc_a * J for the two tangential axes (ascending)
  int ta[2];         // tangential axis ids
  int use_t[2];      // 0: skip (K2D k axis)
};

// Face state from W = [rho, u, p, Y] (spatial.py:42-66); returns false if
// the face temperature is non-positive or non-finite.
template <int NSB>
CSB_DEV bool face_state(const Model& m, const double* W, double& T, double& c, double& et) {
  double R = 0.0, cp = 0.0, yb = 0.0;
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < m.ns) {
      R += W[5 + s] * m.Rs[s];
      cp += W[5 + s] * m.cp[s];
      yb += W[5 + s] * m.bs[s];
    }
  }
  T = W[4] / (W[0] * R);
  const bool ok = (T > 0.0) && finite(T);
  const double gamma = cp / (cp - R);
  c = sqrt(gamma * R * T);
  const double Ek = 0.5 * ((W[1] * W[1] + W[2] * W[2]) + W[3] * W[3]);
  et = yb + (cp - R) * T + Ek;
  return ok;
}

// face_state with the species sums R = sum Y_s R_s, cp = sum Y_s cp_s,
// yb = sum Y_s b_s supplied by the caller (accumulated in species order from
// 0, i.e. bit-identical to face_state's own loop)
CSB_DEV bool face_state_sums(double W0, double W1, double W2, double W3, double W4, double R,
                             double cp, double yb, double& T, double& c, double& et) {
  T = W4 / (W0 * R);
  const bool ok = (T > 0.0) && finite(T);
  const double gamma = cp / (cp - R);
  c = sqrt(gamma * R * T);
  const double Ek = 0.5 * ((W1 * W1 + W2 * W2) + W3 * W3);
  et = yb + (cp - R) * T + Ek;
  return ok;
}

// MUSCL-minmod face values of staged component c (spatial.py:217-226)
CSB_DEV void muscl_pair(const double* sP, int ldP, int imm, int im, int ip, int ipp, int c,
                        bool first_order, double& l, double& r) {
  const double vm = sP[c * ldP + im];
  const double vp = sP[c * ldP + ip];
  if (first_order) {
    l = vm;
    r = vp;
  } else {
    const double vmm = sP[c * ldP + imm];
    const double vpp = sP[c * ldP + ipp];
    const double dc = vp - vm;
    l = vm + 0.5 * minmod(vm - vmm, dc);
    r = vp - 0.5 * minmod(dc, vpp - vp);
  }
}

// Large species counts (NSB > CSB_STREAM_MIN): the face passes stream the species
// instead of holding 2 x (5 + NSB) face values in registers (which spilled:
// ns = 40 residual 6.7 ms per 10^6 cells); species values are recomputed per
// pass from shared memory with the same arithmetic, so results are identical.
#ifndef CSB_STREAM_MIN
#define CSB_STREAM_MIN 8  // measured: streaming from NSB = 12 up, config-4 residual 6.46 -> 4.67 ms
#endif
template <int NSB>
constexpr bool stream_species() { return NSB > CSB_STREAM_MIN; }

// Face flux = convective part (face_conv, writes F) + viscous part
// (face_visc, adds to F), evaluated in two passes so that their register
// footprints do not add up.  sP: staged padded primitives, component plane
// stride ldP; cell offsets im/ip (the two adjacent cells), imm/ipp (MUSCL
// outer cells), tangential strides st[2].

// Convective part: Rusanov on MUSCL-minmod states (spatial.py:217-226,
// rusanov_flux 171-204).
template <int NSB>
CSB_DEV bool face_conv(const Model& m, const double* sP, int ldP, int imm, int im, int ip, int ipp,
                       const double S[3], bool first_order, double* F, int ldF) {
  const int ns = m.ns;
  const int nv = 5 + ns;
  bool ok = true;
  if constexpr (stream_species<NSB>()) {
    double WL[5], WR[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) muscl_pair(sP, ldP, imm, im, ip, ipp, c, first_order, WL[c], WR[c]);
    double RL = 0.0, cpL = 0.0, ybL = 0.0, RR = 0.0, cpR = 0.0, ybR = 0.0;
    for (int sp = 0; sp < ns; ++sp) {
      double yl, yr;
      muscl_pair(sP, ldP, imm, im, ip, ipp, 5 + sp, first_order, yl, yr);
      RL += yl * m.Rs[sp];
      cpL += yl * m.cp[sp];
      ybL += yl * m.bs[sp];
      RR += yr * m.Rs[sp];
      cpR += yr * m.cp[sp];
      ybR += yr * m.bs[sp];
    }
    double TL, cL, eL, TR, cR, eR;
    ok &= face_state_sums(WL[0], WL[1], WL[2], WL[3], WL[4], RL, cpL, ybL, TL, cL, eL);
    ok &= face_state_sums(WR[0], WR[1], WR[2], WR[3], WR[4], RR, cpR, ybR, TR, cR, eR);
    const double UL = WL[1] * S[0] + WL[2] * S[1] + WL[3] * S[2];
    const double UR = WR[1] * S[0] + WR[2] * S[1] + WR[3] * S[2];
    const double area = sqrt((S[0] * S[0] + S[1] * S[1]) + S[2] * S[2]);
    const double lam = npmax(fabs(UL) + cL * area, fabs(UR) + cR * area);
    const double hl = 0.5 * lam;
    {
      const double qL = WL[0], qR = WR[0];
      F[0] = 0.5 * (UL * qL + UR * qR) - hl * (qR - qL);
    }
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const double qL = WL[0] * WL[1 + x], qR = WR[0] * WR[1 + x];
      const double fl = UL * qL + WL[4] * S[x];
      const double fr = UR * qR + WR[4] * S[x];
      F[(1 + x) * ldF] = 0.5 * (fl + fr) - hl * (qR - qL);
    }
    {
      const double qL = WL[0] * eL, qR = WR[0] * eR;
      const double fl = UL * qL + WL[4] * UL;
      const double fr = UR * qR + WR[4] * UR;
      F[4 * ldF] = 0.5 * (fl + fr) - hl * (qR - qL);
    }
    for (int sp = 0; sp < ns; ++sp) {
      double yl, yr;
      muscl_pair(sP, ldP, imm, im, ip, ipp, 5 + sp, first_order, yl, yr);
      const double qL = WL[0] * yl, qR = WR[0] * yr;
      F[(5 + sp) * ldF] = 0.5 * (UL * qL + UR * qR) - hl * (qR - qL);
    }
    return ok;
  }
  double WL[5 + NSB], WR[5 + NSB];
#pragma unroll
  for (int c = 0; c < 5 + NSB; ++c) {
    if (c < nv) {
      const double vm = sP[c * ldP + im];
      const double vp = sP[c * ldP + ip];
      if (first_order) {
        WL[c] = vm;
        WR[c] = vp;
      } else {
        const double vmm = sP[c * ldP + imm];
        const double vpp = sP[c * ldP + ipp];
        const double dc = vp - vm;
        WL[c] = vm + 0.5 * minmod(vm - vmm, dc);
        WR[c] = vp - 0.5 * minmod(dc, vpp - vp);
      }
    } else {
      WL[c] = WR[c] = 0.0;
    }
  }
  double TL, cL, eL, TR, cR, eR;
  ok &= face_state<NSB>(m, WL, TL, cL, eL);
  ok &= face_state<NSB>(m, WR, TR, cR, eR);
  const double UL = WL[1] * S[0] + WL[2] * S[1] + WL[3] * S[2];
  const double UR = WR[1] * S[0] + WR[2] * S[1] + WR[3] * S[2];
  const double area = sqrt((S[0] * S[0] + S[1] * S[1]) + S[2] * S[2]);
  const double lam = npmax(fabs(UL) + cL * area, fabs(UR) + cR * area);
  const double hl = 0.5 * lam;
  {
    const double qL = WL[0], qR = WR[0];
    F[0] = 0.5 * (UL * qL + UR * qR) - hl * (qR - qL);
  }
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    const double qL = WL[0] * WL[1 + x], qR = WR[0] * WR[1 + x];
    const double fl = UL * qL + WL[4] * S[x];
    const double fr = UR * qR + WR[4] * S[x];
    F[(1 + x) * ldF] = 0.5 * (fl + fr) - hl * (qR - qL);
  }
  {
    const double qL = WL[0] * eL, qR = WR[0] * eR;
    const double fl = UL * qL + WL[4] * UL;
    const double fr = UR * qR + WR[4] * UR;
    F[4 * ldF] = 0.5 * (fl + fr) - hl * (qR - qL);
  }
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      const double qL = WL[0] * WL[5 + s], qR = WR[0] * WR[5 + s];
      F[(5 + s) * ldF] = 0.5 * (UL * qL + UR * qR) - hl * (qR - qL);
    }
  }
  return ok;
}

// Gradient of staged component c at the face, in the reference's summation
// order: grad = grads[0] + grads[1] + grads[2] with grads[d] the part along
// axis d (spatial.py:227-248).
CSB_DEV void face_grad(const double* sP, int ldP, int im, int ip, const int st[2],
                       const FaceGeom& fg, int c, double g[3]) {
  const double dn = sP[c * ldP + ip] - sP[c * ldP + im];
  double part[3][3];
  int filled[3] = {0, 0, 0};
  const int d = 3 - fg.ta[0] - fg.ta[1];  // normal axis
#pragma unroll
  for (int x = 0; x < 3; ++x) part[d][x] = dn * fg.xn[x];
  filled[d] = 1;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int a = fg.ta[t];
    if (fg.use_t[t]) {
      const int s = st[t];
      const double cdm = 0.5 * (sP[c * ldP + im + s] - sP[c * ldP + im - s]);
      const double cdp = 0.5 * (sP[c * ldP + ip + s] - sP[c * ldP + ip - s]);
      const double dP = 0.5 * (cdm + cdp);
#pragma unroll
      for (int x = 0; x < 3; ++x) part[a][x] = dP * fg.xt[t][x];
      filled[a] = 1;
    }
  }
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    double v = filled[0] ? part[0][x] : 0.0;
    v = filled[1] ? (filled[0] ? v + part[1][x] : part[1][x]) : v;
    v = filled[2] ? ((filled[0] || filled[1]) ? v + part[2][x] : part[2][x]) : v;
    g[x] = v;
  }
}

// Viscous part (spatial.py:227-256, viscous_flux 143-168), added to F.
// The species diffusion fluxes are formed twice (once for their zero-sum
// correction, once for the fluxes) instead of being kept in registers.
template <int NSB>
CSB_DEV bool face_visc(const Model& m, const double* sP, int ldP, int im, int ip, const int st[2],
                       const FaceGeom& fg, double* F, int ldF) {
  const int ns = m.ns;
  const int nv = 5 + ns;
  const int iT = 5 + ns;
  double Wf[5 + NSB];
#pragma unroll
  for (int c = 0; c < 5 + NSB; ++c) Wf[c] = c < nv ? 0.5 * (sP[c * ldP + im] + sP[c * ldP + ip]) : 0.0;
  double Tf, cf, ef;
  const bool ok = face_state<NSB>(m, Wf, Tf, cf, ef);
  const double rho = Wf[0];
  double mu, kc, D;
  transport<NSB>(m, Tf, Wf + 5, rho, mu, kc, D);
  const double* S = fg.S;
  double tS[3];
  {
    double gu[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) face_grad(sP, ldP, im, ip, st, fg, 1 + i, gu[i]);
    const double div = (gu[0][0] + gu[1][1]) + gu[2][2];
    const double tdiv = 2.0 / 3.0 * mu * div;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        double tau = mu * (gu[i][x] + gu[x][i]);
        if (x == i) tau -= tdiv;
        acc = (x == 0) ? tau * S[0] : acc + tau * S[x];
      }
      tS[i] = acc;
    }
  }
  // species diffusion with zero-sum correction
  const double nrd = -(rho * D);
  double jsum[3] = {0.0, 0.0, 0.0};
  for (int s = 0; s < ns; ++s) {
    double gy[3];
    face_grad(sP, ldP, im, ip, st, fg, 5 + s, gy);
#pragma unroll
    for (int x = 0; x < 3; ++x) jsum[x] += nrd * gy[x];
  }
  double hsj[3] = {0.0, 0.0, 0.0};
  for (int s = 0; s < ns; ++s) {
    double gy[3], js[3];
    face_grad(sP, ldP, im, ip, st, fg, 5 + s, gy);
    const double hs = m.bs[s] + m.cp[s] * Tf;
    const double ys = sP[(5 + s) * ldP + im], yp = sP[(5 + s) * ldP + ip];
    const double yf = 0.5 * (ys + yp);
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      js[x] = nrd * gy[x] - yf * jsum[x];
      hsj[x] += hs * js[x];
    }
    F[(5 + s) * ldF] += (js[0] * S[0] + js[1] * S[1]) + js[2] * S[2];
  }
  double gT[3];
  face_grad(sP, ldP, im, ip, st, fg, iT, gT);
  double qv[3];
#pragma unroll
  for (int x = 0; x < 3; ++x) qv[x] = -kc * gT[x] + hsj[x];
  F[1 * ldF] += -tS[0];
  F[2 * ldF] += -tS[1];
  F[3 * ldF] += -tS[2];
  const double utS = (Wf[1] * tS[0] + Wf[2] * tS[1]) + Wf[3] * tS[2];
  const double qS = (qv[0] * S[0] + qv[1] * S[1]) + qv[2] * S[2];
  F[4 * ldF] += -utS + qS;
  return ok;
}

// 2-D (K2D) viscous face of direction D (0: i-face, 1: j-face): the same
// arithmetic as face_grad/face_visc with the axis bookkeeping resolved at
// compile time.  grad = part_0 + part_1 (axis order), the normal part along
// axis D and the central tangential part along the other in-plane axis.
template <int D>
CSB_DEV void face_grad2d(const double* sP, int ldP, int im, int ip, int st, const double xn[3],
                         const double xt[3], int c, double g[3]) {
  const double dn = sP[c * ldP + ip] - sP[c * ldP + im];
  const double cdm = 0.5 * (sP[c * ldP + im + st] - sP[c * ldP + im - st]);
  const double cdp = 0.5 * (sP[c * ldP + ip + st] - sP[c * ldP + ip - st]);
  const double dP = 0.5 * (cdm + cdp);
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    const double pn = dn * xn[x], pt = dP * xt[x];
    g[x] = D == 0 ? pn + pt : pt + pn;
  }
}

template <int NSB, int D>
CSB_DEV bool face_visc2d(const Model& m, const double* sP, int ldP, int im, int ip, int st,
                         const double S[3], const double xn[3], const double xt[3], double* F,
                         int ldF) {
  const int ns = m.ns;
  const int nv = 5 + ns;
  if constexpr (stream_species<NSB>()) {
    auto wf = [&](int c) { return 0.5 * (sP[c * ldP + im] + sP[c * ldP + ip]); };
    const double W0 = wf(0), W1 = wf(1), W2 = wf(2), W3 = wf(3), W4 = wf(4);
    double R = 0.0, cpf = 0.0, yb = 0.0;
    for (int sp = 0; sp < ns; ++sp) {
      const double y = wf(5 + sp);
      R += y * m.Rs[sp];
      cpf += y * m.cp[sp];
      yb += y * m.bs[sp];
    }
    double Tf, cf, ef;
    const bool ok = face_state_sums(W0, W1, W2, W3, W4, R, cpf, yb, Tf, cf, ef);
    const double rho = W0;
    // transport (mixture.py:354-372) with the species streamed; cp is the
    // same species sum as the face state's
    double acc = 0.0;
    if (m.suth_shared) {
      const double xx = Tf * m.inv_T_mu[0];
      const double Fs = (xx * sqrt(xx)) * m.TS[0] / (Tf + m.S_mu[0]);
      for (int sp = 0; sp < ns; ++sp) acc += wf(5 + sp) * (m.mu_ref[sp] * Fs);
    } else {
      for (int sp = 0; sp < ns; ++sp) acc += wf(5 + sp) * mu_species(m, sp, Tf);
    }
    const double mu = acc, kc = mu * cpf / m.Pr, Dm = mu / (rho * m.Sc);
    double tS[3];
    {
      double gu[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i) face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 1 + i, gu[i]);
      const double div = (gu[0][0] + gu[1][1]) + gu[2][2];
      const double tdiv = 2.0 / 3.0 * mu * div;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double a = 0.0;
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          double tau = mu * (gu[i][x] + gu[x][i]);
          if (x == i) tau -= tdiv;
          a = (x == 0) ? tau * S[0] : a + tau * S[x];
        }
        tS[i] = a;
      }
    }
    const double nrd = -(rho * Dm);
    double jsum[3] = {0.0, 0.0, 0.0};
    for (int sp = 0; sp < ns; ++sp) {
      double gy[3];
      face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + sp, gy);
#pragma unroll
      for (int x = 0; x < 3; ++x) jsum[x] += nrd * gy[x];
    }
    double hsj[3] = {0.0, 0.0, 0.0};
    for (int sp = 0; sp < ns; ++sp) {
      double gy[3], js[3];
      face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + sp, gy);
      const double hs = m.bs[sp] + m.cp[sp] * Tf;
      const double y = wf(5 + sp);
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        js[x] = nrd * gy[x] - y * jsum[x];
        hsj[x] += hs * js[x];
      }
      F[(5 + sp) * ldF] += (js[0] * S[0] + js[1] * S[1]) + js[2] * S[2];
    }
    double gT[3];
    face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + ns, gT);
    double qv[3];
#pragma unroll
    for (int x = 0; x < 3; ++x) qv[x] = -kc * gT[x] + hsj[x];
    F[1 * ldF] += -tS[0];
    F[2 * ldF] += -tS[1];
    F[3 * ldF] += -tS[2];
    const double utS = (W1 * tS[0] + W2 * tS[1]) + W3 * tS[2];
    const double qS = (qv[0] * S[0] + qv[1] * S[1]) + qv[2] * S[2];
    F[4 * ldF] += -utS + qS;
    return ok;
  }
  double Wf[5 + NSB];
#pragma unroll
  for (int c = 0; c < 5 + NSB; ++c) Wf[c] = c < nv ? 0.5 * (sP[c * ldP + im] + sP[c * ldP + ip]) : 0.0;
  double Tf, cf, ef;
  const bool ok = face_state<NSB>(m, Wf, Tf, cf, ef);
  const double rho = Wf[0];
  double mu, kc, Dm;
  transport<NSB>(m, Tf, Wf + 5, rho, mu, kc, Dm);
  double tS[3];
  {
    double gu[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 1 + i, gu[i]);
    const double div = (gu[0][0] + gu[1][1]) + gu[2][2];
    const double tdiv = 2.0 / 3.0 * mu * div;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        double tau = mu * (gu[i][x] + gu[x][i]);
        if (x == i) tau -= tdiv;
        acc = (x == 0) ? tau * S[0] : acc + tau * S[x];
      }
      tS[i] = acc;
    }
  }
  const double nrd = -(rho * Dm);
  double jsum[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      double gy[3];
      face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + s, gy);
#pragma unroll
      for (int x = 0; x < 3; ++x) jsum[x] += nrd * gy[x];
    }
  }
  double hsj[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      double gy[3], js[3];
      face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + s, gy);
      const double hs = m.bs[s] + m.cp[s] * Tf;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        js[x] = nrd * gy[x] - Wf[5 + s] * jsum[x];
        hsj[x] += hs * js[x];
      }
      F[(5 + s) * ldF] += (js[0] * S[0] + js[1] * S[1]) + js[2] * S[2];
    }
  }
  double gT[3];
  face_grad2d<D>(sP, ldP, im, ip, st, xn, xt, 5 + ns, gT);
  double qv[3];
#pragma unroll
  for (int x = 0; x < 3; ++x) qv[x] = -kc * gT[x] + hsj[x];
  F[1 * ldF] += -tS[0];
  F[2 * ldF] += -tS[1];
  F[3 * ldF] += -tS[2];
  const double utS = (Wf[1] * tS[0] + Wf[2] * tS[1]) + Wf[3] * tS[2];
  const double qS = (qv[0] * S[0] + qv[1] * S[1]) + qv[2] * S[2];
  F[4 * ldF] += -utS + qS;
  return ok;
}

// 2-D (K2D) face flux, convective + viscous in one evaluation (the same
// formulas as face_conv + face_visc2d, spatial.py:217-256 and 143-204, with
// the species sums factored so that every species is visited twice instead
// of five times):
//   pass 1 per species: MUSCL states y_L, y_R, face average y_f, normal and
//     tangential differences dn, dP (the gradient is g = dn xn + dP xt), and
//     the sums the face states, the viscosity and the diffusion correction
//     need (sum y R_s, sum y cp_s, sum y b_s on L / R / f, sum y_f mu_ref,
//     sum dn, sum dP, sum b_s dn, ...);
//   pass 2 per species: F_s = y_L C_L + y_R C_R + (-rho D)(g_s . S) - y_f (j . S)
//     with C_L = rho_L (U_L / 2 + lam / 2), C_R = rho_R (U_R / 2 - lam / 2).
// Sums are reassociated against the reference (differences of a few ulp of the
// flux; the parity tests bound R at 1e-10 relative).  PL: planar flow (w == 0
// in every staged cell, checked by the caller): the z components, which are
// exactly zero on a K2D grid (k_check_2d), are not evaluated.
#ifndef CSB_FLUX_UNROLL
#define CSB_FLUX_UNROLL 4  // measured at config 4: 1 3.60, 2 3.58, 4 3.47 ms
#endif
constexpr int FLUX_UNROLL = CSB_FLUX_UNROLL;  // species loops of face_flux2d
#ifndef CSB_FLUX_1DIV
#define CSB_FLUX_1DIV 1
#endif
// face_state_sums with one division: T = p cv / (rho R cv), c^2 = gamma R T =
// cp p R / (rho R cv) (2-3 ulp from the two-division form)
CSB_DEV bool face_state_1div(double W0, double W1, double W2, double W3, double W4, double R,
                             double cp, double yb, double& c, double& et) {
  const double cv = cp - R;
  const double iden = 1.0 / ((W0 * R) * cv);
  const double T = (W4 * cv) * iden;
  const bool ok = (T > 0.0) && finite(T);
  c = sqrt((cp * W4) * (R * iden));
  const double Ek = 0.5 * ((W1 * W1 + W2 * W2) + W3 * W3);
  et = yb + cv * T + Ek;
  return ok;
}
template <int NSB, int D, bool PL>
CSB_DEV bool face_flux2d(const Model& m, const double* sP, int ldP, int im, int ip, int sd, int st,
                         const double* S, const double* xn, const double* xt, bool first_order,
                         double* F, int ldF) {
  constexpr int NX = PL ? 2 : 3;
  const int ns = m.ns;
  const int imm = im - sd, ipp = ip + sd;
  // PL: the caller's staged planes and flux planes have no w component
  // (plane 3 dropped): planes >= 4 sit one plane lower
  const double* sQ = PL ? sP - ldP : sP;
  double* Fq = PL ? F - ldF : F;
  double XNS = 0.0, XTS = 0.0, a2 = 0.0;
#pragma unroll
  for (int x = 0; x < NX; ++x) {
    XNS += xn[x] * S[x];
    XTS += xt[x] * S[x];
    a2 += S[x] * S[x];
  }
  // tangential central difference of component c, face-averaged (spatial.py:241-248)
  auto tang = [&](int c) {
    const double* p = (c >= 4 ? sQ : sP) + c * ldP;
    return 0.5 * (0.5 * (p[im + st] - p[im - st]) + 0.5 * (p[ip + st] - p[ip - st]));
  };
  // ---- flow components: MUSCL states, face averages, velocity gradients
  double WL[5], WR[5], Wf[5];
  double tSm[NX];  // (tau . S) / mu
  {
    double gu[NX][NX];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      if (PL && c == 3) {
        WL[c] = WR[c] = Wf[c] = 0.0;
        continue;
      }
      const double* p = (c >= 4 ? sQ : sP) + c * ldP;
      const double vm = p[im], vp = p[ip];
      const double dc = vp - vm;
      if (first_order) {
        WL[c] = vm;
        WR[c] = vp;
      } else {
        WL[c] = vm + 0.5 * minmod(vm - p[imm], dc);
        WR[c] = vp - 0.5 * minmod(dc, p[ipp] - vp);
      }
      Wf[c] = 0.5 * (vm + vp);
      if (c >= 1 && c <= NX) {
        const double dP = tang(c);
#pragma unroll
        for (int x = 0; x < NX; ++x) gu[c - 1][x] = dc * xn[x] + dP * xt[x];
      }
    }
    double div = 0.0;
#pragma unroll
    for (int i = 0; i < NX; ++i) div += gu[i][i];
    const double td = 2.0 / 3.0 * div;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      double acc = -td * S[i];
#pragma unroll
      for (int x = 0; x < NX; ++x) acc += (gu[i][x] + gu[x][i]) * S[x];
      tSm[i] = acc;
    }
  }
  double GTS;  // grad T . S
  {
    const double* p = sQ + (5 + ns) * ldP;
    GTS = (p[ip] - p[im]) * XNS + tang(5 + ns) * XTS;
  }
  // ---- species pass 1
  double RL = 0.0, cpL = 0.0, ybL = 0.0, RR = 0.0, cpR = 0.0, ybR = 0.0;
  double Rf = 0.0, cpf = 0.0, ybf = 0.0, mua = 0.0;
  double Sdn = 0.0, SdP = 0.0, Bdn = 0.0, BdP = 0.0, Cdn = 0.0, CdP = 0.0;
#pragma unroll FLUX_UNROLL
  for (int sp = 0; sp < ns; ++sp) {
    const double* p = sQ + (5 + sp) * ldP;
    const double vm = p[im], vp = p[ip];
    const double dc = vp - vm;
    double yl = vm, yr = vp;
    if (!first_order) {
      yl = vm + 0.5 * minmod(vm - p[imm], dc);
      yr = vp - 0.5 * minmod(dc, p[ipp] - vp);
    }
    const double yf = 0.5 * (vm + vp);
    const double dP = 0.5 * (0.5 * (p[im + st] - p[im - st]) + 0.5 * (p[ip + st] - p[ip - st]));
    const double Rs = m.Rs[sp], cps = m.cp[sp], bs = m.bs[sp];
    RL += yl * Rs;
    cpL += yl * cps;
    ybL += yl * bs;
    RR += yr * Rs;
    cpR += yr * cps;
    ybR += yr * bs;
    Rf += yf * Rs;
    cpf += yf * cps;
    ybf += yf * bs;
    if (m.suth_shared) mua += yf * m.mu_ref[sp];
    Sdn += dc;
    SdP += dP;
    Bdn += bs * dc;
    BdP += bs * dP;
    Cdn += cps * dc;
    CdP += cps * dP;
  }
  // ---- face states
  double cL, eL, cR, eR;
#if CSB_FLUX_1DIV  // measured at config 4: 3.44 -> 3.32 ms
  bool ok = face_state_1div(WL[0], WL[1], WL[2], WL[3], WL[4], RL, cpL, ybL, cL, eL);
  ok &= face_state_1div(WR[0], WR[1], WR[2], WR[3], WR[4], RR, cpR, ybR, cR, eR);
#else
  double TL, TR;
  bool ok = face_state_sums(WL[0], WL[1], WL[2], WL[3], WL[4], RL, cpL, ybL, TL, cL, eL);
  ok &= face_state_sums(WR[0], WR[1], WR[2], WR[3], WR[4], RR, cpR, ybR, TR, cR, eR);
#endif
  const double rho = Wf[0];
  const double Tf = Wf[4] / (rho * Rf);
  ok &= (Tf > 0.0) && finite(Tf);
  double mu;
  if (m.suth_shared) {
    const double xx = Tf * m.inv_T_mu[0];
    mu = mua * ((xx * sqrt(xx)) * m.TS[0] / (Tf + m.S_mu[0]));
  } else {
    mu = 0.0;
    for (int sp = 0; sp < ns; ++sp) {
      const double* p = sQ + (5 + sp) * ldP;
      mu += (0.5 * (p[im] + p[ip])) * mu_species(m, sp, Tf);
    }
  }
  const double kc = (mu * cpf) * m.iPr;
  const double nrd = -(mu * m.iSc);  // -(rho D), D = mu / (rho Sc)
  double UL = 0.0, UR = 0.0;
#pragma unroll
  for (int x = 0; x < NX; ++x) {
    UL += WL[1 + x] * S[x];
    UR += WR[1 + x] * S[x];
  }
  const double area = sqrt(a2);
  const double hl = 0.5 * npmax(fabs(UL) + cL * area, fabs(UR) + cR * area);
  const double JS = nrd * (Sdn * XNS + SdP * XTS);  // (sum_s j_s) . S
  // ---- flow fluxes
  F[0] = 0.5 * (UL * WL[0] + UR * WR[0]) - hl * (WR[0] - WL[0]);
  double utS = 0.0;
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    if (x >= NX) continue;  // (PL: no w-momentum flux plane)
    const double qL = WL[0] * WL[1 + x], qR = WR[0] * WR[1 + x];
    const double fl = UL * qL + WL[4] * S[x];
    const double fr = UR * qR + WR[4] * S[x];
    const double tS = mu * tSm[x];
    utS += Wf[1 + x] * tS;
    F[(1 + x) * ldF] = (0.5 * (fl + fr) - hl * (qR - qL)) - tS;
  }
  {
    const double qL = WL[0] * eL, qR = WR[0] * eR;
    const double fl = UL * qL + WL[4] * UL;
    const double fr = UR * qR + WR[4] * UR;
    // sum_s h_s (j_s . S), h_s = b_s + cp_s T_f
    const double hsjS = nrd * ((Bdn + Tf * Cdn) * XNS + (BdP + Tf * CdP) * XTS) - JS * (ybf + Tf * cpf);
    const double qS = hsjS - kc * GTS;
    Fq[4 * ldF] = (0.5 * (fl + fr) - hl * (qR - qL)) + (qS - utS);
  }
  // ---- species pass 2
  const double CL = WL[0] * (0.5 * UL + hl), CR = WR[0] * (0.5 * UR - hl);
  const double nXNS = nrd * XNS, nXTS = nrd * XTS;
#pragma unroll FLUX_UNROLL
  for (int sp = 0; sp < ns; ++sp) {
    const double* p = sQ + (5 + sp) * ldP;
    const double vm = p[im], vp = p[ip];
    const double dc = vp - vm;
    double yl = vm, yr = vp;
    if (!first_order) {
      yl = vm + 0.5 * minmod(vm - p[imm], dc);
      yr = vp - 0.5 * minmod(dc, p[ipp] - vp);
    }
    const double yf = 0.5 * (vm + vp);
    const double dP = 0.5 * (0.5 * (p[im + st] - p[im - st]) + 0.5 * (p[ip + st] - p[ip - st]));
    Fq[(5 + sp) * ldF] = (yl * CL + yr * CR) + ((dc * nXNS + dP * nXTS) - yf * JS);
  }
  return ok;
}

// 2-D face enumeration of a tile: thread index f -> face (fi, fj) and its
// flux-buffer slot fi * FY + fj (FY = TJ + (D == 1)).  j-faces enumerate the
// TI x TJ faces in rows of TJ first and the tile's last face column (fj = TJ)
// after them, so that with TJ = 16 every half warp reads one row of 16
// consecutive cells from each staged plane: no shared-memory bank conflicts
// (rows of TJ + 1 = 17 put two words of a half warp on one bank pair; measured
// 1.43 wavefronts per ideal on the species MUSCL loads at config 4).
template <int D>
CSB_DEV void face_of2d(int f, int TI, int TJ, int& fi, int& fj) {
  if (D == 0) {
    fi = f / TJ;
    fj = f % TJ;
  } else {
    const int m = TI * TJ;
    fi = f < m ? f / TJ : f - m;
    fj = f < m ? f % TJ : TJ;
  }
}

template <int NSB, int D>
CSB_DEV void visc_pass2d(const Model& m, const GridDev& g, const double* sP, int ldP, double* sF,
                         int maxf, int i0, int j0, int ci, int cj, int BY, int TIc, int TJc,
                         unsigned long long* flags) {
  // faces enumerated over the full tile shape (compile-time divisor when the
  // tile is fixed), faces beyond a partial edge tile skipped
  const int FX = TIc + (D == 0), FY = TJc + (D == 1);
  const int fx = ci + (D == 0), fy = cj + (D == 1);
  const int nf = FX * FY;
  const int sd = D == 0 ? BY : 1, st = D == 0 ? 1 : BY;
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    int fi, fj;
    face_of2d<D>(f, TIc, TJc, fi, fj);
    if (fi >= fx || fj >= fy) continue;
    const int fs = fi * FY + fj;  // flux-buffer slot
    const int ip = (fi + NG) * BY + (fj + NG);
    const int im = ip - sd;
    const int gi = i0 + fi, gj = j0 + fj;
    double S[3], xn[3], xt[3];
    const long long fidx = face_index(g, D, gi, gj, 0);
    load_S(g, D, fidx, S);
    bool hasm, hasp;
    long long cellm, cellp;
    if (g.fm[D]) {
      // static metric terms, precomputed once per grid (k_face_metrics2d)
      const double* fm = g.fm[D] + fidx;
      const long long nf = g.NF[D];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        xn[x] = __ldg(fm + x * nf);
        xt[x] = __ldg(fm + (3 + x) * nf);
      }
      const int nd = D == 0 ? g.ni : g.nj, pos = D == 0 ? gi : gj;
      hasm = pos > 0;
      hasp = pos < nd;
      cellm = hasm ? cell_index(g, D == 0 ? gi - 1 : gi, D == 0 ? gj : gj - 1, 0) : -1;
      cellp = hasp ? cell_index(g, gi, gj, 0) : -1;
    } else {
      face_metric2d<D>(g, gi, gj, S, xn, xt, hasm, hasp, cellm, cellp);
    }
    if (!face_visc2d<NSB, D>(m, sP, ldP, im, ip, st, S, xn, xt, sF + fs, maxf))
      raise_flag(flags, EB_FACE_T, hasp ? cellp : cellm);
  }
}

// K2D faces of direction D of one tile through face_flux2d (convective +
// viscous in one evaluation); same face enumeration as visc_pass2d.
template <int NSB, int D, bool PL>
CSB_DEV void flux_pass2d(const Model& m, const GridDev& g, const double* sP, int ldP, double* sF,
                         int maxf, int i0, int j0, int ci, int cj, int BY, int TIc, int TJc,
                         bool first_order, unsigned long long* flags) {
  const int FX = TIc + (D == 0), FY = TJc + (D == 1);
  const int fx = ci + (D == 0), fy = cj + (D == 1);
  const int nf = FX * FY;
  const int sd = D == 0 ? BY : 1, st = D == 0 ? 1 : BY;
  for (int f = threadIdx.x; f < nf; f += blockDim.x) {
    int fi, fj;
    face_of2d<D>(f, TIc, TJc, fi, fj);
    if (fi >= fx || fj >= fy) continue;
    const int fs = fi * FY + fj;  // flux-buffer slot
    const int ip = (fi + NG) * BY + (fj + NG);
    const int im = ip - sd;
    const int gi = i0 + fi, gj = j0 + fj;
    double S[3], xn[3], xt[3];
    const long long fidx = face_index(g, D, gi, gj, 0);
    constexpr int NX = PL ? 2 : 3;
    {
      const double* p = g.S[D];
      const long long nfa = g.NF[D];
#pragma unroll
      for (int x = 0; x < 3; ++x) S[x] = x < NX ? __ldg(p + x * nfa + fidx) : 0.0;
    }
    if (g.fm[D]) {
      // static metric terms, precomputed once per grid (k_face_metrics2d)
      const double* fm = g.fm[D] + fidx;
      const long long nfa = g.NF[D];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        xn[x] = x < NX ? __ldg(fm + x * nfa) : 0.0;
        xt[x] = x < NX ? __ldg(fm + (3 + x) * nfa) : 0.0;
      }
    } else {
      bool hasm, hasp;
      long long cellm, cellp;
      load_S(g, D, fidx, S);
      face_metric2d<D>(g, gi, gj, S, xn, xt, hasm, hasp, cellm, cellp);
    }
    if (!face_flux2d<NSB, D, PL>(m, sP, ldP, im, ip, sd, st, S, xn, xt, first_order, sF + fs, maxf)) {
      const int nd = D == 0 ? g.ni : g.nj, pos = D == 0 ? gi : gj;
      raise_flag(flags, EB_FACE_T,
                 pos < nd ? cell_index(g, gi, gj, 0)
                          : cell_index(g, D == 0 ? gi - 1 : gi, D == 0 ? gj : gj - 1, 0));
    }
  }
}

// Net chemical production of one cell (chemistry.py:46-65).
template <int NSB>
CSB_DEV void omega_cell(const Model& m, const Mech& mech, double T, const double* rho_s,
                        double* om) {
  const int ns = m.ns;
  double conc[NSB];
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    om[s] = 0.0;
    if (s < ns) conc[s] = rho_s[s] / m.M[s];
  }
  for (int r = 0; r < mech.nrx; ++r) {
    const Reaction& rx = mech.rx[r];
    double rate = rx.Af * pow(T, rx.bf) * exp(-rx.Eaf / (R_U * T));
    for (int t = 0; t < rx.nr; ++t) {
      const double c = conc[rx.rs[t]];
      const double nu = rx.rn[t];
      rate = rate * (nu == 1.0 ? c : (nu == 2.0 ? c * c : pow(c, nu)));
    }
    if (rx.has_back) {
      double rb = rx.Ab * pow(T, rx.bb) * exp(-rx.Eab / (R_U * T));
      for (int t = 0; t < rx.np; ++t) {
        const double c = conc[rx.ps[t]];
        const double nu = rx.pn[t];
        rb = rb * (nu == 1.0 ? c : (nu == 2.0 ? c * c : pow(c, nu)));
      }
      rate = rate - rb;
    }
    if (!finite(rate)) {
#pragma unroll
      for (int s = 0; s < NSB; ++s)
        if (s < ns) om[s] += 0.0 * rate;
    }
    for (int t = 0; t < rx.nd; ++t) om[rx.ds[t]] += rx.dn[t] * rate;
  }
#pragma unroll
  for (int s = 0; s < NSB; ++s)
    if (s < ns) om[s] = om[s] * m.M[s];
}

// ----------------------------------------------------------------------------
// residual kernel
// ----------------------------------------------------------------------------

// FTI, FTJ: compile-time 2-D tile (0: runtime TI_, TJ_).  With a fixed tile
// every shared-memory plane stride and face / cell index divisor is a
// constant, which removes most of the integer address arithmetic.
#ifndef CSB_RES_FUSED
#define CSB_RES_FUSED 1  // K2D faces through face_flux2d (0: face_conv + face_visc2d)
#endif
template <int NSB, bool K2D, int FTI = 0, int FTJ = 0, bool PL = false>
#ifndef CSB_RES_MINB
#define CSB_RES_MINB 2  // measured: 3 CTAs/SM (80 registers, spills) is 12-29% slower
#endif
__global__ void __launch_bounds__(256, CSB_RES_MINB) k_residual(const Model* __restrict__ mp, GridDev g, BCDev bc,
                                                  Mech mech, const double* __restrict__ q,
                                                  double* __restrict__ R, int first_order, int TI_,
                                                  int TJ_, int TK, unsigned long long* flags,
                                                  NormsOut nrm, int sr_on,
                                                  const unsigned long long* __restrict__ guard,
                                                  int guard_bit, int twobuf) {
  // guarded launch (the general-path fallback queued behind a K2D launch):
  // runs only when that launch raised EB_KSKIP (w != 0 under symmetry
  // k-faces), as a persistent grid over the tiles; otherwise exits at once
  if (guard && !((__ldcg(guard) >> guard_bit) & 1ull)) return;
  const int TI = FTI ? FTI : TI_, TJ = FTJ ? FTJ : TJ_;
  extern __shared__ double smem[];
  __shared__ Model sm;
  {
    // header + the first ns entries of each per-species array (a full copy
    // of the ~5 KB table per block cost ~12% of the kernel)
    static_assert(offsetof(Model, M) % sizeof(double) == 0, "Model layout");
    static_assert(offsetof(Model, inv_T_mu) == offsetof(Model, M) + 8 * MAXNS * sizeof(double),
                  "Model arrays contiguous");
    const double* src = reinterpret_cast<const double*>(mp);
    double* dst = reinterpret_cast<double*>(&sm);
    const int h = (int)(offsetof(Model, M) / sizeof(double));
    const int nsm = __ldg(&mp->ns);
    for (int i = threadIdx.x; i < h + MODEL_NARR * nsm; i += blockDim.x) {
      const int w = i < h ? i : h + ((i - h) / nsm) * MAXNS + (i - h) % nsm;
      dst[w] = __ldg(src + w);
    }
  }
  __syncthreads();
  const Model& m = sm;
  const int ns = m.ns;
  const int nc = 6 + ns;
  const int nv = 5 + ns;
  const int BX = TI + 2 * NG, BY = TJ + 2 * NG, BZ = K2D ? 1 : TK + 2 * NG;
  const int ldP = BX * BY * BZ;
  const int nti = (g.ni + TI - 1) / TI, ntj = (g.nj + TJ - 1) / TJ;
  const int ntiles = nti * ntj * (K2D ? 1 : (g.nk + TK - 1) / TK);
  double n_flow = 0.0, n_sp = 0.0, n_rho = 0.0;  // residual_norms partials of this CTA
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  int b = tile;
  const int ti = b % nti;
  b /= nti;
  const int tj = b % ntj;
  const int tk = b / ntj;
  const int i0 = ti * TI, j0 = tj * TJ, k0 = K2D ? 0 : tk * TK;
  const int ci = min(TI, g.ni - i0), cj = min(TJ, g.nj - j0), ck = K2D ? 1 : min(TK, g.nk - k0);
  double* sP = smem;
  // (K2D: one k layer, so a fixed tile makes maxf -- the flux plane stride -- a constant)
  const int TKc = K2D ? 1 : TK;
  const int maxf = max(max((TI + 1) * TJ * TKc, TI * (TJ + 1) * TKc), TI * TJ * (K2D ? 1 : TK + 1));
  // PL (planar, w == 0): the w plane of the staged primitives and the
  // w-momentum flux plane are not stored; PP maps a component to its plane
  constexpr int NPD = PL ? 1 : 0;
  auto PP = [](int c) { return PL && c > 3 ? c - 1 : c; };
  double* sQ = sP - NPD * ldP;  // planes >= 4
  double* sF = smem + (long long)(nc - NPD) * ldP;
  // twobuf: the two directions' fluxes in separate buffers, one difference
  // pass for both (no partial R between the directions, 3 barriers per tile
  // instead of 5)
  double* sF1 = twobuf ? sF + (long long)(nv - NPD) * maxf : sF;
  // partial residual of the tile, sum over directions in order (0 + dR_0 + ...)
  double* sR = sF + (long long)(twobuf ? 2 : 1) * (nv - NPD) * maxf;

  // ---- stage decoded primitives + halo (padded coordinates = interior + NG)
  for (int l = threadIdx.x; l < ldP; l += blockDim.x) {
    const int lz = K2D ? 0 : l % BZ;
    const int ly = K2D ? l % BY : (l / BZ) % BY;
    const int lx = K2D ? l / BY : l / (BZ * BY);
    const int pi = i0 + lx, pj = j0 + ly, pk = K2D ? NG : k0 + lz;
    const bool inside_pad = pi < g.ni + 2 * NG && pj < g.nj + 2 * NG && pk < g.nk + 2 * NG;
    const bool interior = inside_pad && pi >= NG && pi < g.ni + NG && pj >= NG &&
                          pj < g.nj + NG && pk >= NG && pk < g.nk + NG;
    if (interior && stream_species<NSB>()) {
      // large species counts: decode_from's arithmetic with the mass
      // fractions written straight to (and renormalised in) shared memory
      const long long cell = cell_index(g, pi - NG, pj - NG, pk - NG);
      const double* qc = q + cell;
      const long long N = g.N;
      // loads issued in groups of 8 ahead of their use: the species loop is
      // not unrolled, and one dependent global load per species left the
      // staging latency-bound (~11 % of the kernel's stall samples at
      // config 4, ncu source view)
      const double rho = qc[0], q4 = qc[4 * N];
      double u[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) u[x] = qc[(1 + x) * N];
      bool ok = (rho > 0.0) && finite(rho);
      const double ir = 1.0 / rho;
#pragma unroll
      for (int x = 0; x < 3; ++x) u[x] = u[x] * ir;
      double sum = 0.0;
      const double* qsp = qc + 5 * N;  // running pointer (one 64-bit add per component)
      for (int s0 = 0; s0 < ns; s0 += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k, qsp += N) v[k] = s0 + k < ns ? *qsp : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (s0 + k >= ns) break;
          double y = v[k] * ir;
          if (y < -EPS_NEG) ok = false;
          if (y < 0.0) y = 0.0;
          sQ[(5 + s0 + k) * ldP + l] = y;
          sum += y;
        }
      }
      double R = 0.0, cp = 0.0, yb = 0.0;
      const double isum = 1.0 / sum;
      for (int sp = 0; sp < ns; ++sp) {
        const double y = sQ[(5 + sp) * ldP + l] * isum;
        sQ[(5 + sp) * ldP + l] = y;
        R += y * m.Rs[sp];
        cp += y * m.cp[sp];
        yb += y * m.bs[sp];
      }
      const double Ek = 0.5 * ((u[0] * u[0] + u[1] * u[1]) + u[2] * u[2]);
      const double icv = 1.0 / (cp - R);
      const double e_int = q4 * ir - Ek;
      const double T = (e_int - yb) * icv;
      if (!(T > 0.0) || !finite(T)) ok = false;
      if (!ok) raise_flag(flags, EB_DECODE, cell);
      if (K2D && bc.kind[4] == BC_SYMMETRY && qc[3 * N] != 0.0) raise_flag(flags, EB_KSKIP, cell);
      if (PL && !(qc[3 * N] == 0.0)) raise_flag(flags, EB_NONPLANAR, cell);
      sP[0 * ldP + l] = rho;
      sP[1 * ldP + l] = u[0];
      sP[2 * ldP + l] = u[1];
      if (!PL) sP[3 * ldP + l] = u[2];
      sQ[4 * ldP + l] = rho * R * T;
      sQ[(5 + ns) * ldP + l] = T;
    } else if (interior) {
      const long long cell = cell_index(g, pi - NG, pj - NG, pk - NG);
      Cell<NSB> cs;
      if (!decode<NSB>(m, q + cell, g.N, cs)) raise_flag(flags, EB_DECODE, cell);
      if (K2D && bc.kind[4] == BC_SYMMETRY && q[cell + 3 * g.N] != 0.0)
        raise_flag(flags, EB_KSKIP, cell);
      if (PL && !(q[cell + 3 * g.N] == 0.0)) raise_flag(flags, EB_NONPLANAR, cell);
      sP[0 * ldP + l] = cs.rho;
      sP[1 * ldP + l] = cs.u[0];
      sP[2 * ldP + l] = cs.u[1];
      if (!PL) sP[3 * ldP + l] = cs.u[2];
      sQ[4 * ldP + l] = cs.p;
#pragma unroll
      for (int s = 0; s < NSB; ++s)
        if (s < ns) sQ[(5 + s) * ldP + l] = cs.Y[s];
      sQ[(5 + ns) * ldP + l] = cs.T;
    } else {
      double v[6 + NSB];
      if (!inside_pad) {
#pragma unroll
        for (int c = 0; c < 6 + NSB; ++c) v[c] = 0.0;
      } else {
        padded_value<NSB>(m, g, bc, q, pi, pj, pk, v, flags);
        // (ghosts the reference never fills are NaN and never read)
        if (PL && v[3] != 0.0 && v[3] == v[3]) raise_flag(flags, EB_NONPLANAR, 0);
      }
#pragma unroll
      for (int c = 0; c < 6 + NSB; ++c)
        if (c < nc && !(PL && c == 3)) sP[PP(c) * ldP + l] = v[c];
    }
  }
  __syncthreads();

  auto lidx = [&](int lx, int ly, int lz) { return K2D ? lx * BY + ly : (lx * BY + ly) * BZ + lz; };
  const int strideX = K2D ? BY : BY * BZ, strideY = K2D ? 1 : BZ, strideZ = 1;
  const int ndir = K2D ? 2 : 3;

  // One direction: convective + viscous face passes into sF, then the flux
  // difference into the cells.  dtag is std::integral_constant<int, D> on the
  // 2-D path (every grid-array index static: no local copy of the kernel
  // parameters) and a plain int on the 3-D path.
  auto dir_pass = [&](auto dtag) {
    const int d = dtag;
    // faces of direction d inside the tile: dims (ci+1, cj, ck) etc.  2-D:
    // enumerated over the full tile (FY columns; constant with a fixed tile),
    // faces beyond a partial edge tile skipped; the flux buffer uses the
    // same full-tile face index
    const int fx = ci + (d == 0), fy = cj + (d == 1), fz = ck + (d == 2);
    const int FY = K2D ? TJ + (d == 1) : fy;
    const int nf = K2D ? (TI + (d == 0)) * FY : fx * fy * fz;
    if constexpr (K2D && (CSB_RES_FUSED || PL)) {
      if (d == 0)
        flux_pass2d<NSB, 0, PL>(m, g, sP, ldP, sF, maxf, i0, j0, ci, cj, BY, TI, TJ, first_order != 0, flags);
      else
        flux_pass2d<NSB, 1, PL>(m, g, sP, ldP, sF1, maxf, i0, j0, ci, cj, BY, TI, TJ, first_order != 0, flags);
      if (twobuf && d == 0) return;  // differenced together with direction 1
    } else {
    for (int f = threadIdx.x; f < nf; f += blockDim.x) {
      // (d == 1 ? ... : ...) keeps both divisors compile-time with a fixed tile
      const int fk = K2D ? 0 : f % fz;
      int fi, fj;
      if (K2D) {
        if (d == 0) face_of2d<0>(f, TI, TJ, fi, fj);
        else face_of2d<1>(f, TI, TJ, fi, fj);
      } else {
        fj = (f / fz) % fy;
        fi = f / (fz * fy);
      }
      if (K2D && (fi >= fx || fj >= fy)) continue;
      const int fs = K2D ? fi * FY + fj : f;  // flux-buffer slot
      // local (staged) coordinates of the "p" cell (upper side of the face)
      int lx = fi + NG, ly = fj + NG, lz = K2D ? 0 : fk + NG;
      const int sd = d == 0 ? strideX : (d == 1 ? strideY : strideZ);
      const int ip = lidx(lx, ly, lz);
      const int im = ip - sd, imm = ip - 2 * sd, ipp = ip + sd;
      // global face and the two adjacent cells
      const int gi = i0 + fi, gj = j0 + fj, gk = k0 + fk;
      double S[3];
      load_S(g, d, face_index(g, d, gi, gj, gk), S);
      if (!face_conv<NSB>(m, sP, ldP, imm, im, ip, ipp, S, first_order != 0, sF + fs, maxf)) {
        const int nd = d == 0 ? g.ni : (d == 1 ? g.nj : g.nk);
        const int pos = d == 0 ? gi : (d == 1 ? gj : gk);
        int cm[3] = {gi, gj, gk};
        cm[d] -= 1;
        raise_flag(flags, EB_FACE_T,
                   pos < nd ? cell_index(g, gi, gj, gk) : cell_index(g, cm[0], cm[1], cm[2]));
      }
    }
    // viscous pass over the same faces (same thread -> face map: no barrier)
    if (K2D) {
      if (d == 0) visc_pass2d<NSB, 0>(m, g, sP, ldP, sF, maxf, i0, j0, ci, cj, BY, TI, TJ, flags);
      else visc_pass2d<NSB, 1>(m, g, sP, ldP, sF, maxf, i0, j0, ci, cj, BY, TI, TJ, flags);
    } else {
    for (int f = threadIdx.x; f < nf; f += blockDim.x) {
      const int fk = f % fz;
      const int fj = (f / fz) % fy;
      const int fi = f / (fz * fy);
      int lx = fi + NG, ly = fj + NG, lz = K2D ? 0 : fk + NG;
      const int sd = d == 0 ? strideX : (d == 1 ? strideY : strideZ);
      const int ip = lidx(lx, ly, lz);
      const int im = ip - sd;
      const int gi = i0 + fi, gj = j0 + fj, gk = k0 + fk;
      FaceGeom fg;
      const long long fidx = face_index(g, d, gi, gj, gk);
      load_S(g, d, fidx, fg.S);
      const int nd = d == 0 ? g.ni : (d == 1 ? g.nj : g.nk);
      const int pos = d == 0 ? gi : (d == 1 ? gj : gk);
      int cm[3] = {gi, gj, gk}, cp3[3] = {gi, gj, gk};
      cm[d] -= 1;
      const bool hasm = pos > 0, hasp = pos < nd;
      const long long cellm = hasm ? cell_index(g, cm[0], cm[1], cm[2]) : -1;
      const long long cellp = hasp ? cell_index(g, cp3[0], cp3[1], cp3[2]) : -1;
      const double Vm = hasm ? __ldg(g.vol + cellm) : 0.0;
      const double Vp = hasp ? __ldg(g.vol + cellp) : 0.0;
      const double Vf = (hasm && hasp) ? 0.5 * (Vp + Vm) : (hasm ? Vm : Vp);
#pragma unroll
      for (int x = 0; x < 3; ++x) fg.xn[x] = fg.S[x] / Vf;
      int st[2];
      int t = 0;
      for (int a = 0; a < 3; ++a) {
        if (a == d) continue;
        fg.ta[t] = a;
        fg.use_t[t] = !(K2D && a == 2);
        st[t] = a == 0 ? strideX : (a == 1 ? strideY : strideZ);
        if (fg.use_t[t]) {
          // Sc_a * J at the adjacent cells, face-averaged (spatial.py:241-248)
          double xc[2][3];
          for (int side = 0; side < 2; ++side) {
            const bool has = side == 0 ? hasm : hasp;
            if (!has) continue;
            const int* cc = side == 0 ? cm : cp3;
            double Slo[3], Shi[3];
            int lo[3] = {cc[0], cc[1], cc[2]};
            int hi[3] = {cc[0], cc[1], cc[2]};
            hi[a] += 1;
            load_S(g, a, face_index(g, a, lo[0], lo[1], lo[2]), Slo);
            load_S(g, a, face_index(g, a, hi[0], hi[1], hi[2]), Shi);
            const double J = 1.0 / (side == 0 ? Vm : Vp);
            for (int x = 0; x < 3; ++x) xc[side][x] = (0.5 * (Slo[x] + Shi[x])) * J;
          }
          for (int x = 0; x < 3; ++x)
            fg.xt[t][x] = (hasm && hasp) ? 0.5 * (xc[1][x] + xc[0][x]) : (hasm ? xc[0][x] : xc[1][x]);
        }
        ++t;
      }
      if (!face_visc<NSB>(m, sP, ldP, im, ip, st, fg, sF + f, maxf))
        raise_flag(flags, EB_FACE_T, hasp ? cellp : cellm);
    }
    }
    }  // !(K2D && (CSB_RES_FUSED || PL))
    __syncthreads();
    // difference into R (R = 0 + dR_0 + dR_1 + dR_2, spatial.py:258-259).
    // The last direction also applies the chemistry source (261-267), the
    // finite check (269-271) and, when requested, the residual-norm terms
    // (driver.py:85-90), so R is read back once per direction at most.
    // 2-D: cells over the full tile (index ii * TJ + jj, also the sR index)
    const int ncell = K2D ? TI * TJ : ci * cj * ck;
    const bool last = d == ndir - 1;
    for (int l = threadIdx.x; l < ncell; l += blockDim.x) {
      const int kk = K2D ? 0 : l % ck;
      const int jj = K2D ? l % TJ : (l / ck) % cj;
      const int ii = K2D ? l / TJ : l / (ck * cj);
      if (K2D && (ii >= ci || jj >= cj)) continue;
      const long long cell = cell_index(g, i0 + ii, j0 + jj, k0 + kk);
      int flo, fhi;
      if (d == 0) {
        flo = (ii * FY + jj) * fz + kk;
        fhi = ((ii + 1) * FY + jj) * fz + kk;
      } else if (d == 1) {
        flo = (ii * FY + jj) * fz + kk;
        fhi = (ii * FY + jj + 1) * fz + kk;
      } else {
        flo = (ii * FY + jj) * fz + kk;
        fhi = flo + 1;
      }
      const long long N = g.N;
      double* __restrict__ Rc = R + cell;
      double* __restrict__ sRc = sR + l;
      const double* sFd = (twobuf && d == 1) ? sF1 : sF;  // this direction's fluxes
      // twobuf: direction 0's flux difference of component plane pc
      const int flo0 = ii * TJ + jj, fhi0 = flo0 + TJ;
      // (Rl: the component's R word, a running pointer at the call sites)
      auto prev = [&](int c, int pc, const double* Rl) {
        return twobuf ? sF[pc * maxf + fhi0] - sF[pc * maxf + flo0]
                      : (sr_on ? sRc[c * ncell] : *Rl);
      };
      if (!last) {
        // first / middle direction: partial sums, loads of a group of 8
        // components issued before their stores
        const double* Rl = Rc;  // running pointers: one 64-bit add per component
        double* Rs = Rc;
        for (int c0 = 0; c0 < nv; c0 += 8) {
          double pv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k, Rl += N)
            pv[k] = (d == 0 || c0 + k >= nv) ? 0.0 : (sr_on ? sRc[(c0 + k) * ncell] : *Rl);
#pragma unroll
          for (int k = 0; k < 8; ++k, Rs += N) {
            const int c = c0 + k;
            if (c >= nv) break;
            if (PL && c == 3) continue;  // (R_3 = 0 is written by the last direction)
            const double dR = sFd[PP(c) * maxf + fhi] - sFd[PP(c) * maxf + flo];
            const double v = d == 0 ? dR : pv[k] + dR;
            if (sr_on) sRc[c * ncell] = v;
            else *Rs = v;
          }
        }
        continue;
      }
      // last direction
      double om[NSB];
      double V = 0.0;
      const bool chem = mech.nrx > 0;
      if (chem) {
        const int ls = lidx(ii + NG, jj + NG, K2D ? 0 : kk + NG);
        double rs[NSB];
        const double rho = sP[ls];
#pragma unroll
        for (int s = 0; s < NSB; ++s)
          if (s < ns) rs[s] = rho * sQ[(5 + s) * ldP + ls];
        omega_cell<NSB>(m, mech, sQ[(5 + ns) * ldP + ls], rs, om);
        V = __ldg(g.vol + cell);
      }
      bool fin = true;
      double f = 0.0, sp = 0.0, r0 = 0.0;
      auto fold = [&](int c, double v) {
        fin &= finite(v);
        if (c == 0) {
          r0 = v;
          f = v * v;
        } else if (c < 5) {
          f += v * v;
        } else {
          sp += v;
        }
      };
      if constexpr (stream_species<NSB>()) {
        double* __restrict__ Rp = Rc;  // running pointers (one 64-bit add per component)
        const double* Rl = Rc;
        for (int c0 = 0; c0 < nv; c0 += 8) {
          double pv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k, Rl += N)
            pv[k] = (c0 + k >= nv || (PL && c0 + k == 3)) ? 0.0 : prev(c0 + k, PP(c0 + k), Rl);
#pragma unroll
          for (int k = 0; k < 8; ++k, Rp += N) {
            const int c = c0 + k;
            if (c >= nv) break;
            double v = (PL && c == 3) ? 0.0 : pv[k] + (sFd[PP(c) * maxf + fhi] - sFd[PP(c) * maxf + flo]);
            if (chem && c >= 5) v = v - om[c - 5] * V;
            *Rp = v;
            fold(c, v);
          }
        }
      } else {
        double rv[5 + NSB];
#pragma unroll
        for (int c = 0; c < 5 + NSB; ++c)
          if (c < nv) rv[c] = (PL && c == 3) ? 0.0 : prev(c, PP(c), Rc + (long long)c * N);
        double* __restrict__ Rp = Rc;
#pragma unroll
        for (int c = 0; c < 5 + NSB; ++c, Rp += N)
          if (c < nv) {
            double v = (PL && c == 3) ? 0.0 : rv[c] + (sFd[PP(c) * maxf + fhi] - sFd[PP(c) * maxf + flo]);
            if (chem && c >= 5) v = v - om[c - 5] * V;
            *Rp = v;
            fold(c, v);
          }
      }
      if (!fin) raise_flag(flags, EB_RES_NONFINITE, cell);
      if (nrm.out) {
        n_flow += f;
        n_sp += sp * sp;
        n_rho += r0 * r0;
      }
    }
    __syncthreads();  // next direction rewrites sF; next tile restages sP
  };
  if constexpr (K2D) {
    dir_pass(std::integral_constant<int, 0>{});
    dir_pass(std::integral_constant<int, 1>{});
  } else {
#pragma unroll 1
    for (int d = 0; d < 3; ++d) dir_pass(d);
  }
  }  // tile loop
  if (nrm.out) {
    // block partials, then the last block reduces all partials in fixed order
    __shared__ double red[3][8];
    __shared__ bool last_block;
    double v3[3] = {n_flow, n_sp, n_rho};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double v = v3[k];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < 3; ++k) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[k][w];
        nrm.partial[k * nrm.cap + blockIdx.x] = v;
      }
      __threadfence();
      last_block = atomicAdd(nrm.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last_block) {
      __threadfence();
      const int nb = gridDim.x;
      double acc[3] = {0.0, 0.0, 0.0};
      for (int b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += __ldcg(nrm.partial + k * nrm.cap + b);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double v = acc[k];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = v;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int k = 0; k < 3; ++k) {
          double v = 0.0;
          for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[k][w];
          nrm.out[k] = sqrt(v);
        }
        *nrm.counter = 0u;
      }
    }
  }
}

// Full padded primitive array (API: assemble_residual(return_padded=True)),
// SoA [nc][(ni+4)(nj+4)(nk+4)].
template <int NSB>
__global__ void k_padded(const Model* __restrict__ mp, GridDev g, BCDev bc,
                         const double* __restrict__ q, double* __restrict__ P,
                         unsigned long long* flags) {
  const Model& m = *mp;
  const int nc = 6 + m.ns;
  const int PX = g.ni + 2 * NG, PY = g.nj + 2 * NG, PZ = g.nk + 2 * NG;
  const long long NP = (long long)PX * PY * PZ;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < NP;
       l += (long long)gridDim.x * blockDim.x) {
    const int pk = l % PZ, pj = (l / PZ) % PY, pi = l / ((long long)PZ * PY);
    double v[6 + NSB];
    padded_value<NSB>(m, g, bc, q, pi, pj, pk, v, flags);
    for (int c = 0; c < nc; ++c) P[c * NP + l] = v[c];
  }
}

// ----------------------------------------------------------------------------
// host launchers
// ----------------------------------------------------------------------------

// drop: planes not stored (1 for the planar 2-D variant: w and its flux)
static inline void pick_tile(int ns, bool k2d, int nk, int& TI, int& TJ, int& TK, size_t& smem,
                             int drop = 0) {
  const int nc = 6 + ns - drop, nv = 5 + ns - drop;
  const size_t budget = 200 * 1024;
  if (k2d) {
    // TI x 16 tiles (256 threads cover the (TI + 1) x 16 faces up to TI = 15):
    // the largest TI >= 7 that keeps 2 CTAs per SM (<= 104 KB), else the
    // largest that fits one CTA, else the small fallbacks.  Measured at 1024^2:
    // ns = 40 12 x 16 at 1 CTA/SM 2.55 ms (10 x 16 2.92, 8 x 16 3.07, 7 x 16
    // 3.30; 7 x 8 at 2 CTAs/SM slower still), ns = 20 12 x 16 at 2 CTAs/SM
    // 0.87 ms (11 x 16 0.92; 15 x 16 at 1 CTA/SM is 3x slower per cell than
    // ns = 11).
    auto fits = [&](int ti, int tj, size_t cap) {
      const size_t ldP = (size_t)(ti + 4) * (tj + 4);
      const size_t maxf = std::max((size_t)(ti + 1) * tj, (size_t)ti * (tj + 1));
      smem = (ldP * nc + maxf * nv) * sizeof(double);
      return smem <= cap;
    };
    TK = 1;
    if (const char* e = probe_env("CSB_RHS_TILE")) {  // tuning probe
      if (sscanf(e, "%d,%d", &TI, &TJ) == 2 && TI >= 1 && TJ >= 1 && (TI + 1) * TJ <= 1024 &&
          fits(TI, TJ, budget))
        return;
    }
    TJ = 16;
    for (int pass = 0; pass < 2; ++pass)
      for (TI = 15; TI >= 7; --TI)
        if (fits(TI, TJ, pass == 0 ? (size_t)104 * 1024 : budget)) return;
    const int small[][2] = {{7, 8}, {3, 8}, {3, 4}, {1, 4}};
    for (auto& c : small) {
      TI = c[0];
      TJ = c[1];
      if (fits(TI, TJ, budget)) return;
    }
  } else {
    const int cand[][3] = {{6, 8, 4}, {4, 4, 4}, {4, 4, 2}, {2, 4, 2}, {2, 2, 2}, {1, 2, 1}};
    for (auto& c : cand) {
      TI = c[0];
      TJ = c[1];
      TK = std::min(c[2], nk);
      const size_t ldP = (size_t)(TI + 4) * (TJ + 4) * (TK + 4);
      const size_t maxf = std::max(std::max((size_t)(TI + 1) * TJ * TK, (size_t)TI * (TJ + 1) * TK),
                                   (size_t)TI * TJ * (TK + 1));
      smem = (ldP * nc + maxf * nv) * sizeof(double);
      if (smem <= budget) return;
    }
  }
}

// Accumulate the tile's residual in shared memory (one global write per
// component) when the extra TI*TJ*TK*nv doubles do not cost occupancy
// (2 CTAs/SM under the 128-register bound up to ~104 KB of dynamic smem each).
static inline bool residual_in_smem(size_t smem, int cells, int nv, size_t& total) {
  total = smem + (size_t)cells * nv * sizeof(double);
  // per-SM budget 228 KB including ~5 KB of static shared memory per CTA
  const size_t two = 104 * 1024, one = 200 * 1024;
  return smem <= two ? total <= two : total <= one;
}

cudaError_t CSB_BK(launch_residual)(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                            const Mech& mech, const double* q, double* R, int first_order, int mode,
                            unsigned long long* flags, cudaStream_t st, NormsOut nrm, bool* fused,
                            const unsigned long long* guard, int guard_bit) {
  const bool k2d = mode != RES_GENERAL, planar = mode == RES_K2D_PLANAR;
  int TI, TJ, TK;
  size_t smem;
  pick_tile(ns, k2d, g.nk, TI, TJ, TK, smem, planar ? 1 : 0);
  // planar: both directions' fluxes resident (one difference pass) when the
  // second buffer keeps the tile's CTAs per SM (checked with the occupancy
  // API below: static shared memory and the 1 KB system reservation per CTA
  // come on top of the dynamic size)
#ifndef CSB_RES_TWOBUF
#define CSB_RES_TWOBUF 1
#endif
  const size_t smem1 = smem;  // one flux buffer
  size_t smem2 = 0;
  if (planar && CSB_RES_TWOBUF) {
    const size_t maxf = std::max((size_t)(TI + 1) * TJ, (size_t)TI * (TJ + 1));
    smem2 = smem1 + maxf * (4 + ns) * sizeof(double);
    if (smem2 > (size_t)200 * 1024) smem2 = 0;
  }
  const long long ntiles = (long long)((g.ni + TI - 1) / TI) * ((g.nj + TJ - 1) / TJ) *
                           (k2d ? 1 : (g.nk + TK - 1) / TK);
  // persistent grid: every resident CTA loops over the tiles (the model
  // table, the kernel setup and the block's norms reduction are paid once
  // per CTA instead of once per tile)
  cudaError_t err = cudaSuccess;
  CSB_NS_DISPATCH(ns, {
    const bool fixed = TI == 15 && TJ == 16;
    auto kfn = !k2d    ? k_residual<NSB, false>
               : planar ? (fixed ? k_residual<NSB, true, 15, 16, true> : k_residual<NSB, true, 0, 0, true>)
                        : (fixed ? k_residual<NSB, true, 15, 16> : k_residual<NSB, true>);
    auto occ = [&](size_t bytes) {
      int p = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, kfn, 256, bytes) != cudaSuccess) p = 0;
      return p;
    };
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)std::max(smem1, smem2));
    int twobuf = 0, sr_on = 0;
    int per_sm = occ(smem1);
    if (smem2 && occ(smem2) >= std::max(per_sm, 1)) {
      twobuf = 1;
      smem = smem2;
    } else {
      size_t smem_sr;
      if (residual_in_smem(smem1, TI * TJ * TK, 5 + ns, smem_sr) && occ(smem_sr) >= std::max(per_sm, 1)) {
        sr_on = 1;
        smem = smem_sr;
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      } else {
        smem = smem1;
      }
    }
    if (per_sm < 1) per_sm = 1;
    const long long nblk = std::min<long long>(ntiles, (long long)per_sm * device_sms());
    if (!(nrm.out && nblk <= nrm.cap)) nrm.out = nullptr;
    if (fused) *fused = nrm.out != nullptr;
    kfn<<<(unsigned)nblk, 256, smem, st>>>(mp, g, bc, mech, q, R, first_order, TI, TJ, TK, flags,
                                           nrm, sr_on, guard, guard_bit, twobuf);
    err = cudaGetLastError();
  });
  return err;
}

cudaError_t CSB_BK(launch_padded)(const Model* mp, int ns, const GridDev& g, const BCDev& bc,
                          const double* q, double* P, unsigned long long* flags, cudaStream_t st) {
  const long long NP = (long long)(g.ni + 4) * (g.nj + 4) * (g.nk + 4);
  const int blocks = (int)std::min<long long>((NP + 127) / 128, 148 * 16);
  CSB_NS_DISPATCH(ns, { k_padded<NSB><<<blocks, 128, 0, st>>>(mp, g, bc, q, P, flags); });
  return cudaGetLastError();
}

}  // namespace csb
