// csflow-b200: decode, chemistry Jacobian, local time step and implicit
// operator assembly (reference implicit.py:33-408, chemistry.py:46-104).
#pragma once
#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

// defined in csb_rhs.cu (same translation-unit-free template: re-declared)
template <int NSB>
CSB_DEV void omega_cell_impl(const Model& m, const Mech& mech, double T, const double* rho_s,
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

// ---------------------------------------------------------------- decode (API)
// out: [12 + ns][N] = rho, u0, u1, u2, p, T, c, gamma, h, Ek, R, cp, Y...
template <int NSB>
__global__ void k_decode(const Model* __restrict__ mp, GridDev g, const double* __restrict__ q,
                         double* __restrict__ out, unsigned long long* flags) {
  const Model& m = *mp;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + c, g.N, cs)) raise_flag(flags, EB_DECODE, c);
    const double v[12] = {cs.rho, cs.u[0], cs.u[1], cs.u[2], cs.p, cs.T, cs.c, cs.gamma, cs.h,
                          cs.Ek, cs.R, cs.cp};
    for (int k = 0; k < 12; ++k) out[k * g.N + c] = v[k];
    for (int s = 0; s < m.ns; ++s) out[(12 + s) * g.N + c] = cs.Y[s];
  }
}

// ------------------------------------------------- source Jacobian (FD, T fixed)
// chemistry.py:76-104: dOmega[:, r] = (omega(rho_s + h e_r) - omega(rho_s - h e_r)) / (2 h),
// h = max(1e-8 |rho_r|, 1e-12 rho), T held fixed.  The two perturbed states
// differ only in species r, so only the reactions whose rate depends on
// species r (Mech::sp_off / sp_rx) contribute to column r: each of them is
// evaluated at the two states exactly as the reference evaluates it (rate
// constants, then the concentration factors in stoichiometric order) and the
// difference of the two rates is scattered with the net stoichiometry.  This
// is the reference's finite difference without the rounding noise its two
// full sums leave in the untouched reactions (within the FD-noise
// bound), at O(reactions per species) instead of O(ns x reactions) rate
// evaluations per column.  A non-finite perturbed rate makes the column NaN,
// as it does in the reference.  dom_full: all ns*ns entries ([s*ns+r][N]),
// else the diagonal [s][N].  lamS: row-sum bound max_s sum_r |dOmega_sr|.
// dom_in (optional): injected dOmega instead of the differences.
CSB_DEV double rate_at(const Reaction& rx, double T, const double* conc, int r, double cr) {
  double rate = rx.Af * pow(T, rx.bf) * exp(-rx.Eaf / (R_U * T));
  for (int t = 0; t < rx.nr; ++t) {
    const double c = rx.rs[t] == r ? cr : conc[rx.rs[t]];
    const double nu = rx.rn[t];
    rate = rate * (nu == 1.0 ? c : (nu == 2.0 ? c * c : pow(c, nu)));
  }
  if (rx.has_back) {
    double rb = rx.Ab * pow(T, rx.bb) * exp(-rx.Eab / (R_U * T));
    for (int t = 0; t < rx.np; ++t) {
      const double c = rx.ps[t] == r ? cr : conc[rx.ps[t]];
      const double nu = rx.pn[t];
      rb = rb * (nu == 1.0 ? c : (nu == 2.0 ? c * c : pow(c, nu)));
    }
    rate = rate - rb;
  }
  return rate;
}

template <int NSB>
__global__ void k_source_jac(const Model* __restrict__ mp, GridDev g, Mech mech,
                             const double* __restrict__ q, double* __restrict__ dom, int dom_full,
                             double* __restrict__ lamS, const double* __restrict__ dom_in,
                             unsigned long long* flags) {
  const Model& m = *mp;
  const int ns = m.ns;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + c, g.N, cs)) raise_flag(flags, EB_DECODE, c);
    double rowsum[NSB], rs[NSB], conc[NSB], acc[NSB];
#pragma unroll
    for (int s = 0; s < NSB; ++s) {
      rowsum[s] = 0.0;
      rs[s] = (s < ns) ? cs.rho * cs.Y[s] : 0.0;
      conc[s] = (s < ns) ? rs[s] / m.M[s] : 0.0;
    }
    for (int r = 0; r < ns; ++r) {
      if (dom_in) {
        for (int s = 0; s < ns; ++s) acc[s] = dom_in[((long long)s * ns + r) * g.N + c];
      } else {
        const double h = npmax(1e-8 * fabs(rs[r]), 1e-12 * cs.rho);
        const double cup = (rs[r] + h) / m.M[r], cdn = (rs[r] - h) / m.M[r];
        for (int s = 0; s < ns; ++s) acc[s] = 0.0;
        bool bad = false;
        for (int l = mech.sp_off[r]; l < mech.sp_off[r + 1]; ++l) {
          const Reaction& rx = mech.rx[mech.sp_rx[l]];
          const double a = rate_at(rx, cs.T, conc, r, cup);
          const double b = rate_at(rx, cs.T, conc, r, cdn);
          bad |= !finite(a) || !finite(b);
          const double d = a - b;
          for (int t = 0; t < rx.nd; ++t) acc[rx.ds[t]] += rx.dn[t] * d;
        }
        const double h2 = 2.0 * h;
        for (int s = 0; s < ns; ++s) acc[s] = bad ? NAN : (acc[s] * m.M[s]) / h2;
      }
      for (int s = 0; s < ns; ++s) {
        rowsum[s] += fabs(acc[s]);
        if (dom_full) dom[((long long)s * ns + r) * g.N + c] = acc[s];
      }
      if (!dom_full) dom[(long long)r * g.N + c] = acc[r];
    }
    double mx = rowsum[0];
#pragma unroll
    for (int s = 1; s < NSB; ++s)
      if (s < ns) mx = npmax(mx, rowsum[s]);
    if (lamS) lamS[c] = mx;
  }
}

template <int NSB>
__global__ void k_production(const Model* __restrict__ mp, GridDev g, Mech mech,
                             const double* __restrict__ q, double* __restrict__ out,
                             unsigned long long* flags) {
  const Model& m = *mp;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + c, g.N, cs)) raise_flag(flags, EB_DECODE, c);
    double rs[NSB], om[NSB];
#pragma unroll
    for (int s = 0; s < NSB; ++s) rs[s] = (s < m.ns) ? cs.rho * cs.Y[s] : 0.0;
    if (mech.nrx > 0) omega_cell_impl<NSB>(m, mech, cs.T, rs, om);
    else
      for (int s = 0; s < NSB; ++s) om[s] = 0.0;
    for (int s = 0; s < m.ns; ++s) out[s * g.N + c] = om[s];
  }
}

// ------------------------------------------------------------- local time step
// cell_spectral_radii (implicit.py:152-163) + local_time_step (33-44)
CSB_DEV void cell_metric(const GridDev& g, int d, int i, int j, int k, double Sc[3]) {
  int hi[3] = {i, j, k};
  hi[d] += 1;
  double a[3], b[3];
  load_S(g, d, face_index(g, d, i, j, k), a);
  load_S(g, d, face_index(g, d, hi[0], hi[1], hi[2]), b);
#pragma unroll
  for (int x = 0; x < 3; ++x) Sc[x] = 0.5 * (a[x] + b[x]);
}

template <int NSB>
__global__ void k_time_step(const Model* __restrict__ mp, GridDev g, const double* __restrict__ q,
                            const double* __restrict__ cfl_p, const double* __restrict__ lamS, double* __restrict__ dtau,
                            double* __restrict__ lam_inv, double* __restrict__ lam_vis,
                            unsigned long long* flags) {
  const Model& m = *mp;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    const int k = c % g.nk, j = (c / g.nk) % g.nj, i = c / ((long long)g.nk * g.nj);
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + c, g.N, cs)) raise_flag(flags, EB_DECODE, c);
    double mu, kc, D, nf, nsp, nu;
    transport<NSB>(m, cs.T, cs.Y, cs.rho, mu, kc, D);
    diffusivities(mu, kc, D, cs.rho, cs.cp - cs.R, nf, nsp, nu);
    const double V = __ldg(g.vol + c);
    double li[3], lv[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double Sc[3];
      cell_metric(g, d, i, j, k, Sc);
      const double a2 = (Sc[0] * Sc[0] + Sc[1] * Sc[1]) + Sc[2] * Sc[2];
      li[d] = fabs(cs.u[0] * Sc[0] + cs.u[1] * Sc[1] + cs.u[2] * Sc[2]) + cs.c * sqrt(a2);
      lv[d] = nu * a2 / V;
      if (lam_inv) lam_inv[d * g.N + c] = li[d];
      if (lam_vis) lam_vis[d * g.N + c] = lv[d];
    }
    const double J = 1.0 / V;
    const double den = J * (((li[0] + li[1]) + li[2]) + ((lv[0] + lv[1]) + lv[2])) +
                       (lamS ? lamS[c] : 0.0);
    if (!(den > 0.0)) raise_flag(flags, EB_ZERO_WAVE, c);
    if (dtau) dtau[c] = *cfl_p / den;
  }
}

// ------------------------------------------------------------- assembly (cells)
// assemble_lhs (implicit.py:329-403): per-cell state, diagonals.
template <int NSB>
__global__ void k_assemble_cell(const Model* __restrict__ mp, GridDev g,
                                const double* __restrict__ q, const double* __restrict__ dtau,
                                double theta, double dt, OpDev op, unsigned long long* flags) {
  const Model& m = *mp;
  const int ns = m.ns;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < g.N;
       c += (long long)gridDim.x * blockDim.x) {
    const int k = c % g.nk, j = (c / g.nk) % g.nj, i = c / ((long long)g.nk * g.nj);
    Cell<NSB> cs;
    if (!decode<NSB>(m, q + c, g.N, cs)) raise_flag(flags, EB_DECODE, c);
    double mu, kc, D, nf, nsp, nu;
    transport<NSB>(m, cs.T, cs.Y, cs.rho, mu, kc, D);
    diffusivities(mu, kc, D, cs.rho, cs.cp - cs.R, nf, nsp, nu);
    const double V = __ldg(g.vol + c);
    double base = V / dtau[c];
    if (dt > 0.0 && isfinite(dt)) base = base + (1.0 + theta) * V / dt;
    // directional radii at the cell-averaged metric (implicit.py:166-173)
    double rf = 0.0, rs = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double Sc[3];
      cell_metric(g, d, i, j, k, Sc);
      const double a2 = (Sc[0] * Sc[0] + Sc[1] * Sc[1]) + Sc[2] * Sc[2];
      const double U = fabs(cs.u[0] * Sc[0] + cs.u[1] * Sc[1] + cs.u[2] * Sc[2]);
      const double nuf = op.mode == SCH_CI ? nu : nf;
      const double lf = (U + cs.c * sqrt(a2)) + 2.0 * nuf * a2 / V;
      const double ls = U + 2.0 * nsp * a2 / V;
      rf = d == 0 ? lf : rf + lf;
      rs = d == 0 ? ls : rs + ls;
    }
    const double dflow = base + rf;
    op.d[c] = dflow;
    bool bad = !(fabs(dflow) >= 1e-300) || !isfinite(dflow);
    if (op.mode != SCH_CI) {
      const double dsp = base + rs;
      if (op.dsp_per_species) {
        for (int s = 0; s < ns; ++s) {
          const double vd = op.dom_full ? op.dom[((long long)s * ns + s) * g.N + c] * V
                                        : op.dom[(long long)s * g.N + c] * V;
          const double v = dsp - vd;
          op.dsp[(long long)s * g.N + c] = v;
          op.dinv_sp[(long long)s * g.N + c] = 1.0 / v;
          bad |= !(fabs(v) >= 1e-300) || !isfinite(v);
        }
      } else {
        op.dsp[c] = dsp;
        op.dinv_sp[c] = 1.0 / dsp;
        bad |= !(fabs(dsp) >= 1e-300) || !isfinite(dsp);
      }
    }
    if (bad) raise_flag(flags, EB_SINGULAR, c);
    double* st = op.st;
    const long long N = g.N;
    st[ST_RHO * N + c] = cs.rho;
    st[ST_U0 * N + c] = cs.u[0];
    st[ST_U1 * N + c] = cs.u[1];
    st[ST_U2 * N + c] = cs.u[2];
    st[ST_H * N + c] = cs.h;
    st[ST_BETA * N + c] = cs.gamma - 1.0;
    st[ST_EK * N + c] = cs.Ek;
    st[ST_C * N + c] = cs.c;
    st[ST_NF * N + c] = nf;
    st[ST_NSP * N + c] = nsp;
    st[ST_NU * N + c] = nu;
    st[ST_T * N + c] = cs.T;
    if (op.mode == SCH_CI)
      for (int s = 0; s < ns; ++s) op.Y[(long long)s * N + c] = cs.Y[s];
  }
}

cudaError_t CSB_BK(launch_decode)(const Model* mp, int ns, const GridDev& g, const double* q, double* out,
                          unsigned long long* flags, cudaStream_t st) {
  CSB_NS_DISPATCH(ns, { k_decode<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mp, g, q, out, flags); });
  return cudaGetLastError();
}

cudaError_t CSB_BK(launch_source_jacobian)(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                                   const double* q, double* dom, int dom_full, double* lamS,
                                   const double* dom_in, unsigned long long* flags,
                                   cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_source_jac<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mp, g, mech, q, dom, dom_full, lamS,
                                                          dom_in, flags);
  });
  return cudaGetLastError();
}

cudaError_t CSB_BK(launch_production)(const Model* mp, int ns, const GridDev& g, const Mech& mech,
                              const double* q, double* om, unsigned long long* flags,
                              cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_production<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mp, g, mech, q, om, flags);
  });
  return cudaGetLastError();
}

cudaError_t CSB_BK(launch_time_step)(const Model* mp, int ns, const GridDev& g, const double* q, const double* cfl,
                             const double* lamS, double* dtau, double* lam_inv, double* lam_vis,
                             unsigned long long* flags, cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_time_step<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mp, g, q, cfl, lamS, dtau, lam_inv,
                                                         lam_vis, flags);
  });
  return cudaGetLastError();
}

cudaError_t CSB_BK(launch_assemble_cell)(const Model* mp, int ns, const GridDev& g,
                                          const double* q, const double* dtau, double theta,
                                          double dt, OpDev& op, unsigned long long* flags,
                                          cudaStream_t st) {
  CSB_NS_DISPATCH(ns, {
    k_assemble_cell<NSB><<<grid_for(g.N, 128), 128, 0, st>>>(mp, g, q, dtau, theta, dt, op, flags);
  });
  return cudaGetLastError();
}

}  // namespace csb
