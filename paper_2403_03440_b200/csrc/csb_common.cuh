// csflow-b200: shared device types and closures (sm_100a, FP64).
//
// Layout contract (see include/csflow_b200.h): every cell field is SoA,
// component-major, cell index c = (i*nj + j)*nk + k (the reference's C order
// with the component axis moved to the front).  Face arrays of direction d are
// SoA over the face-shaped grid (n_d + 1 along axis d).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#define CSB_DEV __device__ __forceinline__

namespace csb {

constexpr int MAXNS = 64;
constexpr int NG = 2;  // ghost layers (reference fields.py:14)
constexpr double R_U = 8.314462618;  // mixture.py:26
constexpr double EPS_NEG = 1e-10;    // mixture.py:30

// Error bits of the device flag word.  The host maps them onto the
// reference's exception classes in pipeline order (csflow_b200.h).
enum ErrBit : int {
  EB_DECODE = 0,       // cons_to_prim on the input state (NonPhysicalState)
  EB_FACE_T = 1,       // face temperature <= 0 (spatial.py:54-55)
  EB_RES_NONFINITE = 2,// non-finite residual (spatial.py:269-271)
  EB_ZERO_WAVE = 3,    // local_time_step denominator <= 0 (implicit.py:42-43)
  EB_SINGULAR = 4,     // _check_diag / lusgs underflow (implicit.py:406-408)
  EB_GATE = 5,         // post-update admissibility (driver.py:223-224, 250; implicit.py:138-141)
  EB_KSKIP = 6,        // 2-D fast-path precondition violated (internal)
  EB_BLOCK = 7,        // CI species block not invertible (implicit.py:365-368)
  EB_GATE_DECODE = 8,  // post-update cons_to_prim gate (driver.py:250)
  EB_NONPLANAR = 9,    // planar 2-D residual found w != 0 (internal: the K2D kernel re-runs;
                       // never reported, csb_status masks it)
  EB_COUNT = 10
};
// flag buffer layout (unsigned long long): [0] bits, [1+b] first cell of bit b,
// [15] gate-failure count
constexpr int FLAG_WORDS = 16;
constexpr int FLAG_GATE_COUNT = 15;

struct Model {
  int ns;
  int suth_shared;  // every species has the same (T_mu, S_mu): one Sutherland factor per state
  double Pr, Sc;
  double iPr, iSc;  // 1 / Pr, 1 / Sc (fused 2-D face flux)
  double M[MAXNS], cp[MAXNS], Rs[MAXNS], bs[MAXNS];
  double mu_ref[MAXNS], T_mu[MAXNS], S_mu[MAXNS], TS[MAXNS];  // TS = T_mu + S_mu
  double inv_T_mu[MAXNS];                                      // 1 / T_mu
};
// the per-species arrays of Model, contiguous from M (copied per block by
// the residual kernel, first ns entries of each)
constexpr int MODEL_NARR = 9;

// Reactions in the reference's order; stoichiometry kept as (species, nu)
// pairs in ascending species order (chemistry.py:56-62 iterates np.nonzero).
constexpr int MAXTERM = 6;
struct Reaction {
  double Af, bf, Eaf, Ab, bb, Eab;
  int has_back;
  int nr, np;
  int rs[MAXTERM], ps[MAXTERM];
  double rn[MAXTERM], pn[MAXTERM];
  int nd;                       // species with nonzero (nu'' - nu')
  int ds[2 * MAXTERM];
  double dn[2 * MAXTERM];
};

struct Mech {
  int nrx;  // 0 = frozen
  const Reaction* rx;
  // species -> reactions whose rate depends on it (reactant or product),
  // CSR: reactions of species s at sp_rx[sp_off[s] .. sp_off[s + 1])
  const int* sp_off;
  const int* sp_rx;
};

struct GridDev {
  int ni, nj, nk;
  long long N;
  const double* S[3];   // SoA face vectors, S[d][x*NF_d + f]
  long long NF[3];
  const double* vol;
  const double* fm[2];  // 2-D viscous face metrics [6][NF_d] (xn, xt), or null
  const double* cm;     // static cell metrics [16][N] (cell_metric), or null
};

enum BcKind : int { BC_FARFIELD = 0, BC_OUTFLOW = 1, BC_WALL = 2, BC_SYMMETRY = 3, BC_PERIODIC = 4 };

struct BCDev {
  int kind[6];
  int axis[6];
  double Tw[6];
  const double* fs;  // [6][nc] padded-layout freestream vectors (device)
};

CSB_DEV long long cell_index(const GridDev& g, int i, int j, int k) {
  return ((long long)i * g.nj + j) * g.nk + k;
}

CSB_DEV long long face_index(const GridDev& g, int d, int i, int j, int k) {
  // (i, j, k) with index d ranging over [0, n_d]
  if (d == 0) return ((long long)i * g.nj + j) * g.nk + k;
  if (d == 1) return ((long long)i * (g.nj + 1) + j) * g.nk + k;
  return ((long long)i * g.nj + j) * (g.nk + 1) + k;
}

CSB_DEV void load_S(const GridDev& g, int d, long long f, double S[3]) {
  const double* p = g.S[d];
  const long long nf = g.NF[d];
  S[0] = __ldg(p + f);
  S[1] = __ldg(p + nf + f);
  S[2] = __ldg(p + 2 * nf + f);
}

// Metric terms of a 2-D face of direction D at global face (gi, gj):
// xn = S / Vf, xt = face average of the tangential axis' cell-averaged
// Sc * J (spatial.py:236-248).
template <int D>
CSB_DEV void face_metric2d(const GridDev& g, int gi, int gj, const double S[3], double xn[3],
                           double xt[3], bool& hasm, bool& hasp, long long& cellm,
                           long long& cellp) {
  constexpr int A = 1 - D;  // tangential in-plane axis
  const int nd = D == 0 ? g.ni : g.nj;
  const int pos = D == 0 ? gi : gj;
  const int mi = D == 0 ? gi - 1 : gi, mj = D == 0 ? gj : gj - 1;
  hasm = pos > 0;
  hasp = pos < nd;
  cellm = hasm ? cell_index(g, mi, mj, 0) : -1;
  cellp = hasp ? cell_index(g, gi, gj, 0) : -1;
  const double Vm = hasm ? __ldg(g.vol + cellm) : 0.0;
  const double Vp = hasp ? __ldg(g.vol + cellp) : 0.0;
  const double Vf = (hasm && hasp) ? 0.5 * (Vp + Vm) : (hasm ? Vm : Vp);
#pragma unroll
  for (int x = 0; x < 3; ++x) xn[x] = S[x] / Vf;
  double xc[2][3];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const bool has = side == 0 ? hasm : hasp;
    if (!has) continue;
    const int ci = side == 0 ? mi : gi, cj = side == 0 ? mj : gj;
    double Slo[3], Shi[3];
    load_S(g, A, face_index(g, A, ci, cj, 0), Slo);
    load_S(g, A, face_index(g, A, ci + (A == 0), cj + (A == 1), 0), Shi);
    const double J = 1.0 / (side == 0 ? Vm : Vp);
#pragma unroll
    for (int x = 0; x < 3; ++x) xc[side][x] = (0.5 * (Slo[x] + Shi[x])) * J;
  }
#pragma unroll
  for (int x = 0; x < 3; ++x)
    xt[x] = (hasm && hasp) ? 0.5 * (xc[1][x] + xc[0][x]) : (hasm ? xc[0][x] : xc[1][x]);
}

// Cell-averaged face vector of direction d (grid.py Sc_d), |Sc|^2 and |Sc|
// (implicit.py:152-163), from the static table when present.  Table rows:
// [5d + 0..2] Sc_d, [5d + 3] a2, [5d + 4] sqrt(a2), [15] 1 / V.
CSB_DEV void cell_metric(const GridDev& g, long long c, int i, int j, int k, int d, double Sc[3],
                         double& a2, double& sq) {
  if (g.cm) {
#pragma unroll
    for (int x = 0; x < 3; ++x) Sc[x] = __ldg(g.cm + (5 * d + x) * g.N + c);
    a2 = __ldg(g.cm + (5 * d + 3) * g.N + c);
    sq = __ldg(g.cm + (5 * d + 4) * g.N + c);
    return;
  }
  int hi[3] = {i, j, k};
  hi[d] += 1;
  double a[3], b[3];
  load_S(g, d, face_index(g, d, i, j, k), a);
  load_S(g, d, face_index(g, d, hi[0], hi[1], hi[2]), b);
#pragma unroll
  for (int x = 0; x < 3; ++x) Sc[x] = 0.5 * (a[x] + b[x]);
  a2 = (Sc[0] * Sc[0] + Sc[1] * Sc[1]) + Sc[2] * Sc[2];
  sq = sqrt(a2);
}
CSB_DEV double inv_volume(const GridDev& g, long long c) {
  return g.cm ? __ldg(g.cm + 15 * g.N + c) : 1.0 / __ldg(g.vol + c);
}

// numpy.maximum: NaN-propagating
CSB_DEV double npmax(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : (b > a ? b : a);
}

// minmod with numpy's np.where semantics (spatial.py:22-27): a NaN operand
// fails both comparisons, exactly as in the reference.
CSB_DEV double minmod(double a, double b) {
  double out = (fabs(a) < fabs(b)) ? a : b;
  return (a * b <= 0.0) ? 0.0 : out;
}

CSB_DEV bool finite(double x) { return isfinite(x); }

CSB_DEV void raise_flag(unsigned long long* fl, int bit, long long cell) {
  atomicOr(fl, 1ull << bit);
  atomicMin(fl + 1 + bit, (unsigned long long)cell);
}

// Sutherland viscosity of species s (mixture.py:368); (T/T_mu)^1.5 as x*sqrt(x)
CSB_DEV double mu_species(const Model& m, int s, double T) {
  const double x = T * m.inv_T_mu[s];
  return m.mu_ref[s] * (x * sqrt(x)) * m.TS[s] / (T + m.S_mu[s]);
}

// Decoded cell state (mixture.py:287-307 cons_to_prim with clipping).
template <int NSB>
struct Cell {
  double rho, u[3], p, T, Y[NSB], c, gamma, h, Ek, R, cp;
};

// Decode conservative vector q[c*stride] into primitives.  Returns false on
// the reference's NonPhysicalState conditions (rho, Y < -eps, T).
// QK(k) returns component k (a pointer read or a register array element:
// the register form keeps the caller's array out of local memory).
template <int NSB, class QK>
CSB_DEV bool decode_from(const Model& m, QK qk, Cell<NSB>& o) {
  const int ns = m.ns;
  const double rho = qk(0);
  bool ok = (rho > 0.0) && finite(rho);
  // reciprocal multiplies instead of divisions (last-ulp differences only)
  const double ir = 1.0 / rho;
  o.rho = rho;
#pragma unroll
  for (int x = 0; x < 3; ++x) o.u[x] = qk(1 + x) * ir;
  double sum = 0.0;
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      double y = qk(5 + s) * ir;
      if (y < -EPS_NEG) ok = false;
      if (y < 0.0) y = 0.0;
      o.Y[s] = y;
      sum += y;
    } else {
      o.Y[s] = 0.0;
    }
  }
  double R = 0.0, cp = 0.0, yb = 0.0;
  const double isum = 1.0 / sum;
#pragma unroll
  for (int s = 0; s < NSB; ++s) {
    if (s < ns) {
      const double y = o.Y[s] * isum;
      o.Y[s] = y;
      R += y * m.Rs[s];
      cp += y * m.cp[s];
      yb += y * m.bs[s];
    }
  }
  o.Ek = 0.5 * ((o.u[0] * o.u[0] + o.u[1] * o.u[1]) + o.u[2] * o.u[2]);
  const double cv = cp - R;
  const double icv = 1.0 / cv;
  const double e_int = qk(4) * ir - o.Ek;
  o.T = (e_int - yb) * icv;
  if (!(o.T > 0.0) || !finite(o.T)) ok = false;
  o.R = R;
  o.cp = cp;
  o.p = rho * R * o.T;
  o.gamma = cp * icv;
  o.c = sqrt(o.gamma * R * o.T);
  o.h = yb + cp * o.T + o.Ek;
  return ok;
}

template <int NSB>
CSB_DEV bool decode(const Model& m, const double* __restrict__ q, long long stride, Cell<NSB>& o) {
  if constexpr (NSB <= 8) {
    // all components first, through a running pointer (loads in flight
    // together, one 64-bit add per component instead of a multiply-add)
    double qv[5 + NSB];
    const double* p = q;
    const int nv = 5 + m.ns;
#pragma unroll
    for (int k = 0; k < 5 + NSB; ++k, p += stride) qv[k] = k < nv ? *p : 0.0;
    return decode_from<NSB>(m, [&](int k) { return qv[k]; }, o);
  } else {
    return decode_from<NSB>(m, [&](int k) { return q[k * stride]; }, o);
  }
}

// Transport (mixture.py:354-372): mu, k, D (D identical for all species).
template <int NSB>
CSB_DEV void transport(const Model& m, double T, const double* Y, double rho, double& mu, double& k,
                       double& D) {
  double acc = 0.0, cp = 0.0;
  if (m.suth_shared) {
    // mu_s = mu_ref_s * F(T) with F shared by all species: one sqrt and one
    // division per state instead of ns (reassociated: last-ulp differences)
    const double x = T * m.inv_T_mu[0];
    const double F = (x * sqrt(x)) * m.TS[0] / (T + m.S_mu[0]);
#pragma unroll
    for (int s = 0; s < NSB; ++s) {
      if (s < m.ns) {
        acc += Y[s] * (m.mu_ref[s] * F);
        cp += Y[s] * m.cp[s];
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < NSB; ++s) {
      if (s < m.ns) {
        acc += Y[s] * mu_species(m, s, T);
        cp += Y[s] * m.cp[s];
      }
    }
  }
  mu = acc;
  k = mu * cp / m.Pr;
  D = mu / (rho * m.Sc);
}

// Diffusivities (implicit.py:144-149).
CSB_DEV void diffusivities(double mu, double k, double D, double rho, double cv, double& nf,
                           double& nsp, double& nu) {
  nf = npmax(4.0 * mu / (3.0 * rho), k / (rho * cv));
  nsp = D;
  nu = npmax(nf, nsp);
}

// Deterministic block reduction helper (sum of doubles over a CTA).
template <int NT>
CSB_DEV double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) r += sh[i];
  }
  return r;
}

// ns bucket dispatch: NSB is the compile-time register-array bound.  The
// templated kernels are instantiated once per bucket in separate translation
// units (csb_bucket.cu compiled with -DCSB_BUCKET=<b>); their launchers are
// named <name>_b<b> there (CSB_BK) and routed by csb_dispatch.cu.
#define CSB_BUCKET_LIST(X) X(2) X(4) X(5) X(6) X(8) X(12) X(16) X(20) X(24) X(32) X(40) X(48) X(64)
#define CSB_CAT2(a, b) a##_b##b
#define CSB_CAT(a, b) CSB_CAT2(a, b)
#ifdef CSB_BUCKET
#define CSB_BK(name) CSB_CAT(name, CSB_BUCKET)
#define CSB_NS_DISPATCH(ns, ...)            \
  do {                                      \
    (void)(ns);                             \
    constexpr int NSB = CSB_BUCKET;         \
    __VA_ARGS__;                            \
  } while (0)
#endif

static inline int bucket_of(int ns) {
  return ns <= 2 ? 2 : ns <= 4 ? 4 : ns <= 5 ? 5 : ns <= 6 ? 6 : ns <= 8 ? 8 : ns <= 12 ? 12
       : ns <= 16 ? 16 : ns <= 20 ? 20 : ns <= 24 ? 24 : ns <= 32 ? 32 : ns <= 40 ? 40
       : ns <= 48 ? 48 : 64;
}

// Tuning / timing probe knobs (environment) exist only in builds with
// -DCSB_PROBES; production builds ignore them.  The launch-order knobs
// CSB_NO_OVERLAP / CSB_FORCE_OVERLAP are always honoured (both orders are
// valid and parity-tested).
static inline const char* probe_env(const char* name) {
#ifdef CSB_PROBES
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// SMs of the current device (cached per process).
static inline int device_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  return sms;
}

static inline int grid_for(long long n, int bs) {
  long long b = (n + bs - 1) / bs;
  if (b < 1) b = 1;
  if (b > 148LL * 32) b = 148LL * 32;
  return (int)b;
}

}  // namespace csb
