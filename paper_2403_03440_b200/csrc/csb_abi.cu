// csflow-b200: C-ABI entry points (include/csflow_b200.h).
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/csflow_b200.h"
#include "csb_common.cuh"
#include "csb_kernels.cuh"
#include "csb_march.cuh"

using namespace csb;

// csb_grid.cu
cudaError_t csb_launch_fill_nodes(int mode, int n0, int n1, int n2, const double* a, const double* s,
                                  const double* b, const double* c, double* nodes, cudaStream_t st);
cudaError_t csb_launch_metrics(int ni, int nj, int nk, const double* nodes, double* Si, double* Sj,
                               double* Sk, double* vol, double* scratch,
                               unsigned long long* bad, cudaStream_t st);
cudaError_t csb_launch_primitive(const Model* mp, long long n, const double* rho, const double* u,
                                 const double* p, const double* T, const double* Y, double* out,
                                 double* q, unsigned long long* flags, cudaStream_t st);
cudaError_t csb_launch_wall_flux(const Model* mp, int ns, const GridDev& g, int axis, int side,
                                 double Tw, const double* q, const double* slab, double* qw,
                                 double* pw, unsigned long long* flags, cudaStream_t st);
cudaError_t csb_launch_argmax_pick(long long n, const double* key, const double* val, double* out,
                                   cudaStream_t st);

struct csb_ctx {
  int ns = 0;
  bool has_model = false, has_grid = false, has_ws = false;
  Model host_model{};
  Model* d_model = nullptr;
  std::vector<Reaction> rx;
  Reaction* d_rx = nullptr;
  int* d_sprx = nullptr;  // [ns + 1] offsets | reaction lists (Mech::sp_off / sp_rx)
  int nrx_active = 0;
  GridDev g{};
  int geom2d_ok = 0;
  int k2d_disabled = 0;
  int planar_disabled = 0;  // a step found w != 0: skip the planar residual variant
  int bc_kind[6] = {-1, -1, -1, -1, -1, -1};
  int bc_axis[6] = {-1, -1, -1, -1, -1, -1};
  double bc_Tw[6] = {0, 0, 0, 0, 0, 0};
  std::vector<double> fs;  // [6][nc]
  double* d_fs = nullptr;
  bool fs_dirty = true;
  // workspace carve
  char* ws = nullptr;
  size_t ws_bytes = 0;
  bool ws_block = false;
  unsigned long long* flags = nullptr;
  OpDev op{};
  double *dtau = nullptr, *R = nullptr, *dq = nullptr, *partial = nullptr, *norms = nullptr;
  double* cfl_dev = nullptr;  // the step's CFL on the device (kernels read it: graph-safe)
  bool march_capture = false; // csb_march is capturing: cfl_dev is set by its controller
  // device march (csb_march.cuh): one instantiated graph per buffer set
  MarchState* march_st = nullptr;
  cudaGraphExec_t march_exec = nullptr;
  cudaGraph_t march_graph = nullptr;
  double* dom_scratch = nullptr;
  double* norm_partial = nullptr;
  double* fm_buf[2] = {nullptr, nullptr};  // static 2-D face metrics (workspace)
  bool fm_dirty = true;
  unsigned int* norm_counter = nullptr;
  int npart_cap = 0;
  int assembled_scheme = -1;
  WaveBufs wb{};
  bool wave_ok = false;
  int wave_disabled = 0;
  std::string err;
};

namespace {

int fail(csb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_check(csb_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return CSB_OK;
  return fail(c, CSB_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

Mech mech_of(const csb_ctx* c) {
  Mech m;
  m.nrx = c->nrx_active;
  m.rx = c->d_rx;
  m.sp_off = c->d_sprx;
  m.sp_rx = c->d_sprx ? c->d_sprx + c->ns + 1 : nullptr;
  return m;
}

BCDev bc_of(const csb_ctx* c) {
  BCDev b;
  for (int f = 0; f < 6; ++f) {
    b.kind[f] = c->bc_kind[f];
    b.axis[f] = c->bc_axis[f];
    b.Tw[f] = c->bc_Tw[f];
  }
  b.fs = c->d_fs;
  return b;
}

bool bcs_ready(const csb_ctx* c) {
  for (int f = 0; f < 6; ++f)
    if (c->bc_kind[f] < 0) return false;
  return true;
}

int check_bcs(csb_ctx* c) {
  static const char* names[6] = {"imin", "imax", "jmin", "jmax", "kmin", "kmax"};
  for (int f = 0; f < 6; ++f)
    if (c->bc_kind[f] < 0)
      return fail(c, CSB_E_MISSINGBC, std::string("no boundary condition for face '") + names[f] + "'");
  for (int f = 0; f < 6; ++f) {
    if (c->bc_kind[f] == CSB_BC_PERIODIC && c->bc_kind[f ^ 1] != CSB_BC_PERIODIC)
      return fail(c, CSB_E_MISSINGBC, std::string("periodic face '") + names[f] +
                                          "' requires periodic '" + names[f ^ 1] + "'");
  }
  return CSB_OK;
}

bool use_k2d(const csb_ctx* c) {
  if (c->g.nk != 1 || !c->geom2d_ok || c->k2d_disabled) return false;
  const int a = c->bc_kind[4], b = c->bc_kind[5];
  if (a != b) return false;
  if (a == CSB_BC_OUTFLOW || a == CSB_BC_PERIODIC) return true;
  if (a == CSB_BC_SYMMETRY) {
    const bool ax_ok = (c->bc_axis[4] < 0 || c->bc_axis[4] == 2) &&
                       (c->bc_axis[5] < 0 || c->bc_axis[5] == 2);
    return ax_ok;
  }
  return false;
}

int sync_fs(csb_ctx* c) {
  if (!c->fs_dirty) return CSB_OK;
  const int nc = 6 + c->ns;
  if (!c->d_fs) {
    if (cudaMalloc(&c->d_fs, sizeof(double) * 6 * (size_t)(6 + csb::MAXNS)) != cudaSuccess)
      return fail(c, CSB_E_CUDA, "cudaMalloc(freestream)");
  }
  if (c->fs.size() != (size_t)6 * nc) c->fs.assign((size_t)6 * nc, NAN);
  cudaError_t e = cudaMemcpy(c->d_fs, c->fs.data(), sizeof(double) * 6 * nc, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_check(c, e, "upload freestream");
  c->fs_dirty = false;
  return CSB_OK;
}

int ready(csb_ctx* c, bool need_ws = true) {
  if (!c) return CSB_E_BADARG;
  if (!c->has_model) return fail(c, CSB_E_STATE, "model not set");
  if (!c->has_grid) return fail(c, CSB_E_STATE, "grid not set");
  if (need_ws && !c->has_ws) return fail(c, CSB_E_STATE, "workspace not set");
  return CSB_OK;
}

GridDev with_n(const csb_ctx* c, long long N) {
  GridDev g = c->g;
  if (N > 0) g.N = N;
  return g;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {
  size_t off = 0;
  char* base;
  template <class T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off = align_up(off + count * sizeof(T));
    return p;
  }
};

// planes of the FF / FB record groups: CS flow (30), CI coupled
// (3 NV + 10), plus the ns x ns species block inverses of the coupled
// operator with chemistry when the workspace carries blocks (NSB <= 16)
int flow_planes(int nsb, bool with_block) {
  int n = std::max(30, 3 * (5 + nsb) + 10);
  if (with_block && nsb <= 16) n = std::max(n, 3 * (5 + nsb) + 10 + nsb * nsb);
  return n;
}

size_t carve(csb_ctx* c, char* base, bool with_block) {
  Carve k{0, base};
  const long long N = c->g.N;
  const int ns = c->ns, nv = 5 + ns;
  c->flags = k.take<unsigned long long>(FLAG_WORDS);
  c->op.st = k.take<double>((size_t)NST * N);
  c->op.Y = k.take<double>((size_t)ns * N);
  c->op.d = k.take<double>((size_t)N);
  c->op.dsp = k.take<double>((size_t)ns * N);
  c->op.dinv_sp = k.take<double>((size_t)ns * N);
  for (int d = 0; d < 3; ++d) c->op.lam[d] = k.take<double>((size_t)c->g.NF[d]);
  for (int d = 0; d < 3; ++d) c->op.lamsp[d] = k.take<double>((size_t)c->g.NF[d]);
  c->op.dom = k.take<double>((size_t)(with_block ? ns * ns : ns) * N);
  c->op.lamS = k.take<double>((size_t)N);
  c->op.dinv = with_block ? k.take<double>((size_t)ns * ns * N) : nullptr;
  c->dtau = k.take<double>((size_t)N);
  c->R = k.take<double>((size_t)nv * N);
  c->dq = k.take<double>((size_t)nv * N);
  c->partial = k.take<double>(3 * 512);
  // fused residual-norm partials: one per residual tile (tiles hold >= 64 cells
  // except on tiny grids; larger tile counts fall back to the norms kernels)
  c->npart_cap = (int)std::max<long long>(4096, N / 64 + 1);
  c->norm_partial = k.take<double>((size_t)3 * c->npart_cap);
  c->norm_counter = k.take<unsigned int>(64);
  // (no static cell-metric table: the records kernel forms the cell-averaged
  // face vectors from the face vectors, measured as fast as streaming a
  // 16-plane table and 128 B/cell of workspace lighter)
  if (c->g.nk == 1) {
    c->fm_buf[0] = k.take<double>((size_t)6 * c->g.NF[0]);
    c->fm_buf[1] = k.take<double>((size_t)6 * c->g.NF[1]);
  }
  c->norms = k.take<double>(4);
  c->cfl_dev = k.take<double>(1);
  // 2-D wavefront path buffers (csb_wave.cuh): strip-skewed planes
  c->wave_ok = false;
  if (c->g.nk == 1) {
    Skew sk;
    sk.ni = c->g.ni;
    sk.nj = c->g.nj;
    sk.nstrip = (c->g.nj + 31) / 32;
    sk.T = ((c->g.ni + 31 + TQ - 1) / TQ) * TQ;
    sk.Np = (long long)sk.nstrip * sk.T * 32;  // cells per plane (step-major groups)
    c->wb.sk = sk;
    const int nsb = bucket_of(ns);
    const int nff = flow_planes(nsb, with_block);  // CS flow or CI coupled records
    c->wb.ff = k.take<double>((size_t)nff * sk.Np);
    c->wb.fb = k.take<double>((size_t)nff * sk.Np);
    c->wb.fw = k.take<double>((size_t)5 * sk.Np);
    c->wb.sf = k.take<double>((size_t)(2 * nsb + 2) * sk.Np);
    c->wb.sb = k.take<double>((size_t)(2 * nsb + 2) * sk.Np);
    c->wb.sw = k.take<double>((size_t)nsb * sk.Np);
    c->wb.hand = k.take<double>((size_t)2 * sk.nstrip * (sk.T + 2 * HPAD) * (5 + nsb));
    c->wb.prog = k.take<int>(2);
    c->wb.rdy = k.take<int>((size_t)sk.nstrip * sk.T);
    c->wb.nonplanar = k.take<int>(1);
    c->wb.epoch = k.take<int>(1);
    c->wb.nsI = 0;
    c->wave_ok = true;
  }
  return k.off;
}

// Wavefront padding slots (t - r outside [0, ni), rows beyond nj, padding
// species) are never written by the records kernel: they must hold zeros so
// that padding cells contribute exactly nothing to the sweeps (csb_wave.cuh).
int zero_wave_records(csb_ctx* c, cudaStream_t st) {
  const int nsb = bucket_of(c->ns);
  const WaveBufs& w = c->wb;
  const int nff = flow_planes(nsb, c->ws_block);
  const std::pair<double*, int> groups[] = {{w.ff, nff},         {w.fb, nff},
                                            {w.fw, 5},           {w.sf, 2 * nsb + 2},
                                            {w.sb, 2 * nsb + 2}, {w.sw, nsb}};
  for (const auto& gp : groups)
    if (cudaMemsetAsync(gp.first, 0, (size_t)gp.second * w.sk.Np * sizeof(double), st) !=
        cudaSuccess)
      return 1;
  if (cudaMemsetAsync(w.rdy, 0, (size_t)w.sk.nstrip * w.sk.T * sizeof(int), st) != cudaSuccess)
    return 1;
  if (cudaMemsetAsync(w.nonplanar, 0, sizeof(int), st) != cudaSuccess) return 1;
  if (cudaMemsetAsync(w.epoch, 0, sizeof(int), st) != cudaSuccess) return 1;
  return 0;
}

// The K2D residual reads precomputed static face metrics (recomputed after a
// grid change); without them it evaluates the metrics on the fly.
int ensure_face_metrics(csb_ctx* c, cudaStream_t st) {
  if (!c->fm_dirty) return CSB_OK;
  c->g.fm[0] = c->g.fm[1] = nullptr;
  c->g.cm = nullptr;  // cell metrics are formed from the face vectors where used
  if (c->g.nk == 1 && c->geom2d_ok && c->fm_buf[0]) {
    cudaError_t e = launch_face_metrics2d(c->g, c->fm_buf[0], c->fm_buf[1], st);
    if (e != cudaSuccess) return cuda_check(c, e, "face metrics");
    c->g.fm[0] = c->fm_buf[0];
    c->g.fm[1] = c->fm_buf[1];
  }
  c->fm_dirty = false;
  return CSB_OK;
}

int reset_flags(csb_ctx* c, cudaStream_t st) {
  unsigned long long h[FLAG_WORDS];
  for (int i = 0; i < FLAG_WORDS; ++i) h[i] = 0ull;
  for (int b = 0; b < EB_COUNT; ++b) h[1 + b] = ~0ull;
  return cuda_check(c, cudaMemcpyAsync(c->flags, h, sizeof(h), cudaMemcpyHostToDevice, st),
                    "reset flags");
}

}  // namespace

extern "C" {

int csb_version(void) { return 1; }

unsigned long long csb_launch_count(void) { return launch_count(); }

int csb_create(csb_ctx** out) {
  if (!out) return CSB_E_BADARG;
  *out = new csb_ctx();
  return CSB_OK;
}

void csb_destroy(csb_ctx* c) {
  if (!c) return;
  if (c->d_model) cudaFree(c->d_model);
  if (c->d_rx) cudaFree(c->d_rx);
  if (c->d_sprx) cudaFree(c->d_sprx);
  if (c->d_fs) cudaFree(c->d_fs);
  if (c->wb.s2) cudaStreamDestroy(c->wb.s2);
  if (c->march_exec) cudaGraphExecDestroy(c->march_exec);
  if (c->march_graph) cudaGraphDestroy(c->march_graph);
  if (c->march_st) cudaFree(c->march_st);
  if (c->wb.e1) cudaEventDestroy(c->wb.e1);
  if (c->wb.e2) cudaEventDestroy(c->wb.e2);
  delete c;
}

const char* csb_last_error(const csb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int csb_set_model(csb_ctx* c, int ns, const double* M, const double* cp, const double* hf,
                  const double* Tref, const double* mu_ref, const double* T_mu,
                  const double* S_mu, double Pr, double Sc) {
  if (!c) return CSB_E_BADARG;
  if (ns < 1 || ns > MAXNS) return fail(c, CSB_E_BADARG, "ns must be in [1, 64]");
  Model m{};
  m.ns = ns;
  m.Pr = Pr;
  m.Sc = Sc;
  m.iPr = 1.0 / Pr;
  m.iSc = 1.0 / Sc;
  for (int s = 0; s < ns; ++s) {
    m.M[s] = M[s];
    m.cp[s] = cp[s];
    m.Rs[s] = R_U / M[s];
    m.bs[s] = hf[s] - cp[s] * Tref[s];
    m.mu_ref[s] = mu_ref[s];
    m.T_mu[s] = T_mu[s];
    m.S_mu[s] = S_mu[s];
    m.TS[s] = T_mu[s] + S_mu[s];
    m.inv_T_mu[s] = 1.0 / T_mu[s];
  }
  m.suth_shared = 1;
  for (int s = 1; s < ns; ++s)
    if (T_mu[s] != T_mu[0] || S_mu[s] != S_mu[0]) m.suth_shared = 0;
  if (!c->d_model && cudaMalloc(&c->d_model, sizeof(Model)) != cudaSuccess)
    return fail(c, CSB_E_CUDA, "cudaMalloc(model)");
  cudaError_t e = cudaMemcpy(c->d_model, &m, sizeof(Model), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_check(c, e, "upload model");
  if (c->has_model && c->ns != ns) {
    c->has_ws = false;
    c->fs.clear();
  }
  c->host_model = m;
  c->ns = ns;
  c->has_model = true;
  c->fs_dirty = true;
  return CSB_OK;
}

int csb_set_mechanism(csb_ctx* c, int nrx, const double* nu_r, const double* nu_p,
                      const double* fwd, const double* bwd, int enabled) {
  if (!c || !c->has_model) return fail(c, CSB_E_STATE, "set the model before the mechanism");
  const int ns = c->ns;
  std::vector<Reaction> v;
  for (int r = 0; r < nrx; ++r) {
    Reaction x{};
    x.Af = fwd[3 * r];
    x.bf = fwd[3 * r + 1];
    x.Eaf = fwd[3 * r + 2];
    x.has_back = bwd && !std::isnan(bwd[3 * r]);
    if (x.has_back) {
      x.Ab = bwd[3 * r];
      x.bb = bwd[3 * r + 1];
      x.Eab = bwd[3 * r + 2];
    }
    for (int s = 0; s < ns; ++s) {
      const double a = nu_r[(size_t)r * ns + s], b = nu_p[(size_t)r * ns + s];
      if (a != 0.0) {
        if (x.nr >= MAXTERM) return fail(c, CSB_E_BADARG, "too many reactant terms");
        x.rs[x.nr] = s;
        x.rn[x.nr++] = a;
      }
      if (b != 0.0) {
        if (x.np >= MAXTERM) return fail(c, CSB_E_BADARG, "too many product terms");
        x.ps[x.np] = s;
        x.pn[x.np++] = b;
      }
      if (b - a != 0.0) {
        x.ds[x.nd] = s;
        x.dn[x.nd++] = b - a;
      }
    }
    v.push_back(x);
  }
  if (c->d_rx) {
    cudaFree(c->d_rx);
    c->d_rx = nullptr;
  }
  if (!v.empty()) {
    if (cudaMalloc(&c->d_rx, sizeof(Reaction) * v.size()) != cudaSuccess)
      return fail(c, CSB_E_CUDA, "cudaMalloc(reactions)");
    cudaError_t e = cudaMemcpy(c->d_rx, v.data(), sizeof(Reaction) * v.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_check(c, e, "upload reactions");
  }
  // species -> reactions CSR for the sparse finite-difference Jacobian
  if (c->d_sprx) {
    cudaFree(c->d_sprx);
    c->d_sprx = nullptr;
  }
  if (!v.empty()) {
    std::vector<int> off(ns + 1, 0), lst;
    for (int s = 0; s < ns; ++s) {
      for (int r = 0; r < (int)v.size(); ++r) {
        bool dep = false;
        for (int t = 0; t < v[r].nr; ++t) dep |= v[r].rs[t] == s;
        for (int t = 0; t < v[r].np && v[r].has_back; ++t) dep |= v[r].ps[t] == s;
        if (dep) lst.push_back(r);
      }
      off[s + 1] = (int)lst.size();
    }
    std::vector<int> all(off);
    all.insert(all.end(), lst.begin(), lst.end());
    if (cudaMalloc(&c->d_sprx, sizeof(int) * all.size()) != cudaSuccess)
      return fail(c, CSB_E_CUDA, "cudaMalloc(species-reaction map)");
    cudaError_t e = cudaMemcpy(c->d_sprx, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_check(c, e, "upload species-reaction map");
  }
  c->rx = v;
  c->nrx_active = (enabled && nrx > 0) ? nrx : 0;
  return CSB_OK;
}

int csb_set_grid(csb_ctx* c, int ni, int nj, int nk, const double* Si, const double* Sj,
                 const double* Sk, const double* vol) {
  if (!c) return CSB_E_BADARG;
  if (ni < 1 || nj < 1 || nk < 1) return fail(c, CSB_E_BADARG, "grid dims must be positive");
  const bool changed = !c->has_grid || c->g.ni != ni || c->g.nj != nj || c->g.nk != nk;
  GridDev g{};
  g.ni = ni;
  g.nj = nj;
  g.nk = nk;
  g.N = (long long)ni * nj * nk;
  g.S[0] = Si;
  g.S[1] = Sj;
  g.S[2] = Sk;
  g.NF[0] = (long long)(ni + 1) * nj * nk;
  g.NF[1] = (long long)ni * (nj + 1) * nk;
  g.NF[2] = (long long)ni * nj * (nk + 1);
  g.vol = vol;
  c->g = g;
  c->has_grid = true;
  c->fm_dirty = true;
  if (changed) c->has_ws = false;
  c->geom2d_ok = 0;
  c->k2d_disabled = 0;
  c->planar_disabled = 0;
  if (nk == 1) {
    int* d_ok = nullptr;
    if (cudaMalloc(&d_ok, sizeof(int)) != cudaSuccess) return fail(c, CSB_E_CUDA, "cudaMalloc");
    int one = 1;
    cudaMemcpy(d_ok, &one, sizeof(int), cudaMemcpyHostToDevice);
    launch_check_2d(g, d_ok, 0);
    cudaError_t e = cudaMemcpy(&one, d_ok, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d_ok);
    if (e != cudaSuccess) return cuda_check(c, e, "check 2-D geometry");
    c->geom2d_ok = one;
  }
  return CSB_OK;
}

int csb_set_bc(csb_ctx* c, int face, int kind, double T_wall, int axis, const double* fs_prim) {
  if (!c || !c->has_model) return fail(c, CSB_E_STATE, "set the model before boundary conditions");
  if (face < 0 || face > 5 || kind < 0 || kind > 4) return fail(c, CSB_E_BADARG, "bad face/kind");
  if (kind == CSB_BC_FARFIELD && !fs_prim)
    return fail(c, CSB_E_MISSINGBC, "farfield boundary requires a freestream state");
  if (kind == CSB_BC_WALL && !(T_wall > 0.0))
    return fail(c, CSB_E_MISSINGBC, "isothermal wall requires T_wall > 0");
  c->bc_kind[face] = kind;
  c->bc_axis[face] = axis;
  c->bc_Tw[face] = T_wall;
  const int nc = 6 + c->ns;
  if (c->fs.size() != (size_t)6 * nc) c->fs.assign((size_t)6 * nc, NAN);
  for (int k = 0; k < nc; ++k) c->fs[(size_t)face * nc + k] = fs_prim ? fs_prim[k] : NAN;
  c->fs_dirty = true;
  c->k2d_disabled = 0;
  c->planar_disabled = 0;
  return CSB_OK;
}

size_t csb_workspace_bytes(const csb_ctx* c, int with_block) {
  if (!c || !c->has_model || !c->has_grid) return 0;
  csb_ctx tmp = *c;
  return carve(&tmp, nullptr, with_block != 0) + 256;
}

int csb_set_workspace(csb_ctx* c, void* dev, size_t bytes) {
  int r = ready(c, false);
  if (r) return r;
  const size_t need_plain = csb_workspace_bytes(c, 0);
  const size_t need_block = csb_workspace_bytes(c, 1);
  if (bytes < need_plain) return fail(c, CSB_E_BADARG, "workspace too small");
  char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(dev)));
  c->ws_block = bytes >= need_block;
  carve(c, base, c->ws_block);
  c->ws = reinterpret_cast<char*>(dev);
  c->ws_bytes = bytes;
  c->has_ws = true;
  c->assembled_scheme = -1;
  c->fm_dirty = true;
  if (cudaMemset(c->norm_counter, 0, 64 * sizeof(unsigned int)) != cudaSuccess)
    return fail(c, CSB_E_CUDA, "zero norm counter");
  if (c->wave_ok) {
    // wavefront padding slots (t - r outside [0, ni), rows beyond nj) are never
    // written by the records kernel: they must hold zeros so that padding
    // cells contribute exactly nothing to the sweep (csb_wave.cuh)
    if (zero_wave_records(c, 0)) return fail(c, CSB_E_CUDA, "zero wavefront records");
  }
  return reset_flags(c, 0) ? CSB_E_CUDA : (cudaDeviceSynchronize() == cudaSuccess ? CSB_OK : CSB_E_CUDA);
}

int csb_status(csb_ctx* c, unsigned long long* flags, long long* first_cell, long long* gate_count,
               void* stream) {
  int r = ready(c);
  if (r) return r;
  cudaStream_t st = S(stream);
  unsigned long long h[FLAG_WORDS];
  cudaError_t e = cudaMemcpyAsync(h, c->flags, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_check(c, e, "read status");
  if (flags) *flags = h[0] & ~(1ull << EB_NONPLANAR);
  if (first_cell) {
    *first_cell = -1;  // smallest offending cell over all raised bits
    for (int b = 0; b < EB_COUNT; ++b)
      if ((h[0] & (1ull << b)) && b != EB_KSKIP && b != EB_NONPLANAR) {
        const long long cb = (long long)h[1 + b];
        if (*first_cell < 0 || cb < *first_cell) *first_cell = cb;
      }
  }
  if (gate_count) *gate_count = (long long)h[FLAG_GATE_COUNT];
  if (h[0] & (1ull << EB_KSKIP)) c->k2d_disabled = 1;
  if (h[0] & (1ull << EB_NONPLANAR)) c->planar_disabled = 1;
  return reset_flags(c, st);
}

int csb_residual(csb_ctx* c, const double* q, double* R, double* P, int first_order,
                 void* stream) {
  int r = ready(c);
  if (r) return r;
  if ((r = check_bcs(c))) return r;
  if ((r = sync_fs(c))) return r;
  cudaStream_t st = S(stream);
  if ((r = ensure_face_metrics(c, st))) return r;
  const bool k2d = use_k2d(c), planar = k2d && !c->planar_disabled;
  cudaError_t e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order,
                                  planar ? RES_K2D_PLANAR : (k2d ? RES_K2D : RES_GENERAL), c->flags, st);
  // preconditions checked by the launches themselves; the slower variants
  // re-run on the device when the faster one raised its flag (no-ops
  // otherwise): planar (w == 0 everywhere, EB_NONPLANAR) -> K2D (w == 0
  // under symmetry k-faces, EB_KSKIP) -> general
  const NormsOut none{nullptr, 0, nullptr, nullptr};
  if (e == cudaSuccess && planar)
    e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order, RES_K2D,
                        c->flags, st, none, nullptr, c->flags, EB_NONPLANAR);
  if (e == cudaSuccess && k2d)
    e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order,
                        RES_GENERAL, c->flags, st, none, nullptr, c->flags, EB_KSKIP);
  if (e == cudaSuccess && P) e = launch_padded(c->d_model, c->ns, c->g, bc_of(c), q, P, c->flags, st);
  return cuda_check(c, e, "residual");
}

int csb_cons_to_prim(csb_ctx* c, long long N, const double* q, double* out, void* stream) {
  int r = ready(c);
  if (r) return r;
  return cuda_check(c, launch_decode(c->d_model, c->ns, with_n(c, N), q, out, c->flags, S(stream)),
                    "decode");
}

int csb_production_rates(csb_ctx* c, long long N, const double* q, double* omega, void* stream) {
  int r = ready(c);
  if (r) return r;
  return cuda_check(c, launch_production(c->d_model, c->ns, with_n(c, N), mech_of(c), q, omega, c->flags,
                                         S(stream)),
                    "production");
}

int csb_source_jacobian(csb_ctx* c, long long N, const double* q, double* dOm, double* lamS,
                        void* stream) {
  int r = ready(c);
  if (r) return r;
  const GridDev g = with_n(c, N);
  if (mech_of(c).nrx == 0) {
    cudaStream_t st = S(stream);
    cudaError_t e = cudaMemsetAsync(dOm, 0, sizeof(double) * c->ns * c->ns * g.N, st);
    if (e == cudaSuccess && lamS) e = cudaMemsetAsync(lamS, 0, sizeof(double) * g.N, st);
    return cuda_check(c, e, "source jacobian (frozen)");
  }
  return cuda_check(c, launch_source_jacobian(c->d_model, c->ns, g, mech_of(c), q, dOm, 1, lamS,
                                              nullptr, c->flags, S(stream)),
                    "source jacobian");
}

int csb_spectral_radii(csb_ctx* c, const double* q, double* lam_inv, double* lam_vis,
                       void* stream) {
  int r = ready(c);
  if (r) return r;
  return cuda_check(c, launch_time_step(c->d_model, c->ns, c->g, q, nullptr, nullptr, nullptr, lam_inv,
                                        lam_vis, c->flags, S(stream)),
                    "spectral radii");
}

int csb_local_time_step(csb_ctx* c, long long N, const double* lam_inv, const double* lam_vis,
                        const double* lamS, double lamS_scalar, double cfl, const double* J,
                        double* dtau, void* stream) {
  if (!c || !c->has_ws) return fail(c, CSB_E_STATE, "workspace (flags) not set");
  return cuda_check(c, launch_dtau_arrays(N, lam_inv, lam_vis, lamS, lamS_scalar, cfl, J, dtau,
                                          c->flags, S(stream)),
                    "local_time_step");
}

static int time_step_impl(csb_ctx* c, const double* q, const double* cfl, const double* dOm_in,
                          double* dtau, bool full_dom, cudaStream_t st) {
  const bool chem = mech_of(c).nrx > 0;
  const double* lamS = nullptr;
  cudaError_t e = cudaSuccess;
  if (chem) {
    e = launch_source_jacobian(c->d_model, c->ns, c->g, mech_of(c), q, c->op.dom, full_dom ? 1 : 0,
                               c->op.lamS, dOm_in, c->flags, st);
    lamS = c->op.lamS;
  }
  if (e == cudaSuccess)
    e = launch_time_step(c->d_model, c->ns, c->g, q, cfl, lamS, dtau, nullptr, nullptr, c->flags,
                         st);
  return cuda_check(c, e, "time step");
}

int csb_time_step(csb_ctx* c, const double* q, double cfl, const double* dOm_in, double* dtau,
                  void* stream) {
  int r = ready(c);
  if (r) return r;
  cudaError_t e = launch_set_double(c->cfl_dev, cfl, S(stream));
  if (e != cudaSuccess) return cuda_check(c, e, "time step");
  return time_step_impl(c, q, c->cfl_dev, dOm_in, dtau, c->ws_block, S(stream));
}

static int assemble_impl(csb_ctx* c, const double* q, const double* dtau, int scheme,
                         int offdiag_paper, double theta, double dt, const double* dOm_in,
                         bool dom_ready, cudaStream_t st) {
  if (scheme < 0 || scheme > 2) return fail(c, CSB_E_BADARG, "unknown scheme");
  const bool chem = mech_of(c).nrx > 0;
  if (chem && scheme == SCH_CI && !c->ws_block)
    return fail(c, CSB_E_STATE, "CI with chemistry needs a workspace with blocks");
  OpDev& op = c->op;
  op.mode = scheme;
  op.sp_scale = offdiag_paper ? 1.0 : 0.5;
  op.chem = chem ? 1 : 0;
  op.dsp_per_species = chem ? 1 : 0;
  op.dom_full = (chem && c->ws_block) ? 1 : 0;
  cudaError_t e = cudaSuccess;
  if (chem && !dom_ready)
    e = launch_source_jacobian(c->d_model, c->ns, c->g, mech_of(c), q, op.dom, op.dom_full,
                               op.lamS, dOm_in, c->flags, st);
  if (e == cudaSuccess)
    e = launch_assemble(c->d_model, c->ns, c->g, q, dtau, theta, dt, op, c->flags, st);
  c->assembled_scheme = scheme;
  return cuda_check(c, e, "assemble");
}

int csb_assemble(csb_ctx* c, const double* q, const double* dtau, int scheme, int offdiag_paper,
                 double theta, double dt, const double* dOm_in, void* stream) {
  int r = ready(c);
  if (r) return r;
  return assemble_impl(c, q, dtau, scheme, offdiag_paper, theta, dt, dOm_in, false, S(stream));
}

int csb_operator_field(csb_ctx* c, const double* q, int which, double* dst, void* stream) {
  int r = ready(c);
  if (r) return r;
  if (c->assembled_scheme < 0) return fail(c, CSB_E_STATE, "no operator assembled");
  cudaStream_t st = S(stream);
  const long long N = c->g.N;
  const int ns = c->ns;
  cudaError_t e = cudaSuccess;
  auto cp = [&](const double* src, size_t n) {
    return cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  };
  if (which <= 3) {
    e = launch_export_op(c->d_model, ns, c->g, c->op, q, which, dst, st);
  } else if (which == 4) {
    e = cp(c->op.d, N);
  } else if (which == 5) {
    if (c->op.dsp_per_species) e = cp(c->op.dsp, (size_t)ns * N);
    else
      for (int s = 0; s < ns && e == cudaSuccess; ++s)
        e = cudaMemcpyAsync(dst + (size_t)s * N, c->op.dsp, N * sizeof(double),
                            cudaMemcpyDeviceToDevice, st);
  } else if (which >= 6 && which <= 8) {
    e = cp(c->op.lam[which - 6], c->g.NF[which - 6]);
  } else if (which >= 9 && which <= 11) {
    e = cp(c->op.lamsp[which - 9], c->g.NF[which - 9]);
  } else if (which == 12) {
    if (!c->op.dinv || !(c->op.chem && c->op.mode == SCH_CI))
      return fail(c, CSB_E_STATE, "no CI species block inverse");
    e = cp(c->op.dinv, (size_t)ns * ns * N);
  } else if (which == 13) {
    if (!c->op.dom_full) return fail(c, CSB_E_STATE, "full dOmega not stored");
    e = launch_export_op(c->d_model, ns, c->g, c->op, q, 4, dst, st);
  } else {
    return fail(c, CSB_E_BADARG, "unknown operator field");
  }
  return cuda_check(c, e, "operator field");
}

int csb_lusgs(csb_ctx* c, const double* rhs, double* dq, double* dq_star, void* stream) {
  int r = ready(c);
  if (r) return r;
  if (c->assembled_scheme < 0) return fail(c, CSB_E_STATE, "no operator assembled");
  cudaStream_t st = S(stream);
  cudaError_t e = cudaMemsetAsync(dq, 0, sizeof(double) * (5 + c->ns) * c->g.N, st);
  c->op.neg_rhs = 0;
  if (e == cudaSuccess)
    e = launch_sweeps(c->d_model, c->ns, c->g, c->op, rhs, dq, dq_star, c->flags, st);
  return cuda_check(c, e, "lusgs");
}

int csb_apply_update(csb_ctx* c, long long N, const double* q, const double* dq, int scheme,
                     double* q_new, void* stream) {
  int r = ready(c);
  if (r) return r;
  return cuda_check(c, launch_update(c->d_model, c->ns, with_n(c, N), scheme, q, dq, q_new, c->flags,
                                     S(stream)),
                    "apply update");
}

int csb_correct(csb_ctx* c, int mode, long long rows, int ns, const double* rho_s,
                const double* d_rho_s, const double* d_rho, double* out, void* stream) {
  if (!c || !c->has_ws) return fail(c, CSB_E_STATE, "workspace (flags) not set");
  if (mode != 1 && mode != 2) return fail(c, CSB_E_BADARG, "mode must be 1 (CS1) or 2 (CS2)");
  return cuda_check(c, launch_correct(mode, rows, ns, rho_s, d_rho_s, d_rho, out, c->flags, S(stream)),
                    "correct");
}

int csb_residual_norms(csb_ctx* c, long long N, const double* R, double* out3, void* stream) {
  int r = ready(c);
  if (r) return r;
  return cuda_check(c, launch_norms(c->ns, N > 0 ? N : c->g.N, R, c->partial, out3, S(stream)),
                    "norms");
}

// path: 0 auto, 1 generic (hyperplane sweeps), 2 2-D wavefront
// Residual + grouped norms of one iteration (driver.py:85-90, 279): the
// fused residual kernel, its device-side general-path fallback when the K2D
// precondition fails (EB_KSKIP: w != 0 under symmetry k-faces; a no-op
// launch otherwise), and the standalone norms when they could not be fused.
static cudaError_t residual_norms_impl(csb_ctx* c, const double* q, double* R, int first_order,
                                       double* norms3, cudaStream_t st) {
  bool fused = false, fused2 = true, fused3 = true;
  const bool k2d = use_k2d(c), planar = k2d && !c->planar_disabled;
  const NormsOut nrm{c->norm_partial, c->npart_cap, c->norm_counter, norms3};
  const NormsOut none{nullptr, 0, nullptr, nullptr};
  cudaError_t e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order,
                                  planar ? RES_K2D_PLANAR : (k2d ? RES_K2D : RES_GENERAL), c->flags,
                                  st, nrm, &fused);
  if (e == cudaSuccess && planar)
    e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order, RES_K2D,
                        c->flags, st, fused ? nrm : none, &fused3, c->flags, EB_NONPLANAR);
  if (e == cudaSuccess && k2d)
    e = launch_residual(c->d_model, c->ns, c->g, bc_of(c), mech_of(c), q, R, first_order,
                        RES_GENERAL, c->flags, st, fused ? nrm : none, &fused2, c->flags, EB_KSKIP);
  if (!fused3) fused2 = false;
  if (e == cudaSuccess && (!fused || !fused2))
    e = launch_norms(c->ns, c->g.N, R, c->partial, norms3, st);
  return e;
}

// One implicit step.  rhs_is_R: `R` is the residual (rhs = -R, steady);
// otherwise `R` is the right-hand side itself (dual time, csb_dual_time_rhs)
// and theta, dt add (1 + theta) V / dt to the diagonal (implicit.py:346-348).
static int implicit_impl(csb_ctx* c, const double* q, const double* R, double cfl, int scheme,
                         int offdiag_paper, const double* dOm_in, double* q_new, cudaStream_t st,
                         int path = 0, double* dq_out = nullptr, cudaEvent_t* ev = nullptr,
                         double theta = 0.0, double dt = 0.0, bool rhs_is_R = true) {
  if (int r0 = ensure_face_metrics(c, st)) return r0;
  if (!c->march_capture) {  // (in a captured march the controller kernel sets it)
    cudaError_t e0 = launch_set_double(c->cfl_dev, cfl, st);
    if (e0 != cudaSuccess) return cuda_check(c, e0, "implicit step");
  }
  const bool chem = mech_of(c).nrx > 0;
  const bool full = chem && scheme == SCH_CI;
  const bool dual = dt > 0.0 && std::isfinite(dt);
  if (full && !c->ws_block) return fail(c, CSB_E_STATE, "CI with chemistry needs block workspace");
  // the coupled operator takes the wavefront path when frozen, and with
  // chemistry up to 16 species (the ns x ns block inverses ride in the
  // records); dual-time steps (extra diagonal and rhs terms) take the
  // generic hyperplane path
  const bool ci_wave = scheme != SCH_CI || !chem || (c->ws_block && bucket_of(c->ns) <= 16);
  const bool wave = path != 1 && c->wave_ok && !c->wave_disabled && ci_wave && c->geom2d_ok &&
                    rhs_is_R && !dual;
  if (path == 2 && !wave) return fail(c, CSB_E_STATE, "2-D wavefront path not applicable");
  if (wave) {
    cudaError_t e = cudaSuccess;
    const double* lamS = nullptr;
    const double* domd = nullptr;
    int dstride = 1;
    if (chem) {
      OpDev& op = c->op;
      op.dom_full = c->ws_block ? 1 : 0;
      e = launch_source_jacobian(c->d_model, c->ns, c->g, mech_of(c), q, op.dom, op.dom_full,
                                 op.lamS, dOm_in, c->flags, st);
      lamS = op.lamS;
      domd = op.dom;
      dstride = op.dom_full ? c->ns + 1 : 1;
    }
    const int nsI = scheme == SCH_CI ? (chem ? -2 : -1) : chem ? c->ns : 1;  // record layout key
    c->wb.ci_d = c->op.d;
    c->wb.ci_dinv = c->op.dinv;
    if (e == cudaSuccess && c->wb.nsI != nsI) {
      // species record layout changes with nsI: re-zero the padding slots
      e = zero_wave_records(c, st) ? cudaErrorUnknown : cudaSuccess;
      c->wb.nsI = nsI;
    }
    if (e == cudaSuccess && !c->wb.s2) {
      // high-priority side stream of the overlapped forward sweep
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      if (cudaStreamCreateWithPriority(&c->wb.s2, cudaStreamNonBlocking, hi) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->wb.e1, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->wb.e2, cudaEventDisableTiming) != cudaSuccess)
        e = cudaErrorUnknown;
    }
    if (e == cudaSuccess)
      e = launch_wave_step(c->d_model, c->ns, c->g, c->wb, q, R, c->cfl_dev, lamS, domd, dstride,
                           chem ? 1 : 0, scheme, offdiag_paper ? 1.0 : 0.5, q_new, dq_out, c->flags,
                           st, ev);
    if (e == cudaErrorInvalidConfiguration && path == 0) {
      c->wave_disabled = 1;  // ring does not fit shared memory: generic path
      cudaGetLastError();
    } else {
      return cuda_check(c, e, "implicit step (wavefront)");
    }
  }
  int r = time_step_impl(c, q, c->cfl_dev, dOm_in, c->dtau, full, st);
  if (r) return r;
  OpDev& op = c->op;
  op.dom_full = full ? 1 : 0;
  r = assemble_impl(c, q, c->dtau, scheme, offdiag_paper, theta, dual ? dt : 0.0, dOm_in, true, st);
  if (r) return r;
  // rhs = -R: the sweeps negate on load (exact)
  double* dq = dq_out ? dq_out : c->dq;
  cudaError_t e = cudaMemsetAsync(dq, 0, sizeof(double) * (5 + c->ns) * c->g.N, st);
  op.neg_rhs = rhs_is_R ? 1 : 0;
  if (e == cudaSuccess) e = launch_sweeps(c->d_model, c->ns, c->g, op, R, dq, nullptr, c->flags, st);
  op.neg_rhs = 0;
  if (e == cudaSuccess) e = launch_update(c->d_model, c->ns, c->g, scheme, q, dq, q_new, c->flags, st);
  return cuda_check(c, e, "implicit step");
}

int csb_profile_step(csb_ctx* c, const double* q, const double* R, double cfl, int scheme,
                     double* q_new, float* ms5, void* stream) {
  int r = ready(c);
  if (r) return r;
  cudaStream_t st = S(stream);
  cudaEvent_t ev[6];
  for (int k = 0; k < 6; ++k) cudaEventCreate(&ev[k]);
  cudaEventRecord(ev[5], st);
  r = implicit_impl(c, q, R, cfl, scheme, 0, nullptr, q_new, st, 2, nullptr, ev);
  if (r == CSB_OK) {
    cudaStreamSynchronize(st);
    cudaEventElapsedTime(&ms5[0], ev[5], ev[0]);  // source Jacobian (chemistry) / launch gap
    for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms5[1 + k], ev[k], ev[k + 1]);
  }
  for (int k = 0; k < 6; ++k) cudaEventDestroy(ev[k]);
  return r;
}

int csb_implicit_step_ex(csb_ctx* c, const double* q, const double* R, double cfl, int scheme,
                         int offdiag_paper, const double* dOm_in, double* q_new, double* dq_out,
                         int path, void* stream) {
  int r = ready(c);
  if (r) return r;
  return implicit_impl(c, q, R, cfl, scheme, offdiag_paper, dOm_in, q_new, S(stream), path, dq_out);
}

int csb_implicit_step(csb_ctx* c, const double* q, const double* R, double cfl, int scheme,
                      int offdiag_paper, const double* dOm_in, double* q_new, void* stream) {
  int r = ready(c);
  if (r) return r;
  return implicit_impl(c, q, R, cfl, scheme, offdiag_paper, dOm_in, q_new, S(stream));
}

int csb_iteration(csb_ctx* c, const double* q, double cfl, int scheme, int offdiag_paper,
                  int first_order, double* q_new, double* R_out, double* norms3, void* stream) {
  int r = ready(c);
  if (r) return r;
  if ((r = check_bcs(c))) return r;
  if ((r = sync_fs(c))) return r;
  cudaStream_t st = S(stream);
  if ((r = ensure_face_metrics(c, st))) return r;
  double* R = R_out ? R_out : c->R;
  cudaError_t e = residual_norms_impl(c, q, R, first_order, norms3 ? norms3 : c->norms, st);
  if (e != cudaSuccess) return cuda_check(c, e, "iteration residual");
  return implicit_impl(c, q, R, cfl, scheme, offdiag_paper, nullptr, q_new, st);
}

int csb_dual_time_rhs(csb_ctx* c, long long N, const double* vol, const double* R, const double* q_m,
                      const double* q_n, const double* q_nm1, double theta, double dt, double* rhs,
                      void* stream) {
  int r = ready(c);
  if (r) return r;
  if (N < 0 || !vol || !R || !q_m || !q_n || !q_nm1 || !rhs) return CSB_E_BADARG;
  if (!(dt > 0.0) || !std::isfinite(dt))
    return fail(c, CSB_E_BADARG, "dual_time_rhs: dt must be positive and finite (steady: rhs = -R)");
  if (N == 0) return CSB_OK;
  return cuda_check(c, launch_dual_rhs(N, 5 + c->ns, R, q_m, q_n, q_nm1, vol, theta, dt, rhs,
                                       S(stream)),
                    "dual time rhs");
}

int csb_implicit_step_rhs(csb_ctx* c, const double* q, const double* rhs, double cfl, int scheme,
                          int offdiag_paper, double theta, double dt, double* q_new,
                          void* stream) {
  int r = ready(c);
  if (r) return r;
  return implicit_impl(c, q, rhs, cfl, scheme, offdiag_paper, nullptr, q_new, S(stream), 1, nullptr,
                       nullptr, theta, dt, false);
}

int csb_sum_squares(csb_ctx* c, long long n, const double* x, double* out, void* stream) {
  int r = ready(c);
  if (r) return r;
  if (n < 0 || !x || !out) return CSB_E_BADARG;
  return cuda_check(c, launch_sumsq(n, x, c->partial, out, S(stream)), "sum of squares");
}

int csb_transpose(long long N, int nv, const double* src, double* dst, int to_soa, void* stream) {
  return launch_transpose(N, nv, src, dst, to_soa, S(stream)) == cudaSuccess ? CSB_OK : CSB_E_CUDA;
}

int csb_batched_inverse(int n, long long N, const double* dOm, const double* d, const double* V,
                        double* dinv, unsigned long long* flags, void* stream) {
  if (n < 1 || n > 32 || N < 0 || !dOm || !d || !dinv) return CSB_E_BADARG;
  if (N == 0) return CSB_OK;
  return launch_block_inverse(n, N, dOm, d, V, dinv, flags, S(stream)) == cudaSuccess ? CSB_OK
                                                                                      : CSB_E_CUDA;
}

int csb_fill_nodes(int mode, int n0, int n1, int n2, const double* a, const double* s,
                   const double* b, const double* c, double* nodes, void* stream) {
  if ((mode != 0 && mode != 1) || n0 < 1 || n1 < 1 || n2 < 1 || !a || !b || !c || !nodes ||
      (mode == 1 && !s))
    return CSB_E_BADARG;
  return csb_launch_fill_nodes(mode, n0, n1, n2, a, s, b, c, nodes, S(stream)) == cudaSuccess
             ? CSB_OK
             : CSB_E_CUDA;
}

int csb_grid_metrics(int ni, int nj, int nk, const double* nodes, double* Si, double* Sj,
                     double* Sk, double* vol, double* scratch, unsigned long long* bad,
                     void* stream) {
  if (ni < 1 || nj < 1 || nk < 1 || !nodes || !Si || !Sj || !Sk || !vol || !scratch || !bad)
    return CSB_E_BADARG;
  cudaStream_t st = S(stream);
  const unsigned long long init[2] = {0ull, ~0ull};
  if (cudaMemcpyAsync(bad, init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess)
    return CSB_E_CUDA;
  return csb_launch_metrics(ni, nj, nk, nodes, Si, Sj, Sk, vol, scratch, bad, st) == cudaSuccess
             ? CSB_OK
             : CSB_E_CUDA;
}

int csb_primitive(csb_ctx* c, long long n, const double* rho, const double* u, const double* p,
                  const double* T, const double* Y, double* out, double* q, void* stream) {
  if (!c) return CSB_E_BADARG;
  if (!c->has_model) return fail(c, CSB_E_STATE, "model not set");
  if (!c->has_ws) return fail(c, CSB_E_STATE, "workspace not set");
  const int given = (rho != nullptr) + (p != nullptr) + (T != nullptr);
  if (n < 0 || !u || !Y || given < 2 || (!out && !q))
    return fail(c, CSB_E_BADARG, "primitive: need u, Y and two of (rho, p, T)");
  if (n == 0) return CSB_OK;
  return cuda_check(c, csb_launch_primitive(c->d_model, n, rho, u, p, T, Y, out, q, c->flags, S(stream)),
                    "primitive");
}

int csb_wall_heat_flux(csb_ctx* c, int face, const double* q, const double* slab, double* qw,
                       double* pw, void* stream) {
  int r = ready(c);
  if (r) return r;
  if (face < 0 || face > 5 || !q || !slab || !qw || !pw) return CSB_E_BADARG;
  if (c->bc_kind[face] != CSB_BC_WALL)
    return fail(c, CSB_E_BADARG, "wall_heat_flux: face is not a noslip_isothermal wall");
  const int axis = face / 2, side = face % 2;
  const int dims[3] = {c->g.ni, c->g.nj, c->g.nk};
  if (dims[axis] < 2) return fail(c, CSB_E_BADARG, "wall_heat_flux: need two cells off the wall");
  return cuda_check(c, csb_launch_wall_flux(c->d_model, c->ns, c->g, axis, side, c->bc_Tw[face], q,
                                            slab, qw, pw, c->flags, S(stream)),
                    "wall heat flux");
}

int csb_argmax_pick(long long n, const double* key, const double* val, double* out3, void* stream) {
  if (n < 0 || !key || !val || !out3) return CSB_E_BADARG;
  return csb_launch_argmax_pick(n, key, val, out3, S(stream)) == cudaSuccess ? CSB_OK : CSB_E_CUDA;
}

int csb_fp64_peak(int iters, double* scratch, void* stream) {
  if (iters < 1 || !scratch) return CSB_E_BADARG;
  return launch_fp64_peak(iters, scratch, S(stream)) == cudaSuccess ? CSB_OK : CSB_E_CUDA;
}

// ------------------------------------------------------------ device march
}  // extern "C"

namespace {

// A conditional handle on the graph the stream is capturing into.
cudaError_t new_handle(cudaStream_t s, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  return cudaGraphConditionalHandleCreate(h, g, 0, cudaGraphCondAssignDefault);
}

// Appends a conditional node on handle h after the stream's current capture
// dependencies and returns its body graph.
cudaError_t add_cond_node(cudaStream_t s, cudaGraphConditionalHandle h,
                          cudaGraphConditionalNodeType type, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps;
  size_t nd;
  cudaError_t e = cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd);
  if (e != cudaSuccess) return e;
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, g, deps, nd, &p)) != cudaSuccess) return e;
  *body = p.conditional.phGraph_out[0];
  return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

struct MarchBuild {
  csb_ctx* c;
  MarchCfg cfg;
  int scheme, paper, first_order;
  cudaStream_t lv[6];  // one capture stream per nesting level
};

cudaError_t begin_body(cudaStream_t s, cudaGraph_t body) {
  return cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
}
cudaError_t end_body(cudaStream_t s) {
  cudaGraph_t g;
  return cudaStreamEndCapture(s, &g);
}

// One pseudo-time iteration qin -> qout captured on nesting level L
// (structure in csb_march.cuh).
cudaError_t capture_iteration(MarchBuild& b, int L, const double* qin, double* qout) {
  csb_ctx* c = b.c;
  cudaStream_t s = b.lv[L], s1 = b.lv[L + 1], s2 = b.lv[L + 2];
  cudaError_t e = residual_norms_impl(c, qin, c->R, b.first_order, c->norms, s);
  cudaGraphConditionalHandle hstep, hretry;
  cudaGraph_t gstep, gretry;
  if (e == cudaSuccess) e = new_handle(s, &hstep);
  if (e != cudaSuccess) return e;
  k_march_pre<<<1, 1, 0, s>>>(b.cfg, hstep);
  if ((e = add_cond_node(s, hstep, cudaGraphCondTypeIf, &gstep)) != cudaSuccess) return e;
  // IF(step): retry loop, then the bookkeeping of the accepted step
  if ((e = begin_body(s1, gstep)) != cudaSuccess) return e;
  if ((e = new_handle(s1, &hretry)) == cudaSuccess) {
    k_cond_set<<<1, 1, 0, s1>>>(hretry, 1u);
    e = add_cond_node(s1, hretry, cudaGraphCondTypeWhile, &gretry);
  }
  if (e == cudaSuccess) e = begin_body(s2, gretry);
  if (e == cudaSuccess) {
    int r = implicit_impl(c, qin, c->R, 0.0, b.scheme, b.paper, nullptr, qout, s2);
    if (r != CSB_OK) e = cudaErrorUnknown;
    k_march_after<<<1, 1, 0, s2>>>(b.cfg, hretry);
    cudaError_t e2 = end_body(s2);
    if (e == cudaSuccess) e = e2;
  }
  if (e == cudaSuccess) k_march_post<<<1, 1, 0, s1>>>(b.cfg);
  cudaError_t e1 = end_body(s1);
  return e != cudaSuccess ? e : e1;
}

cudaError_t build_march(MarchBuild& b, const double* q, double* q_alt, cudaGraph_t* out) {
  cudaStream_t s0 = b.lv[0], s1 = b.lv[1], s2 = b.lv[2];
  cudaError_t e = cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle hloop, hb;
  cudaGraph_t gloop, gb;
  if ((e = new_handle(s0, &hloop)) == cudaSuccess) {
    k_march_cond<<<1, 1, 0, s0>>>(b.cfg, hloop);
    e = add_cond_node(s0, hloop, cudaGraphCondTypeWhile, &gloop);
  }
  if (e == cudaSuccess && (e = begin_body(s1, gloop)) == cudaSuccess) {
    e = capture_iteration(b, 1, q, q_alt);  // iteration A (levels 1..3)
    if (e == cudaSuccess && (e = new_handle(s1, &hb)) == cudaSuccess) {
      k_march_cond<<<1, 1, 0, s1>>>(b.cfg, hb);
      e = add_cond_node(s1, hb, cudaGraphCondTypeIf, &gb);
    }
    if (e == cudaSuccess && (e = begin_body(s2, gb)) == cudaSuccess) {
      e = capture_iteration(b, 2, q_alt, const_cast<double*>(q));  // iteration B (levels 2..4)
      cudaError_t e2 = end_body(s2);
      if (e == cudaSuccess) e = e2;
    }
    if (e == cudaSuccess) k_march_cond<<<1, 1, 0, s1>>>(b.cfg, hloop);
    cudaError_t e1 = end_body(s1);
    if (e == cudaSuccess) e = e1;
  }
  cudaGraph_t g = nullptr;
  cudaError_t e0 = cudaStreamEndCapture(s0, &g);
  if (e == cudaSuccess) e = e0;
  if (e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return e;
  }
  *out = g;
  return cudaSuccess;
}

}  // namespace

extern "C" {

void csb_march_end(csb_ctx* c) {
  if (!c) return;
  if (c->march_exec) cudaGraphExecDestroy(c->march_exec);
  if (c->march_graph) cudaGraphDestroy(c->march_graph);
  c->march_exec = nullptr;
  c->march_graph = nullptr;
}

int csb_march_begin(csb_ctx* c, const csb_march_params* p, double* q, double* q_alt, double* hist,
                    int rows, const double* cfl_tab, void* stream) {
  int r = ready(c);
  if (r) return r;
  if (!p || !q || !q_alt || !hist || rows < 1 || !cfl_tab) return CSB_E_BADARG;
  if (p->scheme < 0 || p->scheme > 2) return fail(c, CSB_E_BADARG, "march: unknown scheme");
  if ((r = check_bcs(c))) return r;
  if ((r = sync_fs(c))) return r;
  cudaStream_t st = S(stream);
  if ((r = ensure_face_metrics(c, st))) return r;
  csb_march_end(c);
  if (!c->march_st && cudaMalloc(&c->march_st, sizeof(MarchState)) != cudaSuccess)
    return fail(c, CSB_E_CUDA, "cudaMalloc(march state)");
  // warm-up step outside the capture: lazily created streams, record
  // layouts and padding zeros are in place before the graph is built
  cudaError_t e = residual_norms_impl(c, q, c->R, p->first_order, c->norms, st);
  if (e != cudaSuccess) return cuda_check(c, e, "march warm-up");
  if ((r = implicit_impl(c, q, c->R, 1.0, p->scheme, p->offdiag_paper, nullptr, q_alt, st)))
    return r;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_check(c, e, "march warm-up");
  MarchBuild b{};
  b.c = c;
  b.scheme = p->scheme;
  b.paper = p->offdiag_paper;
  b.first_order = p->first_order;
  b.cfg.st = c->march_st;
  b.cfg.hist = hist;
  b.cfg.rows = rows;
  b.cfg.cfl_tab = cfl_tab;
  b.cfg.norms = c->norms;
  b.cfg.cfl_dev = c->cfl_dev;
  b.cfg.flags = c->flags;
  b.cfg.abs_floor = p->abs_floor;
  b.cfg.drop_factor = p->drop_factor;
  b.cfg.max_retries = p->max_retries;
  for (auto& x : b.lv)
    if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess)
      return fail(c, CSB_E_CUDA, "march: stream");
  c->march_capture = true;
  c->wb.serial = 1;
  cudaGraph_t g = nullptr;
  e = build_march(b, q, q_alt, &g);
  c->march_capture = false;
  c->wb.serial = 0;
  for (auto& x : b.lv) cudaStreamDestroy(x);
  if (e == cudaSuccess) e = cudaGraphInstantiate(&c->march_exec, g, 0);
  if (e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return cuda_check(c, e, "march graph");
  }
  c->march_graph = g;
  k_march_init<<<1, 1, 0, st>>>(c->march_st);
  if ((r = reset_flags(c, st))) return r;
  return cuda_check(c, cudaGetLastError(), "march init");
}

int csb_march_run(csb_ctx* c, int it_last, int plateau_at, int clear_parity, void* stream) {
  if (!c || !c->march_exec) return c ? fail(c, CSB_E_STATE, "march: csb_march_begin first") : CSB_E_BADARG;
  cudaStream_t st = S(stream);
  k_march_chunk<<<1, 1, 0, st>>>(c->march_st, it_last, plateau_at, clear_parity);
  note_launches(1);
  return cuda_check(c, cudaGraphLaunch(c->march_exec, st), "march chunk");
}

int csb_march_state(csb_ctx* c, int* ints4, double* reals4, void* stream) {
  if (!c || !c->march_st || !ints4 || !reals4) return CSB_E_BADARG;
  MarchState h;
  cudaStream_t st = S(stream);
  cudaError_t e = cudaMemcpyAsync(&h, c->march_st, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_check(c, e, "march state");
  ints4[0] = h.it;
  ints4[1] = h.stop;
  ints4[2] = h.parity;
  ints4[3] = h.attempt;
  reals4[0] = h.cfl_scale;
  reals4[1] = h.cfl_try;
  reals4[2] = h.res0;
  reals4[3] = h.cfl_now;
  return CSB_OK;
}

}  // extern "C"
