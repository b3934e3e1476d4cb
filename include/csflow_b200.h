/*
 * csflow_b200.h -- C ABI of the B200-native implicit pseudo-time iteration of
 * arXiv 2403.03440 (component-splitting, CS, and coupled, CI, LU-SGS).
 *
 * The reference (/root/reference/pkg/src/csflow) has no FFI: its boundary is
 * a set of Python functions.  Each entry point below replaces one of them and
 * cites it as <file>:<line>.  The drop-in Python package
 * paper_2403_03440_b200 binds these symbols with ctypes.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers to FP64 data unless stated.
 *  - Cell fields are SoA, component-major: x[c * N + cell], with
 *    cell = (i * nj + j) * nk + k (the reference's C order, component axis
 *    moved to the front) and N = ni * nj * nk.
 *  - Face fields of direction d are SoA over the face-shaped grid
 *    (n_d + 1 along axis d): S_d[x * NF_d + f], f = (i * nj' + j) * nk' + k.
 *  - Padded primitive layout (fields.py:1-20): [rho, u, v, w, p, Y_1..Y_ns, T].
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *    and asynchronous.  Errors inside kernels are recorded in a device flag
 *    word; csb_status() synchronises the stream and reports them.
 *  - Return value: CSB_OK or a CSB_E* code (csb_last_error() has the text).
 */
#ifndef CSFLOW_B200_H
#define CSFLOW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return / status codes (errors.py:4-75) */
#define CSB_OK 0
#define CSB_E_NONPHYSICAL 1   /* NonPhysicalState (mixture.py:169-193, spatial.py:54, 269; driver.py:223, 250) */
#define CSB_E_SINGULAR 2      /* SingularDiagonal (implicit.py:406-408, lusgs.py:253, 267) */
#define CSB_E_ZEROWAVE 3      /* ZeroWavespeed (implicit.py:42-43) */
#define CSB_E_DIVERGED 4      /* Diverged (driver.py:259-262, 282-283) */
#define CSB_E_MISSINGBC 5     /* MissingBC (boundary.py:60-70) */
#define CSB_E_BADARG 10
#define CSB_E_CUDA 11
#define CSB_E_STATE 12        /* call order (model/grid/bc/workspace not set) */

/* device flag bits reported by csb_status (see csb_common.cuh ErrBit) */
#define CSB_F_DECODE (1u << 0)
#define CSB_F_FACE_T (1u << 1)
#define CSB_F_RES_NONFINITE (1u << 2)
#define CSB_F_ZERO_WAVE (1u << 3)
#define CSB_F_SINGULAR (1u << 4)
#define CSB_F_GATE (1u << 5)
#define CSB_F_KSKIP (1u << 6)     /* informational: the 2-D fast residual found w != 0 under
                                      symmetry k-faces and the library re-ran the general path
                                      on the device (R is valid); later calls of the context
                                      skip the fast path */
#define CSB_F_BLOCK (1u << 7)
#define CSB_F_GATE_DECODE (1u << 8)

/* schemes (implicit.py:30 MODES) */
#define CSB_CI 0
#define CSB_CS1 1
#define CSB_CS2 2

/* boundary kinds (boundary.py:22) */
#define CSB_BC_FARFIELD 0
#define CSB_BC_OUTFLOW 1
#define CSB_BC_WALL 2
#define CSB_BC_SYMMETRY 3
#define CSB_BC_PERIODIC 4

typedef struct csb_ctx csb_ctx;

/* ---------------------------------------------------------------- context */
int csb_create(csb_ctx** out);
void csb_destroy(csb_ctx* ctx);
const char* csb_last_error(const csb_ctx* ctx);
int csb_version(void);
/* Kernel launches issued by this library so far (all contexts). */
unsigned long long csb_launch_count(void);

/* Species table, host arrays of length ns (MixtureModel, mixture.py:58-104). */
int csb_set_model(csb_ctx* ctx, int ns, const double* M, const double* cp, const double* hf,
                  const double* Tref, const double* mu_ref, const double* T_mu,
                  const double* S_mu, double Pr, double Sc);

/* Mechanism (Mechanism/Reaction, chemistry.py:21-43), host arrays:
 * nu_r, nu_p: [nrx][ns] stoichiometry; fwd: [nrx][3] (A_f, b_f, Ea_f);
 * bwd: [nrx][3] (A_b, b_b, Ea_b) with NaN A_b for irreversible reactions.
 * enabled = 0 or nrx = 0 freezes the chemistry. */
int csb_set_mechanism(csb_ctx* ctx, int nrx, const double* nu_r, const double* nu_p,
                      const double* fwd, const double* bwd, int enabled);

/* Grid metrics (StructuredGrid, grid.py:20-48), DEVICE SoA arrays owned by
 * the caller: Si [3][ni+1][nj][nk], Sj [3][ni][nj+1][nk], Sk [3][ni][nj][nk+1],
 * vol [ni][nj][nk]. */
int csb_set_grid(csb_ctx* ctx, int ni, int nj, int nk, const double* Si, const double* Sj,
                 const double* Sk, const double* vol);

/* Boundary condition of face 0..5 = imin, imax, jmin, jmax, kmin, kmax
 * (BoundaryCondition, boundary.py:25-38).  fs_prim: HOST padded-layout
 * freestream vector (6 + ns) for farfield, else NULL; axis = -1 for none. */
int csb_set_bc(csb_ctx* ctx, int face, int kind, double T_wall, int axis, const double* fs_prim);

/* Workspace: bytes needed for the current model/grid (with_block != 0 adds
 * the CI+chemistry ns x ns blocks), then hand over a device buffer of at
 * least that size.  No allocation happens on the hot path. */
size_t csb_workspace_bytes(const csb_ctx* ctx, int with_block);
int csb_set_workspace(csb_ctx* ctx, void* dev, size_t bytes);

/* Read and clear the device flag word (synchronises `stream`).  flags: bit
 * set; first_cell: smallest offending cell index over all set bits; gate_count:
 * number of cells that failed the post-update gate. */
int csb_status(csb_ctx* ctx, unsigned long long* flags, long long* first_cell,
               long long* gate_count, void* stream);

/* ---------------------------------------------------------------- stages */

/* assemble_residual (spatial.py:207-274): q [nv][N] -> R [nv][N].
 * P (nullable): padded primitives [6+ns][(ni+4)(nj+4)(nk+4)] (return_padded).
 * On an nk == 1 grid the library runs the fastest variant whose precondition
 * holds and checks the precondition on the device: planar (w == 0 in every
 * cell), then the 2-D form (k-face fluxes cancel; w == 0 under symmetry
 * k-faces, CSB_F_KSKIP), then the general 3-D form.  The slower variants are
 * queued behind the faster one as guarded launches that exit at once unless
 * it raised its flag, so R is always the general path's result. */
int csb_residual(csb_ctx* ctx, const double* q, double* R, double* P, int first_order,
                 void* stream);

/* Grid-free entry points take the cell count N explicitly (N <= 0: the
 * grid's N); they use only the context's model, mechanism and flag word. */

/* cons_to_prim (mixture.py:287-307): q [nv][N] -> out [12+ns][N] =
 * rho, u, v, w, p, T, c, gamma, h, Ek, R, cp, Y_1..Y_ns. */
int csb_cons_to_prim(csb_ctx* ctx, long long N, const double* q, double* out, void* stream);

/* production_rates (chemistry.py:68-73): omega [ns][N]. */
int csb_production_rates(csb_ctx* ctx, long long N, const double* q, double* omega, void* stream);

/* source_jacobian + source_spectral_radius (chemistry.py:76-104):
 * dOm [ns*ns][N] (entry (s, r) at (s*ns + r)), lamS [N] (nullable). */
int csb_source_jacobian(csb_ctx* ctx, long long N, const double* q, double* dOm, double* lamS,
                        void* stream);

/* cell_spectral_radii (implicit.py:152-163): lam_inv, lam_vis [3][N]. */
int csb_spectral_radii(csb_ctx* ctx, const double* q, double* lam_inv, double* lam_vis,
                       void* stream);

/* local_time_step on given radii (implicit.py:33-44): lam_inv, lam_vis
 * AoS [N][3]; lamS [N] or NULL with lamS_scalar; J [N]. */
int csb_local_time_step(csb_ctx* ctx, long long N, const double* lam_inv, const double* lam_vis,
                        const double* lamS, double lamS_scalar, double cfl, const double* J,
                        double* dtau, void* stream);

/* dtau of one implicit step as _implicit_step computes it (driver.py:235-239):
 * radii + (chemistry) source radius -> dtau [N].  dOm_in (nullable): inject
 * the source Jacobian [ns*ns][N] instead of computing it. */
int csb_time_step(csb_ctx* ctx, const double* q, double cfl, const double* dOm_in, double* dtau,
                  void* stream);

/* assemble_lhs (implicit.py:329-403) into the context's operator buffers.
 * offdiag_paper: species_offdiag == "paper"; theta/dt: dual-time diagonal
 * (dt <= 0 or non-finite = steady).  dOm_in as above. */
int csb_assemble(csb_ctx* ctx, const double* q, const double* dtau, int scheme,
                 int offdiag_paper, double theta, double dt, const double* dOm_in, void* stream);

/* Copy one field of the assembled operator (ImplicitOperator, implicit.py:210-241)
 * into dst (device).  which: 0 w [nv][N], 1 b [nv][N], 2 sp_lower [3][N],
 * 3 sp_upper [3][N], 4 d_scal [N], 5 d_species [ns][N] (broadcast when
 * frozen), 6+d lam_face[d], 9+d lam_face_sp[d] (face-shaped), 12 dinv
 * [ns*ns][N], 13 vdom [ns*ns][N].  q must be the state assembled. */
int csb_operator_field(csb_ctx* ctx, const double* q, int which, double* dst, void* stream);

/* lusgs_solve (lusgs.py:250-274) with the assembled operator: rhs [nv][N] ->
 * dq [nv][N]; dq_star (nullable) receives the forward-sweep result. */
int csb_lusgs(csb_ctx* ctx, const double* rhs, double* dq, double* dq_star, void* stream);

/* _apply_update + admissibility gate (driver.py:216-229, 250): q, dq -> q_new. */
int csb_apply_update(csb_ctx* ctx, long long N, const double* q, const double* dq, int scheme,
                     double* q_new, void* stream);

/* correct_increment_cs1 (mode 1) / correct_normalize_cs2 (mode 2)
 * (implicit.py:113-135) on row-major [rows][ns] arrays. */
int csb_correct(csb_ctx* ctx, int mode, long long rows, int ns, const double* rho_s,
                const double* d_rho_s, const double* d_rho, double* out, void* stream);

/* residual_norms (driver.py:85-90): out3 (device) = flow, species, density. */
int csb_residual_norms(csb_ctx* ctx, long long N, const double* R, double* out3, void* stream);

/* _implicit_step (driver.py:232-251), steady: q, R -> q_new (dq kept in the
 * workspace).  dOm_in as above. */
int csb_implicit_step(csb_ctx* ctx, const double* q, const double* R, double cfl, int scheme,
                      int offdiag_paper, const double* dOm_in, double* q_new, void* stream);

/* As csb_implicit_step with a path choice (0 auto, 1 generic hyperplane
 * sweeps, 2 the 2-D wavefront path) and an optional dq output [nv][N]. */
int csb_implicit_step_ex(csb_ctx* ctx, const double* q, const double* R, double cfl, int scheme,
                         int offdiag_paper, const double* dOm_in, double* q_new, double* dq_out,
                         int path, void* stream);

/* Instrumented 2-D wavefront implicit step: ms5 = {source Jacobian, records,
 * forward sweep, backward sweep, epilogue} device milliseconds (synchronises). */
int csb_profile_step(csb_ctx* ctx, const double* q, const double* R, double cfl, int scheme,
                     double* q_new, float* ms5, void* stream);

/* One steady iteration (driver.py:279-308 without the retry/stop logic):
 * R = residual(q) (R_out nullable: internal), norms -> norms3 (device,
 * nullable), q_new = implicit step. */
int csb_iteration(csb_ctx* ctx, const double* q, double cfl, int scheme, int offdiag_paper,
                  int first_order, double* q_new, double* R_out, double* norms3, void* stream);

/* ---------------------------------------------------------- dual time */
/* Unsteady right-hand side (implicit.py:47-56 dual_time_rhs):
 * rhs = -R - V [(1 + theta)(q_m - q_n) - theta (q_n - q_nm1)] / dt for N
 * cells, all SoA (5 + ns) x N, vol[N] the cell volumes; dt > 0 and finite
 * (steady mode, rhs = -R, needs no call). */
int csb_dual_time_rhs(csb_ctx* ctx, long long N, const double* vol, const double* R, const double* q_m,
                      const double* q_n, const double* q_nm1, double theta, double dt, double* rhs,
                      void* stream);
/* One implicit step of the dual-time inner loop (driver.py:232-251 with
 * dt): rhs as formed by csb_dual_time_rhs, (1 + theta) V / dt added to the
 * diagonal (implicit.py:346-348); species closure and gate as
 * csb_implicit_step.  Runs the generic hyperplane sweeps. */
int csb_implicit_step_rhs(csb_ctx* ctx, const double* q, const double* rhs, double cfl, int scheme,
                          int offdiag_paper, double theta, double dt, double* q_new, void* stream);
/* out[0] = sum x^2 over n values (deterministic order; the dual-time inner
 * residual norm, driver.py:341). */
int csb_sum_squares(csb_ctx* ctx, long long n, const double* x, double* out, void* stream);

/* AoS [N][nv] <-> SoA [nv][N] (device). */
int csb_transpose(long long N, int nv, const double* src, double* dst, int to_soa, void* stream);

/* Batched species block inverse of the coupled operator with chemistry:
 * dinv_c = inv(d_c I - V_c dOmega_c) for N cells (implicit.py:362-368,
 * numpy.linalg.inv per cell).  dOm, dinv: [n*n][N] (block row-major, cell
 * minor); d, V: [N] (V may be NULL: 1).  n <= 32.  n <= 23: one thread per
 * cell (block in shared memory); 24 <= n <= 32: one warp per cell, lane =
 * column in registers.  In-place Gauss-Jordan with partial pivoting.  flags (device, may be NULL):
 * the context flag-word layout; singular / non-finite blocks set EB_BLOCK. */
int csb_batched_inverse(int n, long long N, const double* dOm, const double* d, const double* V,
                        double* dinv, unsigned long long* flags, void* stream);

/* FP64 pipe probe: 4 CTAs x 256 threads per SM, 8 independent DFMA chains
 * per thread, iters x 128 DFMA each (2 flops per DFMA).  scratch: 1 double
 * (device).  Used by bench.py as the measured FP64 peak of the roofline. */
int csb_fp64_peak(int iters, double* scratch, void* stream);

/* ------------------------------------------------------- setup on device */
/* Node fill of the grid generators (grid.py:102-111 generate_box, 139-162
 * generate_cylinder_ogrid) from their 1-D axes (host-computed, numpy's
 * linspace / cos / sin / radial distribution): mode 0 (box)
 * node(i,j,k) = (a[i], b[j], c[k]); mode 1 (cylinder)
 * node(i,j,k) = (b[j] a[i], b[j] s[i], c[k]) with a = cos, s = sin, b = r.
 * nodes: device (n0, n1, n2, 3) AoS; a, s, b, c device vectors. */
int csb_fill_nodes(int mode, int n0, int n1, int n2, const double* a, const double* s,
                   const double* b, const double* c, double* nodes, void* stream);

/* Metric terms (grid.py:51-99 compute_metrics) from device nodes
 * (ni+1, nj+1, nk+1, 3) AoS: face vectors Si/Sj/Sk in the library's SoA face
 * layout, volumes vol[N]; numpy's rounding order (bit-identical metrics).
 * scratch: NF0 + NF1 + NF2 doubles; bad: 2 words (device): bad[0] != 0 when a
 * cell has V <= 1e-30 or non-finite V (DegenerateCell), bad[1] = the first
 * such cell. */
int csb_grid_metrics(int ni, int nj, int nk, const double* nodes, double* Si, double* Sj,
                     double* Sk, double* vol, double* scratch, unsigned long long* bad,
                     void* stream);

/* make_primitive / prim_to_cons (mixture.py:310-351) for n states: u (n x 3)
 * and Y (n x ns, used as given) AoS, two of rho, p, T (n each; the third is
 * NULL and derived from p = rho R(Y) T).  out (nullable): the csb_cons_to_prim
 * layout [rho, u0, u1, u2, p, T, c, gamma, h, Ek, R, cp, Y...] x n SoA;
 * q (nullable): conservative vector (5 + ns) x n SoA.  Non-positive rho, p or
 * T sets CSB_F_DECODE (NonPhysicalState).  Needs the model and workspace. */
int csb_primitive(csb_ctx* ctx, long long n, const double* rho, const double* u, const double* p,
                  const double* T, const double* Y, double* out, double* q, void* stream);

/* Wall-normal heat flux on one noslip_isothermal face (driver.py:132-184):
 * one-sided second-order dT/dn through T_wall and the first two cell
 * centres, k at (T_wall, Y of the first cell).  q: device SoA state; slab:
 * the three node planes nearest the wall along the face's axis (plane 0 =
 * wall), AoS (3, m1+1, m2+1, 3) over the two other axes in increasing
 * order.  qw, pw (device, m1 x m2): heat flux (W/m^2, positive into the
 * wall) and the first cell's pressure. */
int csb_wall_heat_flux(csb_ctx* ctx, int face, const double* q, const double* slab, double* qw,
                       double* pw, void* stream);

/* numpy.argmax(key) (first maximum, NaN first) and val at it
 * (driver.py:187-205 stagnation monitor): out3 = [key_max, val_at, index]. */
int csb_argmax_pick(long long n, const double* key, const double* val, double* out3, void* stream);

/* ------------------------------------------------------ device-resident march */
/* Parameters of a steady march (driver.py:266-317, Case fields). */
typedef struct csb_march_params {
  int scheme;          /* CSB_CI / CSB_CS1 / CSB_CS2 */
  int offdiag_paper;   /* species_offdiag == "paper" */
  int first_order;
  int max_retries;     /* CFL halvings per iteration before Diverged (driver.py:35: 5) */
  double abs_floor;    /* stop when the density residual <= this (< 0: off), driver.py:288-291 */
  double drop_factor;  /* stop when it <= first density residual x this (10^-orders; < 0: off) */
} csb_march_params;

/* Stop codes of csb_march_state (ints4[1]). */
#define CSB_MARCH_RUNNING 0
#define CSB_MARCH_CONVERGED_ABSOLUTE 1
#define CSB_MARCH_CONVERGED_DROP 2
#define CSB_MARCH_CONVERGED_PLATEAU 3
#define CSB_MARCH_NAN_NORM 4          /* Diverged (driver.py:281-283) */
#define CSB_MARCH_RETRIES 5           /* Diverged (driver.py:259-262) */
#define CSB_MARCH_ZERO_WAVESPEED 6    /* ZeroWavespeed */
#define CSB_MARCH_SINGULAR 7          /* SingularDiagonal */
#define CSB_MARCH_RESIDUAL 8          /* NonPhysicalState raised by the residual */

/* Build the march graph for these buffers (steady_solve's loop on the
 * device: residual + norms, stop tests, ramped CFL x cfl_scale, the implicit
 * step with device-side halving retries, cfl_scale recovery; one CUDA graph
 * with conditional nodes, iterations alternating q -> q_alt -> q).  Runs one
 * untimed warm-up step (q_alt scratch).  hist: device [rows][6] rows of
 * (res_flow, res_species, res_density, CFL used, retries, stop code) for
 * iterations 1..rows; cfl_tab: device [rows], Case.cfl_at(it) for
 * it = 0..rows-1 (driver.py:71-75).  Resets the march state. */
int csb_march_begin(csb_ctx* ctx, const csb_march_params* params, double* q, double* q_alt,
                    double* hist, int rows, const double* cfl_tab, void* stream);
/* Run iterations until iteration it_last is recorded or the march stops.
 * plateau_at: iteration at which the monitor-plateau stop fires (0: none;
 * decided by the host from the heat-flux samples, driver.py:300-306);
 * clear_parity: the caller copied q_alt into q. */
int csb_march_run(csb_ctx* ctx, int it_last, int plateau_at, int clear_parity, void* stream);
/* Read the march state (synchronises): ints4 = (iterations recorded, stop
 * code, parity [1: the latest state is in q_alt], retries of the last
 * iteration); reals4 = (cfl_scale, last CFL tried, first density residual,
 * CFL of the current iteration). */
int csb_march_state(csb_ctx* ctx, int* ints4, double* reals4, void* stream);
/* Release the march graph. */
void csb_march_end(csb_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* CSFLOW_B200_H */
