// csflow-b200: device-resident steady march (reference driver.py:254-317,
// SURVEY §8(f) row 1), included by csb_abi.cu (it drives the context's
// residual and implicit-step launchers).
//
// One CUDA graph holds a whole chunk of pseudo-time iterations.  Every
// decision of the reference's loop is taken on the device by small
// controller kernels that steer conditional graph nodes:
//
//   top:   k_march_cond(loop)   WHILE(loop): iteration A (q -> q_alt),
//            k_march_cond(b), IF(b): iteration B (q_alt -> q), k_march_cond(loop)
//   iteration X:
//     residual + grouped norms (driver.py:85-90, 279)
//     k_march_pre   NaN norms -> Diverged; CFL of the ramp x cfl_scale
//                   (driver.py:71-75, 308); absolute floor, residual drop and
//                   (host-decided) monitor-plateau stops (driver.py:288-306)
//     IF(step):
//       WHILE(retry): implicit step at the device CFL (csb_implicit_step's
//                     kernels) + k_march_after: decode failure or gate ->
//                     halve the CFL and retry, <= max_retries times, then
//                     Diverged; zero wavespeed / singular diagonal stop the
//                     march (driver.py:254-263)
//       k_march_post  record the iteration (norms, CFL used, retries), update
//                     cfl_scale (x CFL used / CFL tried on retry, else x1.2
//                     capped at 1, driver.py:309-313), continue or end
//
// Iterations A and B alternate the state buffers, so no copy is needed
// inside a chunk.  The host launches one chunk per monitor interval (the
// stagnation heat-flux monitor, driver.py:187-205, is sampled between
// chunks) and reads the history rows once per chunk.
#pragma once

namespace csb {

enum MarchStop : int {
  MS_RUN = 0, MS_ABS = 1, MS_DROP = 2, MS_PLATEAU = 3, MS_NAN = 4, MS_RETRIES = 5, MS_ZERO = 6,
  MS_SINGULAR = 7, MS_RESIDUAL = 8
};

struct MarchState {
  int it;          // iterations recorded so far
  int it_last;     // the chunk ends after recording this iteration
  int stop;        // MarchStop
  int attempt;     // retries of the current iteration
  int parity;      // 0: the current state is in q, 1: in q_alt
  int plateau_at;  // iteration at which the host's plateau test fires (0: none)
  int pad[2];
  double cfl_scale, cfl_now, cfl_try, res0;
  double norms[3];
};

struct MarchCfg {
  MarchState* st;
  double* hist;          // [rows][MARCH_HIST] : flow, species, density, cfl used, retries, stop
  int rows;
  const double* cfl_tab; // cfl_at(it) for it = 0 .. rows - 1 (the host's ramp, driver.py:71-75)
  const double* norms;   // the residual norms of the current iteration
  double* cfl_dev;       // the implicit step's CFL (device)
  unsigned long long* flags;
  double abs_floor;      // < 0: off
  double drop_factor;    // 10^-orders, < 0: off
  int max_retries;
};
constexpr int MARCH_HIST = 6;

CSB_DEV void march_reset_flags(unsigned long long* fl) {
  fl[0] = 0ull;
  for (int b = 0; b < EB_COUNT; ++b) fl[1 + b] = ~0ull;
  fl[FLAG_GATE_COUNT] = 0ull;
}

CSB_DEV void march_record(const MarchCfg& k, int it, const double* n, double cfl, int retries,
                          int stop) {
  if (it - 1 >= k.rows) return;
  double* h = k.hist + (long long)(it - 1) * MARCH_HIST;
  h[0] = n[0];
  h[1] = n[1];
  h[2] = n[2];
  h[3] = cfl;
  h[4] = retries;
  h[5] = stop;
}

// condition of a loop / branch: the march goes on
__global__ void k_march_cond(MarchCfg k, cudaGraphConditionalHandle h) {
  const MarchState& s = *k.st;
  cudaGraphSetConditional(h, (s.stop == MS_RUN && s.it < s.it_last) ? 1u : 0u);
}

__global__ void k_cond_set(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }

// after the residual and its norms: stop tests in the reference's order,
// then the CFL of the step (sets the IF(step) condition)
__global__ void k_march_pre(MarchCfg k, cudaGraphConditionalHandle step) {
  MarchState& s = *k.st;
  const int it = s.it + 1;
  const double n[3] = {k.norms[0], k.norms[1], k.norms[2]};
  // a residual that fails (non-physical state, face temperature, non-finite
  // R) raises out of the reference's loop (spatial.py:207-274)
  const unsigned long long rf = k.flags[0] & ((1ull << EB_DECODE) | (1ull << EB_FACE_T) |
                                              (1ull << EB_RES_NONFINITE));
  if (rf || !isfinite(n[0]) || !isfinite(n[1])) {  // driver.py:281-283 (raised, not recorded)
    s.stop = rf ? MS_RESIDUAL : MS_NAN;
    cudaGraphSetConditional(step, 0u);
    return;
  }
  const double cfl_now = k.cfl_tab[min(it - 1, k.rows - 1)] * s.cfl_scale;
  int stop = MS_RUN;
  if (k.abs_floor >= 0.0 && n[2] <= k.abs_floor) stop = MS_ABS;
  else if (s.it >= 1 && k.drop_factor >= 0.0 && n[2] <= s.res0 * k.drop_factor) stop = MS_DROP;
  else if (s.plateau_at == it) stop = MS_PLATEAU;
  if (stop != MS_RUN) {
    march_record(k, it, n, cfl_now, 0, stop);
    if (it == 1) s.res0 = n[2];
    s.it = it;
    s.stop = stop;
    cudaGraphSetConditional(step, 0u);
    return;
  }
  s.norms[0] = n[0];
  s.norms[1] = n[1];
  s.norms[2] = n[2];
  s.cfl_now = cfl_now;
  s.cfl_try = cfl_now;
  s.attempt = 0;
  *k.cfl_dev = cfl_now;
  march_reset_flags(k.flags);
  cudaGraphSetConditional(step, 1u);
}

// after an implicit-step attempt: accept, retry at half the CFL, or stop
__global__ void k_march_after(MarchCfg k, cudaGraphConditionalHandle retry) {
  MarchState& s = *k.st;
  const unsigned long long f = k.flags[0] & ~((1ull << EB_KSKIP) | (1ull << EB_NONPLANAR));
  bool nonphys;
  if (f & (1ull << EB_DECODE)) {
    nonphys = true;
  } else if (f & (1ull << EB_ZERO_WAVE)) {
    s.stop = MS_ZERO;
    cudaGraphSetConditional(retry, 0u);
    return;
  } else if (f & ((1ull << EB_SINGULAR) | (1ull << EB_BLOCK))) {
    s.stop = MS_SINGULAR;
    cudaGraphSetConditional(retry, 0u);
    return;
  } else {
    nonphys = (f & ((1ull << EB_GATE) | (1ull << EB_GATE_DECODE))) != 0ull;
  }
  if (!nonphys) {
    cudaGraphSetConditional(retry, 0u);
    return;
  }
  if (s.attempt >= k.max_retries) {
    s.stop = MS_RETRIES;
    cudaGraphSetConditional(retry, 0u);
    return;
  }
  s.cfl_try = s.cfl_try * 0.5;
  s.attempt += 1;
  *k.cfl_dev = s.cfl_try;
  march_reset_flags(k.flags);
  cudaGraphSetConditional(retry, 1u);
}

// accepted step: record it, update cfl_scale, flip the state buffers
__global__ void k_march_post(MarchCfg k) {
  MarchState& s = *k.st;
  if (s.stop != MS_RUN) return;
  const int it = s.it + 1;
  march_record(k, it, s.norms, s.cfl_try, s.attempt, MS_RUN);
  if (s.cfl_try < s.cfl_now) s.cfl_scale = s.cfl_scale * (s.cfl_try / s.cfl_now);
  else s.cfl_scale = fmin(1.0, s.cfl_scale * 1.2);
  if (it == 1) s.res0 = s.norms[2];
  s.it = it;
  s.parity ^= 1;
  march_reset_flags(k.flags);
}

__global__ void k_march_chunk(MarchState* st, int it_last, int plateau_at, int clear_parity) {
  st->it_last = it_last;
  st->plateau_at = plateau_at;
  if (clear_parity) st->parity = 0;
}

__global__ void k_march_init(MarchState* st) {
  MarchState s{};
  s.cfl_scale = 1.0;
  s.res0 = NAN;
  *st = s;
}

}  // namespace csb
