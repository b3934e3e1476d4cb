// csflow-b200: sweep dispatch (reference lusgs.py:250-274).
//
// The generic path (3-D grids, and the coupled operator with chemistry)
// sweeps the i+j+k = h hyperplanes in order, one small kernel per plane and
// direction: 2 (ni + nj + nk - 2) launches per solve (4,094 at 1024^2).  Issued
// one by one from the host they are launch-bound, so the whole sequence is
// captured once into a CUDA graph per (operator, buffers) configuration and
// replayed as a single graph launch; the kernels and their order are
// unchanged.  Calls made while the caller's stream is itself being captured
// (an enclosing graph) issue the kernels directly into that capture.
#include <cstring>
#include <mutex>
#include <vector>

#include "csb_common.cuh"
#include "csb_kernels.cuh"

namespace csb {

namespace {

struct SweepKey {
  const Model* mdl;
  int ns;
  GridDev g;
  OpDev op;
  const double* rhs;
  double* dq;
  double* dq_star;
  int device;
};

struct SweepGraph {
  SweepKey key;
  cudaGraphExec_t exec;
  unsigned long long used;
};

std::mutex g_mu;
std::vector<SweepGraph> g_cache;  // small LRU of instantiated sweep graphs
unsigned long long g_tick = 0;
constexpr size_t kMaxGraphs = 8;

bool same(const SweepKey& a, const SweepKey& b) { return std::memcmp(&a, &b, sizeof(SweepKey)) == 0; }

cudaError_t capture(const SweepKey& k, cudaGraphExec_t* out) {
  cudaStream_t cs;
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  cudaGraph_t graph = nullptr;
  e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    cudaError_t el = launch_sweeps_generic(k.mdl, k.ns, k.g, k.op, k.rhs, k.dq, k.dq_star, cs);
    e = cudaStreamEndCapture(cs, &graph);
    if (e == cudaSuccess) e = el;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(out, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  return e;
}

}  // namespace

cudaError_t launch_sweeps(const Model* mdl, int ns, const GridDev& g, const OpDev& op,
                          const double* rhs, double* dq, double* dq_star, unsigned long long* flags,
                          cudaStream_t st) {
  (void)flags;
  const long long nplanes = (long long)(g.ni - 1) + (g.nj - 1) + (g.nk - 1) + 1;
  note_launches(2ull * (unsigned long long)std::max(0LL, nplanes));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
    return launch_sweeps_generic(mdl, ns, g, op, rhs, dq, dq_star, st);
  SweepKey k;
  std::memset(&k, 0, sizeof(k));  // padding bytes take part in the key comparison
  k.mdl = mdl;
  k.ns = ns;
  k.g = g;
  k.op = op;
  k.rhs = rhs;
  k.dq = dq;
  k.dq_star = dq_star;
  cudaGetDevice(&k.device);
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& c : g_cache)
    if (same(c.key, k)) {
      c.used = ++g_tick;
      return cudaGraphLaunch(c.exec, st);
    }
  cudaGraphExec_t exec;
  cudaError_t e = capture(k, &exec);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return launch_sweeps_generic(mdl, ns, g, op, rhs, dq, dq_star, st);  // same kernels, unbatched
  }
  if (g_cache.size() >= kMaxGraphs) {
    size_t old = 0;
    for (size_t i = 1; i < g_cache.size(); ++i)
      if (g_cache[i].used < g_cache[old].used) old = i;
    cudaGraphExecDestroy(g_cache[old].exec);
    g_cache.erase(g_cache.begin() + old);
  }
  g_cache.push_back(SweepGraph{k, exec, ++g_tick});
  return cudaGraphLaunch(exec, st);
}

}  // namespace csb
