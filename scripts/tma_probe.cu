// Microbenchmark: per-SM throughput/latency of cp.async.bulk global->shared
// through an mbarrier ring (producer warp + consumer warp), the data path of
// the wavefront sweep.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool SPIN>
__device__ __forceinline__ void wait_bar(unsigned long long* b, unsigned par) {
  if (SPIN)
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(sa(b)), "r"(par) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(sa(b)), "r"(par) : "memory");
}

template <bool SPIN, int MODE>
__global__ void probe(const double* src, long long nslots, int slot_bytes, int D, int copies,
                      long long* out_cycles, double* sink) {
  extern __shared__ __align__(128) double ring[];
  __shared__ unsigned long long full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < D; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[b])), "r"(MODE == 3 ? 32 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[b])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int slot_dbl = slot_bytes / 8;
  const int piece = slot_bytes / copies;
  long long t0 = clock64();
  if (warp == 0) {
    for (long long ks = 0; ks < nslots; ++ks) {
      const int buf = ks % D;
      if (ks >= D) {
        wait_bar<SPIN>(&empty[buf], (unsigned)(((ks / D) - 1) & 1));
      }
      if (MODE == 3) {
        const char* s2 = (const char*)src + (ks * (long long)slot_bytes);
        char* d2 = (char*)(ring + (long long)buf * slot_dbl);
        const int n2 = slot_bytes / 16;
        for (int e = lane; e < n2; e += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(d2 + 16 * e)), "l"(s2 + 16 * (long long)e) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[buf])) : "memory");
      } else if (MODE == 2) {
        const double2* s2 = (const double2*)((const char*)src + (ks * (long long)slot_bytes));
        double2* d2 = (double2*)(ring + (long long)buf * slot_dbl);
        const int n2 = slot_bytes / 16;
#pragma unroll 8
        for (int e = lane; e < n2; e += 32) d2[e] = __ldcg(s2 + e);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&full[buf])) : "memory");
      } else if (lane == (MODE == 1 ? (int)(ks % 32) : 0)) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[buf])), "r"(slot_bytes) : "memory");
        const char* s = (const char*)src + (ks * (long long)slot_bytes);
        char* d = (char*)(ring + (long long)buf * slot_dbl);
        for (int c = 0; c < copies; ++c)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d + c * piece)), "l"(s + c * piece), "r"(piece), "r"(sa(&full[buf])) : "memory");
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    double acc = 0.0;
    for (long long ks = 0; ks < nslots; ++ks) {
      const int buf = ks % D;
      wait_bar<SPIN>(&full[buf], (unsigned)((ks / D) & 1));
      acc += ring[(long long)buf * slot_dbl + lane];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[buf])) : "memory");
    }
    if (lane == 0) {
      sink[blockIdx.x] = acc;
      out_cycles[blockIdx.x] = clock64() - t0;
    }
  }
}

int main() {
  const long long total = 1ll << 30;  // 1 GiB source
  double* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 0, total);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * sizeof(double));
  int sizes[] = {16384, 33792, 65536};
  int Ds[] = {2, 4, 6};
  for (int mode : {0, 3})
  for (int spin : {0})
  for (int ctas : {1, 296}) {
    for (int sz : sizes) {
      for (int D : Ds) {
        for (int copies : {1, 2}) {
          if ((size_t)sz * D > (ctas > 148 ? 100 : 200) * 1024) continue;
          const long long nslots = (total / ctas) / sz > 2000 ? 2000 : (total / ctas) / sz;
          auto kfn = mode == 0 ? probe<false, 0> : probe<false, 3>;
          cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, sz * D);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          cudaEventRecord(a);
          kfn<<<ctas, 64, sz * D>>>(src, nslots, sz, D, copies, cyc, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          long long hc;
          cudaMemcpy(&hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
          printf("mode %d spin %d ctas %3d slot %6d B D %d copies %d: %8.1f cycles/slot, %7.1f GB/s per CTA, %8.1f GB/s total\n",
                 mode, spin, ctas, sz, D, copies, (double)hc / nslots, (double)sz * nslots / (ms * 1e-3) / 1e9,
                 (double)sz * nslots * ctas / (ms * 1e-3) / 1e9);
        }
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
