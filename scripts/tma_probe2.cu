// Does per-CTA cp.async.bulk throughput scale with the number of independent
// producer warps (each with its own mbarrier ring)?  P producer/consumer warp
// pairs per CTA, slot S bytes, ring depth D per pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_probe2.cu -o tma_probe2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(unsigned long long* b, unsigned par) {
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(sa(b)), "r"(par) : "memory");
}

__global__ void probe(const char* src, long long nslots, int S, int D, int P, long long* cyc, double* sink) {
  extern __shared__ __align__(128) char ring[];
  __shared__ unsigned long long full[4][4], empty[4][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, role = warp & 1;  // role 0 producer, 1 consumer
  if (threadIdx.x == 0) {
    for (int p = 0; p < P; ++p)
      for (int b = 0; b < D; ++b) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[p][b])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[p][b])), "r"(1));
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  char* myring = ring + (long long)pair * D * S;
  const char* mysrc = src + ((long long)blockIdx.x * P + pair) * nslots * S;
  long long t0 = clock64();
  if (role == 0) {
    // lanes take turns issuing (lane ks % LN) -- LN = 1 when issuing from one thread
    const int LN = (P == 1 && D == 4 && S == 16384) ? 4 : 1;
    if (lane < LN)
      for (long long ks = lane; ks < nslots; ks += LN) {
        const int buf = ks % D;
        if (ks >= D) wait_bar(&empty[pair][buf], (unsigned)(((ks / D) - 1) & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[pair][buf])), "r"(S) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(myring + buf * S)), "l"(mysrc + ks * S), "r"(S), "r"(sa(&full[pair][buf])) : "memory");
      }
  } else {
    double acc = 0.0;
    for (long long ks = 0; ks < nslots; ++ks) {
      const int buf = ks % D;
      wait_bar(&full[pair][buf], (unsigned)((ks / D) & 1));
      acc += reinterpret_cast<const double*>(myring + buf * S)[lane];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[pair][buf])) : "memory");
    }
    if (lane == 0) {
      sink[blockIdx.x * 4 + pair] = acc;
      if (pair == 0) cyc[blockIdx.x] = clock64() - t0;
    }
  }
}

int main() {
  const long long total = 1ll << 30;
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 0, total);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, 4096 * 8);
  cudaMalloc(&sink, 4096 * 8 * 4);
  for (int P : {1, 2, 4})
  for (int D : {2, 4}) {
    for (int S : {16384, 32768, 49152}) {
      const size_t smem = (size_t)P * D * S;
      if (smem > 220 * 1024) continue;
      const long long nslots = 1000;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        probe<<<1, 64 * P, smem>>>(src, nslots, S, D, P, cyc, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep)
          printf("P %d slot %6d D %d: %8.1f ns/slot per pair, CTA total %7.1f GB/s\n", P, S, D,
                 ms * 1e6 / nslots, (double)P * S * nslots / (ms * 1e-3) / 1e9);
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
