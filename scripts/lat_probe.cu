// Dependent-chain latency of FP64 ops and warp shuffles on one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat_probe.cu -o lat_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, a, b);
      if (OP == 1) x = x * a;
      if (OP == 2) x = x + b;
      if (OP == 3) x = __shfl_up_sync(0xffffffffu, x, 1) + 0.0;
      if (OP == 4) x = __shfl_up_sync(0xffffffffu, x, 1);
      if (OP == 5) x = __int_as_float(__shfl_up_sync(0xffffffffu, __float_as_int((float)x), 1));
      if (OP == 6) x = fmaf((float)x, (float)a, (float)b);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DMUL", "DADD", "SHFL64+DADD", "SHFL64", "SHFL32", "FFMA"};
  for (int op = 0; op < 7; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      const int n = 1000;
      switch (op) {
        case 0: lat<0><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 1: lat<1><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 2: lat<2><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 3: lat<3><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 4: lat<4><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 5: lat<5><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
        case 6: lat<6><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); break;
      }
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%-12s %.2f cycles/op\n", names[op], (double)h / (n * 16));
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
