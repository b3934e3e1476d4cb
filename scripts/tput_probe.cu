// Issue throughput of independent FP64 ops from ONE warp (and 4 warps on 4 SMSPs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tput_probe.cu -o tput_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void tput(double* out, long long* cyc, double a, double b, int n) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = a + threadIdx.x + k;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (OP == 0) x[k] = fma(x[k], a, b);
        if (OP == 1) x[k] = x[k] * a;
        if (OP == 2) x[k] = x[k] + b;
        if (OP == 3) x[k] = __shfl_up_sync(0xffffffffu, x[k], 1);
        if (OP == 4) x[k] = (double)fmaf((float)x[k], (float)a, (float)b);
      }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 12);
  const char* names[] = {"DFMA", "DMUL", "DADD", "SHFL64", "F2F+FFMA"};
  for (int warps : {1, 4}) {
    for (int op = 0; op < 4; ++op) {
      for (int rep = 0; rep < 2; ++rep) {
        const int n = 2000;
        switch (op) {
          case 0: tput<0><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, n); break;
          case 1: tput<1><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, n); break;
          case 2: tput<2><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, n); break;
          case 3: tput<3><<<1, 32 * warps>>>(out, cyc, 1.0000001, 1e-9, n); break;
        }
        long long h;
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("warps %d %-8s %.2f cycles per warp-instruction (per warp)\n", warps, names[op], (double)h / (n * 32));
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
