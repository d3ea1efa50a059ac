// Microbenchmark: FP64 DFMA issue rate, LDS.64 bandwidth and SM clock under FP64 load on B200.
// Used to derive the "alu" roofline peak in DESIGN.md (the survey flags the FP64 peak as unmeasured).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5) out[0] = s;
}

__global__ void lds_kernel(double* out, int iters) {
  __shared__ double buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = i;
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      acc += buf[(idx + j * 33) & 2047];
    }
    idx = (idx + 7) & 2047;
  }
  if (acc == 1234.5) out[0] = acc;
}

__global__ void clk_kernel(long long* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64(); }

int main() {
  double* d; cudaMalloc(&d, 64);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / threads);
    int iters = 20000;
    dfma_kernel<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ninstr = (double)blocks * threads * iters * 16 * 8;
    printf("DFMA threads=%d: %.3f ms, %.3f T DFMA-lane/s = %.2f TFLOP/s, per SM per clk @1965MHz: %.1f lanes\n", threads, ms,
           ninstr / ms / 1e9, 2 * ninstr / ms / 1e9, ninstr / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  }
  {
    int threads = 512, blocks = p.multiProcessorCount * 4, iters = 20000;
    lds_kernel<<<blocks, threads>>>(d, 100);
    cudaEventRecord(e0);
    lds_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * threads * iters * 16 * 8;
    printf("LDS.64: %.3f ms, %.1f TB/s, per SM per clk @1965MHz: %.1f B\n", ms, bytes / ms / 1e9,
           bytes / (ms * 1e-3) / p.multiProcessorCount / 1.965e9);
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
