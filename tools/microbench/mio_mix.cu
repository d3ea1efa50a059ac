// Microbenchmark: which on-chip datapaths the z-march kernel's instruction classes share on B200.
// Per SM and SM clock cycle (in-kernel clock64, so independent of the clock the GPU runs at):
//   DFMA lanes, LDS.64 bytes, SHFL.32 warp-instructions, STS.64 bytes, and mixes of them.
// If SHFL and LDS add up (a mix runs in max(t_a, t_b)), shuffles are extra bandwidth for stencil
// taps; if they serialise (sum), a shuffle costs the same as the shared-memory wavefront it
// replaces.  Prints one line per test plus the SM clock seen by the events.
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 4096;

__device__ __forceinline__ void report(long long t0, unsigned long long* cyc) {
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cyc, (unsigned long long)(clock64() - t0));
}

template <int MODE>
__global__ void __launch_bounds__(512) mix_kernel(double* out, unsigned long long* cyc, double a, double b) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 1e-3;
  __syncthreads();
  const long long t0 = clock64();
  double x[8];
  int v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = threadIdx.x * 1e-3 + j;
    v[j] = threadIdx.x + j;
  }
  int idx = threadIdx.x;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0 || MODE == 4 || MODE == 6) x[j] = fma(x[j], a, b);                       // DFMA
      if (MODE == 1 || MODE == 3 || MODE == 4) x[j] += buf[(idx + j * 33) & 4095];           // LDS.64
      if (MODE == 2 || MODE == 3) v[j] = __shfl_xor_sync(0xffffffffu, v[j], (j & 3) + 1);   // SHFL.32
      if (MODE == 5) buf[(idx + j * 33 + 17) & 4095] = x[j];                                 // STS.64
      if (MODE == 6) x[j] = __shfl_xor_sync(0xffffffffu, x[j], (j & 3) + 1);                 // SHFL of a double
    }
    idx = (idx + 7) & 4095;
    if (MODE == 4) {  // 3 DFMA per LDS, the z-march kernel's ratio (634 DP : 238 LDS per cell)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, fma(x[j], a, b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j] + v[j];
  if (s == 1234.5) out[0] = s;
  if (MODE == 5 && buf[threadIdx.x] == 1234.5) out[0] = 1;
  report(t0, cyc);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* d;
  unsigned long long* cyc;
  cudaMalloc(&d, 64);
  cudaMalloc(&cyc, 64);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  const char* names[] = {"DFMA", "LDS.64", "SHFL.32", "LDS.64+SHFL.32 (1:1)", "LDS.64+3 DFMA", "STS.64",
                         "DFMA+SHFL.f64 (1:1)"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512}) {
    const int blocks = p.multiProcessorCount * (1024 / threads);  // 2 x 512 or 4 x 256 threads per SM
    for (int mode = 0; mode < 7; ++mode) {
      auto launch = [&] {
        switch (mode) {
          case 0: mix_kernel<0><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 1: mix_kernel<1><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 2: mix_kernel<2><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 3: mix_kernel<3><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 4: mix_kernel<4><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 5: mix_kernel<5><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
          case 6: mix_kernel<6><<<blocks, threads>>>(d, cyc, 0.999999, 1e-7); break;
        }
      };
      launch();
      cudaMemset(cyc, 0, 8);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // per SM: (1024 threads / 32) warps x ITERS x 8 instructions of each class
      const double warp_instr = 1024.0 / 32 * ITERS * 8;
      const double mhz = (double)c / (ms * 1e3);
      printf("%-24s threads=%d: %8.0f SM cycles, %.3f ms -> SM clock %.0f MHz; per SM per cycle: %.3f warp-instr"
             " of each class (DFMA lanes %.1f, LDS B %.1f)\n",
             names[mode], threads, (double)c, ms, mhz, warp_instr / c, 32 * warp_instr / c * (mode == 4 ? 3 : 1),
             mode == 1 || mode == 3 || mode == 4 ? 256 * warp_instr / c : 0.0);
    }
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
