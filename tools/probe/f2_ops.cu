// Probe: do the FP32x2 operations (FADD2 / FMUL2 / FFMA2 via __fadd2_rn, __fmul2_rn, __ffma2_rn)
// round exactly like their scalar counterparts?  Compares lane results against scalar ops on
// random inputs spanning many binades (including subnormal results).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k(const float* a, const float* b, const float* c, unsigned* bad, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i + 1 >= n) return;
  float2 A = make_float2(a[i], a[i + 1]), B = make_float2(b[i], b[i + 1]), C = make_float2(c[i], c[i + 1]);
  float2 s = __fadd2_rn(A, B), m = __fmul2_rn(A, B), f = __ffma2_rn(A, B, C);
  float2 d = __fadd2_rn(A, make_float2(-B.x, -B.y));
  float ss[2] = {__fadd_rn(A.x, B.x), __fadd_rn(A.y, B.y)};
  float mm[2] = {__fmul_rn(A.x, B.x), __fmul_rn(A.y, B.y)};
  float ff[2] = {__fmaf_rn(A.x, B.x, C.x), __fmaf_rn(A.y, B.y, C.y)};
  float dd[2] = {__fsub_rn(A.x, B.x), __fsub_rn(A.y, B.y)};
  float sv[2] = {s.x, s.y}, mv[2] = {m.x, m.y}, fv[2] = {f.x, f.y}, dv[2] = {d.x, d.y};
  for (int l = 0; l < 2; ++l) {
    if (__float_as_uint(sv[l]) != __float_as_uint(ss[l])) atomicAdd(&bad[0], 1);
    if (__float_as_uint(mv[l]) != __float_as_uint(mm[l])) atomicAdd(&bad[1], 1);
    if (__float_as_uint(fv[l]) != __float_as_uint(ff[l])) atomicAdd(&bad[2], 1);
    if (__float_as_uint(dv[l]) != __float_as_uint(dd[l])) atomicAdd(&bad[3], 1);
  }
}

int main() {
  const int n = 1 << 22;
  float *ha = (float*)malloc(n * 4), *hb = (float*)malloc(n * 4), *hc = (float*)malloc(n * 4);
  srand(1);
  for (int i = 0; i < n; ++i) {
    auto r = [] { return ((float)rand() / RAND_MAX - 0.5f) * ldexpf(1.0f, rand() % 60 - 30); };
    ha[i] = r(); hb[i] = r(); hc[i] = r();
  }
  float *a, *b, *c; unsigned* bad;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&bad, 16);
  cudaMemcpy(a, ha, n * 4, cudaMemcpyHostToDevice); cudaMemcpy(b, hb, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(c, hc, n * 4, cudaMemcpyHostToDevice); cudaMemset(bad, 0, 16);
  k<<<n / 512, 256>>>(a, b, c, bad, n);
  unsigned h[4];
  cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
  printf("mismatches of %d lanes: add %u mul %u fma %u sub %u (%s)\n", n, h[0], h[1], h[2], h[3],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
