// TMA matrix probe (libcu++ wrappers): dtype x rank x box, one case per process.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda/barrier>
#include <cstdio>
#include <cstdlib>
namespace cde = cuda::device::experimental;
using barrier = cuda::barrier<cuda::thread_scope_block>;

template <typename T, int RANK>
__global__ void k(const __grid_constant__ CUtensorMap tm, T* out, int c0, int c1, int c2, int n) {
  __shared__ alignas(128) unsigned char smem[16384];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    if (RANK == 2) cde::cp_async_bulk_tensor_2d_global_to_shared(smem, &tm, c0, c1, bar);
    if (RANK == 3) cde::cp_async_bulk_tensor_3d_global_to_shared(smem, &tm, c0, c1, c2, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, n);
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < n / (int)sizeof(T); i += blockDim.x) out[i] = ((T*)smem)[i];
}

template <typename T>
int run(int rank, int bx, int by, int SX, int SY, int SZ, int c0, int c1, int c2) {
  T* g; cudaMalloc(&g, (size_t)SX * SY * SZ * sizeof(T));
  T* h = new T[(size_t)SX * SY * SZ];
  for (size_t i = 0; i < (size_t)SX * SY * SZ; ++i) h[i] = (T)i;
  cudaMemcpy(g, h, (size_t)SX * SY * SZ * sizeof(T), cudaMemcpyHostToDevice);
  T* o; cudaMalloc(&o, 16384);
  CUtensorMap tm;
  const CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t d[3] = {(cuuint64_t)SX, (cuuint64_t)SY, (cuuint64_t)SZ};
  cuuint64_t s[2] = {(cuuint64_t)SX * sizeof(T), (cuuint64_t)SX * SY * sizeof(T)};
  cuuint32_t b[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, e[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, dt, rank, g, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int n = bx * by * (int)sizeof(T);
  if (rank == 2) k<T, 2><<<1, 128>>>(tm, o, c0, c1, 0, n);
  else k<T, 3><<<1, 128>>>(tm, o, c0, c1, c2, n);
  cudaError_t err = cudaDeviceSynchronize();
  int bad = -1;
  if (err == cudaSuccess) {
    T* ho = new T[bx * by];
    cudaMemcpy(ho, o, n, cudaMemcpyDeviceToHost);
    bad = 0;
    for (int y = 0; y < by; ++y)
      for (int x = 0; x < bx; ++x) {
        size_t gi = rank == 2 ? (size_t)(y + c1) * SX + x + c0 : ((size_t)c2 * SY + y + c1) * SX + x + c0;
        T want = (x + c0 < SX) ? (T)gi : (T)0;
        if (ho[y * bx + x] != want) ++bad;
      }
  }
  printf("%s rank %d box %dx%d dims %dx%dx%d at (%d,%d,%d): encode %d, %s, mismatches %d\n",
         sizeof(T) == 8 ? "f64" : "f32", rank, bx, by, SX, SY, SZ, c0, c1, c2, (int)r, cudaGetErrorString(err), bad);
  return err != cudaSuccess;
}

int main(int argc, char** argv) {
  int a[10] = {8, 3, 38, 14, 64, 38, 38, 13, 0, 5};
  for (int i = 1; i < argc && i <= 10; ++i) a[i - 1] = atoi(argv[i]);
  return a[0] == 8 ? run<double>(a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9])
                   : run<float>(a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9]);
}
