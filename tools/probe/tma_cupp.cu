// TMA through the official libcu++ wrappers (CUDA programming guide pattern), sm_100a.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda/barrier>
#include <cstdio>
#include <cstdlib>
namespace cde = cuda::device::experimental;
using barrier = cuda::barrier<cuda::thread_scope_block>;

template <int RANK>
__global__ void k3(const __grid_constant__ CUtensorMap tm, double* out, int c0, int c1, int c2, int n) {
  __shared__ alignas(128) double smem[38 * 14];
#pragma nv_diag_suppress static_var_with_dynamic_init
  __shared__ barrier bar;
  if (threadIdx.x == 0) {
    init(&bar, blockDim.x);
    cde::fence_proxy_async_shared_cta();
  }
  __syncthreads();
  barrier::arrival_token token;
  if (threadIdx.x == 0) {
    cde::cp_async_bulk_tensor_3d_global_to_shared(smem, &tm, c0, c1, c2, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, n);
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < 38 * 14; i += blockDim.x) out[i] = smem[i];
}

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int c0, int c1) {
  __shared__ alignas(128) float smem[32 * 8];
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
    else cde::cp_async_bulk_tensor_1d_global_to_shared(smem, &tm, c0, bar);
    token = cuda::device::barrier_arrive_tx(bar, 1, sizeof(smem));
  } else {
    token = bar.arrive();
  }
  bar.wait(std::move(token));
  for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) out[i] = smem[i];
}

int main(int argc, char** argv) {
  const int rank = argc > 1 ? atoi(argv[1]) : 2;
  if (rank == 3) {
    const int SX = 64, SY = 38, SZ = 38;
    const int bx = argc > 2 ? atoi(argv[2]) : 38, by = argc > 3 ? atoi(argv[3]) : 14;
    double* g3; cudaMalloc(&g3, (size_t)SX * SY * SZ * 8);
    double* h3 = new double[SX * SY * SZ];
    for (int i = 0; i < SX * SY * SZ; ++i) h3[i] = i;
    cudaMemcpy(g3, h3, (size_t)SX * SY * SZ * 8, cudaMemcpyHostToDevice);
    double* o3; cudaMalloc(&o3, 38 * 14 * 8);
    CUtensorMap t3;
    cuuint64_t d3[3] = {SX, SY, SZ}, s3[2] = {SX * 8, (cuuint64_t)SX * SY * 8};
    cuuint32_t b3[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, e3[3] = {1, 1, 1};
    CUresult r3 = cuTensorMapEncodeTiled(&t3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g3, d3, s3, b3, e3,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k3<3><<<1, 128>>>(t3, o3, 13, 0, 5, bx * by * 8);
    cudaError_t e = cudaDeviceSynchronize();
    printf("libcu++ TMA 3d f64 box %dx%d: encode %d, %s\n", bx, by, (int)r3, cudaGetErrorString(e));
    return e != cudaSuccess;
  }
  const int W = 64, H = 32;
  float* g; cudaMalloc(&g, W * H * 4);
  float h[W * H];
  for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 32 * 8 * 4);
  CUtensorMap tm;
  cuuint64_t dims2[2] = {W, H}, str[1] = {W * 4};
  cuuint32_t box2[2] = {32, 8}, es[2] = {1, 1};
  cuuint64_t dims1[1] = {W * H};
  cuuint32_t box1[1] = {256};
  CUresult r = rank == 2 ? cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims2, str, box2, es,
                                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                         : cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, g, dims1, nullptr, box1, es,
                                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rank == 2) k<2><<<1, 128>>>(tm, out, 8, 4);
  else k<1><<<1, 128>>>(tm, out, 64, 0);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[256];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 32; ++x) {
      float want = rank == 2 ? (float)((y + 4) * W + x + 8) : (float)(64 + y * 32 + x);
      if (ho[y * 32 + x] != want) ++bad;
    }
  printf("libcu++ TMA rank %d: encode %d, %s, mismatches %d\n", rank, (int)r, cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
