// Internal (non-ABI) declarations shared by the runtime (mesh.cpp) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mhd_math.cuh"

namespace b2 {

// Origin pointers of the 8 fields of one state: &f[q](x=0, y=0, z=0) of the interior.
template <typename T>
struct Fields {
  T* f[NF];
};

// Local pitched geometry shared by both states: element (x, y, z), x,y,z in [-3, n+3),
// lives at origin + z*sz + y*sy + x.
struct Geom {
  int nx, ny, nz;
  long long sy, sz;
};

// One copy region of the halo machinery: cells of extent ext starting at src
// (interior coordinates) go to dst, or to / from a staging buffer at buf_off values.
struct SegDesc {
  int src[3], dst[3], ext[3];
  long long count;        // ext[0]*ext[1]*ext[2]
  long long buf_off;      // value offset of field 0 of this segment in the staging buffer
  int block0;             // first block of this segment in the launch
};
constexpr int kMaxSeg = 26;
struct SegList {
  int n;
  int nblocks;
  SegDesc s[kMaxSeg];
};
enum SegKind { SEG_SELF = 0, SEG_PACK = 1, SEG_UNPACK = 2 };

struct Region {
  int lo[3];
  int ext[3];
};

// ---- launchers (kernels.cu) ----
template <typename T>
void launch_direct(cudaStream_t st, const Fields<T>& in, const Fields<T>& out, const Geom& g,
                   const Region& r, const Coef<T>& C, int k, T* rhs_out);
template <typename T>
void launch_segments(cudaStream_t st, const Fields<T>& fl, const Geom& g, const SegList& L, int kind, T* buf);
template <typename TS, typename TD>
void launch_copy_in(cudaStream_t st, const TS* src, TD* origin, const Geom& g);
template <typename TS, typename TD>
void launch_copy_out(cudaStream_t st, const TS* origin, TD* dst, const Geom& g);
template <typename T>
void launch_reduce(cudaStream_t st, const T* origin, const Geom& g, double* scratch, int nblocks);

// ---- z-marching shared-memory kernel (zmarch.cu) ----
template <typename T>
bool zmarch_supported(const Geom& g, const Region& r);
template <typename T>
void launch_zmarch(cudaStream_t st, const Fields<T>& in, const Fields<T>& out, const Geom& g,
                   const Region& r, const Coef<T>& C, int k, T* rhs_out);

constexpr int kReduceBlocks = 592;  // 4 x 148 SMs
constexpr int kReduceVals = 5;      // min, max, sum, sum of squares, sum of exp

}  // namespace b2
