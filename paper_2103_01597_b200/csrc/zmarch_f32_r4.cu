// Instantiation of the z-marching kernel for float, stencil radius 4 (order 8).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(float, 4)
}  // namespace b2
