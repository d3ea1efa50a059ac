// Instantiation of the z-marching kernel for float, stencil radius 1 (order 2).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(float, 1)
}  // namespace b2
