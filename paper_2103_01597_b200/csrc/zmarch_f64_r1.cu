// Instantiation of the z-marching kernel for double, stencil radius 1 (order 2).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(double, 1)
}  // namespace b2
