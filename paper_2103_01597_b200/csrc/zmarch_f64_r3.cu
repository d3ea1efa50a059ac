// Instantiation of the z-marching kernel for double, stencil radius 3 (order 6).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(double, 3)
}  // namespace b2
