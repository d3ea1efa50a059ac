// Instantiation of the z-marching kernel for double, stencil radius 2 (order 4).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(double, 2)
}  // namespace b2
