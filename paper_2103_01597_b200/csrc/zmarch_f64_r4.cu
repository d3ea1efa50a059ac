// Instantiation of the z-marching kernel for double, stencil radius 4 (order 8).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(double, 4)
}  // namespace b2
