// Instantiation of the z-marching kernel for float, stencil radius 3 (order 6).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(float, 3)
}  // namespace b2
