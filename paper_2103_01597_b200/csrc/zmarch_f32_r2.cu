// Instantiation of the z-marching kernel for float, stencil radius 2 (order 4).
#include "zmarch.cuh"

namespace b2 {
B2_ZMARCH_INSTANTIATE(float, 2)
}  // namespace b2
