// Instantiation of the warp-specialised z-marching kernel for double, stencil radius 3 (order 6).
#include "zsplit.cuh"

namespace b2 {
B2_ZSPLIT_INSTANTIATE(double, 3)
}  // namespace b2
