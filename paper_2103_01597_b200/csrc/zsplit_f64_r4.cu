// Instantiation of the warp-specialised z-marching kernel for double, stencil radius 4 (order 8).
#include "zsplit.cuh"

namespace b2 {
B2_ZSPLIT_INSTANTIATE(double, 4)
}  // namespace b2
