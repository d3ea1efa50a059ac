// z-marching shared-memory update kernel (placeholder until the tiled kernel lands).
#include "kernels.h"

namespace b2 {
template <typename T>
bool zmarch_supported(const Geom&, const Region&) { return false; }
template <typename T>
void launch_zmarch(cudaStream_t, const Fields<T>&, const Fields<T>&, const Geom&, const Region&, const Coef<T>&, int, T*) {}
template bool zmarch_supported<float>(const Geom&, const Region&);
template bool zmarch_supported<double>(const Geom&, const Region&);
template void launch_zmarch<float>(cudaStream_t, const Fields<float>&, const Fields<float>&, const Geom&, const Region&, const Coef<float>&, int, float*);
template void launch_zmarch<double>(cudaStream_t, const Fields<double>&, const Fields<double>&, const Geom&, const Region&, const Coef<double>&, int, double*);
}  // namespace b2
