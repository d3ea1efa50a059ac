// Peer-memory halo delivery over NVLink / NVSwitch.
//
// With the peer-memory exchange, the kernels that update the outer shell of a subdomain
// store each boundary result both locally and straight into the halo of every
// neighbour that needs it, through CUDA-IPC mapped peer pointers: the halo exchange of the next
// substep (pack -> send/recv -> unpack) is fused into this substep's boundary update.
//
// A cell (x, y, z) of the local interior belongs to the send region of segment o when,
// per axis a:  o_a = +1 and x_a in [0, r);  o_a = -1 and x_a in [n_a - r, n_a);  or o_a = 0.
// It lands in the receiver's halo at x_a + o_a n_a (s' = ((s - r) mod n') + r).
// RAD is the stencil radius r.
#pragma once
#include "mhd_math.cuh"

namespace b2 {

constexpr int kMaxPeers = 7;  // distinct neighbours of a (2,2,2) Morton block

template <typename T>
struct RemoteMap {
  T* f[kMaxPeers][NF];       // origins of the destination state's fields in each peer's workspace
  signed char peer_of[27];   // (ox+1) + 3 (oy+1) + 9 (oz+1)  ->  slot, -1: not stored by the update
  int sys;                   // 1: some slot is another GPU (a system-scope fence ends the kernel);
                             // 0: only this rank's own periodic halo (wrap stores)
};

// Store the 8 new values of cell (x, y, z) into every neighbour halo that holds a copy of it.
template <typename T, int RAD>
__device__ __forceinline__ void remote_store(const RemoteMap<T>& rm, int nx, int ny, int nz, long long sy,
                                             long long sz, int x, int y, int z, const T (&v)[NF]) {
  const int sx = x < RAD ? 1 : (x >= nx - RAD ? -1 : 0);
  const int syy = y < RAD ? 1 : (y >= ny - RAD ? -1 : 0);
  const int szz = z < RAD ? 1 : (z >= nz - RAD ? -1 : 0);
  if ((sx | syy | szz) == 0) return;
#pragma unroll
  for (int m = 1; m < 8; ++m) {
    const int ox = (m & 1) ? sx : 0, oy = (m & 2) ? syy : 0, oz = (m & 4) ? szz : 0;
    if (((m & 1) && !sx) || ((m & 2) && !syy) || ((m & 4) && !szz)) continue;
    const int p = rm.peer_of[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)];
    if (p < 0) continue;
    const long long d = (long long)(z + oz * nz) * sz + (long long)(y + oy * ny) * sy + (x + ox * nx);
#pragma unroll
    for (int q = 0; q < NF; ++q) rm.f[p][q][d] = v[q];
  }
}

}  // namespace b2
