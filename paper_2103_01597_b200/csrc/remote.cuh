// Peer-memory halo delivery over NVLink / NVSwitch.
//
// With the peer-memory exchange, the new boundary cells of a subdomain (the send regions of
// P:705, all inside the outer-shell slabs just updated) are stored straight into the
// halo of every neighbour that needs them, through peer pointers (CUDA IPC across processes, plain
// pointers inside one process): no pack, send/recv or unpack.  A cell of segment o lands
// in the receiver's halo at x_a + o_a n_a per axis (s' = ((s - r) mod n') + r).
#pragma once
#include "mhd_math.cuh"

namespace b2 {

constexpr int kMaxPeers = 7;  // distinct neighbours of a (2,2,2) Morton block

// Origins of the destination state's fields in each neighbour's workspace, by peer slot (the
// order of the mesh's peer list).
template <typename T>
struct RemoteMap {
  T* f[kMaxPeers][NF];
};

}  // namespace b2
