// mpm_ops.cuh -- MLS-MPM transfer ops (P2G / GRID_OP / G2P), see DESIGN.md "MPM ops".
// Filled in by the MPM milestone; until then the ops are rejected by the host.
#pragma once
#include "sg_internal.h"

namespace sg {
__device__ __forceinline__ void mpm_grid_op(const DOp&, const int*, uint32_t*, uint64_t) {}
__device__ __forceinline__ void mpm_p2g(const DevCtx&, const DOp&, int64_t, int) {}
__device__ __forceinline__ void mpm_g2p(const DevCtx&, const DOp&, int64_t) {}
}  // namespace sg
