// kernels_flow.cu -- N2 done with point-to-point dependencies (SURVEY.md s8(f)
// N2; beyond the paper: PAPER.md:367-368 never fuses a task with a dependent
// stencil).  A chain of JACOBI sweeps over the same list of 8^3 dense blocks
// (the C2 solve: 50 ping-pong sweeps, the last one fused with the reduction
// of its output) runs as ONE persistent launch.  No grid-wide barrier between
// sweeps (measured: a grid barrier costs more than a graph-replayed launch,
// DESIGN.md R41): every half block carries a completion flag, and a warp
// starts sweep p of its half block once the 7 half blocks its stencil reads
// (the other half of its block, the x-face half of the x neighbour, the same
// half of the four y / z neighbours) have completed sweep p - 1.  Sweep 0
// needs nothing; one grid barrier after it settles which neighbours are in
// the list at all (an allocated block outside the list reads 0 and never
// publishes a flag).  That one
// condition covers both hazards of the ping-pong: the values it reads were
// written (RAW), and the neighbours finished reading the buffer it is about
// to overwrite (WAR: they read it in sweep p - 1).  Neighbours therefore run
// at most one sweep apart, and the lowest sweep in flight always has its
// dependencies met, so with every CTA resident (cooperative launch) the chain
// cannot deadlock.
//
// Flags: one u32 per half block, indexed by the block's leaf-pool word offset
// (blocks are 512-word runs, so offset >> 9 is unique) -- no extra table.
// Value (epoch << 8) | sweeps completed, the epoch a per-grid launch counter
// bumped by the last CTA, so flags never need resetting (2^24 launches).
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include "sg_internal.h"
#include "jit.h"

namespace sg {
namespace {   // internal linkage: struct_for.cuh's kernels are also compiled in kernels_sf.cu
#include "device_common.cuh"

#include "mpm_ops.cuh"
#include "struct_for.cuh"
}  // namespace

constexpr int FLOW_MAXPH = 128;   // sweeps per launch (kernel-parameter table)

struct JacFlowArgs {
  JacArgs J;               // geometry, block table, reduction target (RED: last sweep)
  uint32_t* flags;         // per half block: (epoch << 8) | sweeps completed
  uint32_t* ctl;           // [0] epoch, [1] CTA done counter, [2] barrier arrivals
  DevCtx C;                // error word (dependency wait timeout)
  int32_t task;
  int32_t nph;
  uint32_t s_dst[FLOW_MAXPH], s_src[FLOW_MAXPH], s_rhs[FLOW_MAXPH];   // field offsets (words) per sweep
};

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool RED>
__global__ void __launch_bounds__(256, 4) k_jacobi8_flow(const __grid_constant__ JacFlowArgs F) {
  const JacArgs& A = F.J;
  const uint32_t* P = A.T.seg[A.T.nseg - 1].base;
  uint32_t* PW = const_cast<uint32_t*>(P);
  const uint32_t E = (F.ctl[0] & 0xFFFFFFu) << 8;   // written by the previous launch's last CTA
  const uint32_t nent = *A.count;
  const bool rows_ok = A.table_ctl[4] != 0u;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), GW = gridDim.x * (blockDim.x >> 5);
  double acc = 0.0;
  for (int p = 0; p < F.nph; p++) {
    const uint32_t* __restrict__ src = P + F.s_src[p];
    const uint32_t* __restrict__ rhs = P + F.s_rhs[p];
    uint32_t* dst = PW + F.s_dst[p];
    const uint32_t need = E | (uint32_t)p, done = E | (uint32_t)(p + 1);
    for (uint32_t wq = gw; wq < nent * 2u; wq += GW) {
      const uint32_t e = wq >> 1, part = wq & 1u;
      uint32_t blk, nb[6];
      if (rows_ok) {
        const uint32_t rv = lane < 12 ? reinterpret_cast<const uint32_t*>(A.table + e)[lane] : 0u;
        blk = __shfl_sync(0xffffffffu, rv, 0);
#pragma unroll
        for (int d = 0; d < 6; d++) nb[d] = __shfl_sync(0xffffffffu, rv, 6 + d);
      } else {
        BlockRow r;
        jac_row_slow(A.T, A.entries[e], &r);
        if (p == 0 && part == 0 && lane == 0) A.table[e] = r;
        blk = r.blk;
#pragma unroll
        for (int d = 0; d < 6; d++) nb[d] = r.nbr[d];
      }
      if (blk == SG_NO_BLOCK) continue;
      const uint32_t self = ((blk >> 9) << 1) | part;
      if (p > 0) {
        // lane 0 watches the other half of the block, lanes 1..6 the face
        // neighbours (x-: its upper half, x+: its lower half, y/z: this half).
        // A neighbour that is allocated but not in the list (its payload
        // reads 0) never publishes: after sweep 0 and the grid barrier every
        // listed half block has a flag >= E | 1, so anything lower is such a
        // non-member and is not waited for.
        uint32_t dep = 0xFFFFFFFFu;
        if (lane == 0) {
          dep = self ^ 1u;
        } else if (lane <= 6) {
          uint32_t nbd = nb[0];   // nb[lane - 1] without a dynamically indexed (local) array
#pragma unroll
          for (int d = 1; d < 6; d++) nbd = lane == d + 1 ? nb[d] : nbd;
          if (nbd != SG_NO_BLOCK) dep = ((nbd >> 9) << 1) | (lane == 1 ? 1u : lane == 2 ? 0u : part);
        }
        if (dep != 0xFFFFFFFFu) {
          uint32_t spins = 0, v;
          while ((v = ld_acquire(F.flags + dep)) < need && v >= (E | 1u)) {
            if (++spins > (1u << 24)) {   // seconds: a broken dependency, not a slow neighbour
              set_err(F.C, SG_ERR_TIMEOUT, F.task);
              break;
            }
            if (spins > 8) __nanosleep(64);
          }
        }
        __syncwarp();
      }
      if (RED && p == F.nph - 1) acc += jac8_half<true>(src, rhs, dst, blk, nb, part, lane, A.inv);
      else jac8_half<false>(src, rhs, dst, blk, nb, part, lane, A.inv);
      __syncwarp();   // the warp's stores, then the flag (release, device scope)
      if (lane == 0) {
        __threadfence();
        st_release(F.flags + self, done);
      }
    }
    if (p == 0 && F.nph > 1) {
      // one grid barrier per launch (all CTAs resident: cooperative launch):
      // after it, list membership of a neighbour is its flag (see above)
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(&F.ctl[2], 1u);
        uint32_t spins = 0;
        while (ld_acquire(&F.ctl[2]) < gridDim.x) {
          if (++spins > (1u << 24)) { set_err(F.C, SG_ERR_TIMEOUT, F.task); break; }
          if (spins > 8) __nanosleep(64);
        }
      }
      __syncthreads();
    }
  }
  if (RED) jac_reduce_tail(A, acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&F.ctl[1], 1u) == gridDim.x - 1) {
      F.ctl[1] = 0u;
      F.ctl[2] = 0u;   // barrier arrivals (every CTA passed it long ago)
      F.ctl[0] = (F.ctl[0] + 1u) & 0xFFFFFFu;
      if (!rows_ok) A.table_ctl[4] = 1u;   // every row was written in sweep 0
      __threadfence();
    }
  }
}

static int flow_grid() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_jacobi8_flow<true>, 256, 0);
    int per2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_jacobi8_flow<false>, 256, 0);
    g = std::max(1, sms) * std::max(1, std::min(std::min(per, per2), 4));
  }
  return g;
}

int jacobi_flow_start(const DTree& t, const DList* drive, const DOp* ops, const int* phase_end, int nph) {
  if (nph < 2 || !drive || !drive->table || t.leaf_bitmasked || t.nd != 3) return -1;
  if (t.nlev - 1 - t.driving != 1) return -1;
  const DLevel& B = t.lev[t.nlev - 1];
  if (B.le[0] != 3 || B.le[1] != 3 || B.le[2] != 3) return -1;   // 8^3 dense blocks
  // walk back from the last phase while phases are flow sweeps
  int first = nph;
  for (int ph = nph - 1; ph >= 0; ph--) {
    const int begin = ph ? phase_end[ph - 1] : 0, n = phase_end[ph] - begin;
    const DOp& j = ops[begin];
    if (j.op != SG_OP_JACOBI || j.dt == SG_I32) break;
    const bool red = n == 2 && ops[begin + 1].op == SG_OP_REDUCE_SUM && ops[begin + 1].f[1] == j.f[0] &&
                     ops[begin + 1].scalar >= 0;
    if (!(n == 1 || (red && ph == nph - 1))) break;
    first = ph;
  }
  if (nph - first < 2) return -1;
  return std::max(first, nph - FLOW_MAXPH);
}

int launch_jacobi_flow(const DevCtx& c, const DTree& t, const DList* drive, const DOp* ops, const int* phase_end,
                       int first, int nph, uint32_t* flags, uint32_t* ctl, int task, void* stream) {
  JacFlowArgs* F = new JacFlowArgs();
  JacArgs& j = F->J;
  j.T = t; j.entries = drive->entries; j.count = drive->count; j.table = drive->table; j.table_ctl = drive->ctl;
  j.inv = 1.0f / 6.0f;
  j.partials = c.partials;
  j.red_done = c.red_done;
  j.red_target = nullptr;
  const uint64_t fs = 1ull << t.ln_leaf;
  int begin = first ? phase_end[first - 1] : 0;
  for (int ph = first; ph < nph; ph++) {
    const DOp& o = ops[begin];
    const int k = ph - first;
    F->s_dst[k] = (uint32_t)(o.slot[0] * fs);
    F->s_src[k] = (uint32_t)(o.slot[1] * fs);
    F->s_rhs[k] = (uint32_t)(o.slot[2] * fs);
    if (phase_end[ph] - begin == 2) j.red_target = c.scalars + ops[begin + 1].scalar;
    begin = phase_end[ph];
  }
  F->flags = flags;
  F->ctl = ctl;
  F->C = c;
  F->task = task;
  F->nph = nph - first;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(flow_grid());
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every CTA resident: the flag waits need it
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = j.red_target ? cudaLaunchKernelEx(&cfg, k_jacobi8_flow<true>, *F)
                               : cudaLaunchKernelEx(&cfg, k_jacobi8_flow<false>, *F);
  delete F;
  return e == cudaSuccess ? 0 : SG_ERR_CUDA;
}

}  // namespace sg
