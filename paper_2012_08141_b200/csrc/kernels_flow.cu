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


// ===========================================================================
// Two sweeps per launch (N2, the variant that wins): temporal blocking of a
// JACOBI chain on 8^3 dense blocks.  A CTA stages one block's x^(k-1) over
// [-2, 10)^3 (its own block, 2-deep faces, the edges; absent or unlisted
// neighbour blocks read 0, R8), computes sweep k on the block and its 1-deep
// face shell (shell cells of listed neighbours only: an unlisted cell is never
// updated), then sweep k+1 on the block -- the SAME float operations in the
// same order as one launch per sweep (jac8_half), so the fields are
// bit-identical.  The race a 2-sweep launch would have with ping-pong buffers
// (x^(k+1) belongs in the buffer other CTAs are still reading x^(k-1) from)
// is avoided with a scratch field T (one 8^3 block per list entry):
//   A-launch (sweeps k, k+1): reads X_(k-1), writes x^(k+1) -> T;
//   B-launch (sweeps k+2, k+3): reads T, writes x^(k+3) -> its field (and,
//   in the chain's last B, x^(k+2) -> its field), so after the last B both
//   ping-pong fields hold exactly what one launch per sweep leaves.
// x^k of an A-launch and x^(k+2) of a non-final B-launch are overwritten
// before anything reads them, so they are not stored.  Neighbour lookups: a
// 27-entry row per list entry (pool offset and list index of every neighbour
// block, NO_BLOCK when absent or unlisted) built by two small kernels per
// chain (an inverse map pool block -> list index tagged with a build epoch,
// then the rows), so list changes between flushes are always picked up.
// ===========================================================================
constexpr int T2_ROW = 54;   // per entry: 27 pool offsets, 27 list indices

struct T2Build {
  DTree T;
  const uint32_t* entries;
  const uint32_t* count;
  const BlockRow* table;
  const uint32_t* table_ctl;
  uint64_t* inv;        // [pool words / 512 + 1]: (tag << 32) | list index
  uint32_t* rows;       // [capacity * T2_ROW]
  uint32_t* ctl;        // [0] build epoch, [1] CTA done counter
};

__device__ __forceinline__ void t2_entry(const T2Build& B, uint32_t e, uint32_t& blk, int org[3]) {
  if (B.table_ctl[4] != 0u) {
    const BlockRow& r = B.table[e];
    blk = r.blk;
    org[0] = r.org[0]; org[1] = r.org[1]; org[2] = r.org[2];
  } else {
    BlockRow r;
    jac_row_slow(B.T, B.entries[e], &r);
    blk = r.blk;
    org[0] = r.org[0]; org[1] = r.org[1]; org[2] = r.org[2];
  }
}

__global__ void __launch_bounds__(256) k_t2_inv(const __grid_constant__ T2Build B) {
  const uint64_t tag = (uint64_t)(B.ctl[0] + 1u) << 32;
  const uint32_t n = *B.count;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    uint32_t blk;
    int org[3];
    t2_entry(B, e, blk, org);
    if (blk != SG_NO_BLOCK) B.inv[blk >> 9] = tag | e;
  }
}

__global__ void __launch_bounds__(256) k_t2_rows(const __grid_constant__ T2Build B) {
  const uint32_t tag = B.ctl[0] + 1u;
  const uint32_t n = *B.count;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), GW = gridDim.x * (blockDim.x >> 5);
  const uint32_t* base = B.T.seg[B.T.nseg - 1].base;
  const DLevel& D = B.T.lev[B.T.driving];
  const uint32_t lowmask = ~((1u << B.T.lblk) - 1u);
  for (uint32_t e = gw; e < n; e += GW) {
    uint32_t blk;
    int org[3];
    t2_entry(B, e, blk, org);
    if (lane < 27) {
      uint32_t off = SG_NO_BLOCK, ent = SG_NO_BLOCK;
      if (blk != SG_NO_BLOCK) {
        const int d[3] = {lane / 9 - 1, (lane / 3) % 3 - 1, lane % 3 - 1};
        int q[3];
#pragma unroll
        for (int a = 0; a < 3; a++) q[a] = org[a] + d[a] * (1 << D.lbelow[a]);
        if (in_domain(B.T, q)) {
          uint32_t idx;
          const uint32_t* c2 = locate(B.T, q, idx);
          if (c2) {
            const uint32_t nb = (uint32_t)(c2 - base) + B.T.payload_off + (idx & lowmask);
            const uint64_t v = B.inv[nb >> 9];
            if ((uint32_t)(v >> 32) == tag) { off = nb; ent = (uint32_t)v; }
          }
        }
      }
      B.rows[(uint64_t)e * T2_ROW + lane] = off;
      B.rows[(uint64_t)e * T2_ROW + 27 + lane] = ent;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&B.ctl[1], 1u) == gridDim.x - 1) {
      B.ctl[1] = 0u;
      B.ctl[0] = tag;   // this build's tag: later builds use a fresh one
      __threadfence();
    }
  }
}

struct T2Args {
  JacArgs J;                 // pool (J.T), count, reduction target / partials
  const uint32_t* rows;
  float* tmp;                // scratch field T: 512 floats per list entry
  uint32_t s_src, s_rhs, s_d1, s_d2;   // pool field offsets (words)
};

// SRC_T: x^(k-1) from T (else the pool field s_src); D1: store sweep k's
// block to s_d1; D2_T: sweep k+1's block to T (else the pool field s_d2).
// Shared layouts, z fastest in rows of ZS = 17 slots (z = zz - 4; the odd
// stride keeps a warp's 32 rows on 32 banks): xs [12 x][12 y][ZS] for x, y in
// [-2, 10); bs, ys [10 x][10 y][ZS] for x, y in [-1, 9).
constexpr int T2_ZS = 17;
template <bool SRC_T, bool D1, bool D2_T, bool RED>
__global__ void __launch_bounds__(256) k_jacobi8_t2(const __grid_constant__ T2Args A) {
  __shared__ float xs[12 * 12 * T2_ZS];
  __shared__ float bs[10 * 10 * T2_ZS];
  __shared__ float ys[10 * 10 * T2_ZS];
  __shared__ uint32_t roff[27], rent[27];
  const uint32_t* P = A.J.T.seg[A.J.T.nseg - 1].base;
  uint32_t* PW = const_cast<uint32_t*>(P);
  const uint32_t n = *A.J.count;
  const float inv = A.J.inv;
  const int tid = threadIdx.x;
  double acc = 0.0;
  for (uint32_t e = blockIdx.x; e < n; e += gridDim.x) {
    if (tid < T2_ROW) {
      const uint32_t v = A.rows[(uint64_t)e * T2_ROW + tid];
      if (tid < 27) roff[tid] = v;
      else rent[tid - 27] = v;
    }
    __syncthreads();
    const uint32_t self = roff[13];
    if (self != SG_NO_BLOCK) {
      // staging: one 16-byte quad per load, every load issued before the
      // first shared store
      uint4 xv[3], bv[2];
#pragma unroll
      for (int it = 0; it < 3; it++) {
        const int q = tid + 256 * it;   // < 576 quads of xs
        xv[it] = make_uint4(0u, 0u, 0u, 0u);
        if (q < 576) {
          const int i = q / 48, r = q - 48 * i, j = r >> 2, zq = r & 3;
          const int x = i - 2, y = j - 2, z0 = zq * 4 - 4;
          const int d = ((x + 8) >> 3) * 9 + ((y + 8) >> 3) * 3 + ((z0 + 8) >> 3);
          const uint32_t loc = (uint32_t)(((x + 8) & 7) * 64 + ((y + 8) & 7) * 8 + ((z0 + 8) & 7));
          if (SRC_T) {
            const uint32_t en = rent[d];
            if (en != SG_NO_BLOCK) xv[it] = *reinterpret_cast<const uint4*>(A.tmp + (uint64_t)en * 512u + loc);
          } else {
            const uint32_t o = roff[d];
            if (o != SG_NO_BLOCK) xv[it] = *reinterpret_cast<const uint4*>(P + A.s_src + o + loc);
          }
        }
      }
#pragma unroll
      for (int it = 0; it < 2; it++) {
        const int q = tid + 256 * it;   // < 400 quads of bs
        bv[it] = make_uint4(0u, 0u, 0u, 0u);
        if (q < 400) {
          const int i = q / 40, r = q - 40 * i, j = r >> 2, zq = r & 3;
          const int x = i - 1, y = j - 1, z0 = zq * 4 - 4;
          const int d = ((x + 8) >> 3) * 9 + ((y + 8) >> 3) * 3 + ((z0 + 8) >> 3);
          const uint32_t loc = (uint32_t)(((x + 8) & 7) * 64 + ((y + 8) & 7) * 8 + ((z0 + 8) & 7));
          const uint32_t o = roff[d];
          if (o != SG_NO_BLOCK) bv[it] = *reinterpret_cast<const uint4*>(P + A.s_rhs + o + loc);
        }
      }
#pragma unroll
      for (int it = 0; it < 3; it++) {
        const int q = tid + 256 * it;
        if (q < 576) {
          float* d = xs + (q >> 2) * T2_ZS + (q & 3) * 4;
          d[0] = __uint_as_float(xv[it].x); d[1] = __uint_as_float(xv[it].y);
          d[2] = __uint_as_float(xv[it].z); d[3] = __uint_as_float(xv[it].w);
        }
      }
#pragma unroll
      for (int it = 0; it < 2; it++) {
        const int q = tid + 256 * it;
        if (q < 400) {
          float* d = bs + (q >> 2) * T2_ZS + (q & 3) * 4;
          d[0] = __uint_as_float(bv[it].x); d[1] = __uint_as_float(bv[it].y);
          d[2] = __uint_as_float(bv[it].z); d[3] = __uint_as_float(bv[it].w);
        }
      }
      __syncthreads();
      // sweep k on the block and its face shell: one thread per (x, y)
      // column of [-1, 9)^2 and z half (z in [-1, 4) or [4, 9)); edge /
      // corner cells are not read by sweep k+1, cells of unlisted neighbours
      // stay 0
      if (tid < 200) {
        const int col = tid >> 1, zh = tid & 1;
        const int i = col / 10, j = col - 10 * i, x = i - 1, y = j - 1;
        const int out = (x < 0 || x > 7) + (y < 0 || y > 7);
        const int dxy = ((x + 8) >> 3) * 9 + ((y + 8) >> 3) * 3;
        const bool mid = out == 0 || (out == 1 && roff[dxy + 1] != SG_NO_BLOCK);
        const bool zlo = out == 0 && roff[dxy] != SG_NO_BLOCK, zhi = out == 0 && roff[dxy + 2] != SG_NO_BLOCK;
        const int xb = ((x + 2) * 12 + (y + 2)) * T2_ZS + 4, yb = col * T2_ZS + 4;   // z = 0 slots
#pragma unroll
        for (int t = 0; t < 5; t++) {
          const int z = zh * 5 - 1 + t;
          const bool need = (z >= 0 && z <= 7) ? mid : (z < 0 ? zlo : zhi);
          float v = 0.0f;
          if (need) {
            const int c = xb + z;
            float sm = xs[c - 1] + xs[c + 1];   // z-1, z+1, then x-1, x+1, y-1, y+1 (jac8_half's order)
            sm += xs[c - 12 * T2_ZS];
            sm += xs[c + 12 * T2_ZS];
            sm += xs[c - T2_ZS];
            sm += xs[c + T2_ZS];
            v = (bs[yb + z] + sm) * inv;
          }
          ys[yb + z] = v;
        }
      }
      __syncthreads();
      // sweep k+1 on the block: one thread per (x, y, z-half)
      if (tid < 128) {
        const int x = tid >> 4, y = (tid >> 1) & 7, zh = tid & 1;
        const int yb = ((x + 1) * 10 + (y + 1)) * T2_ZS + 4 + 4 * zh;
        float o4[4], y4[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const int c = yb + t;
          float sm = ys[c - 1] + ys[c + 1];
          sm += ys[c - 10 * T2_ZS];
          sm += ys[c + 10 * T2_ZS];
          sm += ys[c - T2_ZS];
          sm += ys[c + T2_ZS];
          o4[t] = (bs[c] + sm) * inv;
          y4[t] = ys[c];
        }
        const uint32_t loc = (uint32_t)(x * 64 + y * 8 + 4 * zh);
        if (D1)
          *reinterpret_cast<uint4*>(PW + A.s_d1 + self + loc) =
              make_uint4(__float_as_uint(y4[0]), __float_as_uint(y4[1]), __float_as_uint(y4[2]), __float_as_uint(y4[3]));
        const uint4 ov = make_uint4(__float_as_uint(o4[0]), __float_as_uint(o4[1]), __float_as_uint(o4[2]),
                                    __float_as_uint(o4[3]));
        if (D2_T) *reinterpret_cast<uint4*>(A.tmp + (uint64_t)e * 512u + loc) = ov;
        else *reinterpret_cast<uint4*>(PW + A.s_d2 + self + loc) = ov;
        if (RED) acc += (double)(((o4[0] + o4[1]) + o4[2]) + o4[3]);
      }
    }
    __syncthreads();   // the staging buffers are reused by the next block
  }
  if (RED) jac_reduce_tail(A.J, acc);
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


// Launches of a 2-sweep (temporal) chain tail; see the block comment above.
// Returns the number of launches issued (>= 1), 0 when the chain does not
// have the shape (ping-pong between two fields with one rhs, >= 4 sweeps),
// or a negative sg_status.
bool jacobi_t2_applies(const DOp* ops, const int* phase_end, int first, int nph) {
  if (nph - first < 4) return false;
  auto op_of = [&](int ph) -> const DOp& { return ops[ph ? phase_end[ph - 1] : 0]; };
  const DOp& o0 = op_of(first);
  for (int ph = first; ph < nph; ph++) {
    const DOp& o = op_of(ph);
    if (o.slot[2] != o0.slot[2]) return false;
    if (ph > first && (o.slot[1] != op_of(ph - 1).slot[0] || o.slot[0] != op_of(ph - 1).slot[1])) return false;
  }
  return true;
}

int jacobi_t2_launches(int first, int nph) {
  const int n = nph - first, cycles = n / 4;
  return (n - 4 * cycles) + 2 + 2 * cycles;
}

int launch_jacobi_t2(const DevCtx& c, const DTree& t, const DList* drive, const DOp* ops, const int* phase_end,
                     int first, int nph, const T2Buffers& bf, int task, void* stream) {
  if (!jacobi_t2_applies(ops, phase_end, first, nph)) return 0;
  const int n = nph - first;
  const uint64_t fs = 1ull << t.ln_leaf;
  auto op_of = [&](int ph) -> const DOp& { return ops[ph ? phase_end[ph - 1] : 0]; };
  const DOp& o0 = op_of(first);
  cudaStream_t s = (cudaStream_t)stream;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sms = std::max(sms, 1);
  int launches = 0;
  // the sweeps that do not fill a 4-sweep cycle, one launch each, first
  const int cycles = n / 4, singles = n - 4 * cycles;
  for (int ph = first; ph < first + singles; ph++) {
    const int b = ph ? phase_end[ph - 1] : 0;
    const int rc = launch_struct_for(c, t, 0, drive, ops + b, phase_end[ph] - b, task, stream, sms * 8, nullptr,
                                     nullptr, 1, 0);
    if (rc) return rc;
    launches++;
  }
  // rows of this list version
  T2Build B;
  B.T = t; B.entries = drive->entries; B.count = drive->count; B.table = drive->table; B.table_ctl = drive->ctl;
  B.inv = bf.inv; B.rows = bf.rows; B.ctl = bf.ctl;
  k_t2_inv<<<sms * 4, 256, 0, s>>>(B);
  k_t2_rows<<<sms * 4, 256, 0, s>>>(B);
  launches += 2;
  T2Args A;
  JacArgs& j = A.J;
  j.T = t; j.entries = drive->entries; j.count = drive->count; j.table = drive->table; j.table_ctl = drive->ctl;
  j.inv = 1.0f / 6.0f;
  j.partials = c.partials;
  j.red_done = c.red_done;
  j.red_target = nullptr;
  const int lastb = phase_end[nph - 1] - (nph - 1 ? phase_end[nph - 2] : 0);
  if (lastb == 2) j.red_target = c.scalars + ops[phase_end[nph - 1] - 1].scalar;
  A.rows = bf.rows;
  A.tmp = bf.tmp;
  A.s_rhs = (uint32_t)(o0.slot[2] * fs);
  const int grid = sms * 4;   // one resident wave (57 registers x 256 threads: 4 CTAs / SM)
  for (int cy = 0; cy < cycles; cy++) {
    const int p = first + singles + 4 * cy;   // sweeps p .. p+3
    const bool last = cy == cycles - 1;
    // A: x^(p-1) from its field, x^(p+1) -> T
    A.s_src = (uint32_t)(op_of(p).slot[1] * fs);
    A.s_d1 = 0; A.s_d2 = 0;
    k_jacobi8_t2<false, false, true, false><<<grid, 256, 0, s>>>(A);
    // B: x^(p+1) from T, x^(p+3) -> its field (and x^(p+2) in the last cycle)
    A.s_d1 = (uint32_t)(op_of(p + 2).slot[0] * fs);
    A.s_d2 = (uint32_t)(op_of(p + 3).slot[0] * fs);
    if (last && j.red_target) k_jacobi8_t2<true, true, false, true><<<grid, 256, 0, s>>>(A);
    else if (last) k_jacobi8_t2<true, true, false, false><<<grid, 256, 0, s>>>(A);
    else k_jacobi8_t2<true, false, false, false><<<grid, 256, 0, s>>>(A);
    launches += 2;
  }
  return cudaGetLastError() == cudaSuccess ? launches : SG_ERR_CUDA;
}

}  // namespace sg
