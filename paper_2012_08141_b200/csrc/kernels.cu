// kernels.cu -- sm_100a kernels of the sparse-grid hot path.
//
//   k_activate      explicit activation: CAS-published pointer
//                   allocation from a zeroed pool + atomicOr on bitmask words.
//   k_listgen       element-list generation: 32 children
//                   per thread as one bit word, block scan, single-pass decoupled
//                   look-back for a deterministic order; persistent grid with
//                   dynamic tile order; counts stay on the device.
//   k_struct_for    fused struct-for megakernel:
//                   one tile of leaf blocks per CTA iteration, an op table
//                   interpreted per cell with every identity access kept in the
//                   same thread (atomic demotion).
//   k_deactivate    DEACTIVATE(S): zero payload of active blocks, clear masks,
//                   push pointer children to the free list (zero-on-free).
//   k_serial / k_range_for, export helpers.
// No host synchronization anywhere on the hot path: list counts are read on
// the device and every kernel grid-strides over them.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include "sg_internal.h"
#include "jit.h"

namespace cg = cooperative_groups;

namespace sg {

#include "device_common.cuh"

struct ActArgs {
  DTree T;
  DevCtx C;
  const int32_t* coords;
  int64_t n;
  int task;
};

// Explicit activation: the activating walk with warp-aggregated
// mask updates -- lanes whose cells share a mask word (__match_any_sync on the
// word address) OR their bits together (__reduce_or_sync) and one lane issues
// the atomicOr, skipped when every bit is already set.
__device__ uint32_t* activate_walk_agg(const DevCtx& C, const DTree& T, const int c[3], int task) {
  uint32_t* cont = T.seg[0].base;
  uint32_t idx = 0;
  for (int l = 0; l < T.nlev; l++) {
    const DLevel& L = T.lev[l];
    idx = (idx << L.lE) | local_lin(L, c);
    if (L.kind == SG_BITMASKED) {
      uint32_t* w = cont + L.mask_off + (idx >> 5);
      const uint32_t b = 1u << (idx & 31);
      const unsigned am = __activemask();
      const unsigned peers = __match_any_sync(am, (unsigned long long)w);
      if (peers == (1u << (threadIdx.x & 31))) {
        // alone on its word (random coordinates): no aggregation.  The OR
        // reduction over a partial mask is a loop over the warp's distinct
        // groups (REDUX per group), which made a random-coordinate warp pay 32
        // reductions (ACT-XL: 7.3% of instructions each on the loop's lines)
        if (!(ld_volatile(w) & b)) atomicOr(w, b);
      } else {
        const uint32_t bits = __reduce_or_sync(peers, b);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1 && (ld_volatile(w) & bits) != bits) atomicOr(w, bits);
      }
    } else if (L.kind == SG_POINTER) {
      int32_t s = acquire_child(C, T, L, cont, idx, c, task);
      if (s < 0) return nullptr;
      cont = cont_ptr(T, L.seg + 1, (uint32_t)s);
      idx = 0;
    }
  }
  return cont;
}

__global__ void __launch_bounds__(256) k_activate(const __grid_constant__ ActArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3] = {0, 0, 0};
    for (int d = 0; d < a.T.nd; d++) c[d] = a.coords[i * a.T.nd + d];
    if (!in_domain(a.T, c)) { set_err(a.C, SG_ERR_RANGE, a.task); continue; }
    activate_walk_agg(a.C, a.T, c, a.task);
  }
}

// ---------------------------------------------------------------------------
// Listgen
// ---------------------------------------------------------------------------
struct LGArgs {
  DTree T;
  DevCtx C;
  int ls, lp, mode;     // mode 0: root parent, 1: parent in same segment, 2: parent pointer of previous segment
  int lratio, lcpp, nbits;
  int fast8;            // bitmasked level with >= 8 aligned word-chunks per parent entry
  const uint32_t* pentries;
  const uint32_t* pcount;
  DList out;
  int task;
};

constexpr int LG_TPB = 256, LG_CPT = 8, LG_TILE = LG_TPB * LG_CPT, LG_STAGE = 8192;

__device__ __forceinline__ uint32_t lg_chunk(const LGArgs& a, uint64_t chunk, uint32_t& cslot, uint32_t& first) {
  uint32_t p = (uint32_t)(chunk >> a.lcpp), sub = (uint32_t)(chunk & ((1u << a.lcpp) - 1u));
  const DLevel& S = a.T.lev[a.ls];
  const uint32_t* cont;
  if (a.mode == 0) {
    cslot = 0; first = sub * 32u; cont = a.T.seg[0].base;
  } else {
    const DLevel& P = a.T.lev[a.lp];
    uint32_t e = a.pentries[p];
    uint32_t ps = e >> P.ln, pidx = e & ((1u << P.ln) - 1u);
    if (a.mode == 1) {
      cslot = ps; first = (pidx << a.lratio) + sub * 32u; cont = cont_ptr(a.T, S.seg, ps);
    } else {
      const uint32_t* pc = cont_ptr(a.T, P.seg, ps);
      uint32_t v = pc[P.slot_off + pidx];
      if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) { cslot = 0; first = 0; return 0u; }
      cslot = v - 1u; first = sub * 32u; cont = cont_ptr(a.T, S.seg, cslot);
    }
  }
  uint32_t bits = 0;
  if (S.kind == SG_BITMASKED) {
    uint32_t w = cont[S.mask_off + (first >> 5)];
    bits = a.nbits == 32 ? w : ((w >> (first & 31u)) & ((1u << a.nbits) - 1u));
  } else {
    const uint32_t* sl = cont + S.slot_off + first;
    for (int k = 0; k < a.nbits; k++) bits |= (sl[k] != SG_SLOT_NULL ? 1u : 0u) << k;
  }
  return bits;
}

__device__ __forceinline__ uint64_t lb_pack(uint32_t epoch, uint32_t flag, uint32_t v) {
  return ((uint64_t)(epoch & 0x3FFFFFFFu) << 34) | ((uint64_t)flag << 32) | v;
}

// Single-pass decoupled look-back (deterministic tile order), run by one full
// warp: lane l inspects tiles j-l-32m (m < K), i.e. 32K predecessors per step,
// until the nearest one carrying an inclusive prefix (flag 2).  Returns the
// exclusive prefix of `tile`.  Descriptors of an older epoch read as "not yet
// published".  The inclusive frontier advances at most 32K tiles per L2 round
// trip, so many small tiles in flight need K > 1 (k_listgen_warp).
template <int K = 1, int kSleepNs = 0>
__device__ __forceinline__ uint32_t lb_lookback(const uint64_t* st, uint32_t tile, uint32_t epoch, int lane) {
  uint32_t prefix = 0;
  int64_t j = (int64_t)tile - 1;
  while (j >= 0) {
    uint64_t s[K];
    uint32_t fl[K];
#pragma unroll
    for (int m = 0; m < K; m++) {
      const int64_t q = j - lane - 32 * m;
      s[m] = 0;
      fl[m] = 2u;                             // beyond tile 0: acts as an inclusive zero
      if (q >= 0) {
        s[m] = ld_volatile64(&st[q]);
        fl[m] = ((uint32_t)(s[m] >> 34) == epoch) ? (uint32_t)(s[m] >> 32) & 3u : 0u;
      }
    }
#pragma unroll
    for (int m = 0; m < K; m++) {
      const int64_t q = j - lane - 32 * m;
      while (fl[m] == 0u) {
        if (kSleepNs) __nanosleep(kSleepNs);   // a spinning warp leaves its issue slots to the others
        s[m] = ld_volatile64(&st[q]);
        fl[m] = ((uint32_t)(s[m] >> 34) == epoch) ? (uint32_t)(s[m] >> 32) & 3u : 0u;
      }
    }
    int stop = 32 * K;                        // order index l + 32m of the nearest inclusive
#pragma unroll
    for (int m = K - 1; m >= 0; m--) {
      const uint32_t incl = __ballot_sync(0xffffffffu, fl[m] == 2u);
      if (incl) stop = 32 * m + __ffs(incl) - 1;
    }
    uint32_t v = 0;
#pragma unroll
    for (int m = 0; m < K; m++)
      if (lane + 32 * m <= stop && j - lane - 32 * m >= 0) v += (uint32_t)s[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (stop < 32 * K) break;
    j -= 32 * K;
  }
  return prefix;
}

__global__ void __launch_bounds__(LG_TPB) k_listgen(const __grid_constant__ LGArgs a) {
  __shared__ uint32_t s_warp[LG_TPB / 32];
  __shared__ uint32_t s_tile, s_base, s_total, s_epoch, s_run;
  __shared__ uint32_t s_stage[LG_STAGE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // solo: one CTA walks the tiles in order with a running prefix -- no tile
  // counter, no look-back, no finisher atomics (small lists are a chain of
  // dependent memory round trips, so every one removed counts)
  const bool solo = gridDim.x == 1;
  uint32_t solo_tile = 0;
  if (threadIdx.x == 0) { s_epoch = solo ? 0u : ld_volatile(&a.out.ctl[2]) & 0x3FFFFFFFu; s_run = 0u; }
  uint32_t nparent = a.mode == 0 ? 1u : *a.pcount;
  uint64_t nchunks = (uint64_t)nparent << a.lcpp;
  uint32_t ntiles = (uint32_t)((nchunks + LG_TILE - 1) / LG_TILE);
  const uint32_t lnS = a.T.lev[a.ls].ln;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  while (true) {
    uint32_t tile;
    if (solo) {
      tile = solo_tile++;
    } else {
      if (threadIdx.x == 0) s_tile = atomicAdd(&a.out.ctl[0], 1u);
      __syncthreads();
      tile = s_tile;
    }
    if (tile >= ntiles) break;
    uint32_t bits[LG_CPT], cs[LG_CPT], fs[LG_CPT];
    uint32_t cnt = 0;
    const uint64_t ch0 = (uint64_t)tile * LG_TILE + threadIdx.x * LG_CPT;
    if (a.fast8 && ch0 + LG_CPT <= nchunks) {
      // bitmasked level, >= 8 word-chunks per parent entry: the thread's 8 chunks
      // share one parent, so decode it once and fetch the 8 mask words with two
      // 16-byte loads
      uint32_t c0, f0;
      const uint32_t p = (uint32_t)(ch0 >> a.lcpp), sub = (uint32_t)(ch0 & ((1u << a.lcpp) - 1u));
      const DLevel& S = a.T.lev[a.ls];
      const DLevel& P = a.T.lev[a.lp < 0 ? 0 : a.lp];
      const uint32_t* cont = nullptr;
      if (a.mode == 0) {
        c0 = 0; f0 = sub * 32u; cont = a.T.seg[0].base;
      } else {
        const uint32_t e = a.pentries[p];
        const uint32_t ps = e >> P.ln, pidx = e & ((1u << P.ln) - 1u);
        if (a.mode == 1) {
          c0 = ps; f0 = (pidx << a.lratio) + sub * 32u; cont = cont_ptr(a.T, S.seg, ps);
        } else {
          const uint32_t v = cont_ptr(a.T, P.seg, ps)[P.slot_off + pidx];
          const bool ok = v != SG_SLOT_NULL && v != SG_SLOT_BUSY;
          c0 = ok ? v - 1u : 0u; f0 = sub * 32u; cont = ok ? cont_ptr(a.T, S.seg, c0) : nullptr;
        }
      }
      uint4 w0 = make_uint4(0u, 0u, 0u, 0u), w1 = w0;
      if (cont) {
        const uint4* q = reinterpret_cast<const uint4*>(cont + S.mask_off + (f0 >> 5));
        w0 = q[0];
        w1 = q[1];
      }
      bits[0] = w0.x; bits[1] = w0.y; bits[2] = w0.z; bits[3] = w0.w;
      bits[4] = w1.x; bits[5] = w1.y; bits[6] = w1.z; bits[7] = w1.w;
#pragma unroll
      for (int k = 0; k < LG_CPT; k++) {
        cs[k] = c0;
        fs[k] = f0 + 32u * k;
        cnt += __popc(bits[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < LG_CPT; k++) {
        uint64_t ch = ch0 + k;
        bits[k] = ch < nchunks ? lg_chunk(a, ch, cs[k], fs[k]) : 0u;
        cnt += __popc(bits[k]);
      }
    }
    // block exclusive scan
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < LG_TPB / 32 ? s_warp[lane] : 0u, wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      if (lane < LG_TPB / 32) s_warp[lane] = wi - w;   // exclusive warp offsets
      uint32_t total = __shfl_sync(0xffffffffu, wi, LG_TPB / 32 - 1);
      if (lane == 0) {
        s_total = total;
        // publish the aggregate now, so successors can look back while we stage
        if (!solo)
          atomicExch((unsigned long long*)&a.out.status[tile],
                     (unsigned long long)lb_pack(epoch, tile == 0 ? 2u : 1u, total));
      }
    }
    __syncthreads();
    // stage the tile's first LG_STAGE entries in shared memory (tile-local
    // offsets need no prefix) while warp 0 runs the look-back
    const uint32_t my0 = s_warp[warp] + (inc - cnt);
    if (s_total <= (uint32_t)LG_STAGE) {
      // common case, the whole tile fits: no bound check per bit, highest bit
      // first (FLO without the bit reversal __ffs needs; order within a word
      // is free, reading R2), entry = chunk base + bit (no carry: fs % 32 == 0)
      uint32_t* stg = s_stage + my0;
#pragma unroll
      for (int k = 0; k < LG_CPT; k++) {
        uint32_t b = bits[k];
        const uint32_t hi = (cs[k] << lnS) | fs[k];
        while (b) {
          const uint32_t t = 31u - __clz(b);
          b ^= 1u << t;
          *stg++ = hi + t;
        }
      }
    } else {
      uint32_t off = my0;
#pragma unroll
      for (int k = 0; k < LG_CPT; k++) {
        uint32_t b = bits[k];
        while (b) {
          int t = __ffs(b) - 1;
          b &= b - 1;
          if (off < LG_STAGE) s_stage[off] = (cs[k] << lnS) | (fs[k] + (uint32_t)t);
          off++;
        }
      }
    }
    if (solo) {
      if (threadIdx.x == 0) s_base = s_run;
    } else if (warp == 0) {
      const uint32_t total = s_total;
      uint64_t* st = a.out.status;
      const uint32_t prefix = lb_lookback(st, tile, epoch, lane);
      if (lane == 0) {
        if (tile != 0)
          atomicExch((unsigned long long*)&st[tile], (unsigned long long)lb_pack(epoch, 2u, prefix + total));
        s_base = prefix;
        if (tile == ntiles - 1) {
          uint32_t n = prefix + total;
          if (n > a.out.capacity) { set_err(a.C, SG_ERR_LIST_OVERFLOW, a.task); n = a.out.capacity; }
          *a.out.count = n;
        }
      }
    }
    __syncthreads();
    // coalesced copy of the staged entries; dense tiles take further rounds
    const uint32_t base = s_base, total = s_total;
    for (uint32_t r0 = 0; r0 < total; r0 += LG_STAGE) {
      if (r0 > 0) {
        uint32_t off = my0;
#pragma unroll
        for (int k = 0; k < LG_CPT; k++) {
          uint32_t b = bits[k];
          while (b) {
            int t = __ffs(b) - 1;
            b &= b - 1;
            if (off >= r0 && off < r0 + LG_STAGE) s_stage[off - r0] = (cs[k] << lnS) | (fs[k] + (uint32_t)t);
            off++;
          }
        }
        __syncthreads();
      }
      const uint32_t n = min(total - r0, (uint32_t)LG_STAGE);
      uint32_t* dst = a.out.entries + base + r0;
      if ((uint64_t)base + r0 + n <= a.out.capacity) {
        for (uint32_t i = threadIdx.x; i < n; i += LG_TPB) dst[i] = s_stage[i];
      } else {
        for (uint32_t i = threadIdx.x; i < n; i += LG_TPB)
          if (base + r0 + i < a.out.capacity) dst[i] = s_stage[i];
      }
      __syncthreads();
    }
    if (solo && threadIdx.x == 0) s_run = base + total;
  }
  if (solo) {
    if (threadIdx.x == 0) {
      uint32_t n = s_run;
      if (n > a.out.capacity) { set_err(a.C, SG_ERR_LIST_OVERFLOW, a.task); n = a.out.capacity; }
      *a.out.count = n;
      a.out.ctl[4] = 0u;   // the block table (if any) is stale until a struct-for rebuilds it
    }
    return;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.out.ctl[1], 1u) == gridDim.x - 1) {
      if (ntiles == 0) *a.out.count = 0;
      a.out.ctl[0] = 0;
      a.out.ctl[1] = 0;
      a.out.ctl[2] = a.out.ctl[2] + 1u;
      a.out.ctl[4] = 0u;   // the block table (if any) is stale until a struct-for rebuilds it
      __threadfence();
    }
  }
}


// ---------------------------------------------------------------------------
// Warp-tile listgen for big bitmasked lists (LG-XL).  Same set as
// k_listgen, in a deterministic order (chunk order, highest bit first within a
// word, reading R2), but every warp is an independent tile of LGW_SUB
// consecutive sub-tiles, each 32 lanes x LGW_WPL mask words:
//   * no CTA barriers: a warp grabs its tile, loads all its words up front
//     (two 16-byte loads per lane per sub-tile), scans the sub-tile counts
//     with shuffles, publishes the tile aggregate and runs one decoupled
//     look-back for the whole tile (one look-back per 1024 words: with
//     thousands of warps in flight a per-256-word look-back walked ~5 x 32
//     descriptors back, measured);
//   * the set bits of a lane's 8 words are extracted in ONE loop whose trip
//     count is the lane's own count (not one loop per word run to the
//     per-word maximum over the warp); advancing to the next non-empty word
//     is a single predicated shared load from a per-lane compacted copy;
//   * the staged entries are stored at the destination's 16-byte phase, so
//     the copy to the list is one 16-byte load + one 16-byte store per 4
//     entries.
// Sub-tiles denser than the staging buffer write their entries straight to
// the list (correct, uncoalesced).
// ---------------------------------------------------------------------------
constexpr int LGW_MIN_HINT = 64;   // CTA tiles (2048 chunks) below which the CTA-tile kernel runs
constexpr int LGW_TPB = 128, LGW_WARPS = LGW_TPB / 32, LGW_WPL = 8, LGW_SUBTILE = 32 * LGW_WPL, LGW_SUB = 4,
              LGW_TILE = LGW_SUB * LGW_SUBTILE, LGW_CAP = 1024, LGW_LB = 1, LGW_SLEEP = 128;

__device__ __forceinline__ uint32_t bfind_u32(uint32_t x) {   // index of the highest set bit
  uint32_t r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// dst[0, cnt): the lane's set bits, word by word, highest bit first.  b/hi:
// the first word and its entry base; the lane's other non-empty words are
// compacted at rec[n * 32] = (word, entry base), so advancing to the next word
// is always exactly one predicated 8-byte shared load.  (Two interleaved
// streams per lane to overlap that load measured slower: 1.5x the
// instructions, 350 vs 287 us on LG-XL.)
__device__ __forceinline__ void lgw_extract(uint32_t* dst, uint32_t cnt, uint32_t b, uint32_t hi, const uint2* rec) {
#pragma unroll 4   // (8 measured slower: 297 vs 287 us)
  for (uint32_t i = 0; i < cnt; i++) {
    if (b == 0u) {
      const uint2 r = *rec;
      rec += 32;
      b = r.x;
      hi = r.y;
    }
    const uint32_t t = bfind_u32(b);
    dst[i] = hi + t;
    b ^= 1u << t;
  }
}

// Container and entry base of word-chunk ch0 (lcpp >= 3: the chunk's parent
// entry also holds the next 7 chunks).
__device__ __forceinline__ const uint32_t* lgw_decode(const LGArgs& a, uint64_t ch0, uint32_t& hi) {
  const DLevel& S = a.T.lev[a.ls];
  const DLevel& P = a.T.lev[a.lp < 0 ? 0 : a.lp];
  const uint32_t p = (uint32_t)(ch0 >> a.lcpp), sub = (uint32_t)(ch0 & ((1u << a.lcpp) - 1u));
  const uint32_t* cont = nullptr;
  uint32_t c0 = 0, f0 = sub * 32u;
  if (a.mode == 0) {
    cont = a.T.seg[0].base;
  } else {
    const uint32_t e = a.pentries[p];
    const uint32_t ps = e >> P.ln, pidx = e & ((1u << P.ln) - 1u);
    if (a.mode == 1) {
      c0 = ps; f0 = (pidx << a.lratio) + sub * 32u; cont = cont_ptr(a.T, S.seg, ps);
    } else {
      const uint32_t v = cont_ptr(a.T, P.seg, ps)[P.slot_off + pidx];
      const bool ok = v != SG_SLOT_NULL && v != SG_SLOT_BUSY;
      c0 = ok ? v - 1u : 0u; cont = ok ? cont_ptr(a.T, S.seg, c0) : nullptr;
    }
  }
  hi = (c0 << S.ln) | f0;
  return cont ? cont + S.mask_off + (f0 >> 5) : nullptr;
}

// Loads all LGW_SUB sub-tiles of warp tile `tile`: for sub-tile r this lane's
// LGW_WPL consecutive word-chunks and their entry base.  When one parent entry
// spans the whole tile (lcpp >= 10, e.g. LG-XL's 32^3 leaf containers) the
// parent is decoded once per tile instead of once per sub-tile.
__device__ __forceinline__ void lgw_load_tile(const LGArgs& a, uint64_t nchunks, uint32_t tile, int lane,
                                              uint4 (&w)[LGW_SUB][2], uint32_t (&hi)[LGW_SUB]) {
  const uint64_t t0 = (uint64_t)tile * LGW_TILE;
  if ((1u << a.lcpp) >= (uint32_t)LGW_TILE && t0 + LGW_TILE <= nchunks) {
    uint32_t h;
    const uint32_t* m = lgw_decode(a, t0, h);   // same parent for every lane and sub-tile
#pragma unroll
    for (int r = 0; r < LGW_SUB; r++) {
      const uint32_t off = (uint32_t)(r * LGW_SUBTILE) + (uint32_t)lane * LGW_WPL;
      hi[r] = h + 32u * off;
      if (m) {
        const uint4* q = reinterpret_cast<const uint4*>(m + off);
        w[r][0] = q[0];
        w[r][1] = q[1];
      } else {
        w[r][0] = make_uint4(0u, 0u, 0u, 0u);
        w[r][1] = w[r][0];
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < LGW_SUB; r++) {
    const uint64_t ch0 = t0 + (uint32_t)(r * LGW_SUBTILE) + (uint32_t)lane * LGW_WPL;
    hi[r] = 0;
    w[r][0] = make_uint4(0u, 0u, 0u, 0u);
    w[r][1] = w[r][0];
    if (ch0 < nchunks) {
      const uint32_t* m = lgw_decode(a, ch0, hi[r]);
      if (m) {
        const uint4* q = reinterpret_cast<const uint4*>(m);
        w[r][0] = q[0];
        w[r][1] = q[1];
      }
    }
  }
}

__device__ __forceinline__ uint32_t popc8(const uint4& w0, const uint4& w1) {
  return __popc(w0.x) + __popc(w0.y) + __popc(w0.z) + __popc(w0.w) +
         __popc(w1.x) + __popc(w1.y) + __popc(w1.z) + __popc(w1.w);
}

__global__ void __launch_bounds__(LGW_TPB, 8) k_listgen_warp(const __grid_constant__ LGArgs a) {
  __shared__ __align__(16) uint32_t s_out[LGW_WARPS][LGW_CAP + 4];
  __shared__ uint2 s_rec[LGW_WARPS][LGW_WPL * 32];   // compacted non-empty words 1..7 per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t epoch = ld_volatile(&a.out.ctl[2]) & 0x3FFFFFFFu;
  const uint32_t nparent = a.mode == 0 ? 1u : *a.pcount;
  const uint64_t nchunks = (uint64_t)nparent << a.lcpp;
  const uint32_t ntiles = (uint32_t)((nchunks + LGW_TILE - 1) / LGW_TILE);
  uint2* rec = s_rec[warp];
  uint32_t* so = s_out[warp];
  uint64_t* st = a.out.status;
  while (true) {
    uint32_t tile = 0;
    if (lane == 0) tile = atomicAdd(&a.out.ctl[0], 1u);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= ntiles) break;
    uint4 w[LGW_SUB][2];
    uint32_t hi[LGW_SUB], cnt[LGW_SUB], inc[LGW_SUB], tot[LGW_SUB];
    lgw_load_tile(a, nchunks, tile, lane, w, hi);
    uint32_t agg = 0;
#pragma unroll
    for (int r = 0; r < LGW_SUB; r++) {
      cnt[r] = popc8(w[r][0], w[r][1]);
      inc[r] = cnt[r];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int r = 0; r < LGW_SUB; r++) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc[r], o);
        if (lane >= o) inc[r] += t;
      }
    }
#pragma unroll
    for (int r = 0; r < LGW_SUB; r++) {
      tot[r] = __shfl_sync(0xffffffffu, inc[r], 31);
      agg += tot[r];
    }
    if (lane == 0)
      atomicExch((unsigned long long*)&st[tile], (unsigned long long)lb_pack(epoch, tile == 0 ? 2u : 1u, agg));
    uint32_t base = lb_lookback<LGW_LB, LGW_SLEEP>(st, tile, epoch, lane);
    if (lane == 0) {
      if (tile != 0)
        atomicExch((unsigned long long*)&st[tile], (unsigned long long)lb_pack(epoch, 2u, base + agg));
      if (tile == ntiles - 1) {
        uint32_t n = base + agg;
        if (n > a.out.capacity) { set_err(a.C, SG_ERR_LIST_OVERFLOW, a.task); n = a.out.capacity; }
        *a.out.count = n;
      }
    }
#pragma unroll
    for (int r = 0; r < LGW_SUB; r++) {
      const uint32_t total = tot[r];
      if (total != 0u) {
        // non-empty words 1..7 of the sub-tile, compacted per lane (word 0
        // starts in a register)
        {
          const uint32_t wv[7] = {w[r][0].y, w[r][0].z, w[r][0].w, w[r][1].x, w[r][1].y, w[r][1].z, w[r][1].w};
          uint32_t n = 0;
#pragma unroll
          for (int k = 0; k < 7; k++) {
            if (wv[k]) { rec[n * 32u + lane] = make_uint2(wv[k], hi[r] + 32u * (k + 1)); n++; }
          }
        }
        const uint32_t my0 = inc[r] - cnt[r];
        __syncwarp();
        if (total <= (uint32_t)LGW_CAP) {
          const uint32_t shift = base & 3u;
          lgw_extract(so + shift + my0, cnt[r], w[r][0].x, hi[r], rec + lane);
          __syncwarp();
          // [base, base + total) <- so[shift, shift + total): 16-byte groups at
          // the destination's phase; the partial head / tail groups element-wise
          const uint32_t end = min(base + total, a.out.capacity);
          const uint32_t ga = (base + 3u) & ~3u, gb = end & ~3u;   // full groups: [ga, gb)
          uint32_t* ent = a.out.entries;
          if (ga < gb) {
            uint4* dst = reinterpret_cast<uint4*>(ent + ga);
            const uint4* src = reinterpret_cast<const uint4*>(so + shift + (ga - base));
            const uint32_t ng = (gb - ga) >> 2;
            for (uint32_t j = lane; j < ng; j += 32u) dst[j] = src[j];
            if (lane < ga - base) ent[base + lane] = so[shift + lane];            // head (< 4)
            if (lane < end - gb) ent[gb + lane] = so[shift + (gb - base) + lane];  // tail (< 4)
          } else if (lane < end - min(base, end)) {
            ent[base + lane] = so[shift + lane];                                   // < 8 entries
          }
        } else {
          // dense sub-tile: straight to the list (entries past the capacity are
          // dropped; the overflow is reported with the count)
          const uint32_t o = base + my0, cap = a.out.capacity;
          lgw_extract(a.out.entries + o, o >= cap ? 0u : min(cnt[r], cap - o), w[r][0].x, hi[r], rec + lane);
        }
        __syncwarp();
        base += total;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.out.ctl[1], 1u) == gridDim.x - 1) {
      if (ntiles == 0) *a.out.count = 0;
      a.out.ctl[0] = 0;
      a.out.ctl[1] = 0;
      a.out.ctl[2] = a.out.ctl[2] + 1u;
      a.out.ctl[4] = 0u;   // the block table (if any) is stale until a struct-for rebuilds it
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// Small-list listgen (parent capacity x chunks <= 1024 words: the configs'
// lists, SURVEY 8d.4 "latency-bound").  One CTA of 1024 threads; every thread
// owns ONE unit per pass -- one child slot of a pointer level (a coalesced
// 4-byte load) or one 32-child mask word of a bitmasked level -- so a pass is a
// single round of independent loads (parent entry -> slot -> word) followed by
// one block scan and the writes.  The CTA-tile kernel gave each thread 8 chunks
// (a pointer-level chunk being 32 sequential slot loads) and walked its tiles
// in series: 12-16 us per config listgen.  Entries in unit order, highest bit
// first within a word (reading R2); count, capacity check and the table flag as
// in k_listgen.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_listgen_small(const __grid_constant__ LGArgs a) {
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const DLevel& S = a.T.lev[a.ls];
  const bool ptr = S.kind != SG_BITMASKED;
  const uint32_t nparent = a.mode == 0 ? 1u : *a.pcount;
  const uint64_t nchunks = (uint64_t)nparent << a.lcpp;
  const uint32_t lnb = ptr ? (uint32_t)__ffs(a.nbits) - 1u : 0u;   // units per chunk = 2^lnb
  const uint64_t nunits = nchunks << lnb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lnS = S.ln;
  uint32_t carry = 0;
  for (uint64_t u0 = 0; u0 < nunits; u0 += 1024) {
    const uint64_t u = u0 + threadIdx.x;
    uint32_t bits = 0, hi = 0;
    if (u < nunits) {
      const uint64_t chunk = u >> lnb;
      const uint32_t k = (uint32_t)(u & ((1u << lnb) - 1u));
      const uint32_t p = (uint32_t)(chunk >> a.lcpp), sub = (uint32_t)(chunk & ((1u << a.lcpp) - 1u));
      const uint32_t* cont = nullptr;
      uint32_t cslot = 0, first = sub * 32u;
      if (a.mode == 0) {
        cont = a.T.seg[0].base;
      } else {
        const DLevel& P = a.T.lev[a.lp];
        const uint32_t e = a.pentries[p];
        const uint32_t ps = e >> P.ln, pidx = e & ((1u << P.ln) - 1u);
        if (a.mode == 1) {
          cslot = ps; first = (pidx << a.lratio) + sub * 32u; cont = cont_ptr(a.T, S.seg, ps);
        } else {
          const uint32_t v = cont_ptr(a.T, P.seg, ps)[P.slot_off + pidx];
          if (v != SG_SLOT_NULL && v != SG_SLOT_BUSY) { cslot = v - 1u; cont = cont_ptr(a.T, S.seg, cslot); }
        }
      }
      if (cont) {
        if (ptr) {
          bits = cont[S.slot_off + first + k] != SG_SLOT_NULL ? 1u : 0u;
          first += k;
        } else {
          const uint32_t wd = cont[S.mask_off + (first >> 5)];
          bits = a.nbits == 32 ? wd : ((wd >> (first & 31u)) & ((1u << a.nbits) - 1u));
        }
      }
      hi = (cslot << lnS) | first;
    }
    const uint32_t cnt = __popc(bits);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
      const uint32_t v = s_w[lane];
      uint32_t vi = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, vi, o);
        if (lane >= o) vi += t;
      }
      s_w[lane] = vi - v;
      if (lane == 31) s_carry = vi;
    }
    __syncthreads();
    uint32_t o = carry + s_w[w] + inc - cnt;
    const uint32_t cap = a.out.capacity;
    while (bits) {
      const uint32_t t = 31u - __clz(bits);
      bits ^= 1u << t;
      if (o < cap) a.out.entries[o] = hi + t;
      o++;
    }
    carry += s_carry;
    __syncthreads();   // s_w / s_carry reused by the next pass
  }
  if (threadIdx.x == 0) {
    uint32_t n = carry;
    if (n > a.out.capacity) { set_err(a.C, SG_ERR_LIST_OVERFLOW, a.task); n = a.out.capacity; }
    *a.out.count = n;
    a.out.ctl[4] = 0u;   // the block table (if any) is stale until a struct-for rebuilds it
  }
}

__global__ void k_clear_list(uint32_t* count) { *count = 0; }

#include "mpm_ops.cuh"
#include "struct_for.cuh"
#include "exchange_ops.cuh"
#include "mpm_adj.cuh"
#include "mpm_bin.cuh"

// ---------------------------------------------------------------------------
// Serial and range-for
// ---------------------------------------------------------------------------
struct SerArgs {
  DevCtx C;
  int nops;
  DOp ops[SG_MAXOPS];
  uint64_t aux[SG_MAXOPS];
};

__global__ void k_serial(const __grid_constant__ SerArgs A) {
  for (int o = 0; o < A.nops; o++) {
    if (A.ops[o].op == SG_OP_CLEAR_SCALAR) *(uint32_t*)A.aux[o] = 0u;
    if (A.ops[o].op == SG_OP_COPY_SCALAR)
      *(uint32_t*)A.aux[o] = A.C.scalars[A.C.fields[A.ops[o].f[1]].scalar];
    if (A.ops[o].op == SG_OP_ARRAY_COUNT) *A.C.arrays[A.ops[o].a[0]].dcount = (int32_t)A.ops[o].p[0];
  }
}

struct RFArgs {
  DevCtx C;
  int64_t n;
  const int32_t* dcount;   // device extent (range_n < 0), else null
  int nops;
  int task;
  DOp ops[SG_MAXOPS];
};

__global__ void __launch_bounds__(128) k_range_for(const __grid_constant__ RFArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int o = 0; o < A.nops; o++) {
      const DOp& op = A.ops[o];
      switch (op.op) {
        case SG_OP_P2G: mpm_p2g<0>(A.C, A.C.trees[A.C.fields[op.f[0]].tree], op, i, A.task); break;
        case SG_OP_G2P: mpm_g2p<0>(A.C, A.C.trees[A.C.fields[op.f[0]].tree], op, i); break;
        case SG_OP_HALO_UNPACK: halo_unpack(A.C, op, i, A.task); break;
        case SG_OP_ADJ_INIT: adj_init(A.C, op, i); break;
        default: break;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Deactivate (reading R7): payload zeroed, masks cleared, children freed.
// ---------------------------------------------------------------------------
struct DeArgs {
  DTree T;
  DevCtx C;
  int ls;
  const uint32_t* drive_entries;
  const uint32_t* drive_count;
  const uint32_t* lent[SG_MAXL];
  const uint32_t* lcnt[SG_MAXL];
};

__global__ void __launch_bounds__(256) k_deactivate(const __grid_constant__ DeArgs A) {
  const DTree& T = A.T;
  const uint32_t nblk = A.drive_entries ? *A.drive_count : 1u;
  const uint32_t blk = 1u << T.lblk;
  const uint64_t fstride = 1ull << T.ln_leaf;
  // phase 1: zero the payload (and leaf bits) of every active block
  for (uint32_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    uint32_t* cont;
    uint32_t first;
    int org[3];
    if (!resolve_entry(T, A.drive_entries ? A.drive_entries[b] : 0u, cont, first, org)) continue;
    uint32_t* p0 = cont + T.payload_off + first;
    for (int f = 0; f < T.nfields; f++)
      for (uint32_t i = threadIdx.x; i < blk; i += blockDim.x) p0[(uint64_t)f * fstride + i] = 0u;
    if (T.leaf_bitmasked) {
      const DLevel& LL = T.lev[T.nlev - 1];
      for (uint32_t w = (first >> 5) + threadIdx.x; w < ((first + blk + 31) >> 5); w += blockDim.x)
        cont[LL.mask_off + w] = 0u;
    }
  }
  // phase 2: every listed level at/below S
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gsz = (uint64_t)gridDim.x * blockDim.x;
  for (int l = A.ls; l < T.nlev; l++) {
    if (!A.lent[l]) continue;
    const DLevel& L = T.lev[l];
    uint32_t n = *A.lcnt[l];
    for (uint64_t i = gtid; i < n; i += gsz) {
      uint32_t e = A.lent[l][i];
      uint32_t cs = e >> L.ln, idx = e & ((1u << L.ln) - 1u);
      uint32_t* cont = cont_ptr(T, L.seg, cs);
      if (L.kind == SG_BITMASKED) {
        cont[L.mask_off + (idx >> 5)] = 0u;
      } else if (L.kind == SG_POINTER) {
        uint32_t v = cont[L.slot_off + idx];
        cont[L.slot_off + idx] = SG_SLOT_NULL;
        if (v != SG_SLOT_NULL && v != SG_SLOT_BUSY) {
          const DSeg& S = T.seg[L.seg + 1];
          uint32_t* child = cont_ptr(T, L.seg + 1, v - 1u);
          for (uint32_t w = 0; w < S.header_words; w++) child[w] = 0u;
          int32_t pos = atomicAdd(&S.alloc[1], 1);
          S.free_list[pos] = v - 1u;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Export / handoff helpers (tests and exports only)
// ---------------------------------------------------------------------------
struct FieldIO {
  DTree T;
  int slot;
  uint32_t* dense;
  const uint32_t* src;
  int64_t total;
  int sh[3];
};

__device__ __forceinline__ void dense_coords(const FieldIO& a, int64_t i, int c[3]) {
  c[2] = (int)(i & ((1ll << a.sh[2]) - 1));
  c[1] = (int)((i >> a.sh[2]) & ((1ll << a.sh[1]) - 1));
  c[0] = (int)(i >> (a.sh[1] + a.sh[2]));
}

__global__ void k_read_field(const __grid_constant__ FieldIO a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    dense_coords(a, i, c);
    uint32_t idx;
    uint32_t* cont = locate(a.T, c, idx);
    a.dense[i] = cont ? cont[a.T.payload_off + ((uint64_t)a.slot << a.T.ln_leaf) + idx] : 0u;
  }
}

__global__ void k_load_field(const __grid_constant__ FieldIO a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3];
    dense_coords(a, i, c);
    uint32_t idx;
    uint32_t* cont = locate_active(a.T, c, idx);
    if (cont) cont[a.T.payload_off + ((uint64_t)a.slot << a.T.ln_leaf) + idx] = a.src[i];
  }
}

struct MaskScan {
  DTree T;
  int level;
  uint8_t* flags;
  int64_t total;
  int sh[3];
};

__global__ void k_mask_scan(const __grid_constant__ MaskScan a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.total; i += (int64_t)gridDim.x * blockDim.x) {
    int g[3];
    g[2] = (int)(i & ((1ll << a.sh[2]) - 1));
    g[1] = (int)((i >> a.sh[2]) & ((1ll << a.sh[1]) - 1));
    g[0] = (int)(i >> (a.sh[1] + a.sh[2]));
    const DLevel& S = a.T.lev[a.level];
    int c[3] = {g[0] << S.lbelow[0], g[1] << S.lbelow[1], g[2] << S.lbelow[2]};
    uint32_t* cont = a.T.seg[0].base;
    uint32_t idx = 0;
    uint8_t act = 1;
    for (int l = 0; l <= a.level; l++) {
      const DLevel& L = a.T.lev[l];
      idx = (idx << L.lE) | local_lin(L, c);
      if (L.kind == SG_BITMASKED) {
        if (!((cont[L.mask_off + (idx >> 5)] >> (idx & 31)) & 1u)) { act = 0; break; }
      } else if (L.kind == SG_POINTER) {
        uint32_t v = cont[L.slot_off + idx];
        if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) { act = 0; break; }
        if (l < a.level) { cont = cont_ptr(a.T, L.seg + 1, v - 1u); idx = 0; }
      }
    }
    a.flags[i] = act;
  }
}

struct ListDecode {
  DTree T;
  int level;
  const uint32_t* entries;
  const uint32_t* count;
  int32_t* coords;
};

__global__ void k_list_decode(const __grid_constant__ ListDecode a) {
  uint32_t n = *a.count;
  const DLevel& L = a.T.lev[a.level];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t e = a.entries[i];
    int g[3];
    cell_coords(a.T, a.level, e >> L.ln, e & ((1u << L.ln) - 1u), g);
    for (int d = 0; d < a.T.nd; d++) a.coords[(uint64_t)i * a.T.nd + d] = g[d];
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
static int check_launch() { return cudaGetLastError() == cudaSuccess ? 0 : SG_ERR_CUDA; }
static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

int launch_activate(const DevCtx& c, const DTree& t, int, int, const int32_t* coords, int64_t n, int task,
                    void* stream) {
  if (n <= 0) return 0;
  ActArgs a{t, c, coords, n, task};
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
  k_activate<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_listgen(const DevCtx& c, const DTree& t, int, int level, int parent_level, const DList* parent,
                   const DList& out, int task, void* stream, int grid_hint) {
  LGArgs a;
  a.T = t; a.C = c; a.ls = level; a.lp = parent_level; a.out = out; a.task = task;
  const DLevel& S = t.lev[level];
  int lratio;
  if (parent_level < 0) { a.mode = 0; lratio = S.ln; }
  else if (t.lev[parent_level].seg == S.seg) { a.mode = 1; lratio = S.ln - t.lev[parent_level].ln; }
  else { a.mode = 2; lratio = S.ln; }
  a.lratio = lratio;
  a.lcpp = lratio > 5 ? lratio - 5 : 0;
  a.nbits = lratio >= 5 ? 32 : (1 << lratio);
  // 8 chunks of one parent are 8 consecutive mask words, 16-byte aligned when the
  // level's mask region is (mask_off % 4 == 0) -- see derive_tree
  a.fast8 = S.kind == SG_BITMASKED && a.lcpp >= 3 && (S.mask_off % 4) == 0;
  a.pentries = parent ? parent->entries : nullptr;
  a.pcount = parent ? parent->count : nullptr;
  int grid = grid_hint > 0 ? grid_hint : 1;
  const int resident = num_sms() * 4;
  // big bitmasked lists: warp tiles (k_listgen_warp).  SG_LG_WARP=0 forces the
  // CTA-tile kernel, =1 the warp-tile kernel wherever it applies.
  static const int lg_warp_env = getenv("SG_LG_WARP") ? atoi(getenv("SG_LG_WARP")) : -1;
  if (a.fast8 && (lg_warp_env == 1 || (lg_warp_env != 0 && grid_hint >= LGW_MIN_HINT))) {
    static int wres = 0;
    if (!wres) {
      int per_sm = 0;
      cudaFuncSetAttribute(k_listgen_warp, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_listgen_warp, LGW_TPB, 0);
      wres = num_sms() * std::max(1, per_sm);
    }
    // grid_hint counts 1024-chunk units of the parent list's capacity; tiles
    // are LGW_TILE chunks; a launch never exceeds one resident wave
    const int64_t wt = ((int64_t)grid_hint * 1024 / LGW_TILE + LGW_WARPS - 1) / LGW_WARPS;
    k_listgen_warp<<<(int)std::max<int64_t>(1, std::min<int64_t>(wt, wres)), LGW_TPB, 0, (cudaStream_t)stream>>>(a);
    return check_launch();
  }
  grid = max(1, min(grid, resident));
  // small lists (one CTA tile of parent capacity): k_listgen_small;
  // SG_LG_SMALL=0 keeps the single-CTA path of k_listgen (measurement switch)
  static const bool lg_small = !(getenv("SG_LG_SMALL") && atoi(getenv("SG_LG_SMALL")) == 0);
  if (grid == 1 && lg_small) {
    k_listgen_small<<<1, 1024, 0, (cudaStream_t)stream>>>(a);
    return check_launch();
  }
  k_listgen<<<grid, LG_TPB, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_clear_list(const DList& l, void* stream) {
  k_clear_list<<<1, 1, 0, (cudaStream_t)stream>>>(l.count);
  return check_launch();
}

static int ilog2(uint64_t v) { int r = 0; while ((1ull << r) < v) r++; return r; }

template <typename V, int ND, bool PAIR, int GL>
static void sf_dispatch(SFArgs* a, int grid, cudaStream_t s, const ChainTab* chain) {
  if (!chain) {
    k_struct_for<V, ND, PAIR, GL><<<grid, SF_TPB, 0, s>>>(*a);
    return;
  }
  k_struct_chain<V, ND, PAIR, GL><<<1, SF_TPB, 0, s>>>(*a, *chain);
}

// A group of f32 quad ops on 8^3 dense blocks (k_stream8 / stream8_body).
static bool stream8_group(const DTree& t, const DOp* ops, int nops, int gl, bool i32) {
  if (gl != 1 || i32 || t.leaf_bitmasked) return false;
  for (int o = 0; o < nops; o++) {
    const int op = ops[o].op;
    if (!(op == SG_OP_FILL || op == SG_OP_ADD_CONST || op == SG_OP_INC || op == SG_OP_AXPY || op == SG_OP_STENCIL ||
          op == SG_OP_JACOBI || op == SG_OP_REDUCE_SUM || op == SG_OP_DOT || op == SG_OP_AXPY_RATIO ||
          op == SG_OP_XPAY_RATIO))
      return false;
  }
  return true;
}

// The JIT content of a struct-for group (same geometry decisions as
// launch_struct_for); false when the group runs a dedicated kernel instead.
bool jit_group_of(const DTree& t, const DOp* ops, int nops, JitGroup& G) {
  int lb[3] = {0, 0, 0};
  bool quad = false;
  if (t.nlev - 1 - t.driving == 1) {
    const DLevel& B = t.lev[t.nlev - 1];
    for (int d = 0; d < 3; d++) lb[d] = B.le[d];
    quad = B.le[t.nd - 1] >= 2;
  }
  const int nd = quad ? t.nd : 0;
  int gl = 0;
  if (nd == 3 && lb[0] == 3 && lb[1] == 3 && lb[2] == 3) gl = 1;
  else if (nd == 3 && lb[0] == 2 && lb[1] == 2 && lb[2] == 2) gl = 2;
  else if (nd == 2 && lb[0] == 2 && lb[1] == 2) gl = 3;
  const bool i32 = ops[0].dt == SG_I32;
  const bool jac_red = nops == 2 && ops[0].op == SG_OP_JACOBI && ops[1].op == SG_OP_REDUCE_SUM &&
                       ops[1].f[1] == ops[0].f[0] && ops[1].scalar >= 0;
  if ((nops == 1 || jac_red) && ops[0].op == SG_OP_JACOBI && gl == 1 && !i32 && !t.leaf_bitmasked)
    return false;   // k_jacobi8
  G.nops = nops; G.nd = nd; G.gl = gl; G.i32 = i32 ? 1 : 0;
  G.stream = stream8_group(t, ops, nops, gl, i32) && getenv("SG_NO_STREAM8") == nullptr ? 1 : 0;
  for (int o = 0; o < nops; o++) G.ops[o] = ops[o];
  return true;
}

int launch_struct_for(const DevCtx& c, const DTree& t, int, const DList* drive, const DOp* ops, int nops,
                      int task, void* stream, int grid_hint, const DOp* chain_ops, const int* chain_phase_end,
                      int nphases, int chain_needs_nbr) {
  SFArgs* a = new SFArgs();
  a->T = t; a->C = c; a->task = task; a->nops = nops;
  a->entries = drive ? drive->entries : nullptr;
  a->count = drive ? drive->count : nullptr;
  a->table = drive ? drive->table : nullptr;
  a->table_ctl = drive ? drive->ctl : nullptr;
  a->has_reduce = 0;
  for (int o = 0; o < nops; o++)
    a->has_reduce |= ops[o].op == SG_OP_REDUCE_SUM || ops[o].op == SG_OP_RESID_NORM2 || ops[o].op == SG_OP_DOT;
  a->need_nbr = 0;
  bool i32 = false;
  for (int o = 0; o < nops; o++) {
    a->ops[o] = ops[o];
    int op = ops[o].op;
    if (op == SG_OP_STENCIL || op == SG_OP_JACOBI || op == SG_OP_JITTER || op == SG_OP_SMOOTH_RB ||
        op == SG_OP_RESTRICT || op == SG_OP_RESID_NORM2)
      a->need_nbr = 1;
    a->aux[o] = 0;
  }
  if (chain_needs_nbr) a->need_nbr = 1;
  // dtype of the group (validated uniform by the host)
  i32 = ops[0].dt == SG_I32;
  for (int o = 0; o < nops; o++)
    if (ops[o].scalar >= 0) a->aux[o] = (uint64_t)(c.scalars + ops[o].scalar);
  const int lblk = t.lblk;
  // tile: 2048 cells (at most SF_MAXE blocks); larger blocks span several tiles
  const int TILE_LOG = 11;
  a->ltile = TILE_LOG;
  a->lept = 8;   // entries per tile chosen on the device (<= 256), see sf_tiles
  // QUAD path: the block is a single level whose fastest axis has extent >= 4
  bool quad = false;
  a->lb[0] = a->lb[1] = a->lb[2] = 0;
  if (t.nlev - 1 - t.driving == 1) {
    const DLevel& B = t.lev[t.nlev - 1];
    for (int d = 0; d < 3; d++) a->lb[d] = B.le[d];
    quad = B.le[t.nd - 1] >= 2;
  }
  // one resident wave: 5 CTAs per SM (__launch_bounds__(SF_TPB, 5)); tiles are
  // sized on the device so every CTA gets an equal share
  int grid = num_sms() * 5;
  (void)grid_hint;
  ChainTab* ct = nullptr;
  if (nphases > 1) {   // one-CTA chain (the caller checked the list is small and the table fits)
    ct = new ChainTab();
    const int tot = chain_phase_end[nphases - 1];
    for (int i = 0; i < tot && i < SG_CHAIN_OPS; i++) ct->ops[i] = chain_ops[i];
    for (int i = 0; i < nphases && i < SG_CHAIN_OPS; i++) ct->phase_end[i] = chain_phase_end[i];
    ct->nphases = nphases;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nd = quad ? t.nd : 0;
  static int pair = -1;
  // measured on B200 (profiles/r01_*): one quad per thread at 6 CTAs/SM beats
  // two quads per thread at 3 CTAs/SM (JAC-XL 2.84 vs 1.75 TB/s)
  if (pair < 0) { const char* e = getenv("SG_SF_PAIR"); pair = e ? atoi(e) != 0 : 0; }
  const bool stencil = a->need_nbr;
  // constant-geometry instantiations for the block shapes of the configs
  int gl = 0;
  if (nd == 3 && a->lb[0] == 3 && a->lb[1] == 3 && a->lb[2] == 3) gl = 1;
  else if (nd == 3 && a->lb[0] == 2 && a->lb[1] == 2 && a->lb[2] == 2) gl = 2;
  else if (nd == 2 && a->lb[0] == 2 && a->lb[1] == 2) gl = 3;
  // dedicated kernel: a lone f32 JACOBI over 8^3 dense blocks with a block table
  // dedicated kernel: a lone f32 JACOBI over 8^3 dense blocks with a block
  // table, or JACOBI fused with the reduction of its output
  const bool jac_red = nops == 2 && ops[0].op == SG_OP_JACOBI && ops[1].op == SG_OP_REDUCE_SUM &&
                       ops[1].f[1] == ops[0].f[0] && ops[1].scalar >= 0;
  if ((nops == 1 || jac_red) && ops[0].op == SG_OP_JACOBI && gl == 1 && !i32 && !t.leaf_bitmasked && nphases <= 1 &&
      drive && drive->table && getenv("SG_NO_JAC8") == nullptr) {
    JacArgs j;
    j.T = t; j.entries = drive->entries; j.count = drive->count; j.table = drive->table; j.table_ctl = drive->ctl;
    const uint64_t fs = 1ull << t.ln_leaf;
    j.s_dst = (uint64_t)ops[0].slot[0] * fs; j.s_src = (uint64_t)ops[0].slot[1] * fs;
    j.s_rhs = (uint64_t)ops[0].slot[2] * fs;
    j.inv = 1.0f / 6.0f;
    j.red_target = jac_red ? c.scalars + ops[1].scalar : nullptr;
    j.partials = c.partials;
    j.red_done = c.red_done;
    // (programmatic dependent launch was measured here: 4.36 vs 4.12 us per
    // launch inside the graph -- slower, so plain launches)
    if (jac_red) k_jacobi8<true><<<num_sms() * 4, 256, 0, s>>>(j);
    else k_jacobi8<false><<<num_sms() * 4, 256, 0, s>>>(j);
    delete a;
    return check_launch();
  }
  // groups of quad ops on 8^3 dense blocks: the streaming kernel (k_jacobi8's
  // structure, no shared-memory tiles) instead of the tile interpreter
  const bool stream8 = stream8_group(t, ops, nops, gl, i32) && drive && drive->table && !ct &&
                       getenv("SG_NO_STREAM8") == nullptr;
  // JIT-specialized kernel of this group's content (jit.cpp);
  // the interpreter runs while it compiles
  if (!ct && !(pair && stencil)) {
    JitGroup G;
    const void* k = jit_group_of(t, ops, nops, G) ? jit_lookup(G) : nullptr;
    if (k) {
      void* args[] = {(void*)a};
      cudaLaunchKernel(k, dim3(G.stream ? num_sms() * 4 : grid), dim3(SF_TPB), args, 0, s);
      delete a;
      return check_launch();
    }
  }
  if (stream8) {
    k_stream8<<<num_sms() * 4, 256, 0, s>>>(*a);
    delete a;
    return check_launch();
  }
#define SG_SF_LAUNCH(V)                                                                           \
  switch (nd * 10 + gl) {                                                                         \
    case 10: sf_dispatch<V, 1, false, 0>(a, grid, s, ct); break;   \
    case 20: sf_dispatch<V, 2, false, 0>(a, grid, s, ct); break;   \
    case 23: sf_dispatch<V, 2, false, 3>(a, grid, s, ct); break;   \
    case 30: if (pair && stencil) sf_dispatch<V, 3, true, 0>(a, grid, s, ct); \
             else sf_dispatch<V, 3, false, 0>(a, grid, s, ct); break;          \
    case 31: sf_dispatch<V, 3, false, 1>(a, grid, s, ct); break;   \
    case 32: sf_dispatch<V, 3, false, 2>(a, grid, s, ct); break;   \
    default: sf_dispatch<V, 0, false, 0>(a, grid, s, ct); break;   \
  }
  if (i32) { SG_SF_LAUNCH(int) } else { SG_SF_LAUNCH(float) }
#undef SG_SF_LAUNCH
  delete a;
  delete ct;
  return check_launch();
}

static bool lb2_tree(const DTree& t) {
  const DLevel& d = t.lev[t.driving];
  return d.lbelow[0] == 2 && d.lbelow[1] == 2 && d.lbelow[2] == 2 && t.lblk == 6;
}

uint32_t bin_ntiles(uint32_t nkeys) { return (nkeys + BIN_TILE - 1) / BIN_TILE; }

int launch_bin(const DBins& b, const float* x, int64_t xs, int64_t n, const int32_t* dcount, float inv_dx,
               void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  BinArgs a;
  a.B = b; a.x = x; a.xs = xs; a.n = n; a.dcount = dcount; a.inv_dx = inv_dx;
  a.ntiles = bin_ntiles(b.nkeys);
  const int gp = (int)std::max<int64_t>(1, std::min<int64_t>((n + BIN_TPB - 1) / BIN_TPB, (int64_t)num_sms() * 8));
  const int gt = (int)std::min<uint32_t>(a.ntiles, (uint32_t)num_sms() * 4);
  // (a shared-memory histogram variant, k_bin_count_smem, measured slower on C4:
  // 14.4 vs 10.0 us -- profiles/r01_launches_c4_t31.csv)
  k_bin_count<<<gp, BIN_TPB, 0, s>>>(a);
  k_bin_tiles<<<gt, BIN_TPB, 0, s>>>(a);
  k_bin_top<<<1, 1024, 0, s>>>(a);
  k_bin_apply<<<gt, BIN_TPB, 0, s>>>(a);
  k_bin_scatter<<<gp, BIN_TPB, 0, s>>>(a);
  return check_launch();
}

int launch_range_for(const DevCtx& c, int64_t n, const int32_t* dcount, const DOp* ops, int nops, int task,
                     void* stream, const RangeScratch* rs, const DTree* grid_tree, const DTree* tree2,
                     const DBins* bins) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (nops == 1 && ops[0].op == SG_OP_PERMUTE) {
    PermArgs m;
    m.C = c; m.op = ops[0]; m.n = n; m.dcount = dcount; m.binned = bins != nullptr;
    if (bins) m.B = *bins;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_permute<<<std::max(grid, 1), 256, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && bins) {   // binned MPM kernels (LB = 2 trees; bins built by the caller)
    MpmBinArgs m;
    m.T = *grid_tree; m.TG = tree2 ? *tree2 : *grid_tree; m.C = c; m.op = ops[0]; m.B = *bins; m.task = task;
    // (bin, chunk) grid: x strides over the non-empty bins, y over a bin's chunks
    const dim3 grid((unsigned)num_sms() * MB_BINS_X, MB_CHUNKS_Y);
    switch (ops[0].op) {
      case SG_OP_P2G: k_p2g_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_G2P: k_g2p_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_G2P_ADJ: k_g2p_adj_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      case SG_OP_P2G_ADJ: k_p2g_adj_bin<<<grid, MB_TPB, 0, s>>>(m); break;
      default: return -1;
    }
    return check_launch();
  }
  if (nops == 1 && (ops[0].op == SG_OP_G2P_ADJ || ops[0].op == SG_OP_P2G_ADJ)) {
    Mpm2Args m;
    m.T = *grid_tree; m.TG = tree2 ? *tree2 : *grid_tree; m.C = c; m.op = ops[0]; m.n = n; m.task = task;
    const bool lb2 = lb2_tree(m.T) && lb2_tree(m.TG);
    int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
    if (ops[0].op == SG_OP_G2P_ADJ) {
      if (lb2) k_g2p_adj<2><<<grid, 128, 0, s>>>(m);
      else k_g2p_adj<0><<<grid, 128, 0, s>>>(m);
    } else {
      if (lb2) k_p2g_adj<2><<<grid, 128, 0, s>>>(m);
      else k_p2g_adj<0><<<grid, 128, 0, s>>>(m);
    }
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_LOSS_MEAN) {
    LossArgs m;
    m.C = c; m.op = ops[0]; m.n = n;
    m.target = c.scalars + (ops[0].scalar >= 0 ? ops[0].scalar : 0);
    int grid = (int)std::min<int64_t>((n + LM_TPB - 1) / LM_TPB, (int64_t)std::min(c.max_grid, num_sms() * 4));
    k_loss_mean<<<std::max(grid, 1), LM_TPB, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && grid_tree && (ops[0].op == SG_OP_P2G || ops[0].op == SG_OP_G2P)) {
    MpmArgs m;
    m.T = *grid_tree; m.C = c; m.op = ops[0]; m.n = n; m.dcount = dcount; m.task = task;
    const bool lb2 = lb2_tree(*grid_tree);
    int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
    if (ops[0].op == SG_OP_P2G) {
      if (lb2) k_p2g<2><<<grid, 128, 0, s>>>(m);
      else k_p2g<0><<<grid, 128, 0, s>>>(m);
    } else {
      if (lb2) k_g2p<2><<<grid, 128, 0, s>>>(m);
      else k_g2p<0><<<grid, 128, 0, s>>>(m);
    }
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_G2P_MIGRATE) {
    MigArgs m;
    m.C = c; m.op = ops[0]; m.status = rs->status; m.ctl = rs->ctl; m.task = task;
    m.T = *grid_tree;
    int grid = (int)std::min<int64_t>((n + MG_TPB - 1) / MG_TPB, (int64_t)num_sms() * 6);
    k_g2p_migrate<<<std::max(grid, 1), MG_TPB, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_MIGRATE_COMPACT) {
    CompactArgs m;
    m.C = c; m.op = ops[0]; m.holes = rs->holes; m.tail = rs->tail; m.cap = rs->hole_cap; m.task = task;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_migrate_mark<<<std::max(grid, 1), 256, 0, s>>>(m);
    k_migrate_fill<<<1, 1024, 0, s>>>(m);
    return check_launch();
  }
  if (nops == 1 && ops[0].op == SG_OP_MIGRATE_APPEND) {
    AppArgs m;
    m.C = c; m.op = ops[0]; m.ctl = rs->ctl + 4;
    int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 4);
    k_migrate_append<<<std::max(grid, 1), 256, 0, s>>>(m);
    return check_launch();
  }
  RFArgs* a = new RFArgs();
  a->C = c; a->n = n; a->dcount = dcount; a->nops = nops; a->task = task;
  for (int o = 0; o < nops; o++) a->ops[o] = ops[o];
  int grid = (int)std::min<int64_t>((n + 127) / 128, (int64_t)num_sms() * 16);
  k_range_for<<<grid, 128, 0, s>>>(*a);
  delete a;
  return check_launch();
}

int launch_serial(const DevCtx& c, const DOp* ops, int nops, int, void* stream) {
  SerArgs* a = new SerArgs();
  a->C = c; a->nops = nops;
  for (int o = 0; o < nops; o++) {
    a->ops[o] = ops[o];
    a->aux[o] = (uint64_t)(c.scalars + (ops[o].scalar >= 0 ? ops[o].scalar : 0));
  }
  k_serial<<<1, 1, 0, (cudaStream_t)stream>>>(*a);
  delete a;
  return check_launch();
}

// DEACTIVATE as a pool reset (reading R33): the deactivated level is the
// tree's first sparse level, so every container of every pool is freed -- zero
// the root container and each pool's allocated containers (free-listed ones are
// already zero), then the last CTA resets the bump counters and free lists.
struct ResetArgs {
  DTree T;
};

__global__ void __launch_bounds__(256) k_deactivate_reset(const __grid_constant__ ResetArgs A) {
  const DTree& T = A.T;
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gsz = (uint64_t)gridDim.x * blockDim.x;
  for (int s = 0; s < T.nseg; s++) {
    const DSeg& S = T.seg[s];
    uint64_t n = 1;
    if (s > 0) {
      const int32_t b = S.alloc[0];
      n = (uint64_t)min((uint32_t)max(b, 0), S.capacity);
    }
    const uint64_t words = n * S.stride;   // containers are 128-byte aligned: stride % 4 == 0
    uint4* p = reinterpret_cast<uint4*>(S.base);
    for (uint64_t i = gtid; i < words / 4; i += gsz) p[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (T.nseg < 2) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&T.seg[1].alloc[2], 1) == (int)gridDim.x - 1) {
      for (int s = 1; s < T.nseg; s++) { T.seg[s].alloc[0] = 0; T.seg[s].alloc[1] = 0; }
      T.seg[1].alloc[2] = 0;
      __threadfence();
    }
  }
}

int launch_deactivate_reset(const DTree& t, void* stream) {
  ResetArgs a;
  a.T = t;
  k_deactivate_reset<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_deactivate(const DevCtx& c, const DTree& t, int, int level, const DList* lists, int, void* stream) {
  DeArgs a;
  a.T = t; a.C = c; a.ls = level;
  a.drive_entries = t.driving >= 0 ? lists[t.driving].entries : nullptr;
  a.drive_count = t.driving >= 0 ? lists[t.driving].count : nullptr;
  for (int l = 0; l < SG_MAXL; l++) {
    bool listed = l < t.nlev && (t.lev[l].kind == SG_POINTER ||
                                 (t.lev[l].kind == SG_BITMASKED && !(l == t.nlev - 1)));
    a.lent[l] = listed ? lists[l].entries : nullptr;
    a.lcnt[l] = listed ? lists[l].count : nullptr;
  }
  k_deactivate<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

static void dense_shifts(const DTree& t, int sh[3]) {
  const DLevel& L = t.lev[t.nlev - 1];
  for (int a = 0; a < 3; a++) sh[a] = L.lres[a];
}

int launch_read_field(const DevCtx&, const DTree& t, int, int slot, uint32_t* dense, void* stream) {
  FieldIO a;
  a.T = t; a.slot = slot; a.dense = dense; a.src = nullptr;
  dense_shifts(t, a.sh);
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_read_field<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_load_field(const DevCtx&, const DTree& t, int, int slot, const uint32_t* dense, void* stream) {
  FieldIO a;
  a.T = t; a.slot = slot; a.dense = nullptr; a.src = dense;
  dense_shifts(t, a.sh);
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_load_field<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_mask_scan(const DevCtx&, const DTree& t, int, int level, uint8_t* flags, void* stream) {
  MaskScan a;
  a.T = t; a.level = level; a.flags = flags;
  for (int d = 0; d < 3; d++) a.sh[d] = t.lev[level].lres[d];
  a.total = 1ll << (a.sh[0] + a.sh[1] + a.sh[2]);
  k_mask_scan<<<num_sms() * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

int launch_list_decode(const DTree& t, int level, const DList& l, int32_t* coords, void* stream) {
  ListDecode a{t, level, l.entries, l.count, coords};
  k_list_decode<<<num_sms() * 4, 256, 0, (cudaStream_t)stream>>>(a);
  return check_launch();
}

}  // namespace sg
