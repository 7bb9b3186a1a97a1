// kernels_lg.cu -- activation and element-list generation kernels (split out of
// kernels.cu so the two translation units compile in parallel).
//
//   k_activate      explicit activation: CAS-published pointer
//                   allocation from a zeroed pool + atomicOr on bitmask words.
//   k_listgen*      element-list generation.
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
//     the copy to the list is ONE bulk shared->global copy (cp.async.bulk,
//     the TMA engine reads shared memory: none of the LSU wavefronts the
//     kernel is bound by) plus element-wise head / tail; staging is double
//     buffered so a sub-tile never waits for the previous one's copy.
// Sub-tiles denser than the staging buffer write their entries straight to
// the list (correct, uncoalesced).
// ---------------------------------------------------------------------------
constexpr int LGW_MIN_HINT = 64;   // CTA tiles (2048 chunks) below which the CTA-tile kernel runs
#ifndef LGW_UNROLL
#define LGW_UNROLL 4   // extraction loop unroll (8 measured slower: 297 vs 287 us)
#endif
constexpr int kLgwUnroll = LGW_UNROLL;
#ifndef LGW_SUBN
#define LGW_SUBN 4   // sub-tiles per warp tile (one look-back per tile)
#endif
#ifndef LGW_TPBN
#define LGW_TPBN 128
#endif
constexpr int LGW_TPB = LGW_TPBN, LGW_WARPS = LGW_TPB / 32, LGW_WPL = 8, LGW_SUBTILE = 32 * LGW_WPL, LGW_SUB = LGW_SUBN,
              LGW_TILE = LGW_SUB * LGW_SUBTILE, LGW_CAP = 1024, LGW_LB = 1;
#ifndef LGW_SLEEP
#define LGW_SLEEP 128   // look-back back-off (ns); 0 / 32 / 512 measured the same on LG-XL
#endif
#ifndef LGW_NBUF
#define LGW_NBUF 1   // staging buffers per warp (2: 5 CTAs/SM by shared memory instead of 8)
#endif

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
#pragma unroll kLgwUnroll
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

// Bulk (TMA-engine) shared -> global copies for the staged list entries:
// 16-byte aligned, size a multiple of 16.  Generic-proxy shared stores are
// made visible to the async proxy by fence.proxy.async before the copy.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"((uint32_t)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(LGW_TPB, 8) k_listgen_warp(const __grid_constant__ LGArgs a) {
  __shared__ __align__(16) uint32_t s_out[LGW_WARPS][LGW_NBUF][LGW_CAP + 4];   // staging
  __shared__ uint2 s_rec[LGW_WARPS][LGW_WPL * 32];   // compacted non-empty words 1..7 per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t epoch = ld_volatile(&a.out.ctl[2]) & 0x3FFFFFFFu;
  const uint32_t nparent = a.mode == 0 ? 1u : *a.pcount;
  const uint64_t nchunks = (uint64_t)nparent << a.lcpp;
  const uint32_t ntiles = (uint32_t)((nchunks + LGW_TILE - 1) / LGW_TILE);
  uint2* rec = s_rec[warp];
  uint32_t buf = 0;
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
        const bool staged = total <= (uint32_t)LGW_CAP;
        uint32_t* so = s_out[warp][buf];
        if (staged && lane == 0) bulk_wait_read<LGW_NBUF - 1>();   // the copy that last read this buffer is done
        __syncwarp();
        if (staged) {
          const uint32_t shift = base & 3u;
          lgw_extract(so + shift + my0, cnt[r], w[r][0].x, hi[r], rec + lane);
          // [base, base + total) <- so[shift, shift + total): the full 16-byte
          // groups by one bulk copy (TMA engine: no LSU wavefronts), the
          // partial head / tail groups element-wise
          fence_proxy_async_smem();
          __syncwarp();
          const uint32_t end = min(base + total, a.out.capacity);
          const uint32_t ga = (base + 3u) & ~3u, gb = end & ~3u;   // full groups: [ga, gb)
          uint32_t* ent = a.out.entries;
          if (ga < gb) {
            if (lane == 0) {
              bulk_s2g(ent + ga, so + shift + (ga - base), (gb - ga) * 4u);
              bulk_commit();
            }
            if (lane < ga - base) ent[base + lane] = so[shift + lane];            // head (< 4)
            if (lane < end - gb) ent[gb + lane] = so[shift + (gb - base) + lane];  // tail (< 4)
          } else if (lane < end - min(base, end)) {
            ent[base + lane] = so[shift + lane];                                   // < 8 entries
          }
          buf = (buf + 1u) % LGW_NBUF;
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
  if (lane == 0) bulk_wait_all();   // staging reads done before the CTA's shared memory goes away
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

}  // namespace sg
