// mpm_bin.cuh -- particle binning and the binned MPM transfer kernels
// ("particles are binned by leaf block once per step
// (counting sort); P2G uses a CTA-per-block smem tile").  Included by
// kernels.cu after mpm_adj.cuh.  Only for trees whose leaf blocks are 4^3
// (LB = 2: C3, C4, C5); other trees use the per-particle kernels.
//
// Binning: key = the leaf block holding the particle's base node
// (base = floor(x / dx - 1/2), the same f32 decision as mpm_bspline), or the
// overflow key nkeys-1 for a block outside the domain.  Counting sort in five
// launches: count (rank within the bin), per-tile sums, top-level scan, apply
// (prefix per key + compact list of non-empty bins; resets the histogram), scatter.
//
// Binned kernels: one CTA per (bin, chunk of MB_TPB particles) pair, so a bin
// of ~500 particles spreads over several CTAs.  The 3x3x3 stencils of a bin's
// particles cover the 6^3 nodes [o, o + 6) (o = block origin), i.e. at most the
// 8 blocks b + {0,1}^3.
//   * scatter ops (P2G, the grid-adjoint scatter of G2P_ADJ): each thread
//     stages its particle's record (weights, fx, coefficients) in its warp's
//     shared-memory slice; then the warp walks its 32 records one particle at a
//     time, lane l < 27 owning node l of the particle's stencil, and adds into a
//     warp-PRIVATE 6^3 tile -- the 27 lanes hit 27 distinct nodes and no other
//     warp writes the tile, so plain load-add-store, no atomics (shared-memory
//     f32 atomics are CAS loops on sm_100a).  The warp tiles are summed per
//     node and flushed with one global atomic add per node and field (a node
//     is shared by <= 8 bins and the chunks of its bin).
//   * gather ops (G2P, P2G_ADJ, the particle part of G2P_ADJ) stage the node
//     tile in shared memory once per CTA and gather from it.
#pragma once

constexpr int BIN_TPB = 256;
constexpr int BIN_TILE = 2048;   // keys per scan tile: 8 per thread
constexpr int MB_TPB = 128;      // binned MPM kernels: threads per CTA = particles per chunk
constexpr int MB_NODES = 216;    // 6^3 tile

// DBins: sg_internal.h

struct BinArgs {
  DBins B;
  const float* x;     // particle positions, SoA (3 comps)
  int64_t xs;         // component stride
  int64_t n;
  const int32_t* dcount;
  float inv_dx;
  uint32_t ntiles;
};

__device__ __forceinline__ uint32_t bin_key_of(const DBins& B, const float* x, int64_t xs, int64_t i, float inv_dx) {
  int b[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const float X = __fmul_rn(x[a * xs + i], inv_dx);
    b[a] = ((int)floorf(__fsub_rn(X, 0.5f))) >> 2;
  }
  if (b[0] < 0 || b[1] < 0 || b[2] < 0 || b[0] >= B.nb[0] || b[1] >= B.nb[1] || b[2] >= B.nb[2]) return B.nkeys - 1;
  return ((uint32_t)b[0] * B.nb[1] + (uint32_t)b[1]) * B.nb[2] + (uint32_t)b[2];
}

// Warp-aggregated: lanes with the same key take one atomic (bin-sorted
// particle arrays put whole warps on one key).
__global__ void __launch_bounds__(BIN_TPB) k_bin_count(const __grid_constant__ BinArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)BIN_TPB; i0 < n; i0 += (int64_t)gridDim.x * BIN_TPB) {
    const int64_t i = i0 + threadIdx.x;
    const bool live = i < n;
    const uint32_t k = live ? bin_key_of(A.B, A.x, A.xs, i, A.inv_dx) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (live && lane == leader) base = atomicAdd(&A.B.hist[k], (uint32_t)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (live) {
      A.B.key[i] = k;
      A.B.rank[i] = base + __popc(peers & ((1u << lane) - 1u));
    }
  }
}

// Small key spaces (C4: 4K blocks): per-CTA shared-memory histogram over a
// contiguous particle range, then one global atomic per (CTA, non-empty key);
// the global atomics on a few hundred hot keys were the count kernel's cost.
constexpr int BIN_SMEM_KEYS = 8192;
__global__ void __launch_bounds__(BIN_TPB) k_bin_count_smem(const __grid_constant__ BinArgs A) {
  __shared__ uint32_t sh[BIN_SMEM_KEYS];
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  for (uint32_t k = threadIdx.x; k < A.B.nkeys; k += BIN_TPB) sh[k] = 0u;
  __syncthreads();
  for (int64_t i = i0 + threadIdx.x; i < i1; i += BIN_TPB) {
    const uint32_t k = bin_key_of(A.B, A.x, A.xs, i, A.inv_dx);
    A.B.key[i] = k;
    A.B.rank[i] = atomicAdd(&sh[k], 1u);
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < A.B.nkeys; k += BIN_TPB) {
    const uint32_t c = sh[k];
    sh[k] = c ? atomicAdd(&A.B.hist[k], c) : 0u;
  }
  __syncthreads();
  for (int64_t i = i0 + threadIdx.x; i < i1; i += BIN_TPB) A.B.rank[i] += sh[A.B.key[i]];
}

__device__ __forceinline__ void block_sum2(uint32_t& a, uint32_t& b) {
  __shared__ uint32_t s[2][BIN_TPB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s[0][w] = a; s[1][w] = b; }
  __syncthreads();
  if (w == 0) {
    a = l < BIN_TPB / 32 ? s[0][l] : 0u;
    b = l < BIN_TPB / 32 ? s[1][l] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(BIN_TPB) k_bin_tiles(const __grid_constant__ BinArgs A) {
  for (uint32_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const uint4* h = (const uint4*)(A.B.hist + (size_t)t * BIN_TILE + threadIdx.x * 8);
    const uint4 u0 = h[0], u1 = h[1];
    uint32_t c = u0.x + u0.y + u0.z + u0.w + u1.x + u1.y + u1.z + u1.w;
    uint32_t z = (u0.x > 0) + (u0.y > 0) + (u0.z > 0) + (u0.w > 0) + (u1.x > 0) + (u1.y > 0) + (u1.z > 0) + (u1.w > 0);
    block_sum2(c, z);
    if (threadIdx.x == 0) { A.B.tsum[2 * t] = c; A.B.tsum[2 * t + 1] = z; }
  }
}

// One CTA of 1024 threads: exclusive scan of the per-tile (count, non-empty) pairs.
__global__ void __launch_bounds__(1024) k_bin_top(const __grid_constant__ BinArgs A) {
  __shared__ uint32_t s[2][32];
  __shared__ uint32_t carry[2];
  if (threadIdx.x == 0) { carry[0] = 0; carry[1] = 0; }
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (uint32_t base = 0; base < A.ntiles; base += 1024) {
    const uint32_t t = base + threadIdx.x;
    const uint32_t c = t < A.ntiles ? A.B.tsum[2 * t] : 0u, z = t < A.ntiles ? A.B.tsum[2 * t + 1] : 0u;
    uint32_t ic = c, iz = z;   // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t pc = __shfl_up_sync(0xffffffffu, ic, o), pz = __shfl_up_sync(0xffffffffu, iz, o);
      if (l >= o) { ic += pc; iz += pz; }
    }
    if (l == 31) { s[0][w] = ic; s[1][w] = iz; }
    __syncthreads();
    if (w == 0) {
      uint32_t vc = s[0][l], vz = s[1][l];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t pc = __shfl_up_sync(0xffffffffu, vc, o), pz = __shfl_up_sync(0xffffffffu, vz, o);
        if (l >= o) { vc += pc; vz += pz; }
      }
      s[0][l] = vc; s[1][l] = vz;
    }
    __syncthreads();
    const uint32_t wc = w ? s[0][w - 1] : 0u, wz = w ? s[1][w - 1] : 0u;
    if (t < A.ntiles) {
      A.B.tsum[2 * t] = carry[0] + wc + ic - c;
      A.B.tsum[2 * t + 1] = carry[1] + wz + iz - z;
    }
    __syncthreads();
    if (threadIdx.x == 1023) { carry[0] += wc + ic; carry[1] += wz + iz; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *A.B.nbins = carry[1];
    A.B.off[A.B.nkeys] = carry[0];
  }
}

__global__ void __launch_bounds__(BIN_TPB) k_bin_apply(const __grid_constant__ BinArgs A) {
  __shared__ uint32_t s[2][BIN_TPB / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (uint32_t t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    const uint32_t k0 = t * BIN_TILE + threadIdx.x * 8;
    uint4* h = (uint4*)(A.B.hist + k0);
    const uint4 u0 = h[0], u1 = h[1];
    const uint32_t v[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
    uint32_t c = 0, z = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) { c += v[j]; z += v[j] > 0; }
    uint32_t ic = c, iz = z;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t pc = __shfl_up_sync(0xffffffffu, ic, o), pz = __shfl_up_sync(0xffffffffu, iz, o);
      if (l >= o) { ic += pc; iz += pz; }
    }
    if (l == 31) { s[0][w] = ic; s[1][w] = iz; }
    __syncthreads();
    uint32_t wc = 0, wz = 0;
    for (int j = 0; j < w; j++) { wc += s[0][j]; wz += s[1][j]; }
    uint32_t pc = A.B.tsum[2 * t] + wc + ic - c, pz = A.B.tsum[2 * t + 1] + wz + iz - z;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint32_t k = k0 + j;
      if (k < A.B.nkeys) {
        A.B.off[k] = pc;
        if (v[j]) A.B.bins[pz++] = k;
      }
      pc += v[j];
    }
    h[0] = make_uint4(0, 0, 0, 0);
    h[1] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(BIN_TPB) k_bin_scatter(const __grid_constant__ BinArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  for (int64_t i = blockIdx.x * (int64_t)BIN_TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * BIN_TPB)
    A.B.perm[A.B.off[A.B.key[i]] + A.B.rank[i]] = (uint32_t)i;
}

// ---------------------------------------------------------------------------
// Binned kernels
// ---------------------------------------------------------------------------
constexpr int MB_WARPS = MB_TPB / 32;
constexpr int MB_CHUNKS_Y = 4;   // gridDim.y: chunk slots per bin (grid-strided)
constexpr int MB_BINS_X = 6;     // gridDim.x = MB_BINS_X x SMs: bin slots (grid-strided)

struct MpmBinArgs {
  DTree T;      // grid tree (P2G target / G2P source / G2P_ADJ forward grid)
  DTree TG;     // adjoint tree (G2P_ADJ scatter target, P2G_ADJ source)
  DevCtx C;
  DOp op;
  DBins B;
  int task;
};

// Per-particle fallbacks for the overflow bin (particles whose block lies
// outside the domain), kept out of line so they do not inflate the binned
// kernels' register allocation.
__device__ __noinline__ void p2g_one(const DevCtx& C, const DTree& T, const DOp& op, int64_t i, int task) {
  mpm_p2g<2>(C, T, op, i, task);
}
__device__ __noinline__ void g2p_one(const DevCtx& C, const DTree& T, const DOp& op, int64_t i, int64_t io) {
  mpm_g2p<2>(C, T, op, i, io);
}
__device__ __noinline__ void g2p_adj_one(const DevCtx& C, const DTree& T, const DTree& TG, const DOp& op, int64_t i,
                                         int task) {
  mpm_g2p_adj<2>(C, T, TG, op, i, task);
}
__device__ __noinline__ void p2g_adj_one(const DevCtx& C, const DTree& T, const DOp& op, int64_t i, int task) {
  mpm_p2g_adj<2>(C, T, op, i, task);
}

// Bin geometry: node origin of key k.
__device__ __forceinline__ void bin_origin(const DBins& B, uint32_t k, int o[3]) {
  const uint32_t bz = k % B.nb[2], r = k / B.nb[2];
  o[0] = (int)(r / B.nb[1]) << 2;
  o[1] = (int)(r % B.nb[1]) << 2;
  o[2] = (int)bz << 2;
}

// Offsets of the bin's 8 blocks (bit t of `need`: block o/4 + (t>>2, (t>>1)&1, t&1)).
template <bool ACTIVATE>
__device__ __forceinline__ void bin_blocks(const DevCtx& C, const DTree& T, const int o[3], uint32_t need,
                                           uint32_t* s_off, int task) {
  if (threadIdx.x < 8) {
    const int t = threadIdx.x;
    uint32_t off = SG_NO_BLOCK;
    if ((need >> t) & 1u) {
      int q[3] = {o[0] + ((t >> 2) << 2), o[1] + (((t >> 1) & 1) << 2), o[2] + ((t & 1) << 2)};
      if (in_domain(T, q)) {
        uint32_t idx;
        uint32_t* cont = ACTIVATE ? activate_walk(C, T, q, idx, task) : locate(T, q, idx);
        const uint32_t blkmask = ~((1u << T.lblk) - 1u);
        if (cont) off = (uint32_t)(cont - T.seg[T.nseg - 1].base) + T.payload_off + (idx & blkmask);
      }
    }
    s_off[t] = off;
  }
}

__device__ __forceinline__ uint32_t tile_node_off(const uint32_t* s_off, int q) {
  const int ni = q / 36, nj = (q / 6) % 6, nk = q % 6;
  const uint32_t b = s_off[((ni >> 2) << 2) | ((nj >> 2) << 1) | (nk >> 2)];
  if (b == SG_NO_BLOCK) return SG_NO_BLOCK;
  return b + (((uint32_t)(ni & 3) << 4) | ((uint32_t)(nj & 3) << 2) | (uint32_t)(nk & 3));
}

// 8-block need mask of a particle whose base is r (0..3 per axis) in its bin.
__device__ __forceinline__ uint32_t need_mask(const int r[3]) {
  uint32_t m = 0;
  const int h0 = r[0] >= 2, h1 = r[1] >= 2, h2 = r[2] >= 2;
#pragma unroll
  for (int t = 0; t < 8; t++) {
    const int ix = t >> 2, iy = (t >> 1) & 1, iz = t & 1;
    if ((!ix || h0) && (!iy || h1) && (!iz || h2)) m |= 1u << t;
  }
  return m;
}

// Stage a 6^3 tile of nf fields from the tree (absent blocks read 0).
__device__ __forceinline__ void stage_tile(const DTree& T, const DOp& op, int slot0, int nf, const uint32_t* s_off,
                                           float (*s_tile)[MB_NODES]) {
  const uint32_t* pool = T.seg[T.nseg - 1].base;
  const uint64_t fs = 1ull << T.ln_leaf;
  for (int q = threadIdx.x; q < MB_NODES; q += MB_TPB) {
    const uint32_t off = tile_node_off(s_off, q);
    for (int f = 0; f < nf; f++)
      s_tile[f][q] = off == SG_NO_BLOCK ? 0.0f : __uint_as_float(pool[(uint64_t)op.slot[slot0 + f] * fs + off]);
  }
}

// Warp-private scatter tiles + per-warp particle records.
//   rec: w[3][3] (9), fx (3), coefficient vector q (12), base offset in the tile (as float bits)
constexpr int MB_REC = 25;
// Scatter tiles use padded strides (node (i, j, k) at i*43 + j*7 + k): the 27
// stencil offsets a*43 + b*7 + c (a, b, c < 3) fall in 27 distinct banks, so a
// warp's 27 lanes update their nodes without shared-memory bank conflicts
// (the dense 6x6x6 layout put 2 lanes on one bank for 9 of the offsets).
constexpr int MB_SI = 43, MB_SJ = 7, MB_TP = 6 * MB_SI;
__device__ __forceinline__ int tile_pad(int q) { return (q / 36) * MB_SI + ((q / 6) % 6) * MB_SJ + q % 6; }
struct MbScatter {
  float tile[MB_WARPS][4][MB_TP];
  float rec[MB_WARPS][MB_REC][32];
  uint32_t need;
  uint32_t off[8];
};

__device__ __forceinline__ void zero_tiles(MbScatter& S, int nf) {
  for (int k = threadIdx.x; k < MB_WARPS * 4 * MB_TP; k += MB_TPB) {
    const int f = (k / MB_TP) & 3;
    if (f < nf) (&S.tile[0][0][0])[k] = 0.0f;
  }
}

__device__ __forceinline__ void put_record(MbScatter& S, const MpmKernel& k, const int r[3], const float q[12]) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int o = 0; o < 3; o++)
#pragma unroll
    for (int a = 0; a < 3; a++) S.rec[w][o * 3 + a][l] = k.w[o][a];
#pragma unroll
  for (int a = 0; a < 3; a++) S.rec[w][9 + a][l] = k.fx[a];
#pragma unroll
  for (int j = 0; j < 12; j++) S.rec[w][12 + j][l] = q[j];
  S.rec[w][24][l] = __int_as_float(r[0] * MB_SI + r[1] * MB_SJ + r[2]);
}

// Warp walk over its `m` records: lane l < 27 adds, for node l = (a, b, c) of
// each particle's stencil, y_r = W (q_r + s4q * sum_d q[3+3r+d] dpos_d) for
// r < 3 and y_3 = W * c3 (when nf == 4) into the warp's private tile.
__device__ __forceinline__ void warp_scatter(MbScatter& S, int m, float dx, float s4q, float c3, int nf) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l >= 27) return;
  const int a = l / 9, b = (l / 3) % 3, c = l % 3;
  const int dq = a * MB_SI + b * MB_SJ + c;
  float* t0 = S.tile[w][0];
  float* t1 = S.tile[w][1];
  float* t2 = S.tile[w][2];
  float* t3 = S.tile[w][3];
  for (int p = 0; p < m; p++) {
    const float (*R)[32] = S.rec[w];
    const float W = R[a * 3 + 0][p] * R[b * 3 + 1][p] * R[c * 3 + 2][p];
    const float d0 = ((float)a - R[9][p]) * dx, d1 = ((float)b - R[10][p]) * dx, d2 = ((float)c - R[11][p]) * dx;
    const int nq = __float_as_int(R[24][p]) + dq;
    t0[nq] += W * (R[12][p] + s4q * (R[15][p] * d0 + R[16][p] * d1 + R[17][p] * d2));
    t1[nq] += W * (R[13][p] + s4q * (R[18][p] * d0 + R[19][p] * d1 + R[20][p] * d2));
    t2[nq] += W * (R[14][p] + s4q * (R[21][p] * d0 + R[22][p] * d1 + R[23][p] * d2));
    if (nf == 4) t3[nq] += W * c3;
  }
}

__device__ __forceinline__ float tile_sum(const MbScatter& S, int f, int q) {
  float v = 0.0f;
  const int pq = tile_pad(q);
#pragma unroll
  for (int w = 0; w < MB_WARPS; w++) v += S.tile[w][f][pq];
  return v;
}

#define MB_FOR_CHUNKS                                                                       \
  const uint32_t nbins = *A.B.nbins;                                                        \
  for (uint32_t j = blockIdx.x; j < nbins; j += gridDim.x)                                  \
    for (uint32_t c0 = blockIdx.y * MB_TPB, key = A.B.bins[j], start = A.B.off[key],        \
                  cnt = A.B.off[key + 1] - start;                                           \
         c0 < cnt; c0 += gridDim.y * MB_TPB)

// P2G, binned (op as mpm_p2g; LB = 2).
//
// Record of one particle (P2G_REC floats, record-major, 16-byte aligned): the
// affine momentum folded so a stencil node at offset (a, b, c) from the base
// needs no dpos arithmetic:  mom_r(a,b,c) = b_r + A'_r . (a, b, c), with
// A' = dx * (p_mass C - dt 4 E p_vol (J-1) / dx^2 I) and
// b_r = p_mass v_r - A'_r . fx   (dpos_d = (off_d - fx_d) dx).
//   [0..3] b0 b1 b2 p_mass   [4..7] A'00 A'01 A'02 A'10   [8..11] A'11 A'12 A'20 A'21
//   [12..15] A'22 tile-base (int bits) - -   [16..24] wx0..2 wy0..2 wz0..2
// The warp's 27 lanes read [0..15] as four broadcast 16-byte loads and their
// three weights (distinct banks), then update their node of the warp-private
// tile: ~34 instructions per (particle, node) pair.
constexpr int P2G_REC = 28;
struct MbP2G {
  float tile[MB_WARPS][4][MB_TP];
  float rec[MB_WARPS][32][P2G_REC];
  uint32_t need;
  uint32_t off[8];
};

#ifndef MB_P2G_MINB
#define MB_P2G_MINB 6   // CTAs per SM the P2G register budget is sized for (4: 122 registers, C3 P2G 158 us; 6: 80, 144 us; 8: 148 us)
#endif
__global__ void __launch_bounds__(MB_TPB, MB_P2G_MINB) k_p2g_bin(const __grid_constant__ MpmBinArgs A) {
  __shared__ __align__(16) MbP2G S;
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DTree& T = A.T;
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]];
  const float* x = (const float*)X.ptr;
  const float* v = (const float*)Vv.ptr;
  const float* cm = (const float*)Cm.ptr;
  const float* jj = (const float*)Jj.ptr;
  const float dt = op.p[0], inv_dx = op.p[1], pm = op.p[2], pv = op.p[3], E = op.p[4];
  const float dx = 1.0f / inv_dx;
  uint32_t* pool = T.seg[T.nseg - 1].base;
  const uint64_t fs = 1ull << T.ln_leaf;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // this lane's stencil node (lanes 27..31 idle in the walk)
  const int la = l / 9, lb = (l / 3) % 3, lc = l % 3;
  const float fa = (float)la, fb = (float)lb, fc = (float)lc;
  const int dq = la * MB_SI + lb * MB_SJ + lc;
  MB_FOR_CHUNKS {
    const int m = (int)min((uint32_t)MB_TPB, cnt - c0);
    if (key == A.B.nkeys - 1) {   // outside the domain: per-particle path
      if ((int)threadIdx.x < m) p2g_one(C, T, op, A.B.perm[start + c0 + threadIdx.x], A.task);
      continue;
    }
    int o[3];
    bin_origin(A.B, key, o);
    // the particle records first (their global loads overlap the tile
    // zeroing and the barrier; a warp's record slice is its own, consumed by
    // its own walk of the previous chunk before that chunk's last barrier)
    uint32_t need = 0;
    if ((int)threadIdx.x < m) {
      const int64_t i = A.B.perm[start + c0 + threadIdx.x];
      const float xp[3] = {x[i], x[X.n + i], x[2 * X.n + i]};
      const MpmKernel k = mpm_bspline(xp, inv_dx);
      const int r[3] = {k.base[0] - o[0], k.base[1] - o[1], k.base[2] - o[2]};
      need = need_mask(r);
      const float stress = -dt * 4.0f * E * pv * (jj[i] - 1.0f) * inv_dx * inv_dx;
      float* R = S.rec[w][l];
      float Ap[3][3], b[3];
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
#pragma unroll
        for (int c = 0; c < 3; c++) Ap[rr][c] = (pm * cm[(3 * rr + c) * Cm.n + i] + (rr == c ? stress : 0.0f)) * dx;
        b[rr] = pm * v[rr * Vv.n + i] - (Ap[rr][0] * k.fx[0] + Ap[rr][1] * k.fx[1] + Ap[rr][2] * k.fx[2]);
      }
      *reinterpret_cast<float4*>(R + 0) = make_float4(b[0], b[1], b[2], pm);
      *reinterpret_cast<float4*>(R + 4) = make_float4(Ap[0][0], Ap[0][1], Ap[0][2], Ap[1][0]);
      *reinterpret_cast<float4*>(R + 8) = make_float4(Ap[1][1], Ap[1][2], Ap[2][0], Ap[2][1]);
      *reinterpret_cast<float4*>(R + 12) =
          make_float4(Ap[2][2], __int_as_float(r[0] * MB_SI + r[1] * MB_SJ + r[2]), 0.0f, 0.0f);
#pragma unroll
      for (int oo = 0; oo < 3; oo++)
#pragma unroll
        for (int a = 0; a < 3; a++) R[16 + 3 * a + oo] = k.w[oo][a];
    }
    if (threadIdx.x == 0) S.need = 0;
    for (int k = threadIdx.x; k < MB_WARPS * 4 * MB_TP; k += MB_TPB) (&S.tile[0][0][0])[k] = 0.0f;
    __syncthreads();
    need = __reduce_or_sync(0xffffffffu, need);
    if (l == 0 && need) atomicOr(&S.need, need);
    __syncwarp();
    {
      const int mw = min(32, max(0, m - (int)(threadIdx.x & ~31u)));
      if (l < 27) {
        float* t0 = S.tile[w][0];
        float* t1 = S.tile[w][1];
        float* t2 = S.tile[w][2];
        float* t3 = S.tile[w][3];
        for (int p = 0; p < mw; p++) {
          const float* R = S.rec[w][p];
          const float4 r0 = *reinterpret_cast<const float4*>(R + 0);
          const float4 r1 = *reinterpret_cast<const float4*>(R + 4);
          const float4 r2 = *reinterpret_cast<const float4*>(R + 8);
          const float4 r3 = *reinterpret_cast<const float4*>(R + 12);
          const float W = R[16 + la] * R[19 + lb] * R[22 + lc];
          const int nq = __float_as_int(r3.y) + dq;
          const float m0 = r0.x + r1.x * fa + r1.y * fb + r1.z * fc;
          const float m1 = r0.y + r1.w * fa + r2.x * fb + r2.y * fc;
          const float m2 = r0.z + r2.z * fa + r2.w * fb + r3.x * fc;
          t0[nq] += W * m0;
          t1[nq] += W * m1;
          t2[nq] += W * m2;
          t3[nq] += W * r0.w;
        }
      }
    }
    __syncthreads();
    if (op.act) bin_blocks<true>(C, T, o, S.need, S.off, A.task);
    else bin_blocks<false>(C, T, o, S.need, S.off, A.task);
    __syncthreads();
    for (int q = threadIdx.x; q < MB_NODES; q += MB_TPB) {
      const int pq = tile_pad(q);
      float y[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int ww = 0; ww < MB_WARPS; ww++)
#pragma unroll
        for (int f = 0; f < 4; f++) y[f] += S.tile[ww][f][pq];
      if (y[3] == 0.0f) continue;
      const uint32_t off = tile_node_off(S.off, q);
      if (off == SG_NO_BLOCK) {
        if (C.debug) set_err(C, op.act ? SG_ERR_RANGE : SG_ERR_DEMOTION_TRAP, A.task);
        continue;
      }
#pragma unroll
      for (int r = 0; r < 3; r++)
        if (y[r] != 0.0f) atomicAdd((float*)(pool + (uint64_t)op.slot[r] * fs) + off, y[r]);
      atomicAdd((float*)(pool + (uint64_t)op.slot[3] * fs) + off, y[3]);
    }
    __syncthreads();
  }
}

// G2P, binned: the chunk's 6^3 x 3 velocity tile is staged in shared memory.
#ifndef MB_G2P_MINB
#define MB_G2P_MINB 6
#endif
__global__ void __launch_bounds__(MB_TPB, MB_G2P_MINB) k_g2p_bin(const __grid_constant__ MpmBinArgs A) {
  __shared__ float s_u[3][MB_NODES];
  __shared__ uint32_t s_off[8];
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DTree& T = A.T;
  const int oo = op.a[4] >= 0 ? 4 : 0;
  const DArray X = C.arrays[op.a[0]], Jj = C.arrays[op.a[3]];
  const DArray Xo = C.arrays[op.a[oo]], Vo = C.arrays[op.a[oo + 1]], Co = C.arrays[op.a[oo + 2]],
               Jo = C.arrays[op.a[oo + 3]];
  const float* x = (const float*)X.ptr;
  const float* jin = (const float*)Jj.ptr;
  float* xo = (float*)Xo.ptr;
  float* vo = (float*)Vo.ptr;
  float* co = (float*)Co.ptr;
  float* jo = (float*)Jo.ptr;
  const float dt = op.p[0], inv_dx = op.p[1];
  const float dx = 1.0f / inv_dx, s4 = 4.0f * inv_dx * inv_dx;
  // out of place with p2 != 0: the output state is written in BIN ORDER (the
  // particle at bin position j goes to index j), so the next step's binned
  // kernels read it nearly sequentially; SG_OP_PERMUTE moves the other
  // particle arrays (ids) the same way
  const bool bin_order = oo == 4 && op.p[2] != 0.0f;
  MB_FOR_CHUNKS {
    const int m = (int)min((uint32_t)MB_TPB, cnt - c0);
    if (key == A.B.nkeys - 1) {
      if ((int)threadIdx.x < m) {
        const uint32_t j = start + c0 + threadIdx.x;
        g2p_one(C, T, op, A.B.perm[j], bin_order ? (int64_t)j : (int64_t)A.B.perm[j]);
      }
      continue;
    }
    int o[3];
    bin_origin(A.B, key, o);
    // the particle's loads and weights first: they overlap the block lookups,
    // the tile staging and its barriers
    const bool act = (int)threadIdx.x < m;
    int64_t i = 0;
    float xp[3] = {0.0f, 0.0f, 0.0f}, J = 0.0f;
    if (act) {
      i = A.B.perm[start + c0 + threadIdx.x];
      xp[0] = x[i]; xp[1] = x[X.n + i]; xp[2] = x[2 * X.n + i];
      J = jin[i];
    }
    const MpmKernel k = mpm_bspline(xp, inv_dx);
    bin_blocks<false>(C, T, o, 0xffu, s_off, A.task);
    __syncthreads();
    stage_tile(T, op, 0, 3, s_off, s_u);
    __syncthreads();
    if (act) {
      const int64_t io = bin_order ? (int64_t)(start + c0 + threadIdx.x) : i;
      const int r[3] = {k.base[0] - o[0], k.base[1] - o[1], k.base[2] - o[2]};
      // APIC: C = 4/dx^2 sum w g dpos^T with dpos = (node - fx) dx; the
      // per-axis offsets (a - fx_d) are hoisted and the constant s4 dx applied
      // once at the end (reassociation only: within R29's 1e-5 bound)
      float nv[3] = {0.0f, 0.0f, 0.0f}, nC[3][3] = {{0.0f}};
      float q[3][3];
#pragma unroll
      for (int d = 0; d < 3; d++)
#pragma unroll
        for (int a = 0; a < 3; a++) q[d][a] = (float)a - k.fx[d];
      const int nq0 = (r[0] * 6 + r[1]) * 6 + r[2];
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) {
          const float wab = k.w[a][0] * k.w[b][1];
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const int nq = nq0 + (a * 6 + b) * 6 + c;
            const float wgt = wab * k.w[c][2];
#pragma unroll
            for (int rr = 0; rr < 3; rr++) {
              const float wg = wgt * s_u[rr][nq];
              nv[rr] += wg;
              nC[rr][0] += wg * q[0][a];
              nC[rr][1] += wg * q[1][b];
              nC[rr][2] += wg * q[2][c];
            }
          }
        }
      const float sc = s4 * dx;
#pragma unroll
      for (int rr = 0; rr < 3; rr++)
#pragma unroll
        for (int d = 0; d < 3; d++) nC[rr][d] *= sc;
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
        vo[rr * Vo.n + io] = nv[rr];
        xo[rr * Xo.n + io] = xp[rr] + dt * nv[rr];
#pragma unroll
        for (int d = 0; d < 3; d++) co[(3 * rr + d) * Co.n + io] = nC[rr][d];
      }
      jo[io] = J * (1.0f + dt * (nC[0][0] + nC[1][1] + nC[2][2]));
    }
    __syncthreads();
  }
}

// PERMUTE: dst[c][j] = src[c][perm[j]] for every component -- the bin order of
// the positions a0 (the same binning G2P used), 16-byte stores where the
// arrays allow.  Unbinned grids (SG_NO_BIN, other leaf shapes) copy in place
// order, matching the unbinned G2P.
struct PermArgs {
  DevCtx C;
  DOp op;
  DBins B;
  int64_t n;
  const int32_t* dcount;
  int binned;
};

__global__ void __launch_bounds__(256) k_permute(const __grid_constant__ PermArgs A) {
  const DArray S = A.C.arrays[A.op.a[1]], D = A.C.arrays[A.op.a[2]];
  const uint32_t* src = (const uint32_t*)S.ptr;
  uint32_t* dst = (uint32_t*)D.ptr;
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  const int nc = S.ncomp < D.ncomp ? S.ncomp : D.ncomp;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = A.binned ? (int64_t)A.B.perm[j] : j;
    for (int c = 0; c < nc; c++) dst[c * D.n + j] = src[c * S.n + i];
  }
}

// G2P_ADJ, binned.  Tile: forward grid momentum p (3) and mass m from T, turned
// into the recomputed velocity u, the wall mask and p/m per node.  Particle
// pass (gather): tr C', the x and J adjoints, and the record (v_hat, C_hat);
// warp scatter of g_bar = W (v_hat + s4 C_hat dpos); per node p_bar = (mask
// g_bar)/m and m_bar = -sum_r p_bar_r p_r/m flushed into TG (activating).
struct MbAdj {
  MbScatter S;
  float u[3][MB_NODES];
  float pm[3][MB_NODES];   // p/m (0 where m == 0)
  float m[MB_NODES];
  uint8_t mask[MB_NODES];
  uint32_t offg[8];
};

__global__ void __launch_bounds__(MB_TPB, 3) k_g2p_adj_bin(const __grid_constant__ MpmBinArgs A) {
  __shared__ MbAdj Z;
  MbScatter& S = Z.S;
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DTree& T = A.T;
  const DTree& TG = A.TG;
  const DArray X = C.arrays[op.a[0]];
  const int64_t nx = X.n;
  const float* x = (const float*)X.ptr;
  const float* jj = arr_f(C, op.a[1]);
  const float *xb1 = arr_f(C, op.a[2]), *vb1 = arr_f(C, op.a[3]), *cb1 = arr_f(C, op.a[4]), *jb1 = arr_f(C, op.a[5]);
  const int64_t n1x = C.arrays[op.a[2]].n, n1v = C.arrays[op.a[3]].n, n1c = C.arrays[op.a[4]].n;
  float* xb0 = (float*)C.arrays[op.a[6]].ptr;
  float* jb0 = (float*)C.arrays[op.a[7]].ptr;
  const int64_t n0x = C.arrays[op.a[6]].n;
  const float dt = op.p[0], inv_dx = op.p[1], grav = op.p[2], bound = op.p[3], ng = op.p[4];
  const float dx = 1.0f / inv_dx, s4 = 4.0f * inv_dx * inv_dx;
  uint32_t* poolg = TG.seg[TG.nseg - 1].base;
  const uint64_t fsg = 1ull << TG.ln_leaf;
  MB_FOR_CHUNKS {
    const int m = (int)min((uint32_t)MB_TPB, cnt - c0);
    if (key == A.B.nkeys - 1) {
      if ((int)threadIdx.x < m) g2p_adj_one(C, T, TG, op, A.B.perm[start + c0 + threadIdx.x], A.task);
      continue;
    }
    int o[3];
    bin_origin(A.B, key, o);
    // the particle's loads first (adjoint seeds of state s+1 and its state
    // s): they overlap the block lookups, the tile staging and its barriers
    const bool act = (int)threadIdx.x < m;
    int64_t i = 0;
    float xp[3] = {0.0f, 0.0f, 0.0f}, J = 1.0f, Jb1 = 0.0f, q[12], xb[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int t = 0; t < 12; t++) q[t] = 0.0f;
    if (act) {
      i = A.B.perm[start + c0 + threadIdx.x];
      xp[0] = x[i]; xp[1] = x[nx + i]; xp[2] = x[2 * nx + i];
      J = jj[i];
      Jb1 = jb1[i];
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
        xb[rr] = xb1[rr * n1x + i];
        q[rr] = vb1[rr * n1v + i] + dt * xb[rr];
#pragma unroll
        for (int d = 0; d < 3; d++) q[3 + 3 * rr + d] = cb1[(3 * rr + d) * n1c + i] + (rr == d ? Jb1 * J * dt : 0.0f);
      }
    }
    if (threadIdx.x == 0) S.need = 0;
    bin_blocks<false>(C, T, o, 0xffu, S.off, A.task);
    zero_tiles(S, 3);
    __syncthreads();
    {
      const uint32_t* pool = T.seg[T.nseg - 1].base;
      const uint64_t fs = 1ull << T.ln_leaf;
      for (int q = threadIdx.x; q < MB_NODES; q += MB_TPB) {
        const uint32_t off = tile_node_off(S.off, q);
        float p[3], mm = 0.0f;
#pragma unroll
        for (int r = 0; r < 3; r++)
          p[r] = off == SG_NO_BLOCK ? 0.0f : __uint_as_float(pool[(uint64_t)op.slot[r] * fs + off]);
        if (off != SG_NO_BLOCK) mm = __uint_as_float(pool[(uint64_t)op.slot[3] * fs + off]);
        const int node[3] = {o[0] + q / 36, o[1] + (q / 6) % 6, o[2] + q % 6};
        float u[3];
        uint8_t mk = 0;
#pragma unroll
        for (int r = 0; r < 3; r++) u[r] = mm > 0.0f ? p[r] / mm : p[r];
        u[1] -= dt * grav;
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const bool z = ((float)node[r] < bound && u[r] < 0.0f) || ((float)node[r] > ng - bound && u[r] > 0.0f);
          if (z) u[r] = 0.0f;
          else mk |= (uint8_t)(1u << r);
          Z.u[r][q] = u[r];
          Z.pm[r][q] = mm > 0.0f ? p[r] / mm : 0.0f;
        }
        Z.m[q] = mm;
        Z.mask[q] = mk;
      }
    }
    __syncthreads();
    uint32_t need = 0;
    if (act) {
      const MpmKernel k = mpm_bspline(xp, inv_dx);
      float dw[3][3];
      mpm_dw(k, dw);
      const int r[3] = {k.base[0] - o[0], k.base[1] - o[1], k.base[2] - o[2]};
      need = need_mask(r);
      float trC = 0.0f;
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const int nq = ((r[0] + a) * 6 + (r[1] + b)) * 6 + (r[2] + c);
            const float u[3] = {Z.u[0][nq], Z.u[1][nq], Z.u[2][nq]};
            const float W = k.w[a][0] * k.w[b][1] * k.w[c][2];
            const float gW[3] = {inv_dx * dw[a][0] * k.w[b][1] * k.w[c][2], inv_dx * k.w[a][0] * dw[b][1] * k.w[c][2],
                                 inv_dx * k.w[a][0] * k.w[b][1] * dw[c][2]};
            const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
            trC += s4 * W * (u[0] * dpos[0] + u[1] * dpos[1] + u[2] * dpos[2]);
            float Wbar = 0.0f, dposbar[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int rr = 0; rr < 3; rr++) {
              const float ct = q[3 + 3 * rr] * dpos[0] + q[4 + 3 * rr] * dpos[1] + q[5 + 3 * rr] * dpos[2];
              Wbar += u[rr] * (q[rr] + s4 * ct);
#pragma unroll
              for (int d = 0; d < 3; d++) dposbar[d] += s4 * W * q[3 + 3 * rr + d] * u[rr];
            }
#pragma unroll
            for (int d = 0; d < 3; d++) xb[d] += Wbar * gW[d] - dposbar[d];
          }
#pragma unroll
      for (int d = 0; d < 3; d++) xb0[d * n0x + i] = xb[d];
      jb0[i] = Jb1 * (1.0f + dt * trC);
      put_record(S, k, r, q);
    }
    need = __reduce_or_sync(0xffffffffu, need);
    if ((threadIdx.x & 31) == 0 && need) atomicOr(&S.need, need);
    __syncwarp();
    warp_scatter(S, min(32, max(0, m - (int)(threadIdx.x & ~31u))), dx, s4, 0.0f, 3);
    __syncthreads();
    if (op.act) bin_blocks<true>(C, TG, o, S.need, Z.offg, A.task);
    else bin_blocks<false>(C, TG, o, S.need, Z.offg, A.task);
    __syncthreads();
    for (int q = threadIdx.x; q < MB_NODES; q += MB_TPB) {
      const float g[3] = {tile_sum(S, 0, q), tile_sum(S, 1, q), tile_sum(S, 2, q)};
      if (g[0] == 0.0f && g[1] == 0.0f && g[2] == 0.0f) continue;
      const uint32_t og = tile_node_off(Z.offg, q);
      if (og == SG_NO_BLOCK) {
        if (C.debug) set_err(C, op.act ? SG_ERR_RANGE : SG_ERR_DEMOTION_TRAP, A.task);
        continue;
      }
      const float mm = Z.m[q];
      float mb = 0.0f;
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const float ub = ((Z.mask[q] >> r) & 1) ? g[r] : 0.0f;
        const float pb = mm > 0.0f ? ub / mm : ub;
        if (mm > 0.0f) mb -= pb * Z.pm[r][q];
        if (pb != 0.0f) atomicAdd((float*)(poolg + (uint64_t)op.slot[4 + r] * fsg) + og, pb);
      }
      if (mb != 0.0f) atomicAdd((float*)(poolg + (uint64_t)op.slot[7] * fsg) + og, mb);
    }
    __syncthreads();
  }
}

// P2G_ADJ, binned: the adjoint tile (p_bar 3, m_bar) is staged per CTA.
__global__ void __launch_bounds__(MB_TPB, 4) k_p2g_adj_bin(const __grid_constant__ MpmBinArgs A) {
  __shared__ float s_g[4][MB_NODES];
  __shared__ uint32_t s_off[8];
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DTree& T = A.T;   // the adjoint tree (fields f0..f3)
  const DArray X = C.arrays[op.a[0]];
  const int64_t nx = X.n, nv = C.arrays[op.a[1]].n, nc = C.arrays[op.a[2]].n;
  const float* x = (const float*)X.ptr;
  const float *v = arr_f(C, op.a[1]), *cm = arr_f(C, op.a[2]), *jj = arr_f(C, op.a[3]);
  float* xb = (float*)C.arrays[op.a[4]].ptr;
  float* vb = (float*)C.arrays[op.a[5]].ptr;
  float* cb = (float*)C.arrays[op.a[6]].ptr;
  float* jb = (float*)C.arrays[op.a[7]].ptr;
  const int64_t nxb = C.arrays[op.a[4]].n, nvb = C.arrays[op.a[5]].n, ncb = C.arrays[op.a[6]].n;
  const float dt = op.p[0], inv_dx = op.p[1], pm = op.p[2], pv = op.p[3], E = op.p[4];
  const float dx = 1.0f / inv_dx;
  const float kJ = -dt * 4.0f * E * pv * inv_dx * inv_dx;
  MB_FOR_CHUNKS {
    const int m = (int)min((uint32_t)MB_TPB, cnt - c0);
    if (key == A.B.nkeys - 1) {
      if ((int)threadIdx.x < m) p2g_adj_one(C, T, op, A.B.perm[start + c0 + threadIdx.x], A.task);
      continue;
    }
    int o[3];
    bin_origin(A.B, key, o);
    // the particle's state loads first: they overlap the block lookups, the
    // tile staging and its barriers (as k_g2p_bin)
    const bool act = (int)threadIdx.x < m;
    int64_t i = 0;
    float xp[3] = {0.0f, 0.0f, 0.0f}, J = 1.0f, vv[3] = {0.0f, 0.0f, 0.0f}, Am[3][3];
    float xb0[3] = {0.0f, 0.0f, 0.0f}, jb0 = 0.0f;   // the adjoints this kernel accumulates into
    if (act) {
      i = A.B.perm[start + c0 + threadIdx.x];
      xp[0] = x[i]; xp[1] = x[nx + i]; xp[2] = x[2 * nx + i];
      J = jj[i];
#pragma unroll
      for (int rr = 0; rr < 3; rr++) vv[rr] = v[rr * nv + i];
      // read now, added at the end (ncu: the end-of-kernel read-modify-write
      // of x-bar and J-bar was half of the stall samples)
#pragma unroll
      for (int d = 0; d < 3; d++) xb0[d] = xb[d * nxb + i];
      jb0 = jb[i];
    }
#pragma unroll
    for (int rr = 0; rr < 3; rr++)
#pragma unroll
      for (int c = 0; c < 3; c++)
        Am[rr][c] = (act ? pm * cm[(3 * rr + c) * nc + i] : 0.0f) + (rr == c ? kJ * (J - 1.0f) : 0.0f);
    bin_blocks<false>(C, T, o, 0xffu, s_off, A.task);
    __syncthreads();
    stage_tile(T, op, 0, 4, s_off, s_g);
    __syncthreads();
    if (act) {
      const MpmKernel k = mpm_bspline(xp, inv_dx);
      float dw[3][3];
      mpm_dw(k, dw);
      const int r[3] = {k.base[0] - o[0], k.base[1] - o[1], k.base[2] - o[2]};
      float xbar[3] = {0.0f, 0.0f, 0.0f}, vbar[3] = {0.0f, 0.0f, 0.0f}, Ab[3][3] = {{0.0f}};
#pragma unroll
      for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const int nq = ((r[0] + a) * 6 + (r[1] + b)) * 6 + (r[2] + c);
            const float pb[3] = {s_g[0][nq], s_g[1][nq], s_g[2][nq]};
            const float mb = s_g[3][nq];
            const float W = k.w[a][0] * k.w[b][1] * k.w[c][2];
            const float gW[3] = {inv_dx * dw[a][0] * k.w[b][1] * k.w[c][2], inv_dx * k.w[a][0] * dw[b][1] * k.w[c][2],
                                 inv_dx * k.w[a][0] * k.w[b][1] * dw[c][2]};
            const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
            float Wbar = mb * pm, dposbar[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int rr = 0; rr < 3; rr++) {
              const float mom = pm * vv[rr] + Am[rr][0] * dpos[0] + Am[rr][1] * dpos[1] + Am[rr][2] * dpos[2];
              Wbar += pb[rr] * mom;
              vbar[rr] += W * pm * pb[rr];
#pragma unroll
              for (int d = 0; d < 3; d++) {
                Ab[rr][d] += W * pb[rr] * dpos[d];
                dposbar[d] += W * pb[rr] * Am[rr][d];
              }
            }
#pragma unroll
            for (int d = 0; d < 3; d++) xbar[d] += Wbar * gW[d] - dposbar[d];
          }
#pragma unroll
      for (int d = 0; d < 3; d++) {
        xb[d * nxb + i] = xb0[d] + xbar[d];
        vb[d * nvb + i] = vbar[d];
#pragma unroll
        for (int c = 0; c < 3; c++) cb[(3 * d + c) * ncb + i] = pm * Ab[d][c];
      }
      jb[i] = jb0 + kJ * (Ab[0][0] + Ab[1][1] + Ab[2][2]);
    }
    __syncthreads();
  }
}
