// exchange_ops.cuh -- device side of the x-slab partitioner:
// halo unpack, G2P fused with stable in-place particle compaction + migration
// packing, and the append of received particles.  Included by kernels.cu after
// the tree helpers and the MPM ops.  The transport (NCCL over NVLink, or
// device copies between virtual ranks in tests) lives in parallel.py; every
// buffer carries its record count on the device, so no host sync is needed.
#pragma once

constexpr int PREC_WORDS = 17;   // particle record: x3 v3 C9 J1 id1

// HALO_UNPACK: one thread per cell of a packed block record.
__device__ void halo_unpack(const DevCtx& C, const DOp& op, int64_t i, int task) {
  const DArray B = C.arrays[op.a[0]];
  const DField& F0 = C.fields[op.f[0]];
  const DTree& T = C.trees[F0.tree];
  const uint32_t blk = 1u << T.lblk;
  int nf = 0;
  while (nf < 8 && op.f[nf] >= 0) nf++;
  const uint64_t rec = 4 + (uint64_t)nf * blk;
  const int64_t b = i >> T.lblk;
  const uint32_t j = (uint32_t)(i & (blk - 1));
  if (b >= (int64_t)*B.dcount) return;
  const uint32_t* r = (const uint32_t*)B.ptr + b * rec;
  int bc[3];
  inblock_coords(T, j, bc);
  int c[3] = {(int)r[0] + bc[0], (int)r[1] + bc[1], (int)r[2] + bc[2]};
  if (!in_domain(T, c)) return;
  uint32_t idx;
  uint32_t* cont = op.act ? activate_walk(C, T, c, idx, task) : locate(T, c, idx);
  if (!cont) return;
  const uint64_t fs = 1ull << T.ln_leaf;
  for (int k = 0; k < nf; k++) {
    uint32_t* p = cont + T.payload_off + (uint64_t)C.fields[op.f[k]].slot * fs + idx;
    const uint32_t v = r[4 + (uint64_t)k * blk + j];
    if (op.p[0] == 0.0f) atomicAdd((float*)p, __uint_as_float(v));
    else *p = v;
  }
}

// ---------------------------------------------------------------------------
// G2P + migration: the particle's new state is computed in registers, then
// particles whose cell x stays in [lo, hi) are written back compacted in their
// original order (single-pass scan with decoupled look-back; every tile reads
// its particles before publishing, so in-place writes to lower indices never
// overwrite unread data), leavers are appended to the left / right buffers.
// ---------------------------------------------------------------------------
struct MigArgs {
  DTree T;                // the grid tree (by value: constant bank)
  DevCtx C;
  DOp op;
  uint64_t* status;       // look-back descriptors (one per tile)
  uint32_t* ctl;          // [0] tile counter [1] done [2] epoch [3] new count
  int task;
};

constexpr int MG_TPB = 256;

__device__ __forceinline__ uint64_t mg_pack(uint32_t epoch, uint32_t flag, uint32_t v) {
  return ((uint64_t)(epoch & 0x3FFFFFFFu) << 34) | ((uint64_t)flag << 32) | v;
}

__global__ void __launch_bounds__(MG_TPB) k_g2p_migrate(const __grid_constant__ MigArgs A) {
  __shared__ uint32_t s_warp[MG_TPB / 32];
  __shared__ uint32_t s_tile, s_base, s_epoch;
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]],
               Id = C.arrays[op.a[4]], Lb = C.arrays[op.a[5]], Rb = C.arrays[op.a[6]];
  float* x = (float*)X.ptr;
  float* v = (float*)Vv.ptr;
  float* cm = (float*)Cm.ptr;
  float* jj = (float*)Jj.ptr;
  uint32_t* id = (uint32_t*)Id.ptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_epoch = A.ctl[2] & 0x3FFFFFFFu;   // bumped by an earlier launch
  const uint32_t n = *X.dcount;
  const uint32_t ntiles = (n + MG_TPB - 1) / MG_TPB;
  const float dt = op.p[0], inv_dx = op.p[1], lo = op.p[2], hi = op.p[3];
  const float dx = 1.0f / inv_dx;
  const DTree& T = A.T;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&A.ctl[0], 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t i = tile * MG_TPB + threadIdx.x;
    const bool live = i < n;
    // --- G2P in registers (same arithmetic as mpm_g2p) ---
    float xp[3] = {0, 0, 0}, nv[3] = {0, 0, 0}, nC[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, J = 1.0f;
    uint32_t pid = 0;
    if (live) {
      xp[0] = x[i]; xp[1] = x[X.n + i]; xp[2] = x[2 * X.n + i];
      J = jj[i];
      pid = id[i];
      MpmKernel k = mpm_bspline(xp, inv_dx);
      mpm_gather<0>(C, T, op, k, dx, inv_dx, nv, nC);
      J = J * (1.0f + dt * (nC[0][0] + nC[1][1] + nC[2][2]));
#pragma unroll
      for (int r = 0; r < 3; r++) xp[r] = xp[r] + dt * nv[r];
    }
    const float cx = floorf(__fmul_rn(xp[0], inv_dx));
    const int cat = !live ? 3 : (cx < lo ? 1 : (cx >= hi ? 2 : 0));   // 0 keep 1 left 2 right
    // --- block scan of keeps ---
    const uint32_t keep = cat == 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      uint32_t w = lane < MG_TPB / 32 ? s_warp[lane] : 0u, wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      if (lane < MG_TPB / 32) s_warp[lane] = wi - w;
      const uint32_t total = __shfl_sync(0xffffffffu, wi, MG_TPB / 32 - 1);
      uint64_t* st = A.status;
      if (lane == 0)
        atomicExch((unsigned long long*)&st[tile], (unsigned long long)mg_pack(epoch, tile == 0 ? 2u : 1u, total));
      uint32_t prefix = 0;
      int64_t j = (int64_t)tile - 1;
      while (j >= 0) {
        const int64_t q = j - lane;
        uint64_t s = 0;
        uint32_t fl = 2u;
        if (q >= 0) {
          do {
            s = ld_volatile64(&st[q]);
            fl = ((uint32_t)(s >> 34) == epoch) ? (uint32_t)(s >> 32) & 3u : 0u;
          } while (fl == 0u);
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, fl == 2u);
        const int stop = incl ? __ffs(incl) - 1 : 31;
        uint32_t vv = (lane <= stop && q >= 0) ? (uint32_t)s : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) vv += __shfl_xor_sync(0xffffffffu, vv, o);
        prefix += vv;
        if (incl) break;
        j -= 32;
      }
      if (lane == 0) {
        if (tile != 0)
          atomicExch((unsigned long long*)&st[tile], (unsigned long long)mg_pack(epoch, 2u, prefix + total));
        s_base = prefix;
        if (tile == ntiles - 1) A.ctl[3] = prefix + total;
      }
    }
    __syncthreads();
    if (cat == 0) {
      const uint32_t dst = s_base + s_warp[warp] + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
      for (int r = 0; r < 3; r++) {
        x[r * X.n + dst] = xp[r];
        v[r * Vv.n + dst] = nv[r];
#pragma unroll
        for (int d = 0; d < 3; d++) cm[(3 * r + d) * Cm.n + dst] = nC[r][d];
      }
      jj[dst] = J;
      id[dst] = pid;
    } else if (cat == 1 || cat == 2) {
      const DArray& Bf = cat == 1 ? Lb : Rb;
      const uint32_t s = atomicAdd((uint32_t*)Bf.dcount, 1u);
      if ((uint64_t)(s + 1) * PREC_WORDS <= (uint64_t)Bf.n) {
        uint32_t* rec = (uint32_t*)Bf.ptr + (uint64_t)s * PREC_WORDS;
#pragma unroll
        for (int r = 0; r < 3; r++) {
          rec[r] = __float_as_uint(xp[r]);
          rec[3 + r] = __float_as_uint(nv[r]);
#pragma unroll
          for (int d = 0; d < 3; d++) rec[6 + 3 * r + d] = __float_as_uint(nC[r][d]);
        }
        rec[15] = __float_as_uint(J);
        rec[16] = pid;
      } else {
        set_err(C, SG_ERR_LIST_OVERFLOW, A.task);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&A.ctl[1], 1u) == gridDim.x - 1) {
      *X.dcount = ntiles == 0 ? 0 : (int)A.ctl[3];
      A.ctl[0] = 0;
      A.ctl[1] = 0;
      A.ctl[2] = A.ctl[2] + 1u;
      __threadfence();
    }
  }
}

// MIGRATE_APPEND: received particle records of buffers a5 (left) and a6 (right)
// appended after the current count of a0..a4; the last CTA updates the count.
struct AppArgs {
  DevCtx C;
  DOp op;
  uint32_t* ctl;   // [1] done ticket
};

__global__ void __launch_bounds__(256) k_migrate_append(const __grid_constant__ AppArgs A) {
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]],
               Id = C.arrays[op.a[4]], Lb = C.arrays[op.a[5]], Rb = C.arrays[op.a[6]];
  // received counts are clamped to the buffers' record capacity: a sender whose
  // buffer overflowed latched SG_ERR_LIST_OVERFLOW and kept counting
  const uint32_t n0 = *X.dcount;
  const uint32_t cl = (uint32_t)min((uint64_t)*Lb.dcount, (uint64_t)Lb.n / PREC_WORDS);
  const uint32_t cr = (uint32_t)min((uint64_t)*Rb.dcount, (uint64_t)Rb.n / PREC_WORDS);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cl + cr; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* rec = i < cl ? (const uint32_t*)Lb.ptr + i * PREC_WORDS
                                 : (const uint32_t*)Rb.ptr + (i - cl) * PREC_WORDS;
    const uint64_t dst = n0 + i;
    if (dst >= (uint64_t)X.n) { set_err(C, SG_ERR_LIST_OVERFLOW, 0); continue; }
    float* x = (float*)X.ptr;
    float* v = (float*)Vv.ptr;
    float* cm = (float*)Cm.ptr;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      x[r * X.n + dst] = __uint_as_float(rec[r]);
      v[r * Vv.n + dst] = __uint_as_float(rec[3 + r]);
#pragma unroll
      for (int d = 0; d < 3; d++) cm[(3 * r + d) * Cm.n + dst] = __uint_as_float(rec[6 + 3 * r + d]);
    }
    ((float*)Jj.ptr)[dst] = __uint_as_float(rec[15]);
    ((uint32_t*)Id.ptr)[dst] = rec[16];
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&A.ctl[1], 1u) == gridDim.x - 1) {
      const uint64_t tot = (uint64_t)n0 + cl + cr;
      *X.dcount = (int)(tot < (uint64_t)X.n ? tot : (uint64_t)X.n);
      A.ctl[1] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// MIGRATE_COMPACT: migration for particle arrays kept in the binned kernels'
// order (G2P out of place in bin order, then this op on the new state).  The
// method fixes no particle order, so leavers are removed by HOLE FILLING
// instead of a stable compaction: only O(leavers) particles move.
//   k_migrate_mark: every particle whose cell x left [lo, hi) is appended to
//     the left / right send buffer (17-word record) and its index to the hole
//     list.
//   k_migrate_fill (one CTA): n' = n - holes; the keepers among the tail
//     positions [n', n) move into the holes below n' (k-th tail keeper into the
//     k-th low hole); the count becomes n'.
// ---------------------------------------------------------------------------
struct CompactArgs {
  DevCtx C;
  DOp op;
  uint32_t* holes;    // [0] count, [1..] indices
  uint32_t* tail;     // hole marks of the tail positions
  uint64_t cap;
  int task;
};

__global__ void __launch_bounds__(256) k_migrate_mark(const __grid_constant__ CompactArgs A) {
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]],
               Id = C.arrays[op.a[4]], Lb = C.arrays[op.a[5]], Rb = C.arrays[op.a[6]];
  const float* x = (const float*)X.ptr;
  const uint32_t n = (uint32_t)*X.dcount;
  const float inv_dx = op.p[1], lo = op.p[2], hi = op.p[3];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float xp0 = x[i];
    const float cx = floorf(__fmul_rn(xp0, inv_dx));
    if (cx >= lo && cx < hi) continue;
    const DArray& Bf = cx < lo ? Lb : Rb;
    const uint32_t s = atomicAdd((uint32_t*)Bf.dcount, 1u);
    if ((uint64_t)(s + 1) * PREC_WORDS > (uint64_t)Bf.n) { set_err(C, SG_ERR_LIST_OVERFLOW, A.task); continue; }
    uint32_t* rec = (uint32_t*)Bf.ptr + (uint64_t)s * PREC_WORDS;
    const uint32_t* xv = (const uint32_t*)X.ptr;
    const uint32_t* vv = (const uint32_t*)Vv.ptr;
    const uint32_t* cv = (const uint32_t*)Cm.ptr;
#pragma unroll
    for (int r = 0; r < 3; r++) {
      rec[r] = xv[r * X.n + i];
      rec[3 + r] = vv[r * Vv.n + i];
    }
#pragma unroll
    for (int k = 0; k < 9; k++) rec[6 + k] = cv[k * Cm.n + i];
    rec[15] = ((const uint32_t*)Jj.ptr)[i];
    rec[16] = ((const uint32_t*)Id.ptr)[i];
    const uint32_t h = atomicAdd(A.holes, 1u);
    if (h < A.cap) A.holes[1 + h] = i;
    else set_err(C, SG_ERR_LIST_OVERFLOW, A.task);
  }
}

// Block-wide exclusive scan of one flag per thread (1024 threads).
__device__ __forceinline__ uint32_t block_scan1024(uint32_t f, uint32_t* s_w, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) s_w[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    uint32_t v = s_w[lane], inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    s_w[lane] = inc - v;
    if (lane == 31) s_w[32] = inc;
  }
  __syncthreads();
  const uint32_t r = s_w[w] + __popc(bal & ((1u << lane) - 1u));
  total = s_w[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) k_migrate_fill(const __grid_constant__ CompactArgs A) {
  __shared__ uint32_t s_w[33];
  const DevCtx& C = A.C;
  const DOp& op = A.op;
  const DArray X = C.arrays[op.a[0]];
  const uint32_t n = (uint32_t)*X.dcount;
  const uint32_t L = (uint32_t)min((uint64_t)A.holes[0], A.cap);
  const uint32_t np = n - L;
  // mark the tail positions that are holes
  for (uint32_t t = threadIdx.x; t < L; t += 1024) A.tail[t] = 0u;
  __syncthreads();
  for (uint32_t h = threadIdx.x; h < L; h += 1024) {
    const uint32_t p = A.holes[1 + h];
    if (p >= np) A.tail[p - np] = 1u;
  }
  __syncthreads();
  // k-th low hole (in hole-list order) <- k-th tail keeper (in position order):
  // rank the low holes in place (tail[] is reused below, so first collect the
  // low holes into holes[1..] compacted)
  uint32_t base = 0;
  for (uint32_t h0 = 0; h0 < L; h0 += 1024) {
    const uint32_t h = h0 + threadIdx.x;
    const uint32_t p = h < L ? A.holes[1 + h] : 0xFFFFFFFFu;
    const uint32_t f = h < L && p < np;
    uint32_t tot;
    const uint32_t r = block_scan1024(f, s_w, tot);
    if (f) A.holes[1 + base + r] = p;   // writes only at or below the read position: safe in place
    base += tot;
    __syncthreads();
  }
  // the tail keepers, in order, move into the low holes
  uint32_t kbase = 0;
  for (uint32_t t0 = 0; t0 < L; t0 += 1024) {
    const uint32_t t = t0 + threadIdx.x;
    const uint32_t f = t < L && A.tail[t] == 0u;
    uint32_t tot;
    const uint32_t r = block_scan1024(f, s_w, tot);
    if (f) {
      const uint32_t src = np + t, dst = A.holes[1 + kbase + r];
      for (int a = 0; a < 5; a++) {
        const DArray& Ar = C.arrays[op.a[a]];
        uint32_t* q = (uint32_t*)Ar.ptr;
        for (int c = 0; c < Ar.ncomp; c++) q[(uint64_t)c * Ar.n + dst] = q[(uint64_t)c * Ar.n + src];
      }
    }
    kbase += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *X.dcount = (int)np;
    A.holes[0] = 0u;   // ready for the next step
  }
}
