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
