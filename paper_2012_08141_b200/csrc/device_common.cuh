// device_common.cuh -- device helpers of the sparse-grid layout (tree walks,
// activation, block rows, error word), included INSIDE namespace sg by
// kernels.cu and by every JIT-specialized kernel (jit.cpp).
#pragma once

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Loads of words other CTAs of the SAME launch may be writing (look-back
// descriptors, mask words under activation): device-scope relaxed, so L2 is
// the coherence point (a C++ volatile load compiles to a system-scope strong
// load).  Words written by EARLIER launches (list counts, table flags, pool
// counters) are read with plain loads: the kernel boundary orders them.
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_volatile64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void set_err(const DevCtx& C, int code, int task) {
  if (atomicCAS(&C.err[0], 0u, (uint32_t)code) == 0u) C.err[1] = (uint32_t)task;
}

__device__ __forceinline__ uint32_t local_lin(const DLevel& L, const int c[3]) {
  uint32_t l0 = ((uint32_t)c[0] >> L.lbelow[0]) & ((1u << L.le[0]) - 1u);
  uint32_t l1 = ((uint32_t)c[1] >> L.lbelow[1]) & ((1u << L.le[1]) - 1u);
  uint32_t l2 = ((uint32_t)c[2] >> L.lbelow[2]) & ((1u << L.le[2]) - 1u);
  return (((l0 << L.le[1]) | l1) << L.le[2]) | l2;
}

__device__ __forceinline__ bool in_domain(const DTree& T, const int c[3]) {
  const DLevel& L = T.lev[T.nlev - 1];
#pragma unroll
  for (int a = 0; a < 3; a++)
    if (c[a] < 0 || c[a] >= (1 << L.lres[a])) return false;
  return true;
}

__device__ __forceinline__ uint32_t* cont_ptr(const DTree& T, int seg, uint32_t slot) {
  return T.seg[seg].base + (uint64_t)slot * T.seg[seg].stride;
}

// Non-activating tree walk: leaf container + leaf index of cell c, or null if
// a pointer ancestor is NULL.  Bitmasks are not tested (zero-on-free).
__device__ __forceinline__ uint32_t* locate(const DTree& T, const int c[3], uint32_t& idx) {
  uint32_t* cont = T.seg[0].base;
  idx = 0;
  for (int l = 0; l < T.nlev; l++) {
    const DLevel& L = T.lev[l];
    idx = (idx << L.lE) | local_lin(L, c);
    if (L.kind == SG_POINTER) {
      uint32_t v = cont[L.slot_off + idx];
      if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) return nullptr;
      cont = cont_ptr(T, L.seg + 1, v - 1u);
      idx = 0;
    }
  }
  return cont;
}

// Full activity test: every sparse ancestor set.
__device__ __forceinline__ uint32_t* locate_active(const DTree& T, const int c[3], uint32_t& idx) {
  uint32_t* cont = T.seg[0].base;
  idx = 0;
  for (int l = 0; l < T.nlev; l++) {
    const DLevel& L = T.lev[l];
    idx = (idx << L.lE) | local_lin(L, c);
    if (L.kind == SG_BITMASKED) {
      if (!((cont[L.mask_off + (idx >> 5)] >> (idx & 31)) & 1u)) return nullptr;
    } else if (L.kind == SG_POINTER) {
      uint32_t v = cont[L.slot_off + idx];
      if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) return nullptr;
      cont = cont_ptr(T, L.seg + 1, v - 1u);
      idx = 0;
    }
  }
  return cont;
}

static __device__ int32_t pool_pop(const DSeg& S) {
  int32_t top = atomicSub(&S.alloc[1], 1);
  if (top > 0) return (int32_t)S.free_list[top - 1];
  atomicAdd(&S.alloc[1], 1);
  int32_t b = atomicAdd(&S.alloc[0], 1);
  if (b >= (int32_t)S.capacity) return -1;
  return b;
}

// Pointer child acquisition (PAPER.md:166 allocator; SURVEY.md s7 hard part 1):
// CAS NULL->BUSY, pop the pool, record the origin, publish slot with release.
static __device__ int32_t acquire_child(const DevCtx& C, const DTree& T, const DLevel& L, uint32_t* cont, uint32_t idx,
                                 const int c[3], int task) {
  uint32_t* sp = cont + L.slot_off + idx;
  uint32_t v = ld_acquire(sp);
  if (v != SG_SLOT_NULL && v != SG_SLOT_BUSY) return (int32_t)(v - 1u);
  if (v == SG_SLOT_NULL) {
    uint32_t old = atomicCAS(sp, SG_SLOT_NULL, SG_SLOT_BUSY);
    if (old == SG_SLOT_NULL) {
      const DSeg& S = T.seg[L.seg + 1];
      int32_t got = pool_pop(S);
      if (got < 0) {
        set_err(C, SG_ERR_POOL_EXHAUSTED, task);
        atomicExch(sp, SG_SLOT_NULL);
        return -1;
      }
#pragma unroll
      for (int a = 0; a < 3; a++) S.origin[got * 3 + a] = c[a] >> L.lbelow[a];
      __threadfence();
      atomicExch(sp, (uint32_t)got + 1u);
      return got;
    }
    v = old;
  }
  while (v == SG_SLOT_BUSY) {
    __nanosleep(20);
    v = ld_acquire(sp);
  }
  if (v == SG_SLOT_NULL) return -1;
  return (int32_t)(v - 1u);
}

// Activating walk: every sparse ancestor of c becomes
// active; returns the leaf container + index.  Idempotent; never touches payload.
static __device__ uint32_t* activate_walk(const DevCtx& C, const DTree& T, const int c[3], uint32_t& idx, int task) {
  uint32_t* cont = T.seg[0].base;
  idx = 0;
  for (int l = 0; l < T.nlev; l++) {
    const DLevel& L = T.lev[l];
    idx = (idx << L.lE) | local_lin(L, c);
    if (L.kind == SG_BITMASKED) {
      uint32_t* w = cont + L.mask_off + (idx >> 5);
      uint32_t b = 1u << (idx & 31);
      if (!(ld_volatile(w) & b)) atomicOr(w, b);
    } else if (L.kind == SG_POINTER) {
      int32_t s = acquire_child(C, T, L, cont, idx, c, task);
      if (s < 0) return nullptr;
      cont = cont_ptr(T, L.seg + 1, (uint32_t)s);
      idx = 0;
    }
  }
  return cont;
}

// Level-global coordinates of the level-l cell (container slot cs, index idx).
static __device__ void cell_coords(const DTree& T, int l, uint32_t cs, uint32_t idx, int g[3]) {
  const DLevel& L = T.lev[l];
  const DSeg& S = T.seg[L.seg];
  int acc[3] = {0, 0, 0}, sh[3] = {0, 0, 0};
  for (int m = l; m >= S.first; m--) {
    const DLevel& M = T.lev[m];
    uint32_t d = idx & ((1u << M.lE) - 1u);
    idx >>= M.lE;
    uint32_t d2 = d & ((1u << M.le[2]) - 1u);
    uint32_t d1 = (d >> M.le[2]) & ((1u << M.le[1]) - 1u);
    uint32_t d0 = d >> (M.le[1] + M.le[2]);
    acc[0] |= (int)(d0 << sh[0]); sh[0] += M.le[0];
    acc[1] |= (int)(d1 << sh[1]); sh[1] += M.le[1];
    acc[2] |= (int)(d2 << sh[2]); sh[2] += M.le[2];
  }
  int o[3] = {0, 0, 0};
  if (L.seg > 0) { o[0] = S.origin[cs * 3]; o[1] = S.origin[cs * 3 + 1]; o[2] = S.origin[cs * 3 + 2]; }
#pragma unroll
  for (int a = 0; a < 3; a++) g[a] = (o[a] << sh[a]) | acc[a];
}

// Index of leaf cell c within its block (levels below the driving level).
__device__ __forceinline__ uint32_t inblock_idx(const DTree& T, const int c[3]) {
  uint32_t idx = 0;
  for (int l = T.driving + 1; l < T.nlev; l++) idx = (idx << T.lev[l].lE) | local_lin(T.lev[l], c);
  return idx;
}

// Block-local coordinates of in-block index j.
__device__ __forceinline__ void inblock_coords(const DTree& T, uint32_t j, int c[3]) {
  c[0] = c[1] = c[2] = 0;
  for (int m = T.nlev - 1; m > T.driving; m--) {
    const DLevel& M = T.lev[m];
    uint32_t d = j & ((1u << M.lE) - 1u);
    j >>= M.lE;
    c[2] |= (int)((d & ((1u << M.le[2]) - 1u)) << M.lbelow[2]);
    c[1] |= (int)(((d >> M.le[2]) & ((1u << M.le[1]) - 1u)) << M.lbelow[1]);
    c[0] |= (int)((d >> (M.le[1] + M.le[2])) << M.lbelow[0]);
  }
}

// Resolve a driving-list entry to (leaf container, first leaf idx, origin in leaf units).
__device__ __forceinline__ bool resolve_entry(const DTree& T, uint32_t e, uint32_t*& cont, uint32_t& first,
                                              int org[3]) {
  if (T.driving < 0) {
    cont = T.seg[0].base; first = 0; org[0] = org[1] = org[2] = 0;
    return true;
  }
  const DLevel& D = T.lev[T.driving];
  uint32_t cs = e >> D.ln, idx = e & ((1u << D.ln) - 1u);
  int g[3];
  cell_coords(T, T.driving, cs, idx, g);
#pragma unroll
  for (int a = 0; a < 3; a++) org[a] = g[a] << D.lbelow[a];
  uint32_t* dc = cont_ptr(T, D.seg, cs);
  if (D.kind == SG_POINTER) {
    uint32_t v = dc[D.slot_off + idx];
    if (v == SG_SLOT_NULL || v == SG_SLOT_BUSY) return false;
    cont = cont_ptr(T, D.seg + 1, v - 1u);
    first = 0;
  } else {
    cont = dc;
    first = idx << (T.ln_leaf - D.ln);
  }
  return true;
}

// Block-table row of a driving-list entry: the block and its face neighbours.
__device__ __forceinline__ void make_block_row(const DTree& T, uint32_t e, BlockRow* out) {
  BlockRow r;
  uint32_t* cont = nullptr;
  uint32_t first = 0;
  int org[3] = {0, 0, 0};
  bool ok = resolve_entry(T, e, cont, first, org);
  const uint32_t* base = T.seg[T.nseg - 1].base;
  r.blk = ok ? (uint32_t)(cont - base) + T.payload_off + first : SG_NO_BLOCK;
  r.maskw = ok && T.leaf_bitmasked ? (uint32_t)(cont - base) + T.lev[T.nlev - 1].mask_off + (first >> 5) : 0u;
  r.first = first;
  r.org[0] = org[0]; r.org[1] = org[1]; r.org[2] = org[2];
  const uint32_t lowmask = ~((1u << T.lblk) - 1u);
#pragma unroll
  for (int dir = 0; dir < 6; dir++) {
    r.nbr[dir] = SG_NO_BLOCK;   // absent: reads 0
    int axis = dir >> 1;
    if (!ok || axis >= T.nd || T.driving < 0) continue;
    int q[3] = {org[0], org[1], org[2]};
    q[axis] += (dir & 1) ? (1 << T.lev[T.driving].lbelow[axis]) : -1;
    if (!in_domain(T, q)) continue;
    uint32_t idx;
    uint32_t* c2 = locate(T, q, idx);
    if (c2) r.nbr[dir] = (uint32_t)(c2 - base) + T.payload_off + (idx & lowmask);
  }
  *out = r;
}

// make_block_row by a whole warp (same e on every lane): the entry is resolved
// once per lane, then lanes 0..5 walk to one face neighbour each and the row
// is assembled by shuffles -- two dependent tree walks instead of seven (the
// first struct-for after a listgen builds every row of the table: C2's fused
// FILLs spent ~12 us on serial walks).  Every lane returns the full row.
__device__ __forceinline__ void make_block_row_warp(const DTree& T, uint32_t e, int lane, BlockRow* out) {
  BlockRow r;
  uint32_t* cont = nullptr;
  uint32_t first = 0;
  int org[3] = {0, 0, 0};
  bool ok = resolve_entry(T, e, cont, first, org);
  const uint32_t* base = T.seg[T.nseg - 1].base;
  r.blk = ok ? (uint32_t)(cont - base) + T.payload_off + first : SG_NO_BLOCK;
  r.maskw = ok && T.leaf_bitmasked ? (uint32_t)(cont - base) + T.lev[T.nlev - 1].mask_off + (first >> 5) : 0u;
  r.first = first;
  r.org[0] = org[0]; r.org[1] = org[1]; r.org[2] = org[2];
  const uint32_t lowmask = ~((1u << T.lblk) - 1u);
  uint32_t mine = SG_NO_BLOCK;   // absent: reads 0
  const int axis = lane >> 1;
  if (lane < 6 && ok && axis < T.nd && T.driving >= 0) {
    int q[3] = {org[0], org[1], org[2]};
    q[axis] += (lane & 1) ? (1 << T.lev[T.driving].lbelow[axis]) : -1;
    if (in_domain(T, q)) {
      uint32_t idx;
      uint32_t* c2 = locate(T, q, idx);
      if (c2) mine = (uint32_t)(c2 - base) + T.payload_off + (idx & lowmask);
    }
  }
#pragma unroll
  for (int d = 0; d < 6; d++) r.nbr[d] = __shfl_sync(0xffffffffu, mine, d);
  *out = r;
}

// ---------------------------------------------------------------------------
// Activation
// ---------------------------------------------------------------------------
