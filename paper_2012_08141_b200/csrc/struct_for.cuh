// struct_for.cuh -- the fused struct-for megakernel (included by kernels.cu).
//
// One launch runs a fused group of ops (Figs. 7-8
// "tasks that loop over the active elements of the same tensor") over the
// element list of the tree's driving level.  Each CTA
// iteration takes a tile of leaf blocks whose rows (block, origin, face
// neighbours) come from the list's block table in one coalesced read.  Every
// thread owns a fixed set of cells of the tile and runs the ops of the group on
// them in order (op-outer, cell-inner: one tight loop per op), so an identity
// access never leaves its thread: fused accumulations need no atomics and a
// value written by op k is read back by op k+1 from L1 (PAPER.md:400 atomic
// demotion and store-to-load forwarding).  The planner only fuses groups whose
// shared fields are accessed at the identity, so no cross-thread
// ordering is needed between ops.
//
// Addresses are u32 word offsets from the leaf pool base (a kernel parameter),
// so every access is a global-space load/store.
//
// Two cell paths:
//   QUAD    blocks that are one dense/bitmasked level whose fastest axis has
//           extent >= 4 (C1, C2, C3, C5): a thread owns 4 consecutive cells of a
//           row and moves them with 16-byte loads/stores; neighbour rows along
//           the slower axes are whole quads, the fast-axis neighbours come from
//           the quad itself plus two scalars.  Stencils process two quads per
//           thread with all loads issued before any arithmetic.
//   GENERIC any other block shape: one cell per thread, hierarchical decode.

struct SFArgs {
  DTree T;
  DevCtx C;
  const uint32_t* entries;   // driving list (null when the tree has no driving level)
  const uint32_t* count;
  BlockRow* table;           // the list's block table
  uint32_t* table_ctl;       // the list's ctl words ([3] ticket, [4] rows built)
  int has_reduce;
  int nops;
  int need_nbr;
  int ltile;                 // log2 cells per tile
  int lept;                  // log2 entries per tile (0 when a block spans tiles)
  int task;
  int lb[3];                 // QUAD: log2 block extent per axis
  DOp ops[SG_MAXOPS];
  uint64_t aux[SG_MAXOPS];   // 0-D target address per op
};

constexpr int SF_TPB = 256, SF_MAXE = 256;

// Op sources of a fused group.  OpsRT: the op table of the launch (kernel
// parameters).  A JIT-specialized kernel (jit.cpp) passes a type
// whose operator[] returns compile-time constant DOps and whose size is a
// constant: the op loops unroll, every switch on the op code and every slot /
// parameter folds into the instruction stream.
struct OpsRT {
  static constexpr int kUnroll = 1;
  const DOp* p;
  int n;
  __device__ __forceinline__ const DOp& operator[](int i) const { return p[i]; }
  __device__ __forceinline__ int size() const { return n; }
};

struct SFTile {
  uint32_t blk[SF_MAXE];
  uint32_t maskw[SF_MAXE];
  uint32_t first[SF_MAXE];
  int org[SF_MAXE][3];
  uint32_t nbr[SF_MAXE][6];
  int32_t slot[SF_MAXE];      // HALO_PACK: record slot of each block, -1 = not packed
  uint32_t aux[SF_MAXE];      // RESTRICT / PROLONG: the coarse block (field slot 0) of each block
  uint32_t ne;
};

// HALO_PACK, per-tile part: blocks whose origin x lies in [p0, p1) get a record
// slot (a0's device count) and their header; the payload is copied per cell.
__device__ __forceinline__ void halo_pack_slots(const DevCtx& C, const DOp& op, SFTile& tile, int task) {
  __syncthreads();
  const DArray& B = C.arrays[op.a[0]];
  for (uint32_t e = threadIdx.x; e < tile.ne; e += blockDim.x) {
    int32_t s = -1;
    if (tile.blk[e] != SG_NO_BLOCK && (float)tile.org[e][0] >= op.p[0] && (float)tile.org[e][0] < op.p[1]) {
      s = atomicAdd(B.dcount, 1);
      if (s >= (int32_t)op.p[2]) { set_err(C, SG_ERR_LIST_OVERFLOW, task); s = -1; }
    }
    tile.slot[e] = s;
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t* halo_rec(const DevCtx& C, const DOp& op, int32_t slot, uint32_t lblk, int nf) {
  return (uint32_t*)C.arrays[op.a[0]].ptr + (uint64_t)slot * (4 + ((uint64_t)nf << lblk));
}

template <typename V> __device__ __forceinline__ V ldv(const uint32_t* p);
template <> __device__ __forceinline__ float ldv<float>(const uint32_t* p) { return __uint_as_float(*p); }
template <> __device__ __forceinline__ int ldv<int>(const uint32_t* p) { return (int)*p; }
__device__ __forceinline__ void stv(uint32_t* p, float v) { *p = __float_as_uint(v); }
__device__ __forceinline__ void stv(uint32_t* p, int v) { *p = (uint32_t)v; }
template <typename V> __device__ __forceinline__ bool is_float() { return false; }
template <> __device__ __forceinline__ bool is_float<float>() { return true; }

__device__ __forceinline__ void atomic_add_v(uint32_t* p, float v) { atomicAdd((float*)p, v); }
__device__ __forceinline__ void atomic_add_v(uint32_t* p, int v) { atomicAdd((int*)p, v); }

// Reductions into 0-D fields: per-thread partials -> warp (double) -> CTA
// shared accumulator -> per-CTA partial in global memory -> the last CTA sums
// the partials in CTA order (deterministic, f64) and adds once to the target.
__shared__ double s_red[SG_MAXOPS];

template <typename V>
__device__ __forceinline__ void warp_add(int o, V v) {
  double d = (double)v;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) d += __shfl_xor_sync(0xffffffffu, d, s);
  if ((threadIdx.x & 31) == 0 && d != 0.0) atomicAdd(&s_red[o], d);
}

template <typename V, class OPS>
__device__ void finish_reductions(const SFArgs& A, const OPS& ops) {
  const int nops = ops.size();
  __shared__ bool s_last;
  __shared__ double s_sum[SF_TPB];
  __syncthreads();
  const int G = gridDim.x;
  if (threadIdx.x < SG_MAXOPS) A.C.partials[threadIdx.x * A.C.max_grid + blockIdx.x] = s_red[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(A.C.red_done, 1u) == (uint32_t)G - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll(OPS::kUnroll)
  for (int o = 0; o < nops; o++) {
    if (ops[o].op != SG_OP_REDUCE_SUM && ops[o].op != SG_OP_RESID_NORM2 && ops[o].op != SG_OP_DOT) continue;
    double t = 0.0;   // fixed-order tree sum over CTAs
    for (int b = threadIdx.x; b < G; b += SF_TPB) t += __ldcg(&A.C.partials[o * A.C.max_grid + b]);
    s_sum[threadIdx.x] = t;
    __syncthreads();
    for (int w = SF_TPB / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      uint32_t* tgt = (uint32_t*)A.aux[o];
      V old = ldv<V>(tgt);
      stv(tgt, (V)((double)old + s_sum[0]));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *A.C.red_done = 0u;
}

// ---------------------------------------------------------------------------
// scalar (one cell) helpers
// ---------------------------------------------------------------------------
struct CellCtx {
  const DTree* T;
  const SFTile* tile;
  uint32_t* P;           // leaf pool base
  int e;                 // entry slot in the tile
  uint32_t j;            // in-block index
  int c[3];              // leaf coords
  uint64_t fstride;      // words between field slots
};

__device__ __forceinline__ uint32_t* cell_ptr(const CellCtx& x, int slot) {
  return x.P + x.tile->blk[x.e] + (uint64_t)slot * x.fstride + x.j;
}

template <typename V>
__device__ __forceinline__ V ld_id(const CellCtx& x, int slot) { return ldv<V>(cell_ptr(x, slot)); }
template <typename V>
__device__ __forceinline__ void st_id(const CellCtx& x, int slot, V v) { stv(cell_ptr(x, slot), v); }

// Neighbour value c + d*e_axis (0 when inactive / out of bound).
template <typename V>
__device__ __forceinline__ V ld_nbr(const CellCtx& x, int slot, int axis, int d) {
  const DTree& T = *x.T;
  int n[3] = {x.c[0], x.c[1], x.c[2]};
  n[axis] += d;
  const int bdim = T.driving < 0 ? (1 << T.lev[T.nlev - 1].lres[axis]) : (1 << T.lev[T.driving].lbelow[axis]);
  int rel = n[axis] - x.tile->org[x.e][axis];
  uint32_t base;
  if (rel >= 0 && rel < bdim) {
    base = x.tile->blk[x.e];
  } else {
    if (T.driving < 0) return V(0);
    base = x.tile->nbr[x.e][axis * 2 + (d > 0 ? 1 : 0)];
    if (base == SG_NO_BLOCK) return V(0);
  }
  return ldv<V>(x.P + base + (uint64_t)slot * x.fstride + inblock_idx(T, n));
}

template <typename V>
__device__ __forceinline__ V nbr_sum(const CellCtx& x, int slot) {
  V s = V(0);
  for (int a = 0; a < x.T->nd; a++) s += ld_nbr<V>(x, slot, a, -1) + ld_nbr<V>(x, slot, a, +1);
  return s;
}

template <typename V>
__device__ __noinline__ void apply_downsample(const SFArgs& A, const DOp& op, const int c[3], V val) {
  const DField& tf = A.C.fields[op.f[0]];
  const DTree& T2 = A.C.trees[tf.tree];
  int h[3] = {c[0] >> 1, c[1] >> 1, c[2] >> 1};
  uint32_t idx;
  uint32_t* cont;
  if (op.act & 1u) {
    cont = activate_walk(A.C, T2, h, idx, A.task);
  } else {
    cont = A.C.debug ? locate_active(T2, h, idx) : locate(T2, h, idx);
    if (!cont && A.C.debug) set_err(A.C, SG_ERR_DEMOTION_TRAP, A.task);
  }
  if (!cont) return;
  atomic_add_v(cont + T2.payload_off + ((uint64_t)tf.slot << T2.ln_leaf) + idx, val);
}

// Value of field f (another tree, e.g. the coarse level) at cell h; 0 when inactive.
template <typename V>
__device__ __noinline__ V read_other(const SFArgs& A, int f, const int h[3]) {
  const DField& tf = A.C.fields[f];
  const DTree& T2 = A.C.trees[tf.tree];
  if (!in_domain(T2, h)) return V(0);
  uint32_t idx;
  uint32_t* cont = locate(T2, h, idx);
  if (!cont) return V(0);
  return ldv<V>(cont + T2.payload_off + ((uint64_t)tf.slot << T2.ln_leaf) + idx);
}

// Value of a 0-D field (written by an earlier launch).
template <typename V>
__device__ __forceinline__ V scalar_of(const SFArgs& A, int f) {
  return ldv<V>(A.C.scalars + A.C.fields[f].scalar);
}

// r - A z at the cell (A = -Laplacian, h = 1)
template <typename V>
__device__ __forceinline__ V residual_at(const CellCtx& x, int slot_r, int slot_z) {
  const int D = x.T->nd;
  return ld_id<V>(x, slot_r) - ((V)(2 * D) * ld_id<V>(x, slot_z) - nbr_sum<V>(x, slot_z));
}

// One op on one cell (GENERIC path, and the per-lane ops of the QUAD path).
// Returns the REDUCE contribution.
template <typename V>
__device__ __forceinline__ V apply_cell(const SFArgs& A, const DOp& op, const CellCtx& x) {
  const int D = x.T->nd;
  switch (op.op) {
    case SG_OP_FILL: st_id<V>(x, op.slot[0], (V)op.p[0]); break;
    case SG_OP_ADD_CONST: st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[1]) + (V)op.p[0]); break;
    case SG_OP_INC: st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[0]) + (V)op.p[0]); break;
    case SG_OP_AXPY: st_id<V>(x, op.slot[0], (V)op.p[0] * ld_id<V>(x, op.slot[1]) + ld_id<V>(x, op.slot[2])); break;
    case SG_OP_STENCIL:
      st_id<V>(x, op.slot[0], nbr_sum<V>(x, op.slot[1]) - (V)(2 * D) * ld_id<V>(x, op.slot[1]));
      break;
    case SG_OP_JACOBI:
      st_id<V>(x, op.slot[0], (ld_id<V>(x, op.slot[2]) + nbr_sum<V>(x, op.slot[1])) / (V)(2 * D));
      break;
    case SG_OP_REDUCE_SUM: return ld_id<V>(x, op.slot[1]);
    case SG_OP_DOWNSAMPLE: {
      V v = op.slot[1] >= 0 ? ld_id<V>(x, op.slot[1]) : V(0);
      apply_downsample<V>(A, op, x.c, (V)op.p[0] * v + (V)op.p[1]);
    } break;
    case SG_OP_JITTER:
      if ((x.c[0] & 1) == 0) st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[0]) + ld_nbr<V>(x, op.slot[0], 0, +1));
      break;
    case SG_OP_GRID_OP: mpm_grid_op(op, x.c, cell_ptr(x, 0), x.fstride); break;
    case SG_OP_SMOOTH_RB:
      if (((x.c[0] + x.c[1] + x.c[2]) & 1) == (int)op.p[0])
        st_id<V>(x, op.slot[0], (ld_id<V>(x, op.slot[1]) + nbr_sum<V>(x, op.slot[0])) / (V)(2 * D));
      break;
    case SG_OP_RESTRICT:
      apply_downsample<V>(A, op, x.c, (V)op.p[0] * residual_at<V>(x, op.slot[1], op.slot[2]));
      break;
    case SG_OP_PROLONG: {
      const int h[3] = {x.c[0] >> 1, x.c[1] >> 1, x.c[2] >> 1};
      st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[0]) + read_other<V>(A, op.f[1], h));
    } break;
    case SG_OP_RESID_NORM2: {
      const V r = residual_at<V>(x, op.slot[1], op.slot[2]);
      return r * r;
    }
    case SG_OP_DOT: return (V)op.p[0] * ld_id<V>(x, op.slot[1]) * ld_id<V>(x, op.slot[2]);
    case SG_OP_AXPY_RATIO:
    case SG_OP_XPAY_RATIO: {
      const V ratio = scalar_of<V>(A, op.f[2]) / scalar_of<V>(A, op.f[3]);
      if (op.op == SG_OP_AXPY_RATIO)
        st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[0]) + (V)op.p[0] * ratio * ld_id<V>(x, op.slot[1]));
      else
        st_id<V>(x, op.slot[0], ld_id<V>(x, op.slot[1]) + ratio * ld_id<V>(x, op.slot[0]));
    } break;
    default: break;
  }
  return V(0);
}

// ---------------------------------------------------------------------------
// quad path
// ---------------------------------------------------------------------------
template <typename V>
struct Q4 { V v[4]; };

template <typename V>
__device__ __forceinline__ Q4<V> ld4(const uint32_t* p) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  Q4<V> q;
  if (is_float<V>()) {
    q.v[0] = (V)__uint_as_float(u.x); q.v[1] = (V)__uint_as_float(u.y);
    q.v[2] = (V)__uint_as_float(u.z); q.v[3] = (V)__uint_as_float(u.w);
  } else {
    q.v[0] = (V)(int)u.x; q.v[1] = (V)(int)u.y; q.v[2] = (V)(int)u.z; q.v[3] = (V)(int)u.w;
  }
  return q;
}

__device__ __forceinline__ uint32_t bits_of(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t bits_of(int v) { return (uint32_t)v; }

template <typename V>
__device__ __forceinline__ void st4(uint32_t* p, const Q4<V>& q, uint32_t amask) {
  if (amask == 0xFu) {
    *reinterpret_cast<uint4*>(p) = make_uint4(bits_of(q.v[0]), bits_of(q.v[1]), bits_of(q.v[2]), bits_of(q.v[3]));
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++)
      if ((amask >> k) & 1u) p[k] = bits_of(q.v[k]);
  }
}

struct QuadCtx {
  uint32_t off;            // word offset of lane 0 (field slot 0); SG_NO_BLOCK: skip
  uint32_t j0;             // in-block index of lane 0
  int r[3];                // block-relative coords of lane 0
  int e;
  uint32_t amask;          // active lanes
};

// Block geometry of the QUAD path: log2 extents per axis.  Built once per
// kernel from template constants (common shapes) or the launch parameters.
struct QG {
  int lb[3];
};

template <int GL>
__device__ __forceinline__ QG make_qg(const SFArgs& A) {
  QG g;
  if (GL == 1) { g.lb[0] = 3; g.lb[1] = 3; g.lb[2] = 3; }        // 8^3 (C2, JAC-XL)
  else if (GL == 2) { g.lb[0] = 2; g.lb[1] = 2; g.lb[2] = 2; }   // 4^3 (C3, C5)
  else if (GL == 3) { g.lb[0] = 2; g.lb[1] = 2; g.lb[2] = 0; }   // 4x4 (C1)
  else { g.lb[0] = A.lb[0]; g.lb[1] = A.lb[1]; g.lb[2] = A.lb[2]; }
  return g;
}

template <int ND>
__device__ __forceinline__ QuadCtx quad_ctx(const SFArgs& A, const QG& g, const SFTile& tile, const uint32_t* P,
                                            uint32_t i, uint32_t lq, bool chunked, uint32_t jbase) {
  QuadCtx x;
  x.e = chunked ? 0 : (int)(i >> lq);
  x.j0 = chunked ? jbase + 4 * i : 4 * (i & ((1u << lq) - 1u));
  const uint32_t b = tile.blk[x.e];
  x.off = b == SG_NO_BLOCK ? SG_NO_BLOCK : b + x.j0;
  x.amask = 0xFu;
  if (b != SG_NO_BLOCK && A.T.leaf_bitmasked) {
    uint32_t li = (tile.first[x.e] & 31u) + x.j0;
    x.amask = (P[tile.maskw[x.e] + (li >> 5)] >> (li & 31)) & 0xFu;
  }
  const int lb1 = ND > 1 ? g.lb[1] : 0, lb2 = ND > 2 ? g.lb[2] : 0;
  x.r[0] = (int)(x.j0 >> (lb1 + lb2));
  x.r[1] = ND > 1 ? (int)((x.j0 >> lb2) & ((1u << lb1) - 1u)) : 0;
  x.r[2] = ND > 2 ? (int)(x.j0 & ((1u << lb2) - 1u)) : 0;
  return x;
}

// Gathers the 2*ND face-neighbour values of a quad (loads only, branch-free
// address selection: in-block row, neighbour block row, or absent).
template <typename V, int ND>
struct NbrLoads {
  Q4<V> row[2 * (ND - 1) + 1];   // neighbour rows along the slower axes
  V lo, hi;                      // fast-axis ends
};

// Predicated global loads (no branch; the register keeps 0 when the predicate
// is off -- an absent neighbour reads 0).
__device__ __forceinline__ uint4 ld4_if(const uint32_t* p, bool pred) {
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n @q ld.global.v4.u32 {%0, %1, %2, %3}, [%4];\n}\n"
      : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
      : "l"(p), "r"((int)pred));
  return r;
}
__device__ __forceinline__ uint32_t ld1_if(const uint32_t* p, bool pred) {
  uint32_t r = 0u;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.u32 %0, [%1];\n}\n"
               : "+r"(r)
               : "l"(p), "r"((int)pred));
  return r;
}
template <typename V> __device__ __forceinline__ V bits_to(uint32_t u);
template <> __device__ __forceinline__ float bits_to<float>(uint32_t u) { return __uint_as_float(u); }
template <> __device__ __forceinline__ int bits_to<int>(uint32_t u) { return (int)u; }

// `src` is the field's base (pool + slot * field stride).
template <typename V, int ND>
__device__ __forceinline__ void nbr_load(const QG& g, const SFTile& tile, const uint32_t* __restrict__ src,
                                         const QuadCtx& x, NbrLoads<V, ND>& L) {
  constexpr int f = ND - 1;
  const int Bf = 1 << g.lb[f];
  {
    const uint32_t nbl = tile.nbr[x.e][2 * f], nbh = tile.nbr[x.e][2 * f + 1];
    const bool inl = x.r[f] > 0, inh = x.r[f] + 4 < Bf;
    const uint32_t ol = inl ? x.off - 1 : nbl + x.j0 + (Bf - 1);
    const uint32_t oh = inh ? x.off + 4 : nbh + x.j0 + 4 - Bf;
    L.lo = bits_to<V>(ld1_if(src + ol, inl || nbl != SG_NO_BLOCK));
    L.hi = bits_to<V>(ld1_if(src + oh, inh || nbh != SG_NO_BLOCK));
  }
#pragma unroll
  for (int a = 0; a < f; a++) {
    int sh = 0;
#pragma unroll
    for (int b = a + 1; b < ND; b++) sh += g.lb[b];
    const int B = 1 << g.lb[a];
    const uint32_t stride = 1u << sh;
#pragma unroll
    for (int s = 0; s < 2; s++) {
      const int d = s ? 1 : -1;
      const uint32_t nb = tile.nbr[x.e][2 * a + s];
      const bool in = (unsigned)(x.r[a] + d) < (unsigned)B;
      const uint32_t off = in ? x.off + d * (int)stride : nb + x.j0 - d * (int)((B - 1) * stride);
      const uint4 u = ld4_if(src + off, in || nb != SG_NO_BLOCK);
      Q4<V>& q = L.row[2 * a + s];
      q.v[0] = bits_to<V>(u.x); q.v[1] = bits_to<V>(u.y); q.v[2] = bits_to<V>(u.z); q.v[3] = bits_to<V>(u.w);
    }
  }
}

template <typename V, int ND>
__device__ __forceinline__ Q4<V> nbr_sum4(const NbrLoads<V, ND>& L, const Q4<V>& c) {
  Q4<V> s;
  s.v[0] = L.lo + c.v[1];
  s.v[1] = c.v[0] + c.v[2];
  s.v[2] = c.v[1] + c.v[3];
  s.v[3] = c.v[2] + L.hi;
#pragma unroll
  for (int r = 0; r < 2 * (ND - 1); r++)
#pragma unroll
    for (int k = 0; k < 4; k++) s.v[k] += L.row[r].v[k];
  return s;
}

// Per-lane fallback of the QUAD path: each active lane through apply_cell.
template <typename V, int ND>
__device__ __forceinline__ void run_lanes(const SFArgs& A, const DOp& op, int o, const SFTile& tile, uint32_t* P,
                                          uint32_t nq, uint32_t lq, bool chunked, uint32_t jbase, uint64_t fs,
                                          const QG& g) {
  V acc = V(0);
  for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
    QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
    if (x.off == SG_NO_BLOCK) continue;
    for (int k = 0; k < 4; k++) {
      if (!((x.amask >> k) & 1u)) continue;
      CellCtx c;
      c.T = &A.T; c.tile = &tile; c.P = P; c.e = x.e; c.j = x.j0 + k; c.fstride = fs;
#pragma unroll
      for (int a = 0; a < 3; a++) c.c[a] = tile.org[x.e][a] + x.r[a];
      c.c[ND - 1] += k;
      acc += apply_cell<V>(A, op, c);
    }
  }
  if (op.op == SG_OP_RESID_NORM2 || op.op == SG_OP_DOT) warp_add<V>(o, acc);
}

template <typename V, int ND, bool PAIR, int GL, class OPS>
__device__ __forceinline__ void run_quads(const SFArgs& A, const OPS& ops, const SFTile& tile, uint32_t* P,
                                          uint32_t nq, uint32_t lq, bool chunked, uint32_t jbase, uint64_t fs) {
  const QG g = make_qg<GL>(A);
  const int nops = ops.size();
#pragma unroll(OPS::kUnroll)
  for (int o = 0; o < nops; o++) {
    decltype(auto) op = ops[o];
    const uint64_t s0 = (uint64_t)op.slot[0] * fs, s1 = (uint64_t)(op.slot[1] < 0 ? 0 : op.slot[1]) * fs,
                   s2 = (uint64_t)(op.slot[2] < 0 ? 0 : op.slot[2]) * fs;
    switch (op.op) {
      case SG_OP_FILL: {
        Q4<V> q;
#pragma unroll
        for (int k = 0; k < 4; k++) q.v[k] = (V)op.p[0];
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off != SG_NO_BLOCK && x.amask) st4<V>(P + s0 + x.off, q, x.amask);
        }
      } break;
      case SG_OP_ADD_CONST:
      case SG_OP_INC:
      case SG_OP_AXPY: {
        const V p0 = (V)op.p[0];
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          Q4<V> q;
          if (op.op == SG_OP_AXPY) {
            Q4<V> xx = ld4<V>(P + s1 + x.off), yy = ld4<V>(P + s2 + x.off);
#pragma unroll
            for (int k = 0; k < 4; k++) q.v[k] = p0 * xx.v[k] + yy.v[k];
          } else {
            q = ld4<V>(P + (op.op == SG_OP_INC ? s0 : s1) + x.off);
#pragma unroll
            for (int k = 0; k < 4; k++) q.v[k] += p0;
          }
          st4<V>(P + s0 + x.off, q, x.amask);
        }
      } break;
      case SG_OP_STENCIL:
      case SG_OP_JACOBI: {
        const bool jac = op.op == SG_OP_JACOBI;
        const V inv = V(1) / (V)(2 * ND);
        const uint32_t* __restrict__ src = P + s1;
        const uint32_t* __restrict__ rhs = P + s2;
        uint32_t* dst = P + s0;
        // (PAIR: two quads per thread per trip, every load issued before the arithmetic)
        for (uint32_t i = threadIdx.x; i < nq; i += (PAIR ? 2 : 1) * SF_TPB) {
          const bool two = PAIR && i + SF_TPB < nq;
          QuadCtx x0 = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          QuadCtx x1 = quad_ctx<ND>(A, g, tile, P, two ? i + SF_TPB : i, lq, chunked, jbase);
          const bool ok0 = x0.off != SG_NO_BLOCK && x0.amask, ok1 = two && x1.off != SG_NO_BLOCK && x1.amask;
          Q4<V> c0, c1, r0, r1;
          NbrLoads<V, ND> L0, L1;
          if (ok0) {
            c0 = ld4<V>(src + x0.off);
            if (jac) r0 = ld4<V>(rhs + x0.off);
            nbr_load<V, ND>(g, tile, src, x0, L0);
          }
          if (ok1) {
            c1 = ld4<V>(src + x1.off);
            if (jac) r1 = ld4<V>(rhs + x1.off);
            nbr_load<V, ND>(g, tile, src, x1, L1);
          }
          if (ok0) {
            Q4<V> s = nbr_sum4<V, ND>(L0, c0);
#pragma unroll
            for (int k = 0; k < 4; k++) s.v[k] = jac ? (r0.v[k] + s.v[k]) * inv : s.v[k] - (V)(2 * ND) * c0.v[k];
            st4<V>(dst + x0.off, s, x0.amask);
          }
          if (ok1) {
            Q4<V> s = nbr_sum4<V, ND>(L1, c1);
#pragma unroll
            for (int k = 0; k < 4; k++) s.v[k] = jac ? (r1.v[k] + s.v[k]) * inv : s.v[k] - (V)(2 * ND) * c1.v[k];
            st4<V>(dst + x1.off, s, x1.amask);
          }
        }
      } break;
      case SG_OP_SMOOTH_RB:
      case SG_OP_RESID_NORM2: {
        // red-black half sweep in place (the updated colour reads only the other
        // colour, so concurrent quads never see a value they depend on change),
        // or the squared residual r - A z (reduction)
        const bool rb = op.op == SG_OP_SMOOTH_RB;
        const V inv = V(1) / (V)(2 * ND);
        const uint32_t* __restrict__ zsrc = P + (rb ? s0 : s2);
        const uint32_t* __restrict__ rsrc = P + s1;
        V acc = V(0);
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          const Q4<V> c = ld4<V>(zsrc + x.off), r = ld4<V>(rsrc + x.off);
          NbrLoads<V, ND> L;
          nbr_load<V, ND>(g, tile, zsrc, x, L);
          const Q4<V> sn = nbr_sum4<V, ND>(L, c);
          if (rb) {
            int par = 0;
#pragma unroll
            for (int a = 0; a < ND; a++) par += tile.org[x.e][a] + x.r[a];
            Q4<V> out;
#pragma unroll
            for (int k = 0; k < 4; k++) out.v[k] = (((par + k) & 1) == (int)op.p[0]) ? (r.v[k] + sn.v[k]) * inv : c.v[k];
            st4<V>(P + s0 + x.off, out, x.amask);
          } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
              if ((x.amask >> k) & 1u) {
                const V res = r.v[k] - ((V)(2 * ND) * c.v[k] - sn.v[k]);
                acc += res * res;
              }
          }
        }
        if (!rb) warp_add<V>(o, acc);
      } break;
      case SG_OP_DOT: {
        V acc = V(0);
        const V p0 = (V)op.p[0];
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          const Q4<V> a = ld4<V>(P + s1 + x.off), b = ld4<V>(P + s2 + x.off);
#pragma unroll
          for (int k = 0; k < 4; k++)
            if ((x.amask >> k) & 1u) acc += p0 * a.v[k] * b.v[k];
        }
        warp_add<V>(o, acc);
      } break;
      case SG_OP_AXPY_RATIO:
      case SG_OP_XPAY_RATIO: {
        const V ratio = scalar_of<V>(A, op.f[2]) / scalar_of<V>(A, op.f[3]);
        const V p0 = (V)op.p[0];
        const bool axpy = op.op == SG_OP_AXPY_RATIO;
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          const Q4<V> a = ld4<V>(P + s1 + x.off), o0 = ld4<V>(P + s0 + x.off);
          Q4<V> out;
#pragma unroll
          for (int k = 0; k < 4; k++) out.v[k] = axpy ? o0.v[k] + p0 * ratio * a.v[k] : a.v[k] + ratio * o0.v[k];
          st4<V>(P + s0 + x.off, out, x.amask);
        }
      } break;
      case SG_OP_RESTRICT:
      case SG_OP_PROLONG: {
        // the coarse cells of one block lie in ONE coarse block (coarse blocks
        // at least half as wide): resolve it once per block, not per cell
        const bool restrict_ = op.op == SG_OP_RESTRICT;
        const int cf = restrict_ ? 0 : 1;
        const DField& CF = A.C.fields[op.f[cf]];
        const DTree& T2 = A.C.trees[CF.tree];
        bool fast = !T2.leaf_bitmasked && T2.driving >= 0 && T2.nd == ND;
#pragma unroll
        for (int a = 0; a < ND; a++) fast = fast && T2.lev[T2.driving].lbelow[a] + 1 >= g.lb[a];
        if (!fast) {
          run_lanes<V, ND>(A, op, o, tile, P, nq, lq, chunked, jbase, fs, g);
          break;
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < tile.ne; e += SF_TPB) {
          uint32_t off = SG_NO_BLOCK;
          if (tile.blk[e] != SG_NO_BLOCK) {
            const int h[3] = {tile.org[e][0] >> 1, tile.org[e][1] >> 1, tile.org[e][2] >> 1};
            uint32_t idx;
            uint32_t* cont;
            if (restrict_ && (op.act & 1u)) cont = activate_walk(A.C, T2, h, idx, A.task);
            else cont = locate(T2, h, idx);
            if (cont) off = (uint32_t)(cont - T2.seg[T2.nseg - 1].base) + T2.payload_off + (idx & ~((1u << T2.lblk) - 1u));
            else if (restrict_ && A.C.debug) set_err(A.C, SG_ERR_DEMOTION_TRAP, A.task);
          }
          const_cast<SFTile&>(tile).aux[e] = off;
        }
        __syncthreads();
        uint32_t* cpool = T2.seg[T2.nseg - 1].base + ((uint64_t)CF.slot << T2.ln_leaf);
        const uint32_t* __restrict__ zsrc = P + s2;
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          const uint32_t cb = tile.aux[x.e];
          int h[3];
#pragma unroll
          for (int a = 0; a < 3; a++) h[a] = (tile.org[x.e][a] + x.r[a]) >> 1;
          if (restrict_) {
            if (cb == SG_NO_BLOCK) continue;
            const Q4<V> r = ld4<V>(P + s1 + x.off), c = ld4<V>(zsrc + x.off);
            NbrLoads<V, ND> L;
            nbr_load<V, ND>(g, tile, zsrc, x, L);
            const Q4<V> sn = nbr_sum4<V, ND>(L, c);
            V res[4];
#pragma unroll
            for (int k = 0; k < 4; k++)
              res[k] = ((x.amask >> k) & 1u) ? (V)op.p[0] * (r.v[k] - ((V)(2 * ND) * c.v[k] - sn.v[k])) : V(0);
            // lanes (0,1) and (2,3) share a coarse cell along the fast axis
#pragma unroll
            for (int pr = 0; pr < 2; pr++) {
              int hc[3] = {h[0], h[1], h[2]};
              hc[ND - 1] = (tile.org[x.e][ND - 1] + x.r[ND - 1] + 2 * pr) >> 1;
              if ((x.amask >> (2 * pr)) & 3u)
                atomic_add_v(cpool + cb + inblock_idx(T2, hc), res[2 * pr] + res[2 * pr + 1]);
            }
          } else {
            Q4<V> out = ld4<V>(P + s0 + x.off);
#pragma unroll
            for (int pr = 0; pr < 2; pr++) {
              int hc[3] = {h[0], h[1], h[2]};
              hc[ND - 1] = (tile.org[x.e][ND - 1] + x.r[ND - 1] + 2 * pr) >> 1;
              const V cv = cb == SG_NO_BLOCK ? V(0) : ldv<V>(cpool + cb + inblock_idx(T2, hc));
              out.v[2 * pr] += cv;
              out.v[2 * pr + 1] += cv;
            }
            st4<V>(P + s0 + x.off, out, x.amask);
          }
        }
      } break;
      case SG_OP_REDUCE_SUM: {
        V acc = V(0);
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || !x.amask) continue;
          Q4<V> q = ld4<V>(P + s1 + x.off);
#pragma unroll
          for (int k = 0; k < 4; k++)
            if ((x.amask >> k) & 1u) acc += q.v[k];
        }
        warp_add<V>(o, acc);
      } break;
      case SG_OP_HALO_PACK: {
        int nf = 0;
        while (nf < 8 && op.f[nf] >= 0) nf++;
        halo_pack_slots(A.C, op, const_cast<SFTile&>(tile), A.task);
        const uint32_t lblk = lq + 2;
        for (uint32_t e = threadIdx.x; e < tile.ne; e += SF_TPB)
          if (tile.slot[e] >= 0) {
            uint32_t* r = halo_rec(A.C, op, tile.slot[e], lblk, nf);
            r[0] = (uint32_t)tile.org[e][0]; r[1] = (uint32_t)tile.org[e][1]; r[2] = (uint32_t)tile.org[e][2]; r[3] = 0u;
          }
        for (uint32_t i = threadIdx.x; i < nq; i += SF_TPB) {
          QuadCtx x = quad_ctx<ND>(A, g, tile, P, i, lq, chunked, jbase);
          if (x.off == SG_NO_BLOCK || tile.slot[x.e] < 0) continue;
          uint32_t* r = halo_rec(A.C, op, tile.slot[x.e], lblk, nf) + 4 + x.j0;
          for (int k = 0; k < nf; k++)
            *reinterpret_cast<uint4*>(r + ((uint64_t)k << lblk)) =
                *reinterpret_cast<const uint4*>(P + (uint64_t)op.slot[k] * fs + x.off);
        }
      } break;
      default:
        // per-lane ops (DOWNSAMPLE, JITTER, GRID_OP)
        run_lanes<V, ND>(A, op, o, tile, P, nq, lq, chunked, jbase, fs, g);
        break;
    }
  }
}

template <typename V, class OPS>
__device__ __forceinline__ void run_cells(const SFArgs& A, const OPS& ops, const SFTile& tile, uint32_t* P,
                                          uint32_t tcells, bool chunked, uint32_t jbase, uint64_t fs) {
  const DTree& T = A.T;
  const int lblk = T.lblk;
  const int nops = ops.size();
#pragma unroll(OPS::kUnroll)
  for (int o = 0; o < nops; o++) {
    decltype(auto) op = ops[o];
    V acc = V(0);
    if (op.op == SG_OP_HALO_PACK) {
      int nf = 0;
      while (nf < 8 && op.f[nf] >= 0) nf++;
      halo_pack_slots(A.C, op, const_cast<SFTile&>(tile), A.task);
      for (uint32_t e = threadIdx.x; e < tile.ne; e += SF_TPB)
        if (tile.slot[e] >= 0) {
          uint32_t* r = halo_rec(A.C, op, tile.slot[e], lblk, nf);
          r[0] = (uint32_t)tile.org[e][0]; r[1] = (uint32_t)tile.org[e][1]; r[2] = (uint32_t)tile.org[e][2]; r[3] = 0u;
        }
      for (uint32_t i = threadIdx.x; i < tcells; i += SF_TPB) {
        const int e = chunked ? 0 : (int)(i >> lblk);
        const uint32_t j = chunked ? jbase + i : (i & ((1u << lblk) - 1u));
        if (tile.blk[e] == SG_NO_BLOCK || tile.slot[e] < 0) continue;
        uint32_t* r = halo_rec(A.C, op, tile.slot[e], lblk, nf) + 4 + j;
        for (int k = 0; k < nf; k++) r[(uint64_t)k << lblk] = P[tile.blk[e] + (uint64_t)op.slot[k] * fs + j];
      }
      continue;
    }
    for (uint32_t i = threadIdx.x; i < tcells; i += SF_TPB) {
      CellCtx x;
      x.T = &T;
      x.tile = &tile;
      x.P = P;
      x.e = chunked ? 0 : (int)(i >> lblk);
      x.j = chunked ? jbase + i : (i & ((1u << lblk) - 1u));
      x.fstride = fs;
      if (tile.blk[x.e] == SG_NO_BLOCK) continue;
      if (T.leaf_bitmasked) {
        uint32_t li = (tile.first[x.e] & 31u) + x.j;
        if (!((P[tile.maskw[x.e] + (li >> 5)] >> (li & 31)) & 1u)) continue;
      }
      int bc[3];
      inblock_coords(T, x.j, bc);
      x.c[0] = tile.org[x.e][0] + bc[0];
      x.c[1] = tile.org[x.e][1] + bc[1];
      x.c[2] = tile.org[x.e][2] + bc[2];
      acc += apply_cell<V>(A, op, x);
    }
    if (op.op == SG_OP_REDUCE_SUM || op.op == SG_OP_RESID_NORM2 || op.op == SG_OP_DOT) warp_add<V>(o, acc);
  }
}

// ---------------------------------------------------------------------------
// the kernels
// ---------------------------------------------------------------------------
// One pass over every tile of the list with the given op list.
template <typename V, int ND, bool PAIR, int GL, class OPS>
__device__ __forceinline__ void sf_tiles(const SFArgs& A, const OPS& ops, SFTile& tile, bool rows_ok,
                                         bool tile_cached = false) {
  const DTree& T = A.T;
  uint32_t* P = T.seg[T.nseg - 1].base;
  const uint32_t nent = A.entries ? *A.count : 1u;
  const int lblk = T.lblk;
  const bool chunked = lblk > A.ltile;
  uint64_t ntiles;
  uint32_t tiles_per_entry = 1, ept = 1;
  if (chunked) {
    tiles_per_entry = 1u << (lblk - A.ltile);
    ntiles = (uint64_t)nent * tiles_per_entry;
  } else {
    // entries per tile from the device-side count: k equal waves of tiles over
    // the resident grid (no wave-quantization tail), at most SF_MAXE and at
    // most 2^lept entries per tile
    const uint32_t G = gridDim.x, cap = min((uint32_t)SF_MAXE, 1u << A.lept);
    const uint32_t k = max(1u, (nent + cap * G - 1) / (cap * G));
    ept = max(1u, (nent + k * G - 1) / (k * G));
    ntiles = ((uint64_t)nent + ept - 1) / ept;
  }
  const uint64_t fs = 1ull << T.ln_leaf;

  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint32_t e0, ne, jbase = 0, tcells;
    if (chunked) {
      e0 = (uint32_t)(t / tiles_per_entry);
      ne = 1;
      jbase = (uint32_t)(t % tiles_per_entry) << A.ltile;
      tcells = 1u << A.ltile;
    } else {
      e0 = (uint32_t)t * ept;
      ne = min(ept, nent - e0);
      tcells = ne << lblk;
    }
    // the tile's blocks: one coalesced read of the list's block table, or --
    // first struct-for after a listgen -- built here (tree walks spread over
    // every CTA) and stored for the following launches.  In a chain whose
    // tiles all fit in one wave, every phase reuses the CTA's tile as loaded.
    if (tile_cached && ntiles <= gridDim.x) {
      // shared memory already holds tile t == blockIdx.x from the previous phase
    } else if (A.entries && rows_ok) {
      for (uint32_t i = threadIdx.x; i < ne; i += SF_TPB) {
        const BlockRow r = A.table[e0 + i];
        tile.blk[i] = r.blk;
        tile.maskw[i] = r.maskw;
        tile.first[i] = r.first;
        tile.org[i][0] = r.org[0]; tile.org[i][1] = r.org[1]; tile.org[i][2] = r.org[2];
#pragma unroll
        for (int d = 0; d < 6; d++) tile.nbr[i][d] = r.nbr[d];
      }
      if (threadIdx.x == 0) tile.ne = ne;
    } else if (A.entries) {
      // build the rows: resolve every entry, then one tree walk per (entry, face)
      const uint32_t* base = T.seg[T.nseg - 1].base;
      for (uint32_t i = threadIdx.x; i < ne; i += SF_TPB) {
        uint32_t* cont;
        uint32_t first;
        int org[3];
        bool ok = resolve_entry(T, A.entries[e0 + i], cont, first, org);
        tile.blk[i] = ok ? (uint32_t)(cont - base) + T.payload_off + first : SG_NO_BLOCK;
        tile.maskw[i] = ok && T.leaf_bitmasked ? (uint32_t)(cont - base) + T.lev[T.nlev - 1].mask_off + (first >> 5) : 0u;
        tile.first[i] = first;
        tile.org[i][0] = org[0]; tile.org[i][1] = org[1]; tile.org[i][2] = org[2];
      }
      if (threadIdx.x == 0) tile.ne = ne;
      __syncthreads();
      const uint32_t lowmask = ~((1u << lblk) - 1u);
      for (uint32_t i = threadIdx.x; i < ne * 6; i += SF_TPB) {
        const uint32_t e = i / 6;
        const int dir = i % 6, axis = dir >> 1;
        uint32_t nb = SG_NO_BLOCK;
        if (axis < T.nd && tile.blk[e] != SG_NO_BLOCK && T.driving >= 0) {
          int q[3] = {tile.org[e][0], tile.org[e][1], tile.org[e][2]};
          q[axis] += (dir & 1) ? (1 << T.lev[T.driving].lbelow[axis]) : -1;
          if (in_domain(T, q)) {
            uint32_t idx;
            uint32_t* c2 = locate(T, q, idx);
            if (c2) nb = (uint32_t)(c2 - base) + T.payload_off + (idx & lowmask);
          }
        }
        tile.nbr[e][dir] = nb;
      }
      __syncthreads();
      if (A.table)
        for (uint32_t i = threadIdx.x; i < ne; i += SF_TPB) {
          BlockRow r;
          r.blk = tile.blk[i]; r.maskw = tile.maskw[i]; r.first = tile.first[i];
          r.org[0] = tile.org[i][0]; r.org[1] = tile.org[i][1]; r.org[2] = tile.org[i][2];
#pragma unroll
          for (int d = 0; d < 6; d++) r.nbr[d] = tile.nbr[i][d];
          A.table[e0 + i] = r;
        }
    } else if (threadIdx.x == 0) {   // no driving level: the single root block
      tile.ne = 1;
      tile.blk[0] = (uint32_t)T.payload_off;
      tile.maskw[0] = T.leaf_bitmasked ? T.lev[T.nlev - 1].mask_off : 0u;
      tile.first[0] = 0;
      tile.org[0][0] = tile.org[0][1] = tile.org[0][2] = 0;
#pragma unroll
      for (int d = 0; d < 6; d++) tile.nbr[0][d] = SG_NO_BLOCK;
    }
    __syncthreads();
    if (ND > 0)
      run_quads<V, (ND > 0 ? ND : 1), PAIR, GL>(A, ops, tile, P, tcells >> 2, (uint32_t)lblk - 2, chunked, jbase,
                                                fs);
    else run_cells<V>(A, ops, tile, P, tcells, chunked, jbase, fs);
    __syncthreads();
  }
}

// Marks the block table built (last CTA) when this launch built it.
__device__ __forceinline__ void sf_mark_table(const SFArgs& A, bool rows_ok) {
  if (A.table && !rows_ok && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&A.table_ctl[3], 1u) == gridDim.x - 1) {
      A.table_ctl[3] = 0u;
      __threadfence();
      A.table_ctl[4] = 1u;
    }
  }
}

// ND = 0: GENERIC cell path; 1..3: QUAD path.  PAIR: two stencil quads in
// flight per thread (more registers, fewer resident CTAs).
// GL: 0 runtime block shape, 1 = 8^3, 2 = 4^3, 3 = 4x4 (constant index math).
template <typename V, int ND, bool PAIR, int GL>
__global__ void __launch_bounds__(SF_TPB, PAIR ? 3 : 5) k_struct_for(const __grid_constant__ SFArgs A) {
  __shared__ SFTile tile;
  if (A.has_reduce && threadIdx.x < SG_MAXOPS) s_red[threadIdx.x] = 0.0;
  const bool rows_ok = A.table && A.table_ctl[4] != 0u;   // set by an earlier launch
  const OpsRT ops{A.ops, A.nops};
  sf_tiles<V, ND, PAIR, GL>(A, ops, tile, rows_ok);
  if (A.has_reduce) finish_reductions<V>(A, ops);
  sf_mark_table(A, rows_ok);
}

// Beyond the paper (SG_PASS_CHAIN): a chain of struct-for phases
// over one SMALL list in ONE launch of ONE CTA; phase p+1 starts after a CTA
// barrier, so dependent stencils (the multigrid bottom smoother's 64 half
// sweeps) chain without a kernel boundary.  The op table travels in the
// kernel parameters (graph-capturable, no upload); reductions are allowed in
// the last phase only (their aux / s_red slots are that phase's).  Larger
// lists launch their phases one by one (sg_api.cu: a grid-wide barrier costs
// more than a graph-replayed launch).
constexpr int SG_CHAIN_OPS = 96;
struct ChainTab {
  DOp ops[SG_CHAIN_OPS];
  int phase_end[SG_CHAIN_OPS];
  int nphases;
};

template <typename V, int ND, bool PAIR, int GL>
__global__ void __launch_bounds__(SF_TPB, 1)
    k_struct_chain(const __grid_constant__ SFArgs A, const __grid_constant__ ChainTab CT) {
  __shared__ SFTile tile;
  if (A.has_reduce && threadIdx.x < SG_MAXOPS) s_red[threadIdx.x] = 0.0;
  const bool rows_ok0 = A.table && A.table_ctl[4] != 0u;
  int begin = 0;
  int last_n = 0;
  for (int p = 0; p < CT.nphases; p++) {
    const int end = CT.phase_end[p], n = end - begin;
    // rows built by phase 0 are visible to the later phases after the barrier
    sf_tiles<V, ND, PAIR, GL>(A, OpsRT{CT.ops + begin, n}, tile, rows_ok0 || p > 0, p > 0);
    last_n = n;
    if (p + 1 < CT.nphases) {
      __syncthreads();
      begin = end;
    }
  }
  if (A.has_reduce) finish_reductions<V>(A, OpsRT{CT.ops + begin, last_n});
  sf_mark_table(A, rows_ok0);
}

// ---------------------------------------------------------------------------
// Dedicated JACOBI for 8^3 dense leaf blocks (C2, JAC-XL): a lone f32 JACOBI
// op is the solve's hot loop (89% of the C2 step), so it gets a kernel without
// the op-table interpreter or shared-memory tiles.  One warp per half block
// (two quads of 4 cells along z per lane, 64 per warp).
// Block rows (block + 6 face neighbours) come from the list's block table (one
// 12-word row read by 12 lanes, broadcast by shuffles); the fast-axis
// neighbours inside the block come from the partner lane by one shuffle, the
// rest are uint4 rows (in-block, or the neighbour block's facing plane,
// predicated off -- reading 0 -- when the neighbour is absent).
// Same arithmetic order as the interpreter's quad path.
// ---------------------------------------------------------------------------
struct JacArgs {
  DTree T;
  const uint32_t* entries;
  const uint32_t* count;
  BlockRow* table;
  uint32_t* table_ctl;
  uint64_t s_dst, s_src, s_rhs;   // field offsets (words) from the pool base
  float inv;
  // RED: the group JACOBI + REDUCE_SUM(s += dst) fused ("fuse the
  // Jacobi smoothing and reduction kernels"): per-CTA f64 partials, summed in
  // CTA order by the last CTA (deterministic, as finish_reductions)
  uint32_t* red_target;
  double* partials;
  uint32_t* red_done;
};

// out of line: the slow path must not shape the hot loop's register allocation
__device__ __noinline__ void jac_row_slow(const DTree& T, uint32_t entry, BlockRow* out) {
  make_block_row(T, entry, out);
}
// The same row built by the whole warp (every lane calls it with the same entry)
__device__ __noinline__ void jac_row_warp(const DTree& T, uint32_t entry, int lane, BlockRow* out) {
  make_block_row_warp(T, entry, lane, out);
}

__device__ __forceinline__ float4 u2f(uint4 u) {
  return make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w));
}

// One warp's half block of a JACOBI sweep on an 8^3 dense block (k_jacobi8
// and the flag-chained k_jacobi8_flow): a lane owns the quads at
// x0 = 4*part + 2*(lane/16) and x0 + 1 (same y, z-half), their shared x face
// loaded once; every load of both quads issued before the arithmetic.
// Returns the lane's sum of the written values (RED).
template <bool RED>
__device__ __forceinline__ double jac8_half(const uint32_t* __restrict__ src, const uint32_t* __restrict__ rhs,
                                            uint32_t* dst, uint32_t blk, const uint32_t (&nb)[6], uint32_t part,
                                            int lane, float inv) {
  double acc = 0.0;
  const int xp2 = (lane >> 4) * 2, y = (lane >> 1) & 7, zh = lane & 1;
  const int x0 = (int)part * 4 + xp2;
  const uint32_t j0 = ((uint32_t)x0 << 6) | ((uint32_t)y << 3) | ((uint32_t)zh << 2), j1 = j0 + 64u;
  const uint32_t o0 = blk + j0, o1 = o0 + 64u;
  // every load of both quads issued before the arithmetic
  const uint4 c0u = *reinterpret_cast<const uint4*>(src + o0);
  const uint4 c1u = *reinterpret_cast<const uint4*>(src + o1);
  const uint4 r0u = *reinterpret_cast<const uint4*>(rhs + o0);
  const uint4 r1u = *reinterpret_cast<const uint4*>(rhs + o1);
  const uint32_t nz = zh ? nb[5] : nb[4];
  const uint32_t zo = zh ? 0u : 7u;
  const float z0 = __uint_as_float(ld1_if(src + nz + (j0 & ~7u) + zo, nz != SG_NO_BLOCK));
  const float z1 = __uint_as_float(ld1_if(src + nz + (j1 & ~7u) + zo, nz != SG_NO_BLOCK));
  const uint4 xmu = ld4_if(src + (x0 > 0 ? o0 - 64u : nb[0] + j0 + 448u), x0 > 0 || nb[0] != SG_NO_BLOCK);
  const uint4 xpu = ld4_if(src + (x0 + 1 < 7 ? o1 + 64u : nb[1] + j1 - 448u), x0 + 1 < 7 || nb[1] != SG_NO_BLOCK);
  const bool ym_in = y > 0, yp_in = y < 7;
  const uint32_t ym0 = ym_in ? o0 - 8u : nb[2] + j0 + 56u, yp0 = yp_in ? o0 + 8u : nb[3] + j0 - 56u;
  const uint4 ym0u = ld4_if(src + ym0, ym_in || nb[2] != SG_NO_BLOCK);
  const uint4 yp0u = ld4_if(src + yp0, yp_in || nb[3] != SG_NO_BLOCK);
  const uint4 ym1u = ld4_if(src + ym0 + 64u, ym_in || nb[2] != SG_NO_BLOCK);
  const uint4 yp1u = ld4_if(src + yp0 + 64u, yp_in || nb[3] != SG_NO_BLOCK);
  const float4 c0 = u2f(c0u), c1 = u2f(c1u);
  const float p0 = __shfl_xor_sync(0xffffffffu, zh ? c0.x : c0.w, 1);
  const float p1 = __shfl_xor_sync(0xffffffffu, zh ? c1.x : c1.w, 1);
  {
    const float lo = zh ? p0 : z0, hi = zh ? z0 : p0;
    const float4 xm = u2f(xmu), xp = c1, ym = u2f(ym0u), yp = u2f(yp0u), r = u2f(r0u);
    float s0 = lo + c0.y, s1 = c0.x + c0.z, s2 = c0.y + c0.w, s3 = c0.z + hi;
    s0 += xm.x; s1 += xm.y; s2 += xm.z; s3 += xm.w;
    s0 += xp.x; s1 += xp.y; s2 += xp.z; s3 += xp.w;
    s0 += ym.x; s1 += ym.y; s2 += ym.z; s3 += ym.w;
    s0 += yp.x; s1 += yp.y; s2 += yp.z; s3 += yp.w;
    const float4 out = make_float4((r.x + s0) * inv, (r.y + s1) * inv, (r.z + s2) * inv, (r.w + s3) * inv);
    *reinterpret_cast<uint4*>(dst + o0) = make_uint4(__float_as_uint(out.x), __float_as_uint(out.y),
                                                     __float_as_uint(out.z), __float_as_uint(out.w));
    if (RED) acc += (double)(((out.x + out.y) + out.z) + out.w);
  }
  {
    const float lo = zh ? p1 : z1, hi = zh ? z1 : p1;
    const float4 xm = c0, xp = u2f(xpu), ym = u2f(ym1u), yp = u2f(yp1u), r = u2f(r1u);
    float s0 = lo + c1.y, s1 = c1.x + c1.z, s2 = c1.y + c1.w, s3 = c1.z + hi;
    s0 += xm.x; s1 += xm.y; s2 += xm.z; s3 += xm.w;
    s0 += xp.x; s1 += xp.y; s2 += xp.z; s3 += xp.w;
    s0 += ym.x; s1 += ym.y; s2 += ym.z; s3 += ym.w;
    s0 += yp.x; s1 += yp.y; s2 += yp.z; s3 += yp.w;
    const float4 out = make_float4((r.x + s0) * inv, (r.y + s1) * inv, (r.z + s2) * inv, (r.w + s3) * inv);
    *reinterpret_cast<uint4*>(dst + o1) = make_uint4(__float_as_uint(out.x), __float_as_uint(out.y),
                                                     __float_as_uint(out.z), __float_as_uint(out.w));
    if (RED) acc += (double)(((out.x + out.y) + out.z) + out.w);
  }
  return acc;
}

// A quarter block (x in [2 part, 2 part + 2)) per warp: one quad per lane;
// lanes l and l ^ 16 hold x-adjacent quads, so each lane loads only its OUTER
// x neighbour and takes the inner one from its partner (same loads per cell
// as jac8_half, twice the units: 13,120 on C2 instead of 6,560 over 4,736
// resident warps).  Same float operations in the same order as jac8_half.
template <bool RED>
__device__ __forceinline__ double jac8_quarter(const uint32_t* __restrict__ src, const uint32_t* __restrict__ rhs,
                                               uint32_t* dst, uint32_t blk, const uint32_t (&nb)[6], uint32_t part,
                                               int lane, float inv) {
  const int xh = lane >> 4, x = (int)part * 2 + xh, y = (lane >> 1) & 7, zh = lane & 1;
  const uint32_t j = ((uint32_t)x << 6) | ((uint32_t)y << 3) | ((uint32_t)zh << 2);
  const uint32_t o = blk + j;
  const uint4 cu = *reinterpret_cast<const uint4*>(src + o);
  const uint4 ru = *reinterpret_cast<const uint4*>(rhs + o);
  const uint32_t nz = zh ? nb[5] : nb[4];
  const uint32_t zo = zh ? 0u : 7u;
  const float zv = __uint_as_float(ld1_if(src + nz + (j & ~7u) + zo, nz != SG_NO_BLOCK));
  // outer x neighbour: x - 1 for the lower lane half, x + 1 for the upper
  const bool xin = xh ? x < 7 : x > 0;
  const uint32_t xnb = xh ? nb[1] : nb[0];
  const uint4 xou = ld4_if(src + (xin ? (xh ? o + 64u : o - 64u) : (xh ? xnb + j - 448u : xnb + j + 448u)),
                           xin || xnb != SG_NO_BLOCK);
  const bool ym_in = y > 0, yp_in = y < 7;
  const uint4 ymu = ld4_if(src + (ym_in ? o - 8u : nb[2] + j + 56u), ym_in || nb[2] != SG_NO_BLOCK);
  const uint4 ypu = ld4_if(src + (yp_in ? o + 8u : nb[3] + j - 56u), yp_in || nb[3] != SG_NO_BLOCK);
  const float4 c = u2f(cu);
  const float p = __shfl_xor_sync(0xffffffffu, zh ? c.x : c.w, 1);
  float4 pc;   // the partner's quad: the inner x neighbour
  pc.x = __shfl_xor_sync(0xffffffffu, c.x, 16);
  pc.y = __shfl_xor_sync(0xffffffffu, c.y, 16);
  pc.z = __shfl_xor_sync(0xffffffffu, c.z, 16);
  pc.w = __shfl_xor_sync(0xffffffffu, c.w, 16);
  const float4 xo = u2f(xou);
  const float4 xm = xh ? pc : xo, xp = xh ? xo : pc, ym = u2f(ymu), yp = u2f(ypu), r = u2f(ru);
  const float lo = zh ? p : zv, hi = zh ? zv : p;
  float s0 = lo + c.y, s1 = c.x + c.z, s2 = c.y + c.w, s3 = c.z + hi;
  s0 += xm.x; s1 += xm.y; s2 += xm.z; s3 += xm.w;
  s0 += xp.x; s1 += xp.y; s2 += xp.z; s3 += xp.w;
  s0 += ym.x; s1 += ym.y; s2 += ym.z; s3 += ym.w;
  s0 += yp.x; s1 += yp.y; s2 += yp.z; s3 += yp.w;
  const float4 out = make_float4((r.x + s0) * inv, (r.y + s1) * inv, (r.z + s2) * inv, (r.w + s3) * inv);
  *reinterpret_cast<uint4*>(dst + o) =
      make_uint4(__float_as_uint(out.x), __float_as_uint(out.y), __float_as_uint(out.z), __float_as_uint(out.w));
  return RED ? (double)(((out.x + out.y) + out.z) + out.w) : 0.0;
}

// Deterministic end of a fused JACOBI + REDUCE_SUM (k_jacobi8<true>,
// k_jacobi8_flow<true>): per-CTA f64 partials summed in CTA order by the last
// CTA into the 0-D target.
__device__ __forceinline__ void jac_reduce_tail(const JacArgs& A, double acc) {
  const int lane = threadIdx.x & 31;
  __shared__ double s_acc;
  __shared__ bool s_last;
  __shared__ double s_sum[256];
  if (threadIdx.x == 0) s_acc = 0.0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc != 0.0) atomicAdd(&s_acc, acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    A.partials[blockIdx.x] = s_acc;
    __threadfence();
    s_last = atomicAdd(A.red_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double t = 0.0;   // fixed-order tree sum over CTAs
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 256) t += __ldcg(&A.partials[b]);
    s_sum[threadIdx.x] = t;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (threadIdx.x < w) s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const float old = __uint_as_float(*A.red_target);
      *A.red_target = __float_as_uint((float)((double)old + s_sum[0]));
      *A.red_done = 0u;
    }
  }
}

#ifndef SG_JAC8_QUARTER
#define SG_JAC8_QUARTER 0   // k_jacobi8 unit: 0 half block per warp, 1 quarter block
#endif
#ifndef SG_JAC8_MINB
#define SG_JAC8_MINB 4   // CTAs per SM k_jacobi8 is register-sized for (grid = SMs x this)
#endif
template <bool RED>
__global__ void __launch_bounds__(256, SG_JAC8_MINB) k_jacobi8(const __grid_constant__ JacArgs A) {
  double acc = 0.0;
  const uint32_t* P = A.T.seg[A.T.nseg - 1].base;
  const uint32_t* __restrict__ src = P + A.s_src;
  const uint32_t* __restrict__ rhs = P + A.s_rhs;
  uint32_t* dst = const_cast<uint32_t*>(P) + A.s_dst;
  const uint32_t nent = *A.count;
  const bool rows_ok = A.table_ctl[4] != 0u;   // set by an earlier launch
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), GW = gridDim.x * (blockDim.x >> 5);
  // one warp per half block (jac8_half) or per quarter block (jac8_quarter)
  constexpr uint32_t UPB = SG_JAC8_QUARTER ? 4u : 2u, USH = SG_JAC8_QUARTER ? 2u : 1u;
  for (uint32_t wq = gw; wq < nent * UPB; wq += GW) {
    const uint32_t e = wq >> USH, part = wq & (UPB - 1u);
    uint32_t blk, nb[6];
    if (rows_ok) {
      const uint32_t rv = lane < 12 ? reinterpret_cast<const uint32_t*>(A.table + e)[lane] : 0u;
      blk = __shfl_sync(0xffffffffu, rv, 0);
#pragma unroll
      for (int d = 0; d < 6; d++) nb[d] = __shfl_sync(0xffffffffu, rv, 6 + d);
    } else {
      // no table yet (first struct-for after a listgen): every lane resolves
      // the row; the part-0 warp stores it for the following launches
      BlockRow r;
      jac_row_warp(A.T, A.entries[e], lane, &r);
      if (part == 0 && lane == 0) A.table[e] = r;
      blk = r.blk;
#pragma unroll
      for (int d = 0; d < 6; d++) nb[d] = r.nbr[d];
    }
    if (blk == SG_NO_BLOCK) continue;
    if (SG_JAC8_QUARTER) acc += jac8_quarter<RED>(src, rhs, dst, blk, nb, part, lane, A.inv);
    else acc += jac8_half<RED>(src, rhs, dst, blk, nb, part, lane, A.inv);
  }
  if (RED) jac_reduce_tail(A, acc);
  // the rows built here (no table yet) become the list's block table
  if (!rows_ok) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&A.table_ctl[3], 1u) == gridDim.x - 1) {
        A.table_ctl[3] = 0u;
        __threadfence();
        A.table_ctl[4] = 1u;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Streaming kernel for fused groups of quad ops on 8^3 dense blocks (the
// k_jacobi8 structure for any group of FILL / ADD_CONST / INC / AXPY /
// STENCIL / JACOBI / REDUCE_SUM / DOT / AXPY_RATIO / XPAY_RATIO): one warp per
// half block, a lane owns two quads, block rows by shuffles from the table,
// no shared-memory tiles and no CTA barriers in the loop.  Ops run in group
// order on the lane's quads; an identity operand written by an earlier op of
// the group is re-read by the same thread (L1).  Reductions go through the
// interpreter's warp_add / finish_reductions (deterministic per-CTA f64
// partials).  Same arithmetic order as the quad path.  Used by the launcher
// (OpsRT) and by the JIT-specialized kernels (OpsJit).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool stream8_op(int op) {
  return op == SG_OP_FILL || op == SG_OP_ADD_CONST || op == SG_OP_INC || op == SG_OP_AXPY || op == SG_OP_STENCIL ||
         op == SG_OP_JACOBI || op == SG_OP_REDUCE_SUM || op == SG_OP_DOT || op == SG_OP_AXPY_RATIO ||
         op == SG_OP_XPAY_RATIO;
}

__device__ __forceinline__ void st4f(uint32_t* p, float a, float b, float c, float d) {
  *reinterpret_cast<uint4*>(p) = make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d));
}

// Neighbour sums of the lane's two quads of field `src` (k_jacobi8's loads and
// order): s[q][k] = sum of the 6 face neighbours of cell k of quad q.
__device__ __forceinline__ void stream8_nbr(const uint32_t* __restrict__ src, uint32_t o0, uint32_t o1, uint32_t j0,
                                            uint32_t j1, int x0, int y, int zh, const uint32_t nb[6], float4& c0,
                                            float4& c1, float s[2][4]) {
  const uint4 c0u = *reinterpret_cast<const uint4*>(src + o0);
  const uint4 c1u = *reinterpret_cast<const uint4*>(src + o1);
  const uint32_t nz = zh ? nb[5] : nb[4];
  const uint32_t zo = zh ? 0u : 7u;
  const float z0 = __uint_as_float(ld1_if(src + nz + (j0 & ~7u) + zo, nz != SG_NO_BLOCK));
  const float z1 = __uint_as_float(ld1_if(src + nz + (j1 & ~7u) + zo, nz != SG_NO_BLOCK));
  const uint4 xmu = ld4_if(src + (x0 > 0 ? o0 - 64u : nb[0] + j0 + 448u), x0 > 0 || nb[0] != SG_NO_BLOCK);
  const uint4 xpu = ld4_if(src + (x0 + 1 < 7 ? o1 + 64u : nb[1] + j1 - 448u), x0 + 1 < 7 || nb[1] != SG_NO_BLOCK);
  const bool ym_in = y > 0, yp_in = y < 7;
  const uint32_t ym0 = ym_in ? o0 - 8u : nb[2] + j0 + 56u, yp0 = yp_in ? o0 + 8u : nb[3] + j0 - 56u;
  const uint4 ym0u = ld4_if(src + ym0, ym_in || nb[2] != SG_NO_BLOCK);
  const uint4 yp0u = ld4_if(src + yp0, yp_in || nb[3] != SG_NO_BLOCK);
  const uint4 ym1u = ld4_if(src + ym0 + 64u, ym_in || nb[2] != SG_NO_BLOCK);
  const uint4 yp1u = ld4_if(src + yp0 + 64u, yp_in || nb[3] != SG_NO_BLOCK);
  c0 = u2f(c0u);
  c1 = u2f(c1u);
  const float p0 = __shfl_xor_sync(0xffffffffu, zh ? c0.x : c0.w, 1);
  const float p1 = __shfl_xor_sync(0xffffffffu, zh ? c1.x : c1.w, 1);
  {
    const float lo = zh ? p0 : z0, hi = zh ? z0 : p0;
    const float4 xm = u2f(xmu), xp = c1, ym = u2f(ym0u), yp = u2f(yp0u);
    s[0][0] = lo + c0.y; s[0][1] = c0.x + c0.z; s[0][2] = c0.y + c0.w; s[0][3] = c0.z + hi;
    s[0][0] += xm.x; s[0][1] += xm.y; s[0][2] += xm.z; s[0][3] += xm.w;
    s[0][0] += xp.x; s[0][1] += xp.y; s[0][2] += xp.z; s[0][3] += xp.w;
    s[0][0] += ym.x; s[0][1] += ym.y; s[0][2] += ym.z; s[0][3] += ym.w;
    s[0][0] += yp.x; s[0][1] += yp.y; s[0][2] += yp.z; s[0][3] += yp.w;
  }
  {
    const float lo = zh ? p1 : z1, hi = zh ? z1 : p1;
    const float4 xm = c0, xp = u2f(xpu), ym = u2f(ym1u), yp = u2f(yp1u);
    s[1][0] = lo + c1.y; s[1][1] = c1.x + c1.z; s[1][2] = c1.y + c1.w; s[1][3] = c1.z + hi;
    s[1][0] += xm.x; s[1][1] += xm.y; s[1][2] += xm.z; s[1][3] += xm.w;
    s[1][0] += xp.x; s[1][1] += xp.y; s[1][2] += xp.z; s[1][3] += xp.w;
    s[1][0] += ym.x; s[1][1] += ym.y; s[1][2] += ym.z; s[1][3] += ym.w;
    s[1][0] += yp.x; s[1][1] += yp.y; s[1][2] += yp.z; s[1][3] += yp.w;
  }
}

template <class OPS>
__device__ __forceinline__ void stream8_body(const SFArgs& A, const OPS& ops) {
  uint32_t* P = A.T.seg[A.T.nseg - 1].base;
  const uint64_t fs = 1ull << A.T.ln_leaf;
  const uint32_t nent = *A.count;
  const bool rows_ok = A.table_ctl[4] != 0u;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), GW = gridDim.x * (blockDim.x >> 5);
  const int xp2 = (lane >> 4) * 2, y = (lane >> 1) & 7, zh = lane & 1;
  const int nops = ops.size();
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
      make_block_row_warp(A.T, A.entries[e], lane, &r);
      if (part == 0 && lane == 0) A.table[e] = r;
      blk = r.blk;
#pragma unroll
      for (int d = 0; d < 6; d++) nb[d] = r.nbr[d];
    }
    if (blk == SG_NO_BLOCK) continue;
    const int x0 = (int)part * 4 + xp2;
    const uint32_t j0 = ((uint32_t)x0 << 6) | ((uint32_t)y << 3) | ((uint32_t)zh << 2), j1 = j0 + 64u;
    const uint32_t o0 = blk + j0, o1 = o0 + 64u;
#pragma unroll(OPS::kUnroll)
    for (int o = 0; o < nops; o++) {
      decltype(auto) op = ops[o];
      uint32_t* f0 = P + (uint64_t)(op.slot[0] < 0 ? 0 : op.slot[0]) * fs;
      const uint32_t* f1 = P + (uint64_t)(op.slot[1] < 0 ? 0 : op.slot[1]) * fs;
      const uint32_t* f2 = P + (uint64_t)(op.slot[2] < 0 ? 0 : op.slot[2]) * fs;
      const float p0 = op.p[0];
      switch (op.op) {
        case SG_OP_FILL:
          st4f(f0 + o0, p0, p0, p0, p0);
          st4f(f0 + o1, p0, p0, p0, p0);
          break;
        case SG_OP_ADD_CONST:
        case SG_OP_INC: {
          const uint32_t* src = op.op == SG_OP_INC ? f0 : f1;
          const float4 a = u2f(*reinterpret_cast<const uint4*>(src + o0)), b = u2f(*reinterpret_cast<const uint4*>(src + o1));
          st4f(f0 + o0, a.x + p0, a.y + p0, a.z + p0, a.w + p0);
          st4f(f0 + o1, b.x + p0, b.y + p0, b.z + p0, b.w + p0);
        } break;
        case SG_OP_AXPY: {
          const float4 a0 = u2f(*reinterpret_cast<const uint4*>(f1 + o0)), a1 = u2f(*reinterpret_cast<const uint4*>(f1 + o1));
          const float4 b0 = u2f(*reinterpret_cast<const uint4*>(f2 + o0)), b1 = u2f(*reinterpret_cast<const uint4*>(f2 + o1));
          st4f(f0 + o0, p0 * a0.x + b0.x, p0 * a0.y + b0.y, p0 * a0.z + b0.z, p0 * a0.w + b0.w);
          st4f(f0 + o1, p0 * a1.x + b1.x, p0 * a1.y + b1.y, p0 * a1.z + b1.z, p0 * a1.w + b1.w);
        } break;
        case SG_OP_STENCIL:
        case SG_OP_JACOBI: {
          float4 c0, c1;
          float s[2][4];
          const bool jac = op.op == SG_OP_JACOBI;
          float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
          if (jac) {
            r0 = u2f(*reinterpret_cast<const uint4*>(f2 + o0));
            r1 = u2f(*reinterpret_cast<const uint4*>(f2 + o1));
          }
          stream8_nbr(f1, o0, o1, j0, j1, x0, y, zh, nb, c0, c1, s);
          const float inv = 1.0f / 6.0f;
          if (jac) {
            st4f(f0 + o0, (r0.x + s[0][0]) * inv, (r0.y + s[0][1]) * inv, (r0.z + s[0][2]) * inv, (r0.w + s[0][3]) * inv);
            st4f(f0 + o1, (r1.x + s[1][0]) * inv, (r1.y + s[1][1]) * inv, (r1.z + s[1][2]) * inv, (r1.w + s[1][3]) * inv);
          } else {
            st4f(f0 + o0, s[0][0] - 6.0f * c0.x, s[0][1] - 6.0f * c0.y, s[0][2] - 6.0f * c0.z, s[0][3] - 6.0f * c0.w);
            st4f(f0 + o1, s[1][0] - 6.0f * c1.x, s[1][1] - 6.0f * c1.y, s[1][2] - 6.0f * c1.z, s[1][3] - 6.0f * c1.w);
          }
        } break;
        case SG_OP_REDUCE_SUM: {
          const float4 a = u2f(*reinterpret_cast<const uint4*>(f1 + o0)), b = u2f(*reinterpret_cast<const uint4*>(f1 + o1));
          float acc = 0.0f;
          acc += a.x; acc += a.y; acc += a.z; acc += a.w;
          acc += b.x; acc += b.y; acc += b.z; acc += b.w;
          warp_add<float>(o, acc);
        } break;
        case SG_OP_DOT: {
          const float4 a0 = u2f(*reinterpret_cast<const uint4*>(f1 + o0)), a1 = u2f(*reinterpret_cast<const uint4*>(f1 + o1));
          const float4 b0 = u2f(*reinterpret_cast<const uint4*>(f2 + o0)), b1 = u2f(*reinterpret_cast<const uint4*>(f2 + o1));
          float acc = 0.0f;
          acc += p0 * a0.x * b0.x; acc += p0 * a0.y * b0.y; acc += p0 * a0.z * b0.z; acc += p0 * a0.w * b0.w;
          acc += p0 * a1.x * b1.x; acc += p0 * a1.y * b1.y; acc += p0 * a1.z * b1.z; acc += p0 * a1.w * b1.w;
          warp_add<float>(o, acc);
        } break;
        case SG_OP_AXPY_RATIO:
        case SG_OP_XPAY_RATIO: {
          const float ratio = scalar_of<float>(A, op.f[2]) / scalar_of<float>(A, op.f[3]);
          const bool ax = op.op == SG_OP_AXPY_RATIO;
          const float4 a0 = u2f(*reinterpret_cast<const uint4*>(f1 + o0)), a1 = u2f(*reinterpret_cast<const uint4*>(f1 + o1));
          const float4 d0 = u2f(*reinterpret_cast<const uint4*>(f0 + o0)), d1 = u2f(*reinterpret_cast<const uint4*>(f0 + o1));
          if (ax) {
            st4f(f0 + o0, d0.x + p0 * ratio * a0.x, d0.y + p0 * ratio * a0.y, d0.z + p0 * ratio * a0.z, d0.w + p0 * ratio * a0.w);
            st4f(f0 + o1, d1.x + p0 * ratio * a1.x, d1.y + p0 * ratio * a1.y, d1.z + p0 * ratio * a1.z, d1.w + p0 * ratio * a1.w);
          } else {
            st4f(f0 + o0, a0.x + ratio * d0.x, a0.y + ratio * d0.y, a0.z + ratio * d0.z, a0.w + ratio * d0.w);
            st4f(f0 + o1, a1.x + ratio * d1.x, a1.y + ratio * d1.y, a1.z + ratio * d1.z, a1.w + ratio * d1.w);
          }
        } break;
        default: break;
      }
    }
  }
  if (!rows_ok) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&A.table_ctl[3], 1u) == gridDim.x - 1) {
        A.table_ctl[3] = 0u;
        __threadfence();
        A.table_ctl[4] = 1u;
      }
    }
  }
}

__global__ void __launch_bounds__(256, 4) k_stream8(const __grid_constant__ SFArgs A) {
  if (A.has_reduce && threadIdx.x < SG_MAXOPS) s_red[threadIdx.x] = 0.0;
  __syncthreads();
  const OpsRT ops{A.ops, A.nops};
  stream8_body(A, ops);
  if (A.has_reduce) finish_reductions<float>(A, ops);
}
