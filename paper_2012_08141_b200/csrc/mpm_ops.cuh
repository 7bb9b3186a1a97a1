// mpm_ops.cuh -- MLS-MPM transfer ops (hu2018moving, the method PAPER.md:444
// evaluates; P2G "requires atomic add").  Included by kernels.cu
// after the tree helpers.  Quadratic B-spline weights over 3x3x3 nodes; the base
// node is decided in f32 with round-to-nearest intrinsics (no FMA contraction)
// exactly as the oracle does (reading R16).
//
// Arrays: a0 x (3 comps), a1 v (3), a2 C (9, row-major), a3 J (1); SoA with
// component c at ptr + c*n.  Grid fields f0..f2 velocity (momentum during P2G),
// f3 mass; they live in one tree whose leaf blocks are dense (2^LB per axis;
// LB = 2 for the configs' 4^3 blocks, 0 = read from the tree at run time).
//
// The 3x3x3 stencil touches at most 2 blocks per axis.  Their 8 pool offsets
// are resolved once per particle (one tree walk each, activating in P2G) and
// kept in registers; every node picks its block with a 3-level select, so no
// per-node tree walk and no local-memory array.
#pragma once

struct MpmKernel {
  int base[3];
  float fx[3];
  float w[3][3];
};

__device__ __forceinline__ MpmKernel mpm_bspline(const float xp[3], float inv_dx) {
  MpmKernel k;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    float X = __fmul_rn(xp[a], inv_dx);
    k.base[a] = (int)floorf(__fsub_rn(X, 0.5f));
    float fx = __fsub_rn(X, (float)k.base[a]);
    k.fx[a] = fx;
    float q0 = 1.5f - fx, q1 = fx - 1.0f, q2 = fx - 0.5f;
    k.w[0][a] = 0.5f * q0 * q0;
    k.w[1][a] = 0.75f - q1 * q1;
    k.w[2][a] = 0.5f * q2 * q2;
  }
  return k;
}

// Per-particle block set: offsets (words from the leaf pool base) of the <= 8
// blocks, SG_NO_BLOCK when absent; `hi[a]` = bitmask over k=0..2 of nodes
// base+k that fall into the upper block along axis a.
struct MpmBlocks {
  uint32_t o[8];    // index = 4*ix + 2*iy + iz
  uint32_t hi[3];
};

template <int LB>
__device__ __forceinline__ int mpm_lb(const DTree& T, int a) {
  return LB > 0 ? LB : T.lev[T.driving].lbelow[a];
}

template <bool ACTIVATE, int LB>
__device__ __forceinline__ void mpm_blocks(const DevCtx& C, const DTree& T, const int base[3], MpmBlocks& B, int task) {
  const uint32_t* pool = T.seg[T.nseg - 1].base;
  const uint32_t blkmask = ~((1u << T.lblk) - 1u);
  int b0[3], nb[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int lb = mpm_lb<LB>(T, a), m = (1 << lb) - 1;
    b0[a] = base[a] >> lb;
    const int r = base[a] & m;
    B.hi[a] = ((r + 0 > m) ? 1u : 0u) | ((r + 1 > m) ? 2u : 0u) | ((r + 2 > m) ? 4u : 0u);
    nb[a] = B.hi[a] ? 2 : 1;
  }
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int ix = i >> 2, iy = (i >> 1) & 1, iz = i & 1;
    uint32_t off = SG_NO_BLOCK;
    if (ix < nb[0] && iy < nb[1] && iz < nb[2]) {
      int q[3] = {(b0[0] + ix) << mpm_lb<LB>(T, 0), (b0[1] + iy) << mpm_lb<LB>(T, 1), (b0[2] + iz) << mpm_lb<LB>(T, 2)};
      if (in_domain(T, q)) {
        uint32_t idx;
        uint32_t* cont = ACTIVATE ? activate_walk(C, T, q, idx, task) : locate(T, q, idx);
        if (cont) off = (uint32_t)(cont - pool) + T.payload_off + (idx & blkmask);
      }
    }
    B.o[i] = off;
  }
}

// Offset of node base + (a, b, c) (compile-time a, b, c): block by selects.
template <int LB>
__device__ __forceinline__ uint32_t mpm_node_off(const DTree& T, const MpmBlocks& B, const int base[3], int a, int b,
                                                 int c) {
  const int ix = (B.hi[0] >> a) & 1, iy = (B.hi[1] >> b) & 1, iz = (B.hi[2] >> c) & 1;
  const uint32_t o0 = ix ? B.o[4] : B.o[0], o1 = ix ? B.o[5] : B.o[1], o2 = ix ? B.o[6] : B.o[2],
                 o3 = ix ? B.o[7] : B.o[3];
  const uint32_t p0 = iy ? o2 : o0, p1 = iy ? o3 : o1;
  const uint32_t blk = iz ? p1 : p0;
  if (blk == SG_NO_BLOCK) return SG_NO_BLOCK;
  const int n[3] = {base[0] + a, base[1] + b, base[2] + c};
  uint32_t in;
  if (LB > 0) {
    const int m = (1 << LB) - 1;
    in = ((uint32_t)(n[0] & m) << (2 * LB)) | ((uint32_t)(n[1] & m) << LB) | (uint32_t)(n[2] & m);
  } else {
    in = inblock_idx(T, n);
  }
  return blk + in;
}

template <int LB>
__device__ __forceinline__ void mpm_p2g(const DevCtx& C, const DTree& T, const DOp& op, int64_t i, int task) {
  const DArray X = C.arrays[op.a[0]], Vv = C.arrays[op.a[1]], Cm = C.arrays[op.a[2]], Jj = C.arrays[op.a[3]];
  const float* __restrict__ x = (const float*)X.ptr;
  const float* __restrict__ v = (const float*)Vv.ptr;
  const float* __restrict__ cm = (const float*)Cm.ptr;
  const float* __restrict__ jj = (const float*)Jj.ptr;
  const float dt = op.p[0], inv_dx = op.p[1], pm = op.p[2], pv = op.p[3], E = op.p[4];
  const float dx = 1.0f / inv_dx;
  float xp[3] = {x[i], x[X.n + i], x[2 * X.n + i]};
  MpmKernel k = mpm_bspline(xp, inv_dx);
  const float J = jj[i];
  const float stress = -dt * 4.0f * E * pv * (J - 1.0f) * inv_dx * inv_dx;
  float aff[3][3], mv[3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    mv[r] = pm * v[r * Vv.n + i];
#pragma unroll
    for (int c = 0; c < 3; c++) aff[r][c] = pm * cm[(3 * r + c) * Cm.n + i] + (r == c ? stress : 0.0f);
  }
  uint32_t* pool = T.seg[T.nseg - 1].base;
  const uint64_t fs = 1ull << T.ln_leaf;
  float* fv[4];
#pragma unroll
  for (int r = 0; r < 4; r++) fv[r] = (float*)(pool + (uint64_t)op.slot[r] * fs);
  MpmBlocks B;
  if (op.act) mpm_blocks<true, LB>(C, T, k.base, B, task);
  else mpm_blocks<false, LB>(C, T, k.base, B, task);
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t off = mpm_node_off<LB>(T, B, k.base, a, b, c);
        if (off == SG_NO_BLOCK) {
          if (C.debug) set_err(C, op.act ? SG_ERR_RANGE : SG_ERR_DEMOTION_TRAP, task);
          continue;
        }
        const float wgt = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float d0 = ((float)a - k.fx[0]) * dx, d1 = ((float)b - k.fx[1]) * dx, d2 = ((float)c - k.fx[2]) * dx;
#pragma unroll
        for (int r = 0; r < 3; r++)
          atomicAdd(fv[r] + off, wgt * (mv[r] + aff[r][0] * d0 + aff[r][1] * d1 + aff[r][2] * d2));
        atomicAdd(fv[3] + off, wgt * pm);
      }
}

// G2P gather for one particle: new v, C (grid velocities of the 27 nodes).
template <int LB>
__device__ __forceinline__ void mpm_gather(const DevCtx& C, const DTree& T, const DOp& op, const MpmKernel& k,
                                           float dx, float inv_dx, float nv[3], float nC[3][3]) {
  const uint32_t* pool = T.seg[T.nseg - 1].base;
  const uint64_t fs = 1ull << T.ln_leaf;
  const float* fv[3];
#pragma unroll
  for (int r = 0; r < 3; r++) fv[r] = (const float*)(pool + (uint64_t)op.slot[r] * fs);
  MpmBlocks B;
  mpm_blocks<false, LB>(C, T, k.base, B, 0);
  const float s4 = 4.0f * inv_dx * inv_dx;
#pragma unroll
  for (int r = 0; r < 3; r++) {
    nv[r] = 0.0f;
#pragma unroll
    for (int d = 0; d < 3; d++) nC[r][d] = 0.0f;
  }
#pragma unroll
  for (int a = 0; a < 3; a++)
#pragma unroll
    for (int b = 0; b < 3; b++)
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const uint32_t off = mpm_node_off<LB>(T, B, k.base, a, b, c);
        if (off == SG_NO_BLOCK) continue;
        const float wgt = k.w[a][0] * k.w[b][1] * k.w[c][2];
        const float dpos[3] = {((float)a - k.fx[0]) * dx, ((float)b - k.fx[1]) * dx, ((float)c - k.fx[2]) * dx};
#pragma unroll
        for (int r = 0; r < 3; r++) {
          const float g = fv[r][off];
          nv[r] += wgt * g;
#pragma unroll
          for (int d = 0; d < 3; d++) nC[r][d] += s4 * wgt * g * dpos[d];
        }
      }
}

// G2P: in place on a0..a3, or (a4 set) reading state a0..a3 and writing the
// new state to a4..a7 (C4 keeps every substep's state as a checkpoint).
template <int LB>
__device__ __forceinline__ void mpm_g2p(const DevCtx& C, const DTree& T, const DOp& op, int64_t i,
                                        int64_t io = -1) {
  if (io < 0) io = i;   // output index (binned G2P in bin order writes particle i at its bin position)
  const int o = op.a[4] >= 0 ? 4 : 0;
  const DArray X = C.arrays[op.a[0]], Jj = C.arrays[op.a[3]];
  const DArray Xo = C.arrays[op.a[o]], Vo = C.arrays[op.a[o + 1]], Co = C.arrays[op.a[o + 2]],
               Jo = C.arrays[op.a[o + 3]];
  const float* x = (const float*)X.ptr;
  float* xo = (float*)Xo.ptr;
  float* vo = (float*)Vo.ptr;
  float* co = (float*)Co.ptr;
  float* jo = (float*)Jo.ptr;
  const float dt = op.p[0], inv_dx = op.p[1];
  const float dx = 1.0f / inv_dx;
  float xp[3] = {x[i], x[X.n + i], x[2 * X.n + i]};
  const float J = ((const float*)Jj.ptr)[i];
  MpmKernel k = mpm_bspline(xp, inv_dx);
  float nv[3], nC[3][3];
  mpm_gather<LB>(C, T, op, k, dx, inv_dx, nv, nC);
#pragma unroll
  for (int r = 0; r < 3; r++) {
    vo[r * Vo.n + io] = nv[r];
    xo[r * Xo.n + io] = xp[r] + dt * nv[r];
#pragma unroll
    for (int d = 0; d < 3; d++) co[(3 * r + d) * Co.n + io] = nC[r][d];
  }
  jo[io] = J * (1.0f + dt * (nC[0][0] + nC[1][1] + nC[2][2]));
}

// Grid update for one cell (struct-for).  cell0 points at the cell in field slot 0.
__device__ __forceinline__ void mpm_grid_op(const DOp& op, const int c[3], uint32_t* cell0, uint64_t fs) {
  uint32_t* pv[3] = {cell0 + op.slot[0] * fs, cell0 + op.slot[1] * fs, cell0 + op.slot[2] * fs};
  const float m = __uint_as_float(cell0[op.slot[3] * fs]);
  float v[3] = {__uint_as_float(*pv[0]), __uint_as_float(*pv[1]), __uint_as_float(*pv[2])};
  if (m > 0.0f) {
#pragma unroll
    for (int a = 0; a < 3; a++) v[a] = v[a] / m;
  }
  v[1] -= op.p[0] * op.p[1];
  const float bound = op.p[2], n = op.p[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bool cond = ((float)c[a] < bound && v[a] < 0.0f) || ((float)c[a] > n - bound && v[a] > 0.0f);
    if (cond) v[a] = 0.0f;
  }
#pragma unroll
  for (int a = 0; a < 3; a++) *pv[a] = __float_as_uint(v[a]);
}

// Dedicated MPM range-for kernels: the grid tree travels by value.
struct MpmArgs {
  DTree T;
  DevCtx C;
  DOp op;
  int64_t n;
  const int32_t* dcount;
  int task;
};

template <int LB>
__global__ void __launch_bounds__(128, 6) k_p2g(const __grid_constant__ MpmArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mpm_p2g<LB>(A.C, A.T, A.op, i, A.task);
}

template <int LB>
__global__ void __launch_bounds__(128, 6) k_g2p(const __grid_constant__ MpmArgs A) {
  const int64_t n = A.dcount ? (int64_t)*A.dcount : A.n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mpm_g2p<LB>(A.C, A.T, A.op, i);
}
