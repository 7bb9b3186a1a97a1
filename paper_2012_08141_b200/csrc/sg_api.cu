// sg_api.cu -- the C-ABI of libsg (include/sg.h): layout derivation, device
// memory, the task queue and the flush dispatcher.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <vector>

#include "grid.h"
#include "jit.h"
#include "planner.h"
#include "sg_internal.h"

using namespace sg;

static thread_local std::string g_err;

static sg_status fail(sg_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

void sg_internal_set_error(const char* msg) { g_err = msg; }

#define CUDA_TRY(x)                                                               \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) return fail(SG_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

static int ilog2i(int64_t v) {
  int r = 0;
  while ((1ll << r) < v) r++;
  return r;
}

// ---------------------------------------------------------------------------
// Layout validation and derivation
// ---------------------------------------------------------------------------
static sg_status build_layout(const sg_snode_desc* d, int n, HLayout& L) {
  if (n < 1 || !d || d[0].kind != SG_ROOT || d[0].parent != -1) return fail(SG_ERR_LAYOUT, "row 0 must be the root");
  L.nodes.assign(d, d + n);
  std::vector<std::vector<int>> kids(n);
  for (int i = 1; i < n; i++) {
    const sg_snode_desc& s = d[i];
    if (s.kind <= SG_ROOT || s.kind > SG_PLACE) return fail(SG_ERR_LAYOUT, "bad kind at row " + std::to_string(i));
    if (s.parent < 0 || s.parent >= i) return fail(SG_ERR_LAYOUT, "parent must precede child");
    if (d[s.parent].kind == SG_PLACE) return fail(SG_ERR_LAYOUT, "place with children");
    if (s.ndim < 0 || s.ndim > 3) return fail(SG_ERR_LAYOUT, "ndim out of range");
    for (int a = 0; a < 3; a++) {
      int e = s.extent[a];
      if (e < 1 || (e & (e - 1))) return fail(SG_ERR_LAYOUT, "extent not a power of two");
      if (a >= s.ndim && e != 1) return fail(SG_ERR_LAYOUT, "extent on an unused axis");
    }
    if (s.kind == SG_PLACE && s.dtype != SG_F32 && s.dtype != SG_I32) return fail(SG_ERR_LAYOUT, "bad dtype");
    kids[s.parent].push_back(i);
  }
  L.snode_tree.assign(n, -1);
  L.snode_pos.assign(n, -1);
  int nscal = 0;
  std::vector<int> place_tree(n, -1);
  for (int c : kids[0]) {
    HTree T;
    int tid = (int)L.trees.size();
    if (d[c].kind == SG_PLACE) {
      if (d[c].ndim != 0) return fail(SG_ERR_LAYOUT, "place under the root must be 0-D");
      T.nd = 0;
      T.fields.push_back(c);
      place_tree[c] = tid;
    } else {
      T.nd = d[c].ndim;
      if (T.nd < 1) return fail(SG_ERR_LAYOUT, "levels need ndim >= 1");
      int cur = c;
      while (true) {
        if (d[cur].ndim != T.nd) return fail(SG_ERR_LAYOUT, "axis mismatch along a chain");
        L.snode_tree[cur] = tid;
        L.snode_pos[cur] = (int)T.levels.size();
        T.levels.push_back(cur);
        if ((int)T.levels.size() > SG_MAXL) return fail(SG_ERR_LAYOUT, "chain deeper than 6 levels");
        int structural = -1, places = 0;
        for (int k : kids[cur]) {
          if (d[k].kind == SG_PLACE) places++;
          else if (structural >= 0) return fail(SG_ERR_LAYOUT, "a level with two structural children");
          else structural = k;
        }
        if (structural >= 0 && places) return fail(SG_ERR_LAYOUT, "places only at the leaf level");
        if (structural < 0) {
          if (!places) return fail(SG_ERR_LAYOUT, "leaf level without place");
          if (d[cur].kind == SG_POINTER) return fail(SG_ERR_LAYOUT, "a pointer level cannot be the leaf");
          for (int k : kids[cur]) {
            if (d[k].ndim != T.nd) return fail(SG_ERR_LAYOUT, "place ndim mismatch");
            T.fields.push_back(k);
            place_tree[k] = tid;
          }
          break;
        }
        cur = structural;
      }
      for (int k = (int)T.levels.size() - 1; k >= 0; k--) {
        int s = T.levels[k];
        bool sparse = d[s].kind == SG_BITMASKED || d[s].kind == SG_POINTER;
        if (!sparse) continue;
        if (k == (int)T.levels.size() - 1 && d[s].kind == SG_BITMASKED) { T.leaf_bitmasked = true; continue; }
        T.driving = k;
        break;
      }
    }
    L.trees.push_back(T);
  }
  // fields, in order of place rows
  for (int i = 0; i < n; i++) {
    if (d[i].kind != SG_PLACE) continue;
    int tid = place_tree[i];
    if (tid < 0) return fail(SG_ERR_LAYOUT, "place not reachable from the root");
    int fid = (int)L.field_tree.size();
    const HTree& T = L.trees[tid];
    int slot = 0;
    for (size_t k = 0; k < T.fields.size(); k++) if (T.fields[k] == i) slot = (int)k;
    L.field_tree.push_back(T.nd == 0 ? -1 : tid);
    L.field_slot.push_back(slot);
    L.field_dtype.push_back(d[i].dtype);
    L.field_scalar.push_back(T.nd == 0 ? nscal++ : -1);
    (void)fid;
  }
  // trees hold field ids, not place rows
  for (HTree& T : L.trees) {
    for (int& f : T.fields) {
      int fid = 0;
      for (int i = 0; i < f; i++) if (d[i].kind == SG_PLACE) fid++;
      f = fid;
    }
  }
  L.n_scalars = nscal;
  return SG_OK;
}

static sg_status derive_tree(sg_grid* g, int tid, DTree& T) {
  const HLayout& L = g->L;
  const HTree& H = L.trees[tid];
  std::memset(&T, 0, sizeof(T));
  T.nd = H.nd;
  T.nlev = (int)H.levels.size();
  T.driving = H.driving;
  T.leaf_bitmasked = H.leaf_bitmasked;
  T.nfields = (int)H.fields.size();
  int seg = 0;
  for (int k = 0; k < T.nlev; k++) {
    const sg_snode_desc& s = L.nodes[H.levels[k]];
    DLevel& D = T.lev[k];
    D.kind = s.kind;
    D.seg = seg;
    D.lE = 0;
    for (int a = 0; a < 3; a++) { D.le[a] = ilog2i(s.extent[a]); D.lE += D.le[a]; }
    if (s.kind == SG_POINTER) seg++;
  }
  T.nseg = seg + 1;
  for (int k = 0; k < T.nlev; k++) {
    DLevel& D = T.lev[k];
    for (int a = 0; a < 3; a++) {
      D.lbelow[a] = 0;
      for (int m = k + 1; m < T.nlev; m++) D.lbelow[a] += T.lev[m].le[a];
      D.lres[a] = 0;
      for (int m = 0; m <= k; m++) D.lres[a] += T.lev[m].le[a];
    }
  }
  for (int s = 0; s < T.nseg; s++) { T.seg[s].first = -1; T.seg[s].last = -1; }
  for (int k = 0; k < T.nlev; k++) {
    DSeg& S = T.seg[T.lev[k].seg];
    if (S.first < 0) S.first = k;
    S.last = k;
  }
  T.lblk = 0;
  for (int k = T.driving + 1; k < T.nlev; k++) T.lblk += T.lev[k].lE;
  // container layouts
  for (int s = 0; s < T.nseg; s++) {
    DSeg& S = T.seg[s];
    uint64_t words = 0;
    int ln = 0;
    for (int k = S.first; k <= S.last; k++) {
      DLevel& D = T.lev[k];
      ln += D.lE;
      D.ln = ln;
      if (D.kind == SG_BITMASKED) {
        words = (words + 3) & ~3ull;   // 16-byte aligned mask regions (vector loads in listgen)
        D.mask_off = (uint32_t)words;
        words += std::max<uint64_t>(1, ((1ull << ln) + 31) / 32);
      }
      if (D.kind == SG_POINTER) {
        D.slot_off = (uint32_t)words;
        words += 1ull << ln;
      }
    }
    S.header_words = (uint32_t)words;
    if (s == T.nseg - 1) {
      T.ln_leaf = ln;
      T.payload_off = (int32_t)((words + 31) & ~31ull);
      words = (uint64_t)T.payload_off + (uint64_t)T.nfields << 0;
      words = (uint64_t)T.payload_off + ((uint64_t)T.nfields << ln);
    }
    S.stride = (words + 63) & ~63ull;
    if (s == 0) {
      S.capacity = 1;
    } else {
      const DLevel& P = T.lev[T.seg[s - 1].last];
      int64_t cells = 1ll << (P.lres[0] + P.lres[1] + P.lres[2]);
      int64_t cap = cells;
      if (g->opts.pool_capacity > 0) cap = std::min<int64_t>(cap, g->opts.pool_capacity);
      S.capacity = (uint32_t)cap;
    }
    for (int k = S.first; k <= S.last; k++) {
      if (((uint64_t)S.capacity << T.lev[k].ln) > (1ull << 32))
        return fail(SG_ERR_LAYOUT, "list entries would overflow u32: lower opts.pool_capacity");
    }
    if (s == T.nseg - 1) {
      // one extra, never-allocated container stays all-zero: absent neighbours point at it
      if ((uint64_t)(S.capacity + 1) * S.stride >= 0xFFFFFFFFull)
        return fail(SG_ERR_LAYOUT, "leaf pool exceeds 2^32 words (block offsets are u32): lower opts.pool_capacity");
      T.zero_blk = (uint32_t)((uint64_t)S.capacity * S.stride + T.payload_off);
    }
  }
  return SG_OK;
}

static sg_status alloc_tree(sg_grid* g, int tid, DTree& T) {
  for (int s = 0; s < T.nseg; s++) {
    DSeg& S = T.seg[s];
    size_t bytes = (size_t)(S.capacity + (s == T.nseg - 1 ? 1 : 0)) * S.stride * 4;
    S.base = (uint32_t*)g->dev_alloc(bytes);
    if (!S.base) return fail(SG_ERR_CUDA, "pool allocation failed (" + std::to_string(bytes) + " bytes)");
    CUDA_TRY(cudaMemsetAsync(S.base, 0, bytes, g->stream));
    S.origin = (int32_t*)g->dev_alloc((size_t)S.capacity * 3 * 4);
    S.alloc = (int32_t*)g->dev_alloc(16);
    S.free_list = (uint32_t*)g->dev_alloc((size_t)S.capacity * 4);
    if (!S.origin || !S.alloc || !S.free_list) return fail(SG_ERR_CUDA, "allocation failed");
    CUDA_TRY(cudaMemsetAsync(S.origin, 0, (size_t)S.capacity * 12, g->stream));
    CUDA_TRY(cudaMemsetAsync(S.alloc, 0, 16, g->stream));
  }
  (void)tid;
  return SG_OK;
}

static uint64_t list_capacity(const sg_grid* g, const DTree& T, int k) {
  uint64_t cap = (uint64_t)T.seg[T.lev[k].seg].capacity << T.lev[k].ln;
  if (g->opts.list_capacity > 0) cap = std::min<uint64_t>(cap, (uint64_t)g->opts.list_capacity);
  return std::min<uint64_t>(cap, 0xFFFFFFFFull);
}

static int parent_pos(const DTree& T, int k) {
  for (int m = k - 1; m >= 0; m--)
    if (T.lev[m].kind == SG_BITMASKED || T.lev[m].kind == SG_POINTER) return m;
  return -1;
}

static sg_status alloc_list(sg_grid* g, int tid, int k) {
  DTree& T = g->dtrees[tid];
  DList& Ls = g->lists[tid][k];
  if (Ls.entries) return SG_OK;
  uint64_t cap = list_capacity(g, T, k);
  int pk = parent_pos(T, k);
  uint64_t pcap = pk < 0 ? 1 : list_capacity(g, T, pk);
  int lratio;
  if (pk < 0) lratio = T.lev[k].ln;
  else if (T.lev[pk].seg == T.lev[k].seg) lratio = T.lev[k].ln - T.lev[pk].ln;
  else lratio = T.lev[k].ln;
  uint64_t cpp = lratio > 5 ? (1ull << (lratio - 5)) : 1;
  uint64_t max_tiles = (pcap * cpp + 255) / 256 + 1;   // look-back descriptors: tiles of >= 256 chunks
  Ls.capacity = (uint32_t)cap;
  Ls.max_tiles = (uint32_t)std::min<uint64_t>(max_tiles, 0xFFFFFFFFull);
  if (k == T.driving) {
    Ls.table = (BlockRow*)g->dev_alloc(cap * sizeof(BlockRow));
    if (!Ls.table) return fail(SG_ERR_CUDA, "block table allocation failed");
  }
  Ls.entries = (uint32_t*)g->dev_alloc(cap * 4);
  Ls.count = (uint32_t*)g->dev_alloc(16);
  Ls.ctl = (uint32_t*)g->dev_alloc(32);
  Ls.status = (uint64_t*)g->dev_alloc(max_tiles * 8);
  if (!Ls.entries || !Ls.count || !Ls.ctl || !Ls.status) return fail(SG_ERR_CUDA, "list allocation failed");
  CUDA_TRY(cudaMemsetAsync(Ls.count, 0, 16, g->stream));
  CUDA_TRY(cudaMemsetAsync(Ls.ctl, 0, 32, g->stream));
  CUDA_TRY(cudaMemsetAsync(Ls.status, 0, max_tiles * 8, g->stream));
  return SG_OK;
}

static sg_status upload_tables(sg_grid* g) {
  CUDA_TRY(cudaMemcpyAsync(g->d_trees, g->dtrees.data(), g->dtrees.size() * sizeof(DTree), cudaMemcpyHostToDevice, g->stream));
  return SG_OK;
}

extern "C" sg_status sg_create(const sg_snode_desc* nodes, int32_t n, const sg_opts* o, sg_grid** out) {
  if (!out) return fail(SG_ERR_ARG, "out is null");
  *out = nullptr;
  sg_grid* g = new sg_grid();
  if (o) g->opts = *o;
  g->plan_only = g->opts.plan_only != 0;
  g->stream = (cudaStream_t)g->opts.stream;
  g->user_stream = g->stream;
  { const char* e = std::getenv("SG_NO_BIN"); g->no_bin = e && e[0] == '1'; }
  { const char* e = std::getenv("SG_NO_GRAPH"); g->use_graphs = !(e && e[0] == '1'); }
  sg_status rc = build_layout(nodes, n, g->L);
  if (rc) { delete g; return rc; }
  g->dtrees.resize(g->L.trees.size());
  g->lists.assign(g->L.trees.size(), std::vector<DList>(SG_MAXL));
  for (size_t t = 0; t < g->L.trees.size(); t++) {
    if (g->L.trees[t].nd == 0) continue;
    rc = derive_tree(g, (int)t, g->dtrees[t]);
    if (rc) { delete g; return rc; }
  }
  if (!g->plan_only) {
    cudaError_t e = cudaSetDevice(g->opts.device);
    if (e != cudaSuccess) { delete g; return fail(SG_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)); }
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->opts.device);
    for (size_t t = 0; t < g->L.trees.size(); t++) {
      if (g->L.trees[t].nd == 0) continue;
      rc = alloc_tree(g, (int)t, g->dtrees[t]);
      if (rc) { delete g; return rc; }
      for (int s : g->L.listed_levels((int)t)) {
        rc = alloc_list(g, (int)t, g->L.snode_pos[s]);
        if (rc) { delete g; return rc; }
      }
    }
    size_t nf = g->L.field_tree.size();
    std::vector<DField> hf(nf);
    for (size_t f = 0; f < nf; f++) {
      hf[f].tree = g->L.field_tree[f];
      hf[f].slot = g->L.field_slot[f];
      hf[f].dtype = g->L.field_dtype[f];
      hf[f].scalar = g->L.field_scalar[f];
    }
    g->d_trees = (DTree*)g->dev_alloc(std::max<size_t>(1, g->dtrees.size()) * sizeof(DTree));
    g->d_fields = (DField*)g->dev_alloc(std::max<size_t>(1, nf) * sizeof(DField));
    g->ctx.scalars = (uint32_t*)g->dev_alloc(std::max(1, g->L.n_scalars) * 4);
    g->ctx.err = (uint32_t*)g->dev_alloc(16);
    g->ctx.max_grid = g->num_sms * 8;
    g->ctx.partials = (double*)g->dev_alloc((size_t)SG_MAXOPS * g->ctx.max_grid * sizeof(double));
    g->ctx.red_done = (uint32_t*)g->dev_alloc(16);
    if (!g->ctx.partials || !g->ctx.red_done || cudaMemsetAsync(g->ctx.red_done, 0, 16, g->stream) != cudaSuccess) {
      delete g;
      return fail(SG_ERR_CUDA, "reduction scratch allocation failed");
    }
    g->d_arrays_cap = 64;
    g->d_arrays = (DArray*)g->dev_alloc(g->d_arrays_cap * sizeof(DArray));
    if (!g->d_trees || !g->d_fields || !g->ctx.scalars || !g->ctx.err || !g->d_arrays) {
      delete g;
      return fail(SG_ERR_CUDA, "table allocation failed");
    }
    if ((rc = upload_tables(g))) { delete g; return rc; }
    if (cudaMemcpyAsync(g->d_fields, hf.data(), nf * sizeof(DField), cudaMemcpyHostToDevice, g->stream) != cudaSuccess ||
        cudaMemsetAsync(g->ctx.scalars, 0, std::max(1, g->L.n_scalars) * 4, g->stream) != cudaSuccess ||
        cudaMemsetAsync(g->ctx.err, 0, 16, g->stream) != cudaSuccess ||
        cudaStreamSynchronize(g->stream) != cudaSuccess) {
      delete g;
      return fail(SG_ERR_CUDA, "table upload failed");
    }
    g->ctx.trees = g->d_trees;
    g->ctx.fields = g->d_fields;
    g->ctx.arrays = g->d_arrays;
    g->ctx.debug = g->opts.debug;
  }
  *out = g;
  return SG_OK;
}

extern "C" sg_status sg_destroy(sg_grid* g) {
  if (!g) return SG_OK;
  if (!g->plan_only) cudaStreamSynchronize(g->stream);
  sg_dist_destroy(g);
  for (auto& kv : g->gexec)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  delete g;
  return SG_OK;
}

extern "C" sg_status sg_register_array(sg_grid* g, void* ptr, int64_t n, int32_t dtype, int32_t ncomp, int32_t* id) {
  if (!g || !id || n < 0 || ncomp < 1) return fail(SG_ERR_ARG, "bad array");
  if ((int)g->arrays.size() >= g->d_arrays_cap && !g->plan_only) {
    // grow the device table (C4 registers one state per substep); the old
    // table stays allocated: launches already enqueued still point at it
    const int cap = g->d_arrays_cap * 2;
    DArray* t = (DArray*)g->dev_alloc((size_t)cap * sizeof(DArray));
    if (!t) return fail(SG_ERR_CUDA, "array table allocation failed");
    CUDA_TRY(cudaMemcpyAsync(t, g->d_arrays, (size_t)g->d_arrays_cap * sizeof(DArray), cudaMemcpyDeviceToDevice,
                             g->stream));
    g->d_arrays = t;
    g->d_arrays_cap = cap;
    g->ctx.arrays = t;
  }
  DArray a{ptr, n, ncomp, dtype, nullptr};
  g->arrays.push_back(a);
  g->arr_epoch.push_back(0);
  *id = (int32_t)g->arrays.size() - 1;
  if (!g->plan_only)
    CUDA_TRY(cudaMemcpyAsync(g->d_arrays + *id, &a, sizeof(DArray), cudaMemcpyHostToDevice, g->stream));
  return SG_OK;
}

extern "C" sg_status sg_set_array_count(sg_grid* g, int32_t id, int32_t* dev_count) {
  if (!g || id < 0 || id >= (int)g->arrays.size()) return fail(SG_ERR_ARG, "bad array id");
  g->arrays[id].dcount = dev_count;
  if (!g->plan_only)
    CUDA_TRY(cudaMemcpyAsync(g->d_arrays + id, &g->arrays[id], sizeof(DArray), cudaMemcpyHostToDevice, g->stream));
  return SG_OK;
}

// ---------------------------------------------------------------------------
// Enqueue (tasks are queued until synchronization)
// ---------------------------------------------------------------------------
static sg_status enqueue(sg_grid* g, const UserCall& c) {
  std::string err;
  size_t before = g->eager.size();
  int rc = lower_call(g->L, c, g->ncalls, g->opts.lowering == 1, g->eager, err);
  if (rc) { g->eager.resize(before); return fail(rc, err); }
  for (size_t i = before; i < g->eager.size(); i++) {
    PTask& t = g->eager[i];
    t.pos = (int)i;
    if (t.type == TT_ACTIVATE) {
      int cls = -1;
      for (size_t k = 0; k < g->coords_seen.size(); k++)
        if (g->coords_seen[k].first == t.coords && g->coords_seen[k].second == t.n) cls = (int)k;
      if (cls < 0) { cls = (int)g->coords_seen.size(); g->coords_seen.push_back({t.coords, t.n}); }
      t.coords_class = cls;
    }
    task_meta(g->L, t);
  }
  g->ncalls++;
  return SG_OK;
}

extern "C" sg_status sg_activate(sg_grid* g, int32_t field, const int32_t* coords, int64_t n) {
  if (!g || n < 0 || (n > 0 && !coords)) return fail(SG_ERR_ARG, "bad activate arguments");
  UserCall c;
  c.kind = 0; c.field = field; c.coords = coords; c.n = n;
  return enqueue(g, c);
}

extern "C" sg_status sg_listgen(sg_grid* g, int32_t snode) {
  if (!g) return fail(SG_ERR_ARG, "null grid");
  UserCall c;
  c.kind = 1; c.snode = snode;
  return enqueue(g, c);
}

extern "C" sg_status sg_struct_for(sg_grid* g, const sg_task* t) {
  if (!g || !t) return fail(SG_ERR_ARG, "null task");
  UserCall c;
  c.kind = 2; c.t = *t;
  return enqueue(g, c);
}

extern "C" sg_status sg_clear(sg_grid* g, int32_t target, int32_t mode) {
  if (!g) return fail(SG_ERR_ARG, "null grid");
  UserCall c;
  c.kind = 3; c.mode = mode;
  if (mode == SG_CLEAR_VALUES) c.field = target; else c.snode = target;
  return enqueue(g, c);
}

// ---------------------------------------------------------------------------
// Flush: plan (cached) and launch one kernel per group
// ---------------------------------------------------------------------------
static void make_op(const sg_grid* g, const PTask& t, uint32_t act, int loop_tree, DOp& o) {
  std::memset(&o, 0, sizeof(o));
  o.op = t.t.op;
  o.act = act;
  o.scalar = -1;
  o.dt = SG_F32;
  bool dt_set = false;
  for (int i = 0; i < 8; i++) {
    int f = t.t.fields[i];
    o.f[i] = f;
    o.a[i] = t.t.arrays[i];
    o.p[i] = t.t.params[i];
    o.slot[i] = -1;
    if (f >= 0 && f < (int)g->L.field_tree.size()) {
      o.nf = i + 1;
      if (!dt_set) { o.dt = g->L.field_dtype[f]; dt_set = true; }
      // struct-for: slot in the iterated tree; range-for / serial: slot in the field's own tree
      if (g->L.field_tree[f] >= 0 && (loop_tree < 0 || g->L.field_tree[f] == loop_tree)) o.slot[i] = g->L.field_slot[f];
      if (g->L.field_tree[f] < 0 && o.scalar < 0) o.scalar = g->L.field_scalar[f];
    }
  }
}

constexpr uint64_t CHAIN_SOLO_CELLS = 8192;

// The device op table of a plan group.
static void group_ops(const sg_grid* g, const std::vector<int>& members, const std::vector<uint32_t>& acts, int tree,
                      std::vector<DOp>& all) {
  all.resize(members.size());
  for (size_t i = 0; i < members.size(); i++) make_op(g, g->eager[members[i]], acts[i], tree, all[i]);
}

// A chain's tail of JACOBI sweeps on 8^3 blocks, two opt-in variants, both
// bit-identical to one launch per sweep and both measured SLOWER than one
// graph-replayed launch per sweep on C2 (~4.4 us each) -- negative results
// kept with their tests (kernels_flow.cu):
//   SG_T2=1   two sweeps per launch (temporal blocking through shared
//             memory): 1,840 vs 3,954 solves/s -- a CTA stages one block with
//             its 2-deep halo per iteration, so only ~4 blocks per SM are in
//             flight (registers, 23.6 KB of shared memory each) and every
//             block pays its L2 round trips in series: ~20 us per 2 sweeps;
//   SG_FLOW=1 one flag-chained launch: 1,866 vs 3,974 solves/s (every sweep
//             of a half block pays a flag poll, its loads and a release fence
//             in series, ~10 us per sweep).
// The phases before the tail launch one by one.
static bool t2_on() {
  static const bool on = getenv("SG_T2") && atoi(getenv("SG_T2")) != 0;
  return on;
}

static bool flow_on() {
  static const bool on = getenv("SG_FLOW") && atoi(getenv("SG_FLOW")) != 0;
  return on;
}

// The first phase of a chain's tail of JACOBI sweeps on 8^3 blocks, or -1.
static int chain_jacobi_start(const sg_grid* g, const PTask& t0, const std::vector<DOp>& all,
                              const std::vector<int>& phase_end) {
  if (phase_end.size() < 2) return -1;
  const DTree& T = g->dtrees[t0.tree];
  const DList* drive = T.driving >= 0 ? &g->lists[t0.tree][T.driving] : nullptr;
  return jacobi_flow_start(T, drive, all.data(), phase_end.data(), (int)phase_end.size());
}

// Scratch of the 2-sweep chain kernels for a tree's driving list (first use
// is never inside a CUDA-graph capture, as for the flag buffers).
static bool t2_buffers(sg_grid* g, int tree, const DList* drive, T2Buffers* bf) {
  if ((int)g->t2_bufs.size() <= tree) g->t2_bufs.resize(tree + 1, T2Buffers{nullptr, nullptr, nullptr, nullptr});
  T2Buffers& b = g->t2_bufs[tree];
  if (!b.ctl) {
    const DSeg& S = g->dtrees[tree].seg[g->dtrees[tree].nseg - 1];
    const size_t ninv = ((size_t)S.capacity + 1) * S.stride / 512 + 1, cap = drive->capacity;
    b.inv = (uint64_t*)g->dev_alloc(ninv * 8);
    b.rows = (uint32_t*)g->dev_alloc(cap * 54 * 4);
    b.tmp = (float*)g->dev_alloc(cap * 512 * 4);
    b.ctl = (uint32_t*)g->dev_alloc(16);
    if (!b.inv || !b.rows || !b.tmp || !b.ctl || cudaMemsetAsync(b.inv, 0, ninv * 8, g->stream) != cudaSuccess ||
        cudaMemsetAsync(b.ctl, 0, 16, g->stream) != cudaSuccess) {
      b.ctl = nullptr;
      return false;
    }
  }
  *bf = b;
  return true;
}

// Flag buffers of a tree (allocated and zeroed on first use: a plan's first
// run is never captured, so this happens outside any CUDA-graph capture).
static bool flow_buffers(sg_grid* g, int tree, uint32_t** flags, uint32_t** ctl) {
  if ((int)g->flow_flags.size() <= tree) g->flow_flags.resize(tree + 1, nullptr);
  if (!g->flow_flags[tree]) {
    const DSeg& S = g->dtrees[tree].seg[g->dtrees[tree].nseg - 1];
    const size_t n = 2 * (((size_t)S.capacity + 1) * S.stride / 512 + 1);
    uint32_t* f = (uint32_t*)g->dev_alloc(n * 4);
    if (!f || cudaMemsetAsync(f, 0, n * 4, g->stream) != cudaSuccess) return false;
    g->flow_flags[tree] = f;
  }
  if (!g->flow_ctl) {
    uint32_t* c = (uint32_t*)g->dev_alloc(16);
    if (!c || cudaMemsetAsync(c, 0, 16, g->stream) != cudaSuccess) return false;
    g->flow_ctl = c;
  }
  *flags = g->flow_flags[tree];
  *ctl = g->flow_ctl;
  return true;
}

// A chained group over a list of more than CHAIN_SOLO_CELLS cells launches its
// phases one by one (see launch_group).
static bool chain_is_split(const sg_grid* g, const PTask& t0, size_t nops = 0, size_t nphases = 0) {
  if (nops > 96 || nphases > 96) return true;   // SG_CHAIN_OPS: the table must fit the kernel parameters
  const DTree& T = g->dtrees[t0.tree];
  const DList* drive = T.driving >= 0 ? &g->lists[t0.tree][T.driving] : nullptr;
  const uint64_t cap = drive && drive->entries ? (uint64_t)drive->capacity : (T.driving >= 0 ? 0xFFFFFFFFull : 1ull);
  return (cap << T.lblk) > CHAIN_SOLO_CELLS;
}

static int grid_hint_struct(const sg_grid* g, const DTree& T) {
  (void)T;
  return g->num_sms * 8;
}

static bool tree_lb2(const DTree& t) {
  if (t.nd != 3 || t.driving < 0 || t.lblk != 6) return false;
  const DLevel& d = t.lev[t.driving];
  return d.lbelow[0] == 2 && d.lbelow[1] == 2 && d.lbelow[2] == 2;
}

// Bins of the particles in position array xa over tree `tree` (4^3 leaf
// blocks); rebuilt unless the cache holds the same (array, epoch, range) over
// the same bin geometry (blocks per axis, cell size).  The geometry, not the
// tree id: C4's adjoint tree has the grid tree's shape, so P2G, G2P_ADJ and
// P2G_ADJ of one substep share one binning of its positions.
constexpr int BIN_SLOTS = 160;   // C4: 65 states (T = 64) x forward + backward fit

static sg_status ensure_bins(sg_grid* g, int tree, int xa, float inv_dx, int64_t n, const int32_t* dcount,
                             int64_t& aux) {
  const DTree& T = g->dtrees[tree];
  const DLevel& leaf = T.lev[T.nlev - 1];
  int nb[3];
  for (int a = 0; a < 3; a++) nb[a] = (1 << leaf.lres[a]) >> 2;
  const uint64_t nk = (uint64_t)nb[0] * nb[1] * nb[2] + 1;
  if (nk > 0x7fffffffull) return fail(SG_ERR_ARG, "too many leaf blocks for particle binning");
  const uint32_t nkeys = (uint32_t)nk;
  const int64_t cap = g->arrays[xa].n;
  // shared scratch of the binning kernels
  if (cap > g->bin_cap) {
    g->bins.rank = (uint32_t*)g->dev_alloc((size_t)cap * 4);
    g->bins.key = (uint32_t*)g->dev_alloc((size_t)cap * 4);
    if (!g->bins.rank || !g->bins.key) return fail(SG_ERR_CUDA, "bin allocation failed");
    g->bin_cap = cap;
    g->bin_gen++;
  }
  if (nkeys > g->bin_keys_cap) {
    const uint32_t nt = bin_ntiles(nkeys);
    g->bins.hist = (uint32_t*)g->dev_alloc((size_t)nt * 2048 * 4);
    g->bins.tsum = (uint32_t*)g->dev_alloc((size_t)nt * 8);
    if (!g->bins.hist || !g->bins.tsum) return fail(SG_ERR_CUDA, "bin allocation failed");
    CUDA_TRY(cudaMemsetAsync(g->bins.hist, 0, (size_t)nt * 2048 * 4, g->stream));
    g->bin_keys_cap = nkeys;
    g->bin_gen++;
  }
  auto use = [&](const sg_grid::BinSlot& sl) {
    g->bins_cur = g->bins;
    g->bins_cur.perm = sl.perm;
    g->bins_cur.off = sl.off;
    g->bins_cur.bins = sl.bins;
    g->bins_cur.nbins = sl.nbins;
    g->bins_cur.nkeys = nkeys;
    for (int a = 0; a < 3; a++) g->bins_cur.nb[a] = nb[a];
  };
  for (const sg_grid::BinSlot& sl : g->bin_slots)
    if (sl.valid && sl.xa == xa && sl.epoch == g->arr_epoch[xa] && sl.nb[0] == nb[0] && sl.nb[1] == nb[1] &&
        sl.nb[2] == nb[2] && sl.inv_dx == inv_dx && sl.n == n && sl.dcount == dcount) {
      use(sl);
      return SG_OK;
    }
  const int si = g->bin_next++ % BIN_SLOTS;
  if ((int)g->bin_slots.size() <= si) g->bin_slots.resize(si + 1);
  sg_grid::BinSlot& sl = g->bin_slots[si];
  if (sl.cap < cap) {
    sl.perm = (uint32_t*)g->dev_alloc((size_t)cap * 4);
    if (!sl.perm) return fail(SG_ERR_CUDA, "bin allocation failed");
    sl.cap = cap;
    g->bin_gen++;
  }
  if (sl.kcap < nkeys) {
    sl.off = (uint32_t*)g->dev_alloc(((size_t)nkeys + 1) * 4);
    sl.bins = (uint32_t*)g->dev_alloc((size_t)nkeys * 4);
    if (!sl.nbins) sl.nbins = (uint32_t*)g->dev_alloc(16);
    if (!sl.off || !sl.bins || !sl.nbins) return fail(SG_ERR_CUDA, "bin allocation failed");
    sl.kcap = nkeys;
    g->bin_gen++;
  }
  use(sl);
  if (launch_bin(g->bins_cur, (const float*)g->arrays[xa].ptr, g->arrays[xa].n, n, dcount, inv_dx, g->stream))
    return fail(SG_ERR_CUDA, std::string("binning launch failed: ") + cudaGetErrorString(cudaGetLastError()));
  aux += BIN_KERNELS;
  sl.valid = true;
  sl.xa = xa; sl.epoch = g->arr_epoch[xa]; sl.n = n; sl.dcount = dcount; sl.inv_dx = inv_dx;
  for (int a = 0; a < 3; a++) sl.nb[a] = nb[a];
  return SG_OK;
}

static sg_status launch_group(sg_grid* g, const std::vector<int>& members, const std::vector<uint32_t>& acts,
                              const std::vector<int>& phase_end, sg_stats& st) {
  const PTask& t0 = g->eager[members[0]];
  int task = (int)(g->task_counter++ & 0x7FFFFFFF);   // launch index in the flush: stable across replays
  int rc = 0;
  switch (t0.type) {
    case TT_ACTIVATE: {
      rc = launch_activate(g->ctx, g->dtrees[t0.tree], t0.tree, t0.field, t0.coords, t0.n, task, g->stream);
    } break;
    case TT_LISTGEN: {
      const DTree& T = g->dtrees[t0.tree];
      int k = g->L.snode_pos[t0.snode];
      if ((rc = alloc_list(g, t0.tree, k))) return rc;
      int pk = parent_pos(T, k);
      const DList* parent = pk >= 0 ? &g->lists[t0.tree][pk] : nullptr;
      // upper bound on the listgen's tiles: parent entries x 32-child chunks / tile
      const int lratio = pk >= 0 && T.lev[pk].seg == T.lev[k].seg ? T.lev[k].ln - T.lev[pk].ln : T.lev[k].ln;
      const uint64_t pcap = parent ? parent->capacity : 1;
      const uint64_t ptiles = (pcap * (1ull << std::max(0, lratio - 5)) + 1023) / 1024;
      // (the launcher clamps the grid; an uncapped hint lets it pick the two-pass scheme for big lists)
      int hint = (int)std::max<uint64_t>(1, std::min<uint64_t>(ptiles, 0x7fffffffull));
      rc = launch_listgen(g->ctx, T, t0.tree, k, pk, parent, g->lists[t0.tree][k], task, g->stream, hint);
      st.listgen_launched++;
    } break;
    case TT_CLEAR_LIST: {
      int k = g->L.snode_pos[t0.snode];
      if ((rc = alloc_list(g, t0.tree, k))) return rc;
      rc = launch_clear_list(g->lists[t0.tree][k], g->stream);
      st.clear_list_launched++;
    } break;
    case TT_STRUCT_FOR: {
      const DTree& T = g->dtrees[t0.tree];
      const DList* drive = T.driving >= 0 ? &g->lists[t0.tree][T.driving] : nullptr;
      const int nops = (int)members.size();
      if (phase_end.size() <= 1) {
        DOp ops[SG_MAXOPS];
        for (int i = 0; i < nops; i++) make_op(g, g->eager[members[i]], acts[i], t0.tree, ops[i]);
        rc = launch_struct_for(g->ctx, T, t0.tree, drive, ops, nops, task, g->stream, grid_hint_struct(g, T),
                               nullptr, nullptr, 1, 0);
      } else {
        // chain (SG_PASS_CHAIN): whole op table + phase ends to the device
        std::vector<DOp> all(nops);
        int nbr = 0;
        for (int i = 0; i < nops; i++) make_op(g, g->eager[members[i]], acts[i], t0.tree, all[i]);
        uint32_t *ffl = nullptr, *fct = nullptr;
        const int fs = chain_jacobi_start(g, t0, all, phase_end);
        T2Buffers bf;
        if (fs >= 0 && !flow_on() && t2_on() &&
            jacobi_t2_applies(all.data(), phase_end.data(), fs, (int)phase_end.size()) &&
            t2_buffers(g, t0.tree, drive, &bf)) {
          int begin = 0;
          for (int ph = 0; ph < fs && !rc; ph++) {
            rc = launch_struct_for(g->ctx, T, t0.tree, drive, all.data() + begin, phase_end[ph] - begin, task,
                                   g->stream, grid_hint_struct(g, T), nullptr, nullptr, 1, 0);
            begin = phase_end[ph];
            st.launches++;
          }
          if (!rc) {
            const int nl = launch_jacobi_t2(g->ctx, T, drive, all.data(), phase_end.data(), fs,
                                            (int)phase_end.size(), bf, task, g->stream);
            if (nl < 0) rc = nl;
            else st.launches += nl - 1;
          }
          st.launches_chained++;
          break;
        }
        if (fs >= 0 && flow_on() && flow_buffers(g, t0.tree, &ffl, &fct)) {
          // leading phases (e.g. the fused FILLs of a solve) one launch each,
          // then the sweeps as one flag-chained launch
          int begin = 0;
          for (int ph = 0; ph < fs && !rc; ph++) {
            rc = launch_struct_for(g->ctx, T, t0.tree, drive, all.data() + begin, phase_end[ph] - begin, task,
                                   g->stream, grid_hint_struct(g, T), nullptr, nullptr, 1, 0);
            begin = phase_end[ph];
            st.launches++;
          }
          if (!rc)
            rc = launch_jacobi_flow(g->ctx, T, drive, all.data(), phase_end.data(), fs, (int)phase_end.size(), ffl,
                                    fct, task, g->stream);
          st.launches_chained++;
          break;
        }
        for (int i = 0; i < nops; i++) {
          int op = all[i].op;
          nbr |= op == SG_OP_STENCIL || op == SG_OP_JACOBI || op == SG_OP_JITTER || op == SG_OP_SMOOTH_RB ||
                 op == SG_OP_RESTRICT || op == SG_OP_RESID_NORM2;
        }
        // a chain pays off only when its barriers are CTA barriers: lists of at
        // most CHAIN_SOLO_CELLS cells (the MG bottom level) run as ONE CTA with
        // every phase in it; larger lists launch the phases one by one (a
        // grid-wide barrier costs more than a graph-replayed launch, measured)
        if (chain_is_split(g, t0, (size_t)nops, phase_end.size())) {
          int begin = 0;
          for (size_t ph = 0; ph < phase_end.size() && !rc; ph++) {
            const int end = phase_end[ph];
            rc = launch_struct_for(g->ctx, T, t0.tree, drive, all.data() + begin, end - begin, task, g->stream,
                                   grid_hint_struct(g, T), nullptr, nullptr, 1, 0);
            begin = end;
            if (ph + 1 < phase_end.size()) st.launches++;
          }
          break;
        }
        // one-CTA chain: the whole op table travels in the kernel parameters
        const int last0 = phase_end[phase_end.size() - 2], nlast = nops - last0;
        rc = launch_struct_for(g->ctx, T, t0.tree, drive, all.data() + last0, nlast, task, g->stream, 1, all.data(),
                               phase_end.data(), (int)phase_end.size(), nbr);
        st.launches_chained++;
      }
    } break;
    case TT_RANGE_FOR: {
      DOp ops[SG_MAXOPS];
      int nops = (int)members.size();
      for (int i = 0; i < nops; i++) make_op(g, g->eager[members[i]], acts[i], -1, ops[i]);
      const sg_task& tk = t0.t;
      auto arr = [&](int slot) -> const DArray* {
        int id = tk.arrays[slot];
        return id >= 0 && id < (int)g->arrays.size() ? &g->arrays[id] : nullptr;
      };
      for (int s = 0; s < 8; s++)
        if (tk.arrays[s] >= (int)g->arrays.size()) return fail(SG_ERR_ARG, "array id not registered");
      int64_t n = t0.n;
      const int32_t* dcount = nullptr;
      if (tk.op == SG_OP_HALO_UNPACK) {
        const DTree& T = g->dtrees[g->L.field_tree[tk.fields[0]]];
        int nf = 0;
        while (nf < 8 && tk.fields[nf] >= 0) nf++;
        int64_t rec = 4 + ((int64_t)nf << T.lblk);
        n = (arr(0)->n / rec) << T.lblk;
        if (!arr(0)->dcount) return fail(SG_ERR_ARG, "HALO_UNPACK buffer needs a device count");
      } else if (tk.op == SG_OP_MIGRATE_APPEND) {
        n = (arr(5)->n + arr(6)->n) / 17;
      } else if (n < 0) {
        const DArray* a0 = arr(0);
        if (!a0 || !a0->dcount) return fail(SG_ERR_ARG, "range_n < 0 needs arrays[0] with a device count");
        n = a0->n;
        dcount = a0->dcount;
      }
      if (tk.op == SG_OP_MIGRATE_COMPACT) {
        for (int s = 0; s < 7; s++)
          if (!arr(s) || ((s == 0 || s >= 5) && !arr(s)->dcount)) return fail(SG_ERR_ARG, "migration arrays need device counts");
        const uint64_t cap = (uint64_t)(arr(5)->n + arr(6)->n) / 17 + 1;
        if (cap > g->mig_hole_cap) {
          g->mig_holes = (uint32_t*)g->dev_alloc((cap + 1) * 4);
          g->mig_tail = (uint32_t*)g->dev_alloc(cap * 4);
          if (!g->mig_holes || !g->mig_tail) return fail(SG_ERR_CUDA, "migration scratch allocation failed");
          CUDA_TRY(cudaMemsetAsync(g->mig_holes, 0, 4, g->stream));
          g->mig_hole_cap = cap;
        }
      }
      if (tk.op == SG_OP_G2P_MIGRATE || tk.op == SG_OP_MIGRATE_APPEND) {
        for (int s = 0; s < 7; s++)
          if (!arr(s) || ((s == 0 || s >= 5) && !arr(s)->dcount)) return fail(SG_ERR_ARG, "migration arrays need device counts");
        uint64_t tiles = (uint64_t)n / 256 + 2;
        if (tiles > g->mig_tiles) {
          g->mig_status = (uint64_t*)g->dev_alloc(tiles * 8);
          if (!g->mig_status) return fail(SG_ERR_CUDA, "migration scratch allocation failed");
          CUDA_TRY(cudaMemsetAsync(g->mig_status, 0, tiles * 8, g->stream));
          g->mig_tiles = tiles;
        }
        if (!g->mig_ctl) {
          g->mig_ctl = (uint32_t*)g->dev_alloc(64);
          if (!g->mig_ctl) return fail(SG_ERR_CUDA, "migration scratch allocation failed");
          CUDA_TRY(cudaMemsetAsync(g->mig_ctl, 0, 64, g->stream));
        }
      }
      RangeScratch rs{g->mig_status, g->mig_ctl, g->mig_holes, g->mig_tail, g->mig_hole_cap};
      const DTree* gt = nullptr;
      if (tk.fields[0] >= 0 && tk.fields[0] < (int)g->L.field_tree.size() && g->L.field_tree[tk.fields[0]] >= 0)
        gt = &g->dtrees[g->L.field_tree[tk.fields[0]]];
      const DTree* gt2 = nullptr;   // G2P_ADJ: the adjoint tree
      if (tk.op == SG_OP_G2P_ADJ) gt2 = &g->dtrees[g->L.field_tree[tk.fields[4]]];
      const DBins* bp = nullptr;
      const bool mpm_op = tk.op == SG_OP_P2G || tk.op == SG_OP_G2P || tk.op == SG_OP_G2P_ADJ || tk.op == SG_OP_P2G_ADJ ||
                          tk.op == SG_OP_PERMUTE;
      if (n > 0 && nops == 1 && mpm_op && gt && !g->no_bin && tree_lb2(*gt) && (!gt2 || tree_lb2(*gt2))) {
        if ((rc = ensure_bins(g, g->L.field_tree[tk.fields[0]], tk.arrays[0], ops[0].p[1], n, dcount, st.aux_kernels)))
          return rc;
        bp = &g->bins_cur;
      }
      rc = launch_range_for(g->ctx, n, dcount, ops, nops, task, g->stream, &rs, gt, gt2, bp);
    } break;
    case TT_SERIAL: {
      if (t0.t.op == SG_OP_DIST_SIGNAL || t0.t.op == SG_OP_DIST_WAIT) {
        rc = sg_dist_launch(g, t0.t.op, (int)t0.t.params[0], task);
        if (rc) return rc;
        break;
      }
      DOp ops[SG_MAXOPS];
      int nops = (int)members.size();
      for (int i = 0; i < nops; i++) make_op(g, g->eager[members[i]], acts[i], -1, ops[i]);
      rc = launch_serial(g->ctx, ops, nops, task, g->stream);
    } break;
    case TT_DEACTIVATE: {
      const DTree& T = g->dtrees[t0.tree];
      if (g->L.deactivate_resets(t0.snode)) rc = launch_deactivate_reset(T, g->stream);
      else rc = launch_deactivate(g->ctx, T, t0.tree, g->L.snode_pos[t0.snode], g->lists[t0.tree].data(), task, g->stream);
    } break;
    default: rc = SG_ERR_ARG;
  }
  if (rc) return fail(rc, std::string("launch failed: ") + cudaGetErrorString(cudaGetLastError()));
  if (t0.type == TT_RANGE_FOR || t0.type == TT_SERIAL || t0.type == TT_STRUCT_FOR) {
    for (int m : members) {
      const sg_task& tk = g->eager[m].t;
      const uint32_t w = task_array_writes(tk);
      for (int s = 0; s < 8; s++)
        if (((w >> s) & 1u) && tk.arrays[s] >= 0 && tk.arrays[s] < (int)g->arr_epoch.size()) g->arr_epoch[tk.arrays[s]]++;
    }
  }
  st.launches++;
  return SG_OK;
}

// Makes the grid's device current for the scope of a call (lazy allocations
// and launches inside sg_flush), restoring the caller's device afterwards.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const sg_grid* g) {
    if (g->plan_only) return;
    if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; return; }
    if (prev == g->opts.device) prev = -1;
    else cudaSetDevice(g->opts.device);
  }
  ~DeviceScope() { if (prev >= 0) cudaSetDevice(prev); }
};

static int plan_op(const PTask& t) {
  return (t.type == TT_STRUCT_FOR || t.type == TT_RANGE_FOR || t.type == TT_SERIAL) ? t.t.op : 0;
}

extern "C" sg_status sg_flush(sg_grid* g, uint32_t passes, const int32_t* observed, int32_t n_observed, sg_stats* out) {
  if (!g) return fail(SG_ERR_ARG, "null grid");
  DeviceScope dev_scope(g);
  sg_stats st;
  std::memset(&st, 0, sizeof(st));
  auto t0 = std::chrono::steady_clock::now();
  size_t nf = g->L.field_tree.size();
  std::vector<char> obs(nf, 1);
  if (observed && n_observed >= 0) {
    std::fill(obs.begin(), obs.end(), 0);
    for (int i = 0; i < n_observed; i++)
      if (observed[i] >= 0 && observed[i] < (int)nf) obs[observed[i]] = 1;
  }
  st.tasks_lowered = (int64_t)g->eager.size();
  g->last_plan.clear();
  // arrays may have been rewritten outside the library since the last flush:
  // no binning carries over; slots are reassigned in this window's order
  for (sg_grid::BinSlot& sl : g->bin_slots) sl.valid = false;
  g->bin_next = 0;
  if (g->eager.empty()) {
    if (out) *out = st;
    return SG_OK;
  }
  uint64_t key = stream_hash(g->eager, passes, obs);
  auto it = g->cache.find(key);
  const Plan* plan;
  if (it != g->cache.end()) {
    st.plan_cache_hits = 1;
    plan = &it->second;
  } else {
    st.plan_cache_misses = 1;
    Plan p = optimize(g->L, g->eager, passes, obs);
    plan = &(g->cache[key] = std::move(p));
  }
  st.listgens_removed = plan->stats.listgens_removed;
  st.demotions = plan->stats.demotions;
  st.tasks_fused = plan->stats.fused;
  st.dead_removed = plan->stats.dead;
  st.tasks_chained = plan->stats.chained;
  auto t1 = std::chrono::steady_clock::now();
  st.plan_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
  sg_status rc = SG_OK;
  g->task_counter = 0;
  // CUDA graph replay of a plan that already ran once (its allocations done)
  bool capturing = false;
  const cudaStream_t user = g->stream;
  uint64_t sig = 0;
  if (!g->plan_only && g->use_graphs && !g->profiling && g->plan_runs[key]++ > 0) {
    // (chains carry their op tables in the kernel parameters: capturable like any launch)
    const bool chain = false;
    // signature of everything a capture bakes into launch arguments beyond the
    // plan: activation buffers, the array table, list / bin capacities
    sig = 1469598103934665603ull;
    auto mix = [&](uint64_t v) { sig ^= v; sig *= 1099511628211ull; };
    mix(key);
    // task params are baked into the captured kernels' __grid_constant__ op
    // tables (the plan key ignores them: passes never depend on them)
    for (const PTask& t : g->eager) {
      mix((uint64_t)(uintptr_t)t.coords);
      mix((uint64_t)t.n);
      mix((uint64_t)t.t.activating);
      for (int i = 0; i < 8; i++) {
        uint32_t b;
        std::memcpy(&b, &t.t.params[i], 4);
        mix(b);
      }
    }
    mix((uint64_t)(uintptr_t)g->d_arrays);
    mix((uint64_t)g->arrays.size());
    for (const DArray& a : g->arrays) { mix((uint64_t)(uintptr_t)a.ptr); mix((uint64_t)a.n); mix((uint64_t)(uintptr_t)a.dcount); }
    mix((uint64_t)jit_generation());   // a specialized kernel became ready: recapture
    mix((uint64_t)g->bin_gen);   // binning buffers (re)allocated: their pointers are baked into launches
    auto ex = g->gexec.find(key);
    if (!chain && ex != g->gexec.end() && ex->second && g->gsig[key] == sig) {
      // identical window: relaunch the graph as captured
      for (size_t gi = 0; gi < plan->groups.size(); gi++) {
        const auto& mem = plan->groups[gi];
        const auto& acts = plan->acts[gi];
        for (size_t m = 0; m < mem.size(); m++) {
          const PTask& t = g->eager[mem[m]];
          g->last_plan.push_back({(int)gi, t.type, t.call, t.snode, acts[m], plan_op(t)});
        }
        const PTask& t = g->eager[mem[0]];
        st.launches++;
        if (t.type == TT_LISTGEN) st.listgen_launched++;
        if (t.type == TT_CLEAR_LIST) st.clear_list_launched++;
        if (plan->phase_ends[gi].size() > 1) {
          std::vector<DOp> all;
          group_ops(g, mem, acts, t.tree, all);
          const int fs = chain_jacobi_start(g, t, all, plan->phase_ends[gi]);
          const int nph = (int)plan->phase_ends[gi].size();
          if (fs >= 0 && !flow_on() && t2_on() && jacobi_t2_applies(all.data(), plan->phase_ends[gi].data(), fs, nph)) {
            st.launches += fs + jacobi_t2_launches(fs, nph) - 1;
            st.launches_chained++;
          } else if (fs >= 0 && flow_on()) { st.launches += fs; st.launches_chained++; }
          else if (chain_is_split(g, t, mem.size(), plan->phase_ends[gi].size()))
            st.launches += (int64_t)plan->phase_ends[gi].size() - 1;
          else st.launches_chained++;
        }
      }
      st.aux_kernels = g->gaux[key];
      sg_status rc2 = SG_OK;
      if (cudaGraphLaunch(ex->second, g->stream) != cudaSuccess) rc2 = fail(SG_ERR_CUDA, "graph launch failed");
      g->eager.clear();
      g->coords_seen.clear();
      g->ncalls = 0;
      if (out) *out = st;
      return rc2;
    }
    if (!chain) {
      if (!g->cap_stream) cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking);
      if (g->cap_stream && cudaStreamBeginCapture(g->cap_stream, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
        g->stream = g->cap_stream;
        capturing = true;
      } else {
        cudaGetLastError();
      }
    }
  }
  // parallel compilation: submit every struct-for group's
  // specialized kernel before the first launch, so they compile concurrently
  if (!g->plan_only && !g->jit_prefetched[key]) {
    g->jit_prefetched[key] = 1;
    int64_t jm[1] = {0};
    jit_stats(jm, 1);
    if (jm[0])
      for (size_t gi = 0; gi < plan->groups.size(); gi++) {
        const PTask& t0 = g->eager[plan->groups[gi][0]];
        if (t0.type != TT_STRUCT_FOR || plan->phase_ends[gi].size() > 1) continue;
        DOp ops[SG_MAXOPS];
        const int nops = (int)plan->groups[gi].size();
        for (int i = 0; i < nops; i++) make_op(g, g->eager[plan->groups[gi][i]], plan->acts[gi][i], t0.tree, ops[i]);
        JitGroup G;
        if (jit_group_of(g->dtrees[t0.tree], ops, nops, G)) jit_lookup(G, true);
      }
  }
  for (size_t gi = 0; gi < plan->groups.size(); gi++) {
    const auto& mem = plan->groups[gi];
    const auto& acts = plan->acts[gi];
    for (size_t m = 0; m < mem.size(); m++) {
      const PTask& t = g->eager[mem[m]];
      g->last_plan.push_back({(int)gi, t.type, t.call, t.snode, acts[m], plan_op(t)});
    }
    if (g->plan_only) {
      const PTask& t = g->eager[mem[0]];
      st.launches++;
      if (t.type == TT_LISTGEN) st.listgen_launched++;
      if (t.type == TT_CLEAR_LIST) st.clear_list_launched++;
      continue;
    }
    if (!rc) {
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (g->profiling) { e0 = g->get_event(); cudaEventRecord(e0, g->stream); }
      rc = launch_group(g, mem, acts, plan->phase_ends[gi], st);
      if (g->profiling) {
        e1 = g->get_event();
        cudaEventRecord(e1, g->stream);
        const PTask& t = g->eager[mem[0]];
        int key = t.type == TT_STRUCT_FOR ? 100 + t.t.op : t.type == TT_LISTGEN ? 200 + t.snode
                : t.type == TT_RANGE_FOR ? 300 + t.t.op : t.type;
        g->prof_pending.push_back({key, {e0, e1}});
      }
    }
  }
  if (capturing) {
    g->stream = user;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(g->cap_stream, &graph);
    if (e != cudaSuccess || rc) {
      if (graph) cudaGraphDestroy(graph);
      if (!rc) rc = fail(SG_ERR_CUDA, std::string("graph capture failed: ") + cudaGetErrorString(e));
    } else {
      cudaGraphExec_t& ex = g->gexec[key];
      bool ok = false;
      if (ex) {
        cudaGraphExecUpdateResultInfo info;
        ok = cudaGraphExecUpdate(ex, graph, &info) == cudaSuccess;
        if (!ok) { cudaGetLastError(); cudaGraphExecDestroy(ex); ex = nullptr; }
      }
      if (!ok && cudaGraphInstantiate(&ex, graph, 0) != cudaSuccess) {
        ex = nullptr;
        rc = fail(SG_ERR_CUDA, "graph instantiation failed");
      }
      if (ex && cudaGraphLaunch(ex, g->stream) != cudaSuccess) rc = fail(SG_ERR_CUDA, "graph launch failed");
      if (ex) { g->gsig[key] = sig; g->gaux[key] = st.aux_kernels; }
      cudaGraphDestroy(graph);
    }
  }
  g->eager.clear();
  g->coords_seen.clear();
  g->ncalls = 0;
  if (out) *out = st;
  return rc;
}

extern "C" sg_status sg_sync(sg_grid* g) {
  if (!g) return fail(SG_ERR_ARG, "null grid");
  if (g->plan_only) return SG_OK;
  CUDA_TRY(cudaStreamSynchronize(g->stream));
  uint32_t e[2] = {0, 0};
  CUDA_TRY(cudaMemcpy(e, g->ctx.err, 8, cudaMemcpyDeviceToHost));
  if (e[0]) {
    int code = (int)(int32_t)e[0];
    const char* what = code == SG_ERR_POOL_EXHAUSTED ? "pool exhausted"
                       : code == SG_ERR_LIST_OVERFLOW ? "list overflow"
                       : code == SG_ERR_DEMOTION_TRAP ? "non-activating write to an inactive cell"
                       : code == SG_ERR_RANGE ? "coordinate out of range"
                       : code == SG_ERR_TIMEOUT ? "a neighbour rank's exchange signal never arrived" : "device error";
    return fail(code, std::string("device: ") + what + " (task " + std::to_string(e[1]) + ")");
  }
  return SG_OK;
}

static sg_status flush_sync(sg_grid* g) {
  if (g->plan_only) return fail(SG_ERR_STATE, "plan-only grid has no device state");
  sg_status rc = sg_flush(g, SG_PASS_ALL, nullptr, -1, nullptr);
  if (rc) return rc;
  return sg_sync(g);
}

extern "C" sg_status sg_export_mask(sg_grid* g, int32_t snode, int32_t* host, int64_t cap, int64_t* count) {
  if (!g || !count) return fail(SG_ERR_ARG, "null argument");
  if (snode <= 0 || snode >= (int)g->L.nodes.size() || !g->L.is_sparse(snode)) return fail(SG_ERR_ARG, "bad snode");
  sg_status rc = flush_sync(g);
  if (rc) return rc;
  int tid = g->L.snode_tree[snode], k = g->L.snode_pos[snode];
  const DTree& T = g->dtrees[tid];
  const DLevel& D = T.lev[k];
  int lt = D.lres[0] + D.lres[1] + D.lres[2];
  if (lt > 30) return fail(SG_ERR_ARG, "level too large to export");
  int64_t total = 1ll << lt;
  uint8_t* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, total));
  int lrc = launch_mask_scan(g->ctx, T, tid, k, d, g->stream);
  std::vector<uint8_t> h(total);
  cudaError_t e = cudaMemcpyAsync(h.data(), d, total, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(d);
  if (lrc || e != cudaSuccess) return fail(SG_ERR_CUDA, "mask scan failed");
  int64_t n = 0;
  for (int64_t i = 0; i < total; i++) {
    if (!h[i]) continue;
    if (n < cap && host) {
      int64_t c[3] = {i >> (D.lres[1] + D.lres[2]), (i >> D.lres[2]) & ((1ll << D.lres[1]) - 1), i & ((1ll << D.lres[2]) - 1)};
      for (int a = 0; a < T.nd; a++) host[n * T.nd + a] = (int32_t)c[a];
    }
    n++;
  }
  *count = n;
  return SG_OK;
}

extern "C" sg_status sg_export_list(sg_grid* g, int32_t snode, int32_t* host, int64_t cap, int64_t* count) {
  if (!g || !count) return fail(SG_ERR_ARG, "null argument");
  if (snode <= 0 || snode >= (int)g->L.nodes.size() || !g->L.is_sparse(snode)) return fail(SG_ERR_ARG, "bad snode");
  sg_status rc = flush_sync(g);
  if (rc) return rc;
  int tid = g->L.snode_tree[snode], k = g->L.snode_pos[snode];
  const DList& Ls = g->lists[tid][k];
  if (!Ls.entries) { *count = 0; return SG_OK; }
  uint32_t n = 0;
  CUDA_TRY(cudaMemcpy(&n, Ls.count, 4, cudaMemcpyDeviceToHost));
  *count = n;
  if (!host || cap <= 0 || n == 0) return SG_OK;
  const DTree& T = g->dtrees[tid];
  int32_t* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, (size_t)n * T.nd * 4));
  int lrc = launch_list_decode(T, k, Ls, d, g->stream);
  std::vector<int32_t> h((size_t)n * T.nd);
  cudaError_t e = cudaMemcpyAsync(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(d);
  if (lrc || e != cudaSuccess) return fail(SG_ERR_CUDA, "list decode failed");
  int64_t m = std::min<int64_t>(cap, n);
  std::memcpy(host, h.data(), (size_t)m * T.nd * 4);
  return SG_OK;
}

static int64_t field_cells(const sg_grid* g, int f, const DTree** T) {
  int tid = g->L.field_tree[f];
  if (tid < 0) { *T = nullptr; return 1; }
  *T = &g->dtrees[tid];
  const DLevel& L = (*T)->lev[(*T)->nlev - 1];
  return 1ll << (L.lres[0] + L.lres[1] + L.lres[2]);
}

extern "C" sg_status sg_struct_for_batch(sg_grid* g, const sg_task* tasks, int32_t n) {
  if (!g || (n > 0 && !tasks) || n < 0) return fail(SG_ERR_ARG, "bad batch");
  for (int32_t i = 0; i < n; i++) {
    sg_status rc = sg_struct_for(g, tasks + i);
    if (rc) return rc;
  }
  return SG_OK;
}

extern "C" sg_status sg_read_scalar_async(sg_grid* g, int32_t f, void* host) {
  if (!g || !host || f < 0 || f >= (int)g->L.field_tree.size() || g->L.field_tree[f] >= 0)
    return fail(SG_ERR_ARG, "sg_read_scalar_async needs a 0-D field");
  if (g->plan_only) return fail(SG_ERR_STATE, "plan-only grid has no device state");
  CUDA_TRY(cudaMemcpyAsync(host, g->ctx.scalars + g->L.field_scalar[f], 4, cudaMemcpyDeviceToHost, g->stream));
  return SG_OK;
}

extern "C" sg_status sg_read_field(sg_grid* g, int32_t f, void* host, int64_t bytes) {
  if (!g || !host || f < 0 || f >= (int)g->L.field_tree.size()) return fail(SG_ERR_ARG, "bad field");
  sg_status rc = flush_sync(g);
  if (rc) return rc;
  const DTree* T;
  int64_t n = field_cells(g, f, &T);
  if (bytes != n * 4) return fail(SG_ERR_ARG, "size mismatch: expected " + std::to_string(n * 4) + " bytes");
  if (!T) {
    CUDA_TRY(cudaMemcpy(host, g->ctx.scalars + g->L.field_scalar[f], 4, cudaMemcpyDeviceToHost));
    return SG_OK;
  }
  uint32_t* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, n * 4));
  int lrc = launch_read_field(g->ctx, *T, g->L.field_tree[f], g->L.field_slot[f], d, g->stream);
  cudaError_t e = cudaMemcpyAsync(host, d, n * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(d);
  if (lrc || e != cudaSuccess) return fail(SG_ERR_CUDA, "read_field failed");
  return SG_OK;
}

extern "C" sg_status sg_load_field(sg_grid* g, int32_t f, const void* host, int64_t bytes) {
  if (!g || !host || f < 0 || f >= (int)g->L.field_tree.size()) return fail(SG_ERR_ARG, "bad field");
  sg_status rc = flush_sync(g);
  if (rc) return rc;
  const DTree* T;
  int64_t n = field_cells(g, f, &T);
  if (bytes != n * 4) return fail(SG_ERR_ARG, "size mismatch");
  if (!T) {
    CUDA_TRY(cudaMemcpy(g->ctx.scalars + g->L.field_scalar[f], host, 4, cudaMemcpyHostToDevice));
    return SG_OK;
  }
  uint32_t* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, n * 4));
  cudaError_t e = cudaMemcpyAsync(d, host, n * 4, cudaMemcpyHostToDevice, g->stream);
  int lrc = e == cudaSuccess ? launch_load_field(g->ctx, *T, g->L.field_tree[f], g->L.field_slot[f], d, g->stream) : 1;
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(d);
  if (lrc || e != cudaSuccess) return fail(SG_ERR_CUDA, "load_field failed");
  return SG_OK;
}

extern "C" sg_status sg_last_plan(sg_grid* g, int32_t* out, int64_t cap, int64_t* count) {
  if (!g || !count) return fail(SG_ERR_ARG, "null argument");
  *count = (int64_t)g->last_plan.size();
  for (int64_t i = 0; i < std::min<int64_t>(cap, *count) && out; i++) {
    const PlanRecord& r = g->last_plan[i];
    out[i * 6 + 0] = r.group; out[i * 6 + 1] = r.type; out[i * 6 + 2] = r.call;
    out[i * 6 + 3] = r.snode; out[i * 6 + 4] = (int32_t)r.act; out[i * 6 + 5] = r.flags;
  }
  return SG_OK;
}

// [0] num trees, then per tree i: [1+4i] pool base of the leaf segment, [2+4i] leaf stride words,
// [3+4i] leaf capacity, [4+4i] payload offset words.
extern "C" sg_status sg_device_info(sg_grid* g, int64_t* out, int32_t n) {
  if (!g || !out) return fail(SG_ERR_ARG, "null argument");
  int nt = (int)g->dtrees.size();
  if (n > 0) out[0] = nt;
  for (int i = 0; i < nt; i++) {
    const DTree& T = g->dtrees[i];
    int64_t v[4] = {0, 0, 0, 0};
    if (T.nlev > 0) {
      const DSeg& S = T.seg[T.nseg - 1];
      v[0] = (int64_t)(uintptr_t)S.base; v[1] = (int64_t)S.stride; v[2] = S.capacity; v[3] = T.payload_off;
    }
    for (int k = 0; k < 4; k++) if (1 + 4 * i + k < n) out[1 + 4 * i + k] = v[k];
  }
  return SG_OK;
}

extern "C" sg_status sg_set_profiling(sg_grid* g, int32_t on) {
  if (!g) return fail(SG_ERR_ARG, "null grid");
  if (g->plan_only) return fail(SG_ERR_STATE, "plan-only grid");
  g->profiling = on != 0;
  return SG_OK;
}

extern "C" sg_status sg_profile_read(sg_grid* g, double* ms, int64_t* count, int32_t n_kinds) {
  if (!g || !ms || !count) return fail(SG_ERR_ARG, "null argument");
  CUDA_TRY(cudaStreamSynchronize(g->stream));
  for (int i = 0; i < n_kinds; i++) { ms[i] = 0; count[i] = 0; }
  for (auto& p : g->prof_pending) {
    float t = 0;
    cudaEventElapsedTime(&t, p.second.first, p.second.second);
    int key = p.first;
    int kinds[2] = {key >= 300 ? TT_RANGE_FOR : key >= 200 ? TT_LISTGEN : key >= 100 ? TT_STRUCT_FOR : key,
                    key >= 100 ? key : -1};
    for (int k : kinds) {
      if (k >= 0 && k < n_kinds) { ms[k] += t; count[k]++; }
    }
    g->event_pool.push_back(p.second.first);
    g->event_pool.push_back(p.second.second);
  }
  g->prof_pending.clear();
  return SG_OK;
}

extern "C" const char* sg_last_error(void) { return g_err.c_str(); }

extern "C" sg_status sg_jit_info(int64_t* out, int32_t n) {
  if (!out || n < 1) return fail(SG_ERR_ARG, "null output");
  jit_stats(out, n);
  return SG_OK;
}

extern "C" sg_status sg_jit_set_mode(int32_t mode) {
  if (mode < -1 || mode > 2) return fail(SG_ERR_ARG, "JIT mode is -1 (env), 0, 1 or 2");
  jit_set_mode(mode);
  return SG_OK;
}

extern "C" sg_status sg_jit_shutdown(void) {
  jit_shutdown();
  return SG_OK;
}

extern "C" sg_status sg_jit_selftest(int32_t nd, int32_t gl, int32_t i32, const int32_t* ops, int32_t nops,
                                     char* log, int64_t cap) {
  if (!ops || nops < 1 || nops > SG_MAXOPS) return fail(SG_ERR_ARG, "bad op list");
  const int rc = jit_selftest(nd, gl, i32, ops, nops, log, cap);
  return rc == 0 ? SG_OK : fail(SG_ERR_STATE, "NVRTC compile failed (" + std::to_string(rc) + ")");
}
