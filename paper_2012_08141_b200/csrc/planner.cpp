// planner.cpp -- lowering, state-flow graph and the four whole-program passes.
//
//   * Lowering ("kernels are decomposed into tasks"; PAPER.md:316
//     "3 tasks per such a small kernel"): a struct-for over a sparse tree emits
//     one listgen per listed sparse level (optionally preceded by clear-list,
//     the paper-faithful count), then the body.
//   * SFG: tasks carry input/output states; insertion adds
//     RAW edges from the latest writer, WAW edges on the main branch and WAR
//     edges from readers (Fig. 4 caption).  Deletion is
//     "topologically sort, remove, rebuild": every pass below
//     produces a filtered / reordered sequence that is rebuilt from scratch.
//   * Passes, run to a fixpoint in the order listgen removal -> activation
//     demotion -> listgen removal -> fusion -> DSE:
//       listgen removal  PAPER.md:338, 390 (section 6.2, 7.1)
//       act. demotion    PAPER.md:346 (section 6.3)
//       task fusion      PAPER.md:367-370, 392 (section 6.4)
//       dead stores      PAPER.md:374-377 (section 6.5)
//   * Plan cache keyed by a hash of the task stream (the IR bank's role,
//     PAPER.md:395).
#include "planner.h"

#include <algorithm>
#include <cstring>
#include <unordered_set>

namespace sg {

std::vector<int> HLayout::listed_levels(int t) const {
  std::vector<int> out;
  const HTree& T = trees[t];
  for (size_t k = 0; k < T.levels.size(); k++) {
    int s = T.levels[k];
    if (!is_sparse(s)) continue;
    if (k + 1 == T.levels.size() && nodes[s].kind == SG_BITMASKED) continue;
    out.push_back(s);
  }
  return out;
}

bool HLayout::deactivate_resets(int snode) const {
  if (snode <= 0 || snode >= (int)nodes.size() || snode_tree[snode] < 0) return false;
  const HTree& T = trees[snode_tree[snode]];
  int first = -1;
  for (int s : T.levels)
    if (is_sparse(s)) { first = s; break; }
  if (first != snode) return false;
  double cells = 1.0;
  for (int s : T.levels) cells *= (double)nodes[s].extent[0] * nodes[s].extent[1] * nodes[s].extent[2];
  return cells * 4.0 * std::max<size_t>(1, T.fields.size()) <= 64.0 * 1024 * 1024;
}

std::vector<int> HLayout::sparse_levels(int t) const {
  std::vector<int> out;
  for (int s : trees[t].levels)
    if (is_sparse(s)) out.push_back(s);
  return out;
}

// ---------------------------------------------------------------------------
// Op vocabulary: operand roles and access patterns (include/sg.h).
// ---------------------------------------------------------------------------
enum { R_READ = 1, R_WRITE = 2, R_RW = 3 };
struct OpUse {
  int slot;       // operand slot
  bool array;     // arrays[] instead of fields[]
  int role;
  int access;
  bool complete;
};

static std::vector<OpUse> op_uses(const sg_task& t) {
  std::vector<OpUse> u;
  auto F = [&](int slot, int role, int acc, bool complete = false) { u.push_back({slot, false, role, acc, complete}); };
  auto A = [&](int slot, int role, int acc, bool complete = false) { u.push_back({slot, true, role, acc, complete}); };
  switch (t.op) {
    case SG_OP_FILL: F(0, R_WRITE, AC_ID, true); break;
    case SG_OP_ADD_CONST: F(1, R_READ, AC_ID); F(0, R_WRITE, AC_ID, true); break;
    case SG_OP_INC: F(0, R_RW, AC_ID); break;
    case SG_OP_AXPY: F(1, R_READ, AC_ID); F(2, R_READ, AC_ID); F(0, R_WRITE, AC_ID, true); break;
    case SG_OP_STENCIL: F(1, R_READ, AC_NBR); F(0, R_WRITE, AC_ID, true); break;
    case SG_OP_JACOBI: F(1, R_READ, AC_NBR); F(2, R_READ, AC_ID); F(0, R_WRITE, AC_ID, true); break;
    case SG_OP_REDUCE_SUM: F(1, R_READ, AC_ID); F(0, R_RW, AC_CONST); break;
    case SG_OP_DOWNSAMPLE:
      if (t.fields[1] >= 0) F(1, R_READ, AC_ID);
      F(0, R_RW, AC_DIV2);
      break;
    case SG_OP_JITTER: F(0, R_RW, AC_NBR); break;
    case SG_OP_CLEAR_SCALAR: F(0, R_WRITE, AC_CONST, true); break;
    case SG_OP_P2G:
      for (int i = 0; i < 4; i++) A(i, R_READ, AC_ID);
      for (int i = 0; i < 4; i++) F(i, R_RW, AC_DATA);
      break;
    case SG_OP_GRID_OP:
      for (int i = 0; i < 3; i++) F(i, R_RW, AC_ID);
      F(3, R_READ, AC_ID);
      break;
    case SG_OP_G2P:
      for (int i = 0; i < 3; i++) F(i, R_READ, AC_DATA);
      if (t.arrays[4] >= 0) {   // out of place: state a0..a3 -> a4..a7
        A(0, R_READ, AC_ID); A(3, R_READ, AC_ID);
        for (int i = 4; i < 8; i++) A(i, R_WRITE, AC_ID, true);
      } else {
        A(0, R_RW, AC_ID); A(1, R_WRITE, AC_ID, true); A(2, R_WRITE, AC_ID, true); A(3, R_RW, AC_ID);
      }
      break;
    case SG_OP_LOSS_MEAN: A(0, R_READ, AC_ID); F(0, R_RW, AC_CONST); break;
    case SG_OP_SMOOTH_RB: F(1, R_READ, AC_ID); F(0, R_RW, AC_NBR); break;
    case SG_OP_RESTRICT: F(1, R_READ, AC_ID); F(2, R_READ, AC_NBR); F(0, R_RW, AC_DIV2); break;
    case SG_OP_PROLONG: F(1, R_READ, AC_DIV2); F(0, R_RW, AC_ID); break;
    case SG_OP_RESID_NORM2: F(1, R_READ, AC_ID); F(2, R_READ, AC_NBR); F(0, R_RW, AC_CONST); break;
    case SG_OP_DOT: F(1, R_READ, AC_ID); F(2, R_READ, AC_ID); F(0, R_RW, AC_CONST); break;
    case SG_OP_AXPY_RATIO:
    case SG_OP_XPAY_RATIO: F(1, R_READ, AC_ID); F(2, R_READ, AC_CONST); F(3, R_READ, AC_CONST); F(0, R_RW, AC_ID); break;
    case SG_OP_COPY_SCALAR: F(1, R_READ, AC_CONST); F(0, R_WRITE, AC_CONST, true); break;
    case SG_OP_ADJ_INIT:
      for (int i = 0; i < 4; i++) A(i, R_WRITE, AC_ID, true);
      break;
    case SG_OP_G2P_ADJ:
      for (int i = 0; i < 4; i++) F(i, R_READ, AC_DATA);
      for (int i = 4; i < 8; i++) F(i, R_RW, AC_DATA);
      for (int i = 0; i < 6; i++) A(i, R_READ, AC_ID);
      A(6, R_WRITE, AC_ID, true); A(7, R_WRITE, AC_ID, true);
      break;
    case SG_OP_P2G_ADJ:
      for (int i = 0; i < 4; i++) F(i, R_READ, AC_DATA);
      for (int i = 0; i < 4; i++) A(i, R_READ, AC_ID);
      A(4, R_RW, AC_ID); A(5, R_WRITE, AC_ID, true); A(6, R_WRITE, AC_ID, true); A(7, R_RW, AC_ID);
      break;
    case SG_OP_ARRAY_COUNT: A(0, R_WRITE, AC_CONST); break;
    case SG_OP_HALO_PACK:
      for (int i = 0; i < 8 && t.fields[i] >= 0; i++) F(i, R_READ, AC_ID);
      A(0, R_RW, AC_DATA);
      break;
    case SG_OP_HALO_UNPACK:
      A(0, R_READ, AC_DATA);
      for (int i = 0; i < 8 && t.fields[i] >= 0; i++) F(i, R_RW, AC_DATA);
      break;
    case SG_OP_G2P_MIGRATE:
      for (int i = 0; i < 3; i++) F(i, R_READ, AC_DATA);
      for (int i = 0; i < 5; i++) A(i, R_RW, AC_DATA);     // compaction moves particles
      A(5, R_RW, AC_DATA); A(6, R_RW, AC_DATA);
      break;
    case SG_OP_MIGRATE_APPEND:
      for (int i = 0; i < 5; i++) A(i, R_RW, AC_DATA);
      A(5, R_READ, AC_DATA); A(6, R_READ, AC_DATA);
      break;
    case SG_OP_MIGRATE_COMPACT:
      for (int i = 0; i < 7; i++) A(i, R_RW, AC_DATA);
      break;
    case SG_OP_PERMUTE: A(0, R_READ, AC_DATA); A(1, R_READ, AC_DATA); A(2, R_WRITE, AC_DATA, true); break;
    case SG_OP_DIST_SIGNAL:   // send buffers complete -> the neighbours' receive buffers
      A(0, R_READ, AC_DATA); A(1, R_READ, AC_DATA); A(2, R_WRITE, AC_DATA); A(3, R_WRITE, AC_DATA);
      break;
    case SG_OP_DIST_WAIT:
      A(0, R_READ, AC_DATA); A(1, R_READ, AC_DATA); A(2, R_RW, AC_DATA); A(3, R_RW, AC_DATA);
      break;
    default: break;
  }
  return u;
}

uint32_t task_array_writes(const sg_task& t) {
  uint32_t m = 0;
  for (const OpUse& u : op_uses(t))
    if (u.array && (u.role & R_WRITE)) m |= 1u << u.slot;
  return m;
}

static int op_min_fields(int op) {
  switch (op) {
    case SG_OP_FILL: case SG_OP_INC: case SG_OP_JITTER: case SG_OP_CLEAR_SCALAR: case SG_OP_DOWNSAMPLE: return 1;
    case SG_OP_ADD_CONST: case SG_OP_STENCIL: case SG_OP_REDUCE_SUM: return 2;
    case SG_OP_AXPY: case SG_OP_JACOBI: return 3;
    case SG_OP_P2G: case SG_OP_GRID_OP: case SG_OP_G2P: case SG_OP_G2P_MIGRATE: return 4;
    case SG_OP_ARRAY_COUNT: case SG_OP_MIGRATE_APPEND: case SG_OP_ADJ_INIT: case SG_OP_MIGRATE_COMPACT: return 0;
    case SG_OP_DIST_SIGNAL: case SG_OP_DIST_WAIT: return 0;
    case SG_OP_PERMUTE: return 1;
    case SG_OP_LOSS_MEAN: return 1;
    case SG_OP_SMOOTH_RB: case SG_OP_PROLONG: return 2;
    case SG_OP_RESTRICT: case SG_OP_RESID_NORM2: case SG_OP_DOT: return 3;
    case SG_OP_AXPY_RATIO: case SG_OP_XPAY_RATIO: return 4;
    case SG_OP_COPY_SCALAR: return 2;
    case SG_OP_G2P_ADJ: return 8;
    case SG_OP_P2G_ADJ: return 4;
    case SG_OP_HALO_PACK: case SG_OP_HALO_UNPACK: return 1;
    default: return -1;
  }
}

static void add_activation_states(const HLayout& L, int tree, std::vector<Use>& in, std::vector<Use>& out) {
  for (int s : L.sparse_levels(tree)) {
    in.push_back({skey(ST_MASK, s), AC_NONE, false});
    out.push_back({skey(ST_MASK, s), AC_NONE, false});
    if (L.nodes[s].kind == SG_POINTER) {
      in.push_back({skey(ST_ALLOC, s), AC_NONE, false});
      out.push_back({skey(ST_ALLOC, s), AC_NONE, false});
    }
  }
}

void task_meta(const HLayout& L, PTask& t) {
  t.in.clear();
  t.out.clear();
  switch (t.type) {
    case TT_ACTIVATE:
      add_activation_states(L, t.tree, t.in, t.out);
      break;
    case TT_LISTGEN: {
      const HTree& T = L.trees[t.tree];
      int pos = L.snode_pos[t.snode];
      t.in.push_back({skey(ST_MASK, t.snode), AC_NONE, false});
      for (int k = pos - 1; k >= 0; k--) {
        int s = T.levels[k];
        if (!L.is_sparse(s)) continue;
        t.in.push_back({skey(ST_MASK, s), AC_NONE, false});
      }
      for (int k = pos - 1; k >= 0; k--) {
        int s = T.levels[k];
        if (L.is_sparse(s)) { t.in.push_back({skey(ST_LIST, s), AC_NONE, false}); break; }
      }
      t.out.push_back({skey(ST_LIST, t.snode), AC_NONE, true});
    } break;
    case TT_CLEAR_LIST:
      t.out.push_back({skey(ST_LIST, t.snode), AC_NONE, true});
      break;
    case TT_DEACTIVATE: {
      const HTree& T = L.trees[t.tree];
      const bool reset = L.deactivate_resets(t.snode);
      if (!reset)
        for (int s : L.listed_levels(t.tree)) t.in.push_back({skey(ST_LIST, s), AC_NONE, false});
      int pos = L.snode_pos[t.snode];
      for (size_t k = pos; k < T.levels.size(); k++) {
        int s = T.levels[k];
        if (!L.is_sparse(s)) continue;
        if (!reset) t.in.push_back({skey(ST_MASK, s), AC_NONE, false});
        t.out.push_back({skey(ST_MASK, s), AC_NONE, true});
        if (L.nodes[s].kind == SG_POINTER) {
          if (!reset) t.in.push_back({skey(ST_ALLOC, s), AC_NONE, false});
          t.out.push_back({skey(ST_ALLOC, s), AC_NONE, reset});
        }
      }
      for (int f : T.fields) t.out.push_back({skey(ST_VALUE, f), AC_ID, true});
    } break;
    case TT_STRUCT_FOR: case TT_RANGE_FOR: case TT_SERIAL: {
      if (t.type == TT_STRUCT_FOR) {
        const HTree& T = L.trees[t.tree];
        if (T.driving >= 0) t.in.push_back({skey(ST_LIST, T.levels[T.driving]), AC_NONE, false});
        if (T.leaf_bitmasked) t.in.push_back({skey(ST_MASK, T.levels.back()), AC_NONE, false});
      }
      for (const OpUse& u : op_uses(t.t)) {
        int id = u.array ? t.t.arrays[u.slot] : t.t.fields[u.slot];
        if (id < 0) continue;
        int64_t s = skey(u.array ? ST_ARRAY : ST_VALUE, id);
        if (u.role & R_READ) t.in.push_back({s, u.access, false});
        if (u.role & R_WRITE) {
          t.out.push_back({s, u.access, u.complete});
          if (!u.complete && !(u.role & R_READ)) t.in.push_back({s, u.access, false});
          if (!u.array && ((t.act >> u.slot) & 1u) && L.field_tree[id] >= 0)
            add_activation_states(L, L.field_tree[id], t.in, t.out);
        }
      }
      const int64_t seq = skey(ST_ARRAY, 0x7ffffff0);
      if (t.t.op == SG_OP_DIST_SIGNAL || t.t.op == SG_OP_DIST_WAIT) {
        // every exchange task reads and writes one sequence state: the passes
        // keep exchanges in program order on every rank (no cross-rank
        // deadlock from a reordered wait)
        t.in.push_back({seq, AC_NONE, false});
        t.out.push_back({seq, AC_NONE, false});
      } else {
        // a write into a send buffer (pack, count reset, migration) reads the
        // sequence: it stays after the exchange before it and before the one
        // after it.  On the peer transport it lands in the neighbour's receive
        // buffer, which the neighbour may still be consuming until then.
        bool ordered = false;
        for (const OpUse& u : op_uses(t.t)) {
          int id = u.array ? t.t.arrays[u.slot] : -1;
          if (id >= 0 && (u.role & R_WRITE) && id < (int)L.seq_arrays.size() && L.seq_arrays[id]) ordered = true;
        }
        if (ordered) t.in.push_back({seq, AC_NONE, false});
      }
    } break;
    default: break;
  }
}

// ---------------------------------------------------------------------------
// Lowering
// ---------------------------------------------------------------------------
static void emit_lists(const HLayout& L, const std::vector<int>& levels, int tree, int call, bool faithful,
                       bool pinned, std::vector<PTask>& out) {
  for (int s : levels) {
    if (faithful) {
      PTask c;
      c.type = TT_CLEAR_LIST; c.snode = s; c.tree = tree; c.call = call; c.pinned = pinned;
      out.push_back(c);
    }
    PTask g;
    g.type = TT_LISTGEN; g.snode = s; g.tree = tree; g.call = call; g.pinned = pinned;
    out.push_back(g);
  }
}

static bool valid_field(const HLayout& L, int f) { return f >= 0 && f < (int)L.field_tree.size(); }

static int validate_task(const HLayout& L, const sg_task& t, std::string& err) {
  int need = op_min_fields(t.op);
  if (need < 0) { err = "unknown op"; return SG_ERR_ARG; }
  for (int i = 0; i < need; i++) {
    if (t.op == SG_OP_DOWNSAMPLE && i == 1) continue;
    if (!valid_field(L, t.fields[i])) { err = "missing or bad field operand"; return SG_ERR_ARG; }
  }
  const bool sf = t.kind == SG_TASK_STRUCT_FOR;
  if (t.kind == SG_TASK_RANGE_FOR && t.range_n < 0 && t.arrays[0] < 0) {
    err = "range_n < 0 needs arrays[0] with a device count"; return SG_ERR_ARG;
  }
  switch (t.op) {
    case SG_OP_ARRAY_COUNT:
      if (t.kind != SG_TASK_SERIAL || t.arrays[0] < 0) { err = "ARRAY_COUNT is a serial op on arrays[0]"; return SG_ERR_ARG; }
      return SG_OK;
    case SG_OP_PERMUTE: {
      if (t.kind != SG_TASK_RANGE_FOR) { err = "PERMUTE is a range-for op"; return SG_ERR_ARG; }
      for (int i = 0; i < 3; i++) if (t.arrays[i] < 0) { err = "PERMUTE needs arrays a0 (positions), a1 (src), a2 (dst)"; return SG_ERR_ARG; }
      if (t.arrays[1] == t.arrays[2]) { err = "PERMUTE is out of place"; return SG_ERR_ARG; }
      int tree = L.field_tree[t.fields[0]];
      if (tree < 0 || L.trees[tree].nd != 3 || L.trees[tree].driving < 0) { err = "PERMUTE field must live in a 3-D sparse tree"; return SG_ERR_ARG; }
      return SG_OK;
    }
    case SG_OP_DIST_SIGNAL:
    case SG_OP_DIST_WAIT:
      if (t.kind != SG_TASK_SERIAL) { err = "exchange tasks are serial ops"; return SG_ERR_ARG; }
      if (!(t.params[0] == 0.0f || t.params[0] == 1.0f || t.params[0] == 2.0f)) { err = "exchange kind (p0) must be 0, 1 or 2"; return SG_ERR_ARG; }
      return SG_OK;
    case SG_OP_MIGRATE_APPEND:
    case SG_OP_MIGRATE_COMPACT:
    case SG_OP_HALO_UNPACK:
    case SG_OP_G2P_MIGRATE:
      if (t.kind != SG_TASK_RANGE_FOR) { err = "migration / unpack ops are range-for ops"; return SG_ERR_ARG; }
      for (int i = 0; i < (t.op == SG_OP_HALO_UNPACK ? 1 : 7); i++)
        if (t.arrays[i] < 0) { err = "missing array operand"; return SG_ERR_ARG; }
      if (t.op == SG_OP_HALO_UNPACK) {
        int tree = L.field_tree[t.fields[0]];
        if (tree < 0 || L.trees[tree].driving < 0) { err = "HALO_UNPACK fields must live in a sparse tree"; return SG_ERR_ARG; }
        for (int i = 0; i < 8 && t.fields[i] >= 0; i++)
          if (!valid_field(L, t.fields[i]) || L.field_tree[t.fields[i]] != tree) { err = "HALO_UNPACK fields must share a tree"; return SG_ERR_ARG; }
        return SG_OK;
      }
      if (t.op == SG_OP_MIGRATE_APPEND || t.op == SG_OP_MIGRATE_COMPACT) return SG_OK;
      break;   // G2P_MIGRATE: grid checks below
    case SG_OP_LOSS_MEAN:
      if (t.kind != SG_TASK_RANGE_FOR || t.arrays[0] < 0) { err = "LOSS_MEAN is a range-for op over arrays[0]"; return SG_ERR_ARG; }
      if (L.field_tree[t.fields[0]] >= 0 || L.field_dtype[t.fields[0]] != SG_F32) { err = "LOSS_MEAN target must be a 0-D f32 field"; return SG_ERR_ARG; }
      return SG_OK;
    case SG_OP_ADJ_INIT:
      if (t.kind != SG_TASK_RANGE_FOR) { err = "ADJ_INIT is a range-for op"; return SG_ERR_ARG; }
      for (int i = 0; i < 4; i++) if (t.arrays[i] < 0) { err = "ADJ_INIT needs 4 arrays"; return SG_ERR_ARG; }
      return SG_OK;
    case SG_OP_G2P_ADJ:
    case SG_OP_P2G_ADJ: {
      if (t.kind != SG_TASK_RANGE_FOR) { err = "MPM adjoints are range-for ops"; return SG_ERR_ARG; }
      for (int i = 0; i < 8; i++) if (t.arrays[i] < 0) { err = "MPM adjoints need 8 arrays"; return SG_ERR_ARG; }
      const int ng = t.op == SG_OP_G2P_ADJ ? 2 : 1;
      int trees[2];
      for (int k = 0; k < ng; k++) {
        int tree = L.field_tree[t.fields[4 * k]];
        if (tree < 0 || L.trees[tree].nd != 3 || L.trees[tree].driving < 0) { err = "MPM grid fields must live in a 3-D sparse tree"; return SG_ERR_ARG; }
        for (int i = 4 * k; i < 4 * k + 4; i++)
          if (L.field_tree[t.fields[i]] != tree || L.field_dtype[t.fields[i]] != SG_F32) { err = "MPM grid fields must be f32 fields of one tree"; return SG_ERR_ARG; }
        trees[k] = tree;
      }
      if (ng == 2) {
        if (trees[0] == trees[1]) { err = "G2P_ADJ adjoint fields need their own tree"; return SG_ERR_ARG; }
        for (int a = 0; a < 3; a++) {
          int64_t ra = 1, rb = 1;
          for (int s : L.trees[trees[0]].levels) ra *= L.nodes[s].extent[a];
          for (int s : L.trees[trees[1]].levels) rb *= L.nodes[s].extent[a];
          if (ra != rb) { err = "G2P_ADJ trees must have the same resolution"; return SG_ERR_ARG; }
        }
        if (L.trees[trees[0]].levels.size() != L.trees[trees[1]].levels.size()) { err = "G2P_ADJ trees must have the same shape"; return SG_ERR_ARG; }
        for (size_t k = 0; k < L.trees[trees[0]].levels.size(); k++) {
          const auto& A = L.nodes[L.trees[trees[0]].levels[k]];
          const auto& B = L.nodes[L.trees[trees[1]].levels[k]];
          if (A.kind != B.kind || A.extent[0] != B.extent[0] || A.extent[1] != B.extent[1] || A.extent[2] != B.extent[2]) {
            err = "G2P_ADJ trees must have the same shape"; return SG_ERR_ARG;
          }
        }
      }
      return SG_OK;
    }
    case SG_OP_HALO_PACK:
      if (!sf || t.arrays[0] < 0) { err = "HALO_PACK is a struct-for op with a buffer in arrays[0]"; return SG_ERR_ARG; }
      break;
    default: break;
  }
  if (t.op == SG_OP_CLEAR_SCALAR) {
    if (t.kind != SG_TASK_SERIAL || L.field_tree[t.fields[0]] >= 0) { err = "CLEAR_SCALAR is a serial op on a 0-D field"; return SG_ERR_ARG; }
    return SG_OK;
  }
  if (t.op == SG_OP_COPY_SCALAR) {
    if (t.kind != SG_TASK_SERIAL || L.field_tree[t.fields[0]] >= 0 || L.field_tree[t.fields[1]] >= 0 ||
        L.field_dtype[t.fields[0]] != L.field_dtype[t.fields[1]]) {
      err = "COPY_SCALAR is a serial op on two 0-D fields of one dtype"; return SG_ERR_ARG;
    }
    return SG_OK;
  }
  if (t.op == SG_OP_P2G || t.op == SG_OP_G2P || t.op == SG_OP_GRID_OP || t.op == SG_OP_G2P_MIGRATE) {
    if (t.op != SG_OP_GRID_OP && t.kind != SG_TASK_RANGE_FOR) { err = "P2G/G2P are range-for ops"; return SG_ERR_ARG; }
    int tree = L.field_tree[t.fields[0]];
    if (tree < 0 || L.trees[tree].nd != 3 || L.trees[tree].driving < 0) {
      err = "MPM grid fields must live in a 3-D sparse tree"; return SG_ERR_ARG;
    }
    for (int i = 0; i < 4; i++) {
      if (L.field_tree[t.fields[i]] != tree || L.field_dtype[t.fields[i]] != SG_F32) {
        err = "MPM grid fields must be f32 fields of one tree"; return SG_ERR_ARG;
      }
      if (t.op != SG_OP_GRID_OP && t.arrays[i] < 0) { err = "MPM ops need 4 particle arrays"; return SG_ERR_ARG; }
    }
    if (t.op != SG_OP_GRID_OP) return SG_OK;
  }
  if (!sf) { err = "op must be launched as a struct-for"; return SG_ERR_ARG; }
  if (t.snode <= 0 || t.snode >= (int)L.nodes.size() || L.nodes[t.snode].kind == SG_PLACE ||
      L.snode_tree[t.snode] < 0) { err = "struct-for snode must be a level"; return SG_ERR_ARG; }
  int tree = L.snode_tree[t.snode];
  if (L.trees[tree].levels.back() != t.snode) { err = "struct-for snode must be the leaf level of its tree"; return SG_ERR_ARG; }
  int dt = -1;
  for (const OpUse& u : op_uses(t)) {
    if (u.array) continue;
    int f = t.fields[u.slot];
    if (f < 0) continue;
    if (dt < 0) dt = L.field_dtype[f];
    else if (dt != L.field_dtype[f]) { err = "operands of one op must share a dtype"; return SG_ERR_ARG; }
    if (u.access == AC_ID || u.access == AC_NBR) {
      if (L.field_tree[f] != tree) { err = "identity / neighbour operands must live in the iterated tree"; return SG_ERR_ARG; }
    }
    if (u.access == AC_CONST && L.field_tree[f] >= 0) { err = "reduction target must be 0-D"; return SG_ERR_ARG; }
    if (u.access == AC_DIV2) {
      int t2 = L.field_tree[f];
      if (t2 < 0) { err = "DOWNSAMPLE target must be a tree field"; return SG_ERR_ARG; }
      const HTree& A = L.trees[tree];
      const HTree& B = L.trees[t2];
      if (A.nd != B.nd) { err = "DOWNSAMPLE trees differ in ndim"; return SG_ERR_ARG; }
      for (int a = 0; a < A.nd; a++) {
        int64_t ra = 1, rb = 1;
        for (int s : A.levels) ra *= L.nodes[s].extent[a];
        for (int s : B.levels) rb *= L.nodes[s].extent[a];
        if (ra != 2 * rb) { err = "DOWNSAMPLE target must have half the resolution"; return SG_ERR_ARG; }
      }
    }
  }
  if ((t.op == SG_OP_STENCIL || t.op == SG_OP_JACOBI) && (t.fields[0] == t.fields[1])) {
    err = "stencil destination must differ from its source"; return SG_ERR_ARG;
  }
  if (t.op == SG_OP_JACOBI && (t.fields[0] == t.fields[2])) { err = "JACOBI destination must differ from b"; return SG_ERR_ARG; }
  if (t.op == SG_OP_JACOBI && dt == SG_I32) { err = "JACOBI is f32 only"; return SG_ERR_ARG; }
  return SG_OK;
}

int lower_call(const HLayout& L, const UserCall& c, int call, bool faithful, std::vector<PTask>& out,
               std::string& err) {
  switch (c.kind) {
    case 0: {  // activate
      if (!valid_field(L, c.field) || L.field_tree[c.field] < 0) { err = "activate needs a tree field"; return SG_ERR_ARG; }
      PTask t;
      t.type = TT_ACTIVATE; t.field = c.field; t.tree = L.field_tree[c.field]; t.coords = c.coords; t.n = c.n; t.call = call;
      out.push_back(t);
    } break;
    case 1: {  // explicit listgen
      if (c.snode <= 0 || c.snode >= (int)L.nodes.size() || !L.is_sparse(c.snode)) { err = "listgen needs a sparse level"; return SG_ERR_ARG; }
      int tree = L.snode_tree[c.snode];
      std::vector<int> lv;
      for (int s : L.trees[tree].levels) {
        if (L.is_sparse(s)) lv.push_back(s);
        if (s == c.snode) break;
      }
      emit_lists(L, lv, tree, call, faithful, true, out);
    } break;
    case 2: {  // struct-for / range-for / serial
      int rc = validate_task(L, c.t, err);
      if (rc) return rc;
      PTask t;
      t.call = call; t.t = c.t; t.act = c.t.activating;
      if (c.t.kind == SG_TASK_STRUCT_FOR) {
        t.type = TT_STRUCT_FOR; t.snode = c.t.snode; t.tree = L.snode_tree[c.t.snode];
        emit_lists(L, L.listed_levels(t.tree), t.tree, call, faithful, false, out);
      } else if (c.t.kind == SG_TASK_RANGE_FOR) {
        t.type = TT_RANGE_FOR; t.n = c.t.range_n;
      } else {
        t.type = TT_SERIAL;
        // exchanges are collective with the neighbour ranks: never removed
        t.pinned = c.t.op == SG_OP_DIST_SIGNAL || c.t.op == SG_OP_DIST_WAIT;
      }
      out.push_back(t);
    } break;
    case 3: {  // clear
      if (c.mode == SG_CLEAR_VALUES) {
        if (!valid_field(L, c.field)) { err = "bad field"; return SG_ERR_ARG; }
        PTask t;
        t.call = call;
        std::memset(&t.t, 0, sizeof(t.t));
        for (int i = 0; i < 8; i++) { t.t.fields[i] = -1; t.t.arrays[i] = -1; }
        t.t.fields[0] = c.field;
        int tree = L.field_tree[c.field];
        if (tree < 0) {
          t.type = TT_SERIAL; t.t.kind = SG_TASK_SERIAL; t.t.op = SG_OP_CLEAR_SCALAR;
        } else {
          t.type = TT_STRUCT_FOR; t.t.kind = SG_TASK_STRUCT_FOR; t.t.op = SG_OP_FILL;
          t.tree = tree; t.snode = L.trees[tree].levels.back(); t.t.snode = t.snode;
          emit_lists(L, L.listed_levels(tree), tree, call, faithful, false, out);
        }
        out.push_back(t);
      } else if (c.mode == SG_DEACTIVATE) {
        if (c.snode <= 0 || c.snode >= (int)L.nodes.size() || !L.is_sparse(c.snode)) { err = "deactivate needs a sparse level"; return SG_ERR_ARG; }
        int tree = L.snode_tree[c.snode];
        emit_lists(L, L.listed_levels(tree), tree, call, faithful, false, out);
        PTask t;
        t.type = TT_DEACTIVATE; t.snode = c.snode; t.tree = tree; t.call = call;
        out.push_back(t);
      } else {
        err = "bad clear mode";
        return SG_ERR_ARG;
      }
    } break;
    default:
      err = "bad call";
      return SG_ERR_ARG;
  }
  return SG_OK;
}

// ---------------------------------------------------------------------------
// State-flow graph
// ---------------------------------------------------------------------------
static bool has_state(const std::vector<Use>& v, int64_t s) {
  for (const Use& u : v) if (u.state == s) return true;
  return false;
}
static bool complete_out(const PTask& t, int64_t s) {
  for (const Use& u : t.out) if (u.state == s && u.complete) return true;
  return false;
}

Graph build_graph(const std::vector<PTask>& seq) {
  Graph G;
  G.n = (int)seq.size();
  G.succ.assign(G.n, {}); G.pred.assign(G.n, {});
  G.in_ver.assign(G.n, {}); G.next_writer.assign(G.n, {}); G.readers.assign(G.n, {}); G.edges_to.assign(G.n, {});
  std::unordered_map<int64_t, int> latest;
  std::unordered_map<int64_t, std::vector<int>> readers_since;
  std::vector<std::unordered_set<int>> succ_set(G.n);
  auto edge = [&](int a, int b, int64_t s) {
    if (a < 0 || a == b) return;
    G.edges_to[b].push_back({a, s});
    if (succ_set[a].insert(b).second) { G.succ[a].push_back(b); G.pred[b].push_back(a); }
  };
  for (int i = 0; i < G.n; i++) {
    const PTask& t = seq[i];
    std::unordered_set<int64_t> seen;
    for (const Use& u : t.in) {
      if (!seen.insert(u.state).second) continue;
      auto it = latest.find(u.state);
      int p = it == latest.end() ? -1 : it->second;
      G.in_ver[i][u.state] = p;
      edge(p, i, u.state);                                  // RAW
      if (p >= 0) G.readers[p][u.state]++;
      readers_since[u.state].push_back(i);
    }
    seen.clear();
    for (const Use& u : t.out) {
      if (!seen.insert(u.state).second) continue;
      auto it = latest.find(u.state);
      int p = it == latest.end() ? -1 : it->second;
      if (p >= 0) { edge(p, i, u.state); G.next_writer[p][u.state] = i; }   // WAW
      for (int r : readers_since[u.state]) edge(r, i, u.state);              // WAR
      readers_since[u.state].clear();
      latest[u.state] = i;
      G.next_writer[i][u.state] = -1;
      G.readers[i].emplace(u.state, 0);
    }
  }
  return G;
}

// ---------------------------------------------------------------------------
// Passes
// ---------------------------------------------------------------------------
struct Stream {
  std::vector<PTask> seq;
  std::vector<std::unordered_map<int64_t, int>> ver;   // input versions of kept tasks
  std::unordered_map<int64_t, int> latest;
  int cur(int64_t s) const { auto it = latest.find(s); return it == latest.end() ? -1 : it->second; }
  void push(const PTask& t) {
    int i = (int)seq.size();
    std::unordered_map<int64_t, int> v;
    for (const Use& u : t.in) v[u.state] = cur(u.state);
    seq.push_back(t);
    ver.push_back(std::move(v));
    for (const Use& u : t.out) latest[u.state] = i;
  }
};

// Section 6.2: "Two list generation tasks with the same parent
// list and the same mask as the input outputs the same list, and we can
// eliminate one of them."  Versions = producing task ids (reading R12).
static bool pass_listgen_removal(std::vector<PTask>& seq, PlanStats& st) {
  Stream S;
  bool changed = false;
  for (const PTask& t : seq) {
    if (t.type == TT_LISTGEN && t.members.size() == 1 && !t.pinned) {
      int a = S.cur(skey(ST_LIST, t.snode));
      if (a >= 0 && S.seq[a].type == TT_LISTGEN && S.seq[a].snode == t.snode) {
        bool same = true;
        for (const Use& u : t.in) {
          auto it = S.ver[a].find(u.state);
          int av = it == S.ver[a].end() ? -2 : it->second;
          if (av != S.cur(u.state)) { same = false; break; }
        }
        if (same) { st.listgens_removed++; changed = true; continue; }
      }
    }
    S.push(t);
  }
  seq.swap(S.seq);
  return changed;
}

static int operand_access(const sg_task& t, int slot) {
  for (const OpUse& u : op_uses(t))
    if (!u.array && u.slot == slot && (u.role & R_WRITE)) return u.access;
  return AC_NONE;
}

static bool same_task(const sg_task& a, const sg_task& b) {
  if (a.kind != b.kind || a.op != b.op || a.snode != b.snode) return false;
  for (int i = 0; i < 8; i++) if (a.fields[i] != b.fields[i]) return false;
  return true;
}

// Section 6.3: "If two struct-for tasks are identical, the loop
// lists are the same, and the activation statement in the second task depends
// only on the loop indices, then the activation in the second task can be
// removed."  Plus reading R9: nothing between them writes the target's masks.
static bool pass_demotion(const HLayout& L, std::vector<PTask>& seq, PlanStats& st) {
  Stream S;
  bool changed = false;
  for (PTask t : seq) {
    if (t.type == TT_STRUCT_FOR && t.members.size() == 1 && t.act) {
      const HTree& T = L.trees[t.tree];
      int64_t list_state = T.driving >= 0 ? skey(ST_LIST, T.levels[T.driving]) : 0;
      int64_t leafmask = T.leaf_bitmasked ? skey(ST_MASK, T.levels.back()) : 0;
      uint32_t act = t.act;
      for (int i = 0; i < 8; i++) {
        if (!((act >> i) & 1u)) continue;
        int acc = operand_access(t.t, i);
        if (acc != AC_ID && acc != AC_DIV2) continue;      // only loop-index addresses
        int f = t.t.fields[i];
        if (f < 0 || L.field_tree[f] < 0) continue;
        std::vector<int> masks = L.sparse_levels(L.field_tree[f]);
        for (int a = (int)S.seq.size() - 1; a >= 0; a--) {
          const PTask& A = S.seq[a];
          if (A.type != TT_STRUCT_FOR || A.members.size() != 1 || !same_task(A.t, t.t) || !((A.act >> i) & 1u)) continue;
          if (list_state && S.ver[a].count(list_state) && S.ver[a].at(list_state) != S.cur(list_state)) continue;
          if (leafmask && S.ver[a].count(leafmask) && S.ver[a].at(leafmask) != S.cur(leafmask)) continue;
          bool latest_writer = true;
          for (int m : masks) if (S.cur(skey(ST_MASK, m)) != a) { latest_writer = false; break; }
          if (!latest_writer) continue;
          act &= ~(1u << i);
          st.demotions++;
          break;
        }
      }
      if (act != t.act) {
        t.act = act;
        t.member_act[0] = act;
        task_meta(L, t);
        changed = true;
      }
    } else if (t.type == TT_ACTIVATE && t.members.size() == 1) {
      // reading R9 extension: a repeated explicit activation of the same
      // coordinate buffer with no intervening mask writer is a no-op.
      std::vector<int> masks = L.sparse_levels(t.tree);
      bool drop = false;
      for (int a = (int)S.seq.size() - 1; a >= 0 && !drop; a--) {
        const PTask& A = S.seq[a];
        if (A.type != TT_ACTIVATE || A.field != t.field || A.coords_class != t.coords_class) continue;
        bool latest_writer = true;
        for (int m : masks) if (S.cur(skey(ST_MASK, m)) != a) { latest_writer = false; break; }
        drop = latest_writer;
      }
      if (drop) { st.demotions++; changed = true; continue; }
    }
    S.push(t);
  }
  seq.swap(S.seq);
  return changed;
}

static int task_dtype(const HLayout& L, const PTask& t) {
  for (int i = 0; i < 8; i++)
    if (t.t.fields[i] >= 0 && t.t.fields[i] < (int)L.field_dtype.size()) return L.field_dtype[t.t.fields[i]];
  return SG_F32;
}

static void fuse_meta(PTask& A, const PTask& B) {
  std::unordered_set<int64_t> a_complete;
  for (const Use& u : A.out) if (u.complete) a_complete.insert(u.state);
  for (const Use& u : B.in) if (!a_complete.count(u.state)) A.in.push_back(u);
  for (const Use& u : B.out) A.out.push_back(u);
}

// Section 6.4: same group (type + SNode & list for struct-fors,
// range for range-fors); no path of length >= 2 between A and B; across an
// edge A->B every access to the shared state is at the same address, unique
// per iteration (identity).
static bool pass_fusion(const HLayout& L, std::vector<PTask>& seq, PlanStats& st) {
  bool changed = false;
  while (true) {
    Graph G = build_graph(seq);
    const int n = G.n;
    const int W = (n + 63) / 64;
    std::vector<uint64_t> reach((size_t)n * W, 0);
    for (int i = n - 1; i >= 0; i--) {
      uint64_t* r = &reach[(size_t)i * W];
      for (int j : G.succ[i]) {
        r[j >> 6] |= 1ull << (j & 63);
        const uint64_t* rj = &reach[(size_t)j * W];
        for (int w = 0; w < W; w++) r[w] |= rj[w];
      }
    }
    auto R = [&](int a, int b) { return (reach[(size_t)a * W + (b >> 6)] >> (b & 63)) & 1ull; };
    int fa = -1, fb = -1;
    for (int a = 0; a < n && fa < 0; a++) {
      const PTask& A = seq[a];
      if (A.type != TT_STRUCT_FOR && A.type != TT_RANGE_FOR && A.type != TT_SERIAL) continue;
      for (int b = a + 1; b < n; b++) {
        const PTask& B = seq[b];
        if (B.type != A.type) continue;
        if (A.members.size() + B.members.size() > SG_MAXOPS) continue;
        if (task_dtype(L, A) != task_dtype(L, B)) continue;
        if (A.type == TT_STRUCT_FOR) {
          if (A.snode != B.snode) continue;
          const HTree& T = L.trees[A.tree];
          bool ok = true;
          if (T.driving >= 0) {
            int64_t ls = skey(ST_LIST, T.levels[T.driving]);
            ok = G.in_ver[a].count(ls) && G.in_ver[b].count(ls) && G.in_ver[a].at(ls) == G.in_ver[b].at(ls);
          }
          if (ok && T.leaf_bitmasked) {
            int64_t lm = skey(ST_MASK, T.levels.back());
            ok = G.in_ver[a].count(lm) && G.in_ver[b].count(lm) && G.in_ver[a].at(lm) == G.in_ver[b].at(lm);
          }
          if (!ok) continue;
        } else if (A.type == TT_RANGE_FOR) {
          // same range: equal host extent, or the same device-counted array
          if (A.n != B.n || (A.n < 0 && A.t.arrays[0] != B.t.arrays[0])) continue;
          // ops with their own kernels (scan / append / unpack, the binned MPM transfers) run alone
          auto solo = [](int op) {
            return op == SG_OP_G2P_MIGRATE || op == SG_OP_MIGRATE_APPEND || op == SG_OP_HALO_UNPACK ||
                   op == SG_OP_MIGRATE_COMPACT ||
                   op == SG_OP_LOSS_MEAN || op == SG_OP_G2P_ADJ || op == SG_OP_P2G_ADJ || op == SG_OP_P2G ||
                   op == SG_OP_G2P || op == SG_OP_PERMUTE;
          };
          if (solo(A.t.op) || solo(B.t.op)) continue;
        } else if (A.type == TT_SERIAL) {
          auto xchg = [](int op) { return op == SG_OP_DIST_SIGNAL || op == SG_OP_DIST_WAIT; };
          if (xchg(A.t.op) || xchg(B.t.op)) continue;
        }
        // no path of length >= 2
        bool long_path = false;
        for (int c = a + 1; c < b && !long_path; c++) long_path = R(a, c) && R(c, b);
        if (long_path) continue;
        // direct edge: every shared state identity-accessed on both sides
        bool ok = true;
        for (const auto& e : G.edges_to[b]) {
          if (e.first != a) continue;
          int k = skind(e.second);
          if (k != ST_VALUE && k != ST_ARRAY) { ok = false; break; }
          for (const Use& u : A.in) if (u.state == e.second && u.access != AC_ID) ok = false;
          for (const Use& u : A.out) if (u.state == e.second && u.access != AC_ID) ok = false;
          for (const Use& u : B.in) if (u.state == e.second && u.access != AC_ID) ok = false;
          for (const Use& u : B.out) if (u.state == e.second && u.access != AC_ID) ok = false;
          if (!ok) break;
        }
        if (!ok) continue;
        fa = a; fb = b;
        break;
      }
    }
    if (fa < 0) break;
    // contract: [0,a) + between-not-reachable-from-a + AB + between-reachable + (b,n)
    std::vector<PTask> out;
    out.reserve(n - 1);
    for (int i = 0; i < fa; i++) out.push_back(seq[i]);
    for (int c = fa + 1; c < fb; c++) if (!R(fa, c)) out.push_back(seq[c]);
    PTask F = seq[fa];
    const PTask& B = seq[fb];
    F.members.insert(F.members.end(), B.members.begin(), B.members.end());
    F.member_act.insert(F.member_act.end(), B.member_act.begin(), B.member_act.end());
    fuse_meta(F, B);
    out.push_back(F);
    for (int c = fa + 1; c < fb; c++) if (R(fa, c)) out.push_back(seq[c]);
    for (int i = fb + 1; i < n; i++) out.push_back(seq[i]);
    seq.swap(out);
    st.fused++;
    changed = true;
  }
  return changed;
}

// Section 6.5: "for cases like this that a field is completely
// overwritten, our optimizer can eliminate the previous dead stores."  A task
// is removed when every version it writes has no reader and is either
// completely overwritten next or unobserved at the sync point (reading R11).
static bool pass_dse(std::vector<PTask>& seq, const std::vector<char>& observed, PlanStats& st) {
  bool changed = false;
  while (true) {
    Graph G = build_graph(seq);
    std::vector<char> dead(G.n, 0);
    int ndead = 0;
    for (int i = 0; i < G.n; i++) {
      const PTask& t = seq[i];
      if (t.pinned || t.out.empty()) continue;
      bool all_dead = true;
      for (const auto& kv : G.next_writer[i]) {
        int64_t s = kv.first;
        auto r = G.readers[i].find(s);
        if (r != G.readers[i].end() && r->second > 0) { all_dead = false; break; }
        int nw = kv.second;
        if (nw >= 0) {
          if (!complete_out(seq[nw], s)) { all_dead = false; break; }
        } else {
          int k = skind(s);
          bool obs = k == ST_MASK || k == ST_ALLOC || k == ST_ARRAY ||
                     (k == ST_VALUE && (sid(s) >= (int)observed.size() || observed[sid(s)]));
          if (obs) { all_dead = false; break; }
        }
      }
      if (all_dead) { dead[i] = 1; ndead++; }
    }
    if (!ndead) break;
    std::vector<PTask> out;
    for (int i = 0; i < G.n; i++) if (!dead[i]) out.push_back(seq[i]);
    st.dead += ndead;
    seq.swap(out);
    changed = true;
  }
  return changed;
}

// Beyond the paper (SG_PASS_CHAIN): adjacent struct-for groups over the same
// list version become phases of one cooperative launch (grid barrier between
// phases).  Tasks in between that do not depend on the chain so far are
// hoisted before it; a reduction may only end a chain.
static void pass_chain(const HLayout& L, std::vector<PTask>& seq, const std::vector<PTask>& eager, PlanStats& st) {
  Graph G = build_graph(seq);
  const int n = G.n;
  std::vector<char> used(n, 0);
  std::vector<PTask> out;
  auto list_ver = [&](int i, int64_t& lv, int64_t& mv) {
    const HTree& T = L.trees[seq[i].tree];
    lv = -7; mv = -7;
    if (T.driving >= 0) {
      int64_t s = skey(ST_LIST, T.levels[T.driving]);
      lv = G.in_ver[i].count(s) ? G.in_ver[i].at(s) : -3;
    }
    if (T.leaf_bitmasked) {
      int64_t s = skey(ST_MASK, T.levels.back());
      mv = G.in_ver[i].count(s) ? G.in_ver[i].at(s) : -3;
    }
  };
  auto group_reduces = [&](const PTask& t) {
    for (int m : t.members)
      if (eager[m].t.op == SG_OP_REDUCE_SUM || eager[m].t.op == SG_OP_RESID_NORM2 || eager[m].t.op == SG_OP_DOT)
        return true;
    return false;
  };
  for (int i = 0; i < n; i++) {
    if (used[i]) continue;
    const PTask& A = seq[i];
    if (A.type != TT_STRUCT_FOR) { out.push_back(A); used[i] = 1; continue; }
    int64_t alv, amv;
    list_ver(i, alv, amv);
    std::vector<int> chain{i}, hoist;
    std::vector<char> in_chain(n, 0);
    in_chain[i] = 1;
    bool reduce_seen = group_reduces(A);
    for (int j = i + 1; j < n && !reduce_seen; j++) {
      if (used[j]) continue;
      const PTask& X = seq[j];
      if (X.type == TT_STRUCT_FOR && X.tree == A.tree && X.snode == A.snode &&
          task_dtype(L, X) == task_dtype(L, A)) {
        int64_t xlv, xmv;
        list_ver(j, xlv, xmv);
        if (xlv == alv && xmv == amv) {
          chain.push_back(j);
          in_chain[j] = 1;
          reduce_seen = group_reduces(X);
          continue;
        }
      }
      bool dep = false;
      for (int p : G.pred[j]) if (in_chain[p]) { dep = true; break; }
      if (dep) break;
      hoist.push_back(j);
    }
    if (chain.size() < 2) { out.push_back(A); used[i] = 1; continue; }
    for (int h : hoist) { out.push_back(seq[h]); used[h] = 1; }
    PTask F = seq[chain[0]];
    F.phase_end = {(int)F.members.size()};
    for (size_t c = 1; c < chain.size(); c++) {
      const PTask& X = seq[chain[c]];
      F.members.insert(F.members.end(), X.members.begin(), X.members.end());
      F.member_act.insert(F.member_act.end(), X.member_act.begin(), X.member_act.end());
      F.phase_end.push_back((int)F.members.size());
    }
    for (int c : chain) used[c] = 1;
    st.chained += (int64_t)chain.size() - 1;
    out.push_back(F);
  }
  seq.swap(out);
}

Plan optimize(const HLayout& L, const std::vector<PTask>& eager, uint32_t passes,
              const std::vector<char>& observed) {
  std::vector<PTask> seq = eager;
  for (size_t i = 0; i < seq.size(); i++) {
    seq[i].members = {seq[i].pos};
    seq[i].member_act = {seq[i].act};
  }
  Plan P;
  if (passes) {
    for (int round = 0; round < 10; round++) {
      bool ch = false;
      if (passes & SG_PASS_LISTGEN_REMOVAL) ch |= pass_listgen_removal(seq, P.stats);
      if (passes & SG_PASS_ACT_DEMOTION) {
        ch |= pass_demotion(L, seq, P.stats);
        if (passes & SG_PASS_LISTGEN_REMOVAL) ch |= pass_listgen_removal(seq, P.stats);
      }
      // DSE also runs before fusion so that a dead task is not fused into a
      // live one, which would keep it alive (reading R26).
      if (passes & SG_PASS_DSE) ch |= pass_dse(seq, observed, P.stats);
      if (passes & SG_PASS_FUSION) ch |= pass_fusion(L, seq, P.stats);
      if (passes & SG_PASS_DSE) ch |= pass_dse(seq, observed, P.stats);
      if (!ch) break;
    }
    if (passes & SG_PASS_CHAIN) pass_chain(L, seq, eager, P.stats);
  }
  for (const PTask& t : seq) {
    P.groups.push_back(t.members);
    P.acts.push_back(t.member_act);
    P.phase_ends.push_back(t.phase_end.empty() ? std::vector<int>{(int)t.members.size()} : t.phase_end);
  }
  return P;
}

uint64_t stream_hash(const std::vector<PTask>& eager, uint32_t passes, const std::vector<char>& observed) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](int64_t v) {
    for (int k = 0; k < 8; k++) { h ^= (uint64_t)((v >> (8 * k)) & 0xff); h *= 1099511628211ull; }
  };
  mix(passes);
  mix((int64_t)eager.size());
  for (const PTask& t : eager) {
    mix(t.type); mix(t.snode); mix(t.tree); mix(t.field); mix(t.coords_class); mix(t.act); mix(t.pinned);
    mix(t.n);
    mix(t.t.kind); mix(t.t.op); mix(t.t.snode); mix(t.t.range_n);
    for (int i = 0; i < 8; i++) { mix(t.t.fields[i]); mix(t.t.arrays[i]); }
  }
  for (char c : observed) mix(c);
  return h;
}

}  // namespace sg
