// sg_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU implementation of the sparse-grid
// semantics of AsyncTaichi (arXiv 2012.08141).  It executes the UNOPTIMIZED
// lowered task stream one task at a time, in program order (PAPER.md:84-85
// "eagerly launches"; PAPER.md:97/250 the optimizer must not change results).
// It is the parity reference for the CUDA path in paper_2012_08141_b200/ and
// shares no code, header, table or helper with it.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it.  The product path never does.
//
// Data model (restated from the paper):
//   * SNode tree (Fig. 2): root -> chains of
//     dense / bitmasked / pointer levels -> place leaves.
//   * Mask state: per sparse level, the std::set of active
//     level-global cell coordinates.  A leaf cell is active iff every sparse
//     ancestor covering it is active; dense levels add no mask (PAPER.md:162,
//     Fig. 3 caption "Because of the constraints of the dense node, y[0] and
//     y[2] are also activated").
//   * Value state: per field a map coord -> value; an inactive
//     voxel reads 0 ("the inactive voxel has value 0").
//   * List state ("Lists of each layer are defined to be a
//     collection of active node indices"): per level the last
//     generated list; struct-for iterates that list.
//   * Allocator state: counters of pointer children allocated
//     and freed.
// Float arithmetic (reading R14/R15): storage is f32 (values are
// rounded to float at the end of each task), arithmetic is f64, and every
// element carries a shadow magnitude M (sum of |terms| that produced it) used
// for the 1e-5 tolerance.  Index-deciding f32 expressions are evaluated with the
// same f32 operation order as the device; this file is compiled with
// -ffp-contract=off.
//
// Parity status per function: see DESIGN.md "Oracle pins".  All functions
// below are pinned by tests/test_oracle_*.py except where marked
// "parity unpinned".

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <map>
#include <set>
#include <string>
#include <vector>
#include <array>
#include <algorithm>

namespace {

enum { K_ROOT = 0, K_DENSE = 1, K_BITMASKED = 2, K_POINTER = 3, K_PLACE = 4 };
enum { T_F32 = 0, T_I32 = 1 };
enum {
  OK = 0, E_ARG = -1, E_LAYOUT = -2, E_RANGE = -3, E_TRAP = -6, E_OVERFLOW = -7
};
// Op ids of the oracle's own vocabulary (mapped from names in oracle/__init__.py).
enum {
  OP_FILL = 1, OP_ADD_CONST = 2, OP_INC = 3, OP_AXPY = 4, OP_STENCIL = 5,
  OP_JACOBI = 6, OP_REDUCE_SUM = 7, OP_DOWNSAMPLE = 8, OP_JITTER = 9,
  OP_CLEAR_SCALAR = 10,
  OP_P2G = 20, OP_GRID_OP = 21, OP_G2P = 22,
  OP_LOSS_MEAN = 27, OP_ADJ_INIT = 28, OP_G2P_ADJ = 29, OP_P2G_ADJ = 30,
  OP_SMOOTH_RB = 31, OP_RESTRICT = 32, OP_PROLONG = 33, OP_RESID_NORM2 = 34,
  OP_DOT = 35, OP_AXPY_RATIO = 36, OP_XPAY_RATIO = 37, OP_COPY_SCALAR = 38, OP_PERMUTE = 42
};

typedef std::array<int64_t, 3> Coord;

struct Node {
  int kind, parent, nd, e[3], dtype;
  std::vector<int> children;
  int tree = -1;
  int64_t res[3] = {1, 1, 1};    // level-global resolution
  int64_t below[3] = {1, 1, 1};  // leaf cells per cell of this level (per axis)
};

struct Tree {
  std::vector<int> levels;   // snode ids root->leaf (empty for a 0-D tree)
  std::vector<int> fields;   // field ids placed at the leaf
  int nd = 0;
};

struct Field {
  int snode, tree, dtype;
  std::map<Coord, double> val;   // only active cells have entries
  std::map<Coord, double> mag;   // shadow magnitude M
};

struct Array {
  int64_t n; int ncomp;
  std::vector<double> val, mag;  // [comp][n]
};

struct Grid {
  std::vector<Node> nodes;
  std::vector<Tree> trees;
  std::vector<Field> fields;
  std::vector<Array> arrays;
  std::map<int, std::set<Coord>> active;     // sparse level -> active cells
  std::map<int, std::vector<Coord>> lists;   // level -> last generated list
  std::map<int, int64_t> allocated, freed;   // pointer level -> counters
  int64_t tasks = 0, listgens = 0;
  bool exact = false;   // f64 storage (no f32 rounding): finite-difference pins of the adjoints
  std::string err;
  // per-task bookkeeping: cells whose value must be rounded to storage type
  std::set<std::pair<int, Coord>> touched;
};

inline bool is_pow2(int v) { return v >= 1 && (v & (v - 1)) == 0; }
inline bool sparse(int k) { return k == K_BITMASKED || k == K_POINTER; }

int fail(Grid* g, int code, const std::string& m) { g->err = m; return code; }

// ---------------------------------------------------------------------------
// Layout (SPEC.md:46-51 validation rules; Fig. 2)
// ---------------------------------------------------------------------------
int build_layout(Grid* g, const int32_t* d, int n) {
  if (n < 1 || d[0] != K_ROOT || d[1] != -1) return fail(g, E_LAYOUT, "row 0 must be the root");
  for (int i = 0; i < n; i++) {
    Node nd;
    nd.kind = d[i * 7 + 0]; nd.parent = d[i * 7 + 1]; nd.nd = d[i * 7 + 2];
    for (int a = 0; a < 3; a++) nd.e[a] = d[i * 7 + 3 + a];
    nd.dtype = d[i * 7 + 6];
    if (i > 0) {
      if (nd.kind == K_ROOT) return fail(g, E_LAYOUT, "second root");
      if (nd.kind < 0 || nd.kind > K_PLACE) return fail(g, E_LAYOUT, "bad kind");
      if (nd.parent < 0 || nd.parent >= i) return fail(g, E_LAYOUT, "parent must precede child");
      if (g->nodes[nd.parent].kind == K_PLACE) return fail(g, E_LAYOUT, "place with children");
      if (nd.nd < 0 || nd.nd > 3) return fail(g, E_LAYOUT, "ndim out of range");
      for (int a = 0; a < 3; a++) {
        if (!is_pow2(nd.e[a])) return fail(g, E_LAYOUT, "extent not a power of two");
        if (a >= nd.nd && nd.e[a] != 1) return fail(g, E_LAYOUT, "extent on unused axis");
      }
      if (nd.kind == K_PLACE && (nd.dtype != T_F32 && nd.dtype != T_I32))
        return fail(g, E_LAYOUT, "bad dtype");
      g->nodes[nd.parent].children.push_back(i);
    }
    g->nodes.push_back(nd);
  }
  // Trees: each structural child of the root starts a chain; a place under the
  // root is a 0-D tree.
  for (int c : g->nodes[0].children) {
    Tree t;
    if (g->nodes[c].kind == K_PLACE) {
      if (g->nodes[c].nd != 0) return fail(g, E_LAYOUT, "place under root must be 0-D");
      t.nd = 0;
      t.fields.push_back(c);
    } else {
      int cur = c;
      t.nd = g->nodes[c].nd;
      int64_t res[3] = {1, 1, 1};
      while (true) {
        Node& nn = g->nodes[cur];
        if (nn.nd != t.nd) return fail(g, E_LAYOUT, "axis mismatch along chain");
        for (int a = 0; a < 3; a++) { res[a] *= nn.e[a]; nn.res[a] = res[a]; }
        t.levels.push_back(cur);
        int structural = -1, places = 0;
        for (int ch : nn.children) {
          if (g->nodes[ch].kind == K_PLACE) places++;
          else if (structural >= 0) return fail(g, E_LAYOUT, "level with two structural children");
          else structural = ch;
        }
        if (structural >= 0 && places) return fail(g, E_LAYOUT, "places only at the leaf level");
        if (structural < 0) {
          if (!places) return fail(g, E_LAYOUT, "leaf level without place");
          if (nn.kind == K_POINTER) return fail(g, E_LAYOUT, "pointer level cannot be the leaf");
          for (int ch : nn.children) {
            if (g->nodes[ch].nd != t.nd) return fail(g, E_LAYOUT, "place ndim mismatch");
            t.fields.push_back(ch);
          }
          break;
        }
        cur = structural;
      }
      // below[] of each level: product of extents of deeper levels
      for (size_t k = 0; k < t.levels.size(); k++) {
        Node& nn = g->nodes[t.levels[k]];
        for (int a = 0; a < 3; a++) {
          int64_t b = 1;
          for (size_t m = k + 1; m < t.levels.size(); m++) b *= g->nodes[t.levels[m]].e[a];
          nn.below[a] = b;
        }
      }
    }
    int tid = (int)g->trees.size();
    for (int l : t.levels) g->nodes[l].tree = tid;
    g->trees.push_back(t);
  }
  // fields in order of place rows
  for (int i = 0; i < n; i++) {
    if (g->nodes[i].kind != K_PLACE) continue;
    Field f;
    f.snode = i; f.dtype = g->nodes[i].dtype; f.tree = -1;
    for (size_t t = 0; t < g->trees.size(); t++)
      for (int pl : g->trees[t].fields) if (pl == i) f.tree = (int)t;
    if (f.tree < 0) return fail(g, E_LAYOUT, "place not reachable");
    g->nodes[i].tree = f.tree;
    g->fields.push_back(f);
  }
  return OK;
}

Tree& tree_of_field(Grid* g, int f) { return g->trees[g->fields[f].tree]; }

const int64_t* leaf_res(Grid* g, const Tree& t) {
  static const int64_t one[3] = {1, 1, 1};
  return t.levels.empty() ? one : g->nodes[t.levels.back()].res;
}

bool in_range(Grid* g, const Tree& t, const Coord& c) {
  const int64_t* r = leaf_res(g, t);
  for (int a = 0; a < 3; a++) {
    if (a < t.nd) { if (c[a] < 0 || c[a] >= r[a]) return false; }
    else if (c[a] != 0) return false;
  }
  return true;
}

Coord level_coord(const Node& n, const Coord& c) {
  return Coord{c[0] / n.below[0], c[1] / n.below[1], c[2] / n.below[2]};
}

// is_active: AND over the sparse ancestors
bool is_active(Grid* g, const Tree& t, const Coord& c) {
  for (int l : t.levels) {
    const Node& n = g->nodes[l];
    if (!sparse(n.kind)) continue;
    auto it = g->active.find(l);
    if (it == g->active.end() || !it->second.count(level_coord(n, c))) return false;
  }
  return true;
}

// activate: top-down insertion of every sparse ancestor
void activate_cell(Grid* g, const Tree& t, const Coord& c) {
  for (int l : t.levels) {
    const Node& n = g->nodes[l];
    if (!sparse(n.kind)) continue;
    bool fresh = g->active[l].insert(level_coord(n, c)).second;
    if (fresh && n.kind == K_POINTER) g->allocated[l]++;
  }
}

// read never activates; inactive or out-of-bound reads give 0 (
// reading R8 for out-of-bound stencil neighbours)
double read(Grid* g, int f, const Coord& c) {
  Tree& t = tree_of_field(g, f);
  if (!in_range(g, t, c) || !is_active(g, t, c)) return 0.0;
  auto& m = g->fields[f].val;
  auto it = m.find(c);
  return it == m.end() ? 0.0 : it->second;
}

double read_mag(Grid* g, int f, const Coord& c) {
  Tree& t = tree_of_field(g, f);
  if (!in_range(g, t, c) || !is_active(g, t, c)) return 0.0;
  auto& m = g->fields[f].mag;
  auto it = m.find(c);
  if (it != m.end()) return it->second;
  return std::fabs(read(g, f, c));
}

// write / atomic_add (SPEC.md:74-78 demotion trap)
int prepare_write(Grid* g, int f, const Coord& c, bool activating) {
  Tree& t = tree_of_field(g, f);
  if (!in_range(g, t, c)) return fail(g, E_RANGE, "write out of range");
  if (activating) activate_cell(g, t, c);
  else if (!is_active(g, t, c)) return fail(g, E_TRAP, "non-activating write to an inactive cell");
  g->touched.insert({f, c});
  return OK;
}

int write(Grid* g, int f, const Coord& c, double v, bool activating, double m) {
  int rc = prepare_write(g, f, c, activating);
  if (rc) return rc;
  g->fields[f].val[c] = v;
  g->fields[f].mag[c] = m;
  return OK;
}

int atomic_add(Grid* g, int f, const Coord& c, double v, bool activating) {
  double old = read(g, f, c), om = read_mag(g, f, c);
  int rc = prepare_write(g, f, c, activating);
  if (rc) return rc;
  g->fields[f].val[c] = old + v;
  g->fields[f].mag[c] = om + std::fabs(v);
  return OK;
}

// Scatter-add with an explicit shadow magnitude for the contribution.
int atomic_add_m(Grid* g, int f, const Coord& c, double v, double vm, bool activating) {
  double old = read(g, f, c), om = read_mag(g, f, c);
  int rc = prepare_write(g, f, c, activating);
  if (rc) return rc;
  g->fields[f].val[c] = old + v;
  g->fields[f].mag[c] = om + vm;
  return OK;
}

// End of task: values are stored as f32 / i32 (reading R14).
int end_task(Grid* g) {
  for (auto& tc : g->touched) {
    Field& fl = g->fields[tc.first];
    auto it = fl.val.find(tc.second);
    if (it == fl.val.end()) continue;
    double v = it->second;
    if (fl.dtype == T_F32) {
      if (!g->exact) it->second = (double)(float)v;
    } else {
      if (v != std::floor(v) || v > 2147483647.0 || v < -2147483648.0) {
        g->touched.clear();
        return fail(g, E_OVERFLOW, "i32 overflow or non-integral value");
      }
    }
  }
  g->touched.clear();
  g->tasks++;
  return OK;
}

// Nearest sparse ancestor level of level index k in the chain (-1 = root list).
int parent_sparse(Grid* g, const Tree& t, size_t k) {
  for (int m = (int)k - 1; m >= 0; m--)
    if (sparse(g->nodes[t.levels[m]].kind)) return (int)m;
  return -1;
}

// Enumerate the cells of a box [lo, lo+ext) in ascending lexicographic order.
template <class F>
void for_box(const Coord& lo, const int64_t ext[3], F fn) {
  for (int64_t i = 0; i < ext[0]; i++)
    for (int64_t j = 0; j < ext[1]; j++)
      for (int64_t k = 0; k < ext[2]; k++) fn(Coord{lo[0] + i, lo[1] + j, lo[2] + k});
}

int chain_index(const Tree& t, int snode) {
  for (size_t k = 0; k < t.levels.size(); k++) if (t.levels[k] == snode) return (int)k;
  return -1;
}

// listgen(S): for every entry
// p of the parent's list, every S-cell under p that is active is appended;
// the result is sorted.  The root's list is the constant {root}.
int listgen(Grid* g, int snode) {
  if (snode <= 0 || snode >= (int)g->nodes.size()) return fail(g, E_ARG, "bad snode");
  const Node& n = g->nodes[snode];
  if (!sparse(n.kind)) return fail(g, E_ARG, "listgen on a non-sparse level");
  const Tree& t = g->trees[n.tree];
  int k = chain_index(t, snode);
  int pk = parent_sparse(g, t, k);
  std::vector<Coord> parents;
  int64_t ratio[3];
  if (pk < 0) {
    parents.push_back(Coord{0, 0, 0});
    for (int a = 0; a < 3; a++) ratio[a] = n.res[a];
  } else {
    parents = g->lists[t.levels[pk]];
    for (int a = 0; a < 3; a++) ratio[a] = n.res[a] / g->nodes[t.levels[pk]].res[a];
  }
  std::vector<Coord> out;
  const std::set<Coord>& act = g->active[snode];
  for (const Coord& p : parents) {
    Coord lo{p[0] * ratio[0], p[1] * ratio[1], p[2] * ratio[2]};
    for_box(lo, ratio, [&](const Coord& q) { if (act.count(q)) out.push_back(q); });
  }
  std::sort(out.begin(), out.end());
  g->lists[snode] = out;
  g->listgens++;
  g->tasks++;
  return OK;
}

// Driving level of a struct-for over a tree: the deepest sparse level, except
// a bitmasked leaf whose bits are tested per cell (reading R5).
int driving_level(Grid* g, const Tree& t) {
  for (int m = (int)t.levels.size() - 1; m >= 0; m--) {
    const Node& n = g->nodes[t.levels[m]];
    if (!sparse(n.kind)) continue;
    if (m == (int)t.levels.size() - 1 && n.kind == K_BITMASKED) continue;
    return m;
  }
  return -1;
}

// Visit the cells a struct-for over tree t iterates:
// for every entry of the driving list, every leaf cell below it, testing the
// leaf bit if the leaf is bitmasked.  The list is the one current at task
// start, so cells activated by the task itself are not visited.
template <class F>
void for_struct(Grid* g, const Tree& t, F fn) {
  if (t.levels.empty()) { fn(Coord{0, 0, 0}); return; }
  int leaf = t.levels.back();
  const Node& ln = g->nodes[leaf];
  int dk = driving_level(g, t);
  std::vector<Coord> cells;
  const std::set<Coord>* leafmask = nullptr;
  if (ln.kind == K_BITMASKED) leafmask = &g->active[leaf];
  auto visit = [&](const Coord& c) {
    if (leafmask && !leafmask->count(c)) return;
    cells.push_back(c);
  };
  if (dk < 0) {
    for_box(Coord{0, 0, 0}, ln.res, visit);
  } else {
    const Node& dn = g->nodes[t.levels[dk]];
    std::vector<Coord> entries = g->lists[t.levels[dk]];
    for (const Coord& p : entries) {
      Coord lo{p[0] * dn.below[0], p[1] * dn.below[1], p[2] * dn.below[2]};
      for_box(lo, dn.below, visit);
    }
  }
  for (const Coord& c : cells) fn(c);
}

Coord shift(const Coord& c, int axis, int64_t d) { Coord r = c; r[axis] += d; return r; }

bool act_bit(uint32_t activating, int slot) { return (activating >> slot) & 1u; }

int field_ok(Grid* g, int f) { return f >= 0 && f < (int)g->fields.size(); }

// ---------------------------------------------------------------------------
// Struct-for bodies (the op vocabulary).  Every body is
// race-free by construction, so sequential order equals any parallel order up
// to float reassociation.
// ---------------------------------------------------------------------------
void grid_update(double p[3], double m, const int node[3], double dt, double grav, double bound, double ng, int D,
                 double u[3], double mask[3]);

int struct_for(Grid* g, int op, int leaf_snode, const int32_t* f, int nf, const float* p, int np,
               uint32_t activating) {
  if (leaf_snode <= 0 || leaf_snode >= (int)g->nodes.size()) return fail(g, E_ARG, "bad snode");
  const Node& ln = g->nodes[leaf_snode];
  if (ln.kind == K_PLACE || ln.tree < 0) return fail(g, E_ARG, "struct-for snode must be a level");
  const Tree& t = g->trees[ln.tree];
  if (t.levels.back() != leaf_snode) return fail(g, E_ARG, "struct-for snode must be the leaf level");
  for (int i = 0; i < nf; i++) if (f[i] >= 0 && !field_ok(g, f[i])) return fail(g, E_ARG, "bad field");
  auto P = [&](int i) { return i < np ? (double)p[i] : 0.0; };
  int D = t.nd;
  int rc = OK;
  auto need = [&](int cnt) { return nf >= cnt; };
  switch (op) {
    case OP_FILL:
      if (!need(1)) return fail(g, E_ARG, "FILL needs 1 field");
      for_struct(g, t, [&](const Coord& c) {
        if (!rc) rc = write(g, f[0], c, P(0), act_bit(activating, 0), std::fabs(P(0)));
      });
      break;
    case OP_ADD_CONST:
      if (!need(2)) return fail(g, E_ARG, "ADD_CONST needs 2 fields");
      for_struct(g, t, [&](const Coord& c) {
        double x = read(g, f[1], c);
        if (!rc) rc = write(g, f[0], c, x + P(0), act_bit(activating, 0), read_mag(g, f[1], c) + std::fabs(P(0)));
      });
      break;
    case OP_INC:
      if (!need(1)) return fail(g, E_ARG, "INC needs 1 field");
      for_struct(g, t, [&](const Coord& c) {
        if (!rc) rc = atomic_add(g, f[0], c, P(0), act_bit(activating, 0));
      });
      break;
    case OP_AXPY:
      if (!need(3)) return fail(g, E_ARG, "AXPY needs 3 fields");
      for_struct(g, t, [&](const Coord& c) {
        double x = read(g, f[1], c), y = read(g, f[2], c);
        double m = std::fabs(P(0)) * read_mag(g, f[1], c) + read_mag(g, f[2], c);
        if (!rc) rc = write(g, f[0], c, P(0) * x + y, act_bit(activating, 0), m);
      });
      break;
    case OP_STENCIL:
      // y = sum_{a<D} (x[c+e_a] + x[c-e_a]) - 2D x[c]   (5-/7-point Laplacian)
      if (!need(2)) return fail(g, E_ARG, "STENCIL needs 2 fields");
      for_struct(g, t, [&](const Coord& c) {
        double s = 0, m = 0;
        for (int a = 0; a < D; a++) {
          double u = read(g, f[1], shift(c, a, +1)), d = read(g, f[1], shift(c, a, -1));
          s += u + d;
          m += read_mag(g, f[1], shift(c, a, +1)) + read_mag(g, f[1], shift(c, a, -1));
        }
        s -= 2.0 * D * read(g, f[1], c);
        m += 2.0 * D * read_mag(g, f[1], c);
        if (!rc) rc = write(g, f[0], c, s, act_bit(activating, 0), m);
      });
      break;
    case OP_JACOBI:
      // x1 = (b + sum of neighbours of x0) / (2D): Jacobi for -Lap x = b, h = 1
      if (!need(3)) return fail(g, E_ARG, "JACOBI needs 3 fields");
      for_struct(g, t, [&](const Coord& c) {
        double s = read(g, f[2], c), m = read_mag(g, f[2], c);
        for (int a = 0; a < D; a++) {
          s += read(g, f[1], shift(c, a, +1)) + read(g, f[1], shift(c, a, -1));
          m += read_mag(g, f[1], shift(c, a, +1)) + read_mag(g, f[1], shift(c, a, -1));
        }
        if (!rc) rc = write(g, f[0], c, s / (2.0 * D), act_bit(activating, 0), m / (2.0 * D));
      });
      break;
    case OP_REDUCE_SUM:
      if (!need(2)) return fail(g, E_ARG, "REDUCE_SUM needs 2 fields");
      if (g->trees[g->fields[f[0]].tree].nd != 0) return fail(g, E_ARG, "REDUCE_SUM target must be 0-D");
      for_struct(g, t, [&](const Coord& c) {
        if (!rc) rc = atomic_add(g, f[0], Coord{0, 0, 0}, read(g, f[1], c), act_bit(activating, 0));
      });
      break;
    case OP_DOWNSAMPLE:
      // y[c // 2] += p0 * x[c] + p1   (PAPER.md:350 restriction; Fig. 3 with p0=0,p1=1)
      if (!need(1)) return fail(g, E_ARG, "DOWNSAMPLE needs a target");
      for_struct(g, t, [&](const Coord& c) {
        Coord h{c[0] / 2, c[1] / 2, c[2] / 2};
        double x = (nf > 1 && f[1] >= 0) ? read(g, f[1], c) : 0.0;
        if (!rc) rc = atomic_add(g, f[0], h, P(0) * x + P(1), act_bit(activating, 0));
      });
      break;
    // --- multigrid (PAPER.md:348-361 restriction, PAPER.md:438-441 MGPCG
    // after hu2019taichi: red-black smoothing, residual restriction, prolongation).
    // A = -Laplacian with h = 1 on the level's grid; inactive / out-of-bound reads 0.
    case OP_SMOOTH_RB:
      // red-black Gauss-Seidel half sweep: cells with (sum c) % 2 == p0 get
      // z = (r + sum_nbr z) / (2D); the other colour is only read
      if (!need(2)) return fail(g, E_ARG, "SMOOTH_RB needs 2 fields");
      for_struct(g, t, [&](const Coord& c) {
        const long par = ((long)c[0] + c[1] + c[2]) & 1;
        if (par != (long)P(0)) return;
        double s = read(g, f[1], c), m = read_mag(g, f[1], c);
        for (int a = 0; a < D; a++) {
          s += read(g, f[0], shift(c, a, +1)) + read(g, f[0], shift(c, a, -1));
          m += read_mag(g, f[0], shift(c, a, +1)) + read_mag(g, f[0], shift(c, a, -1));
        }
        if (!rc) rc = write(g, f[0], c, s / (2.0 * D), act_bit(activating, 0), m / (2.0 * D));
      });
      break;
    case OP_RESTRICT:
      // coarse r[c // 2] += p0 * (r[c] - A z[c])   (fields: f0 coarse target, f1 r, f2 z)
      if (!need(3)) return fail(g, E_ARG, "RESTRICT needs 3 fields");
      for_struct(g, t, [&](const Coord& c) {
        double az = 2.0 * D * read(g, f[2], c), m = 2.0 * D * read_mag(g, f[2], c);
        for (int a = 0; a < D; a++) {
          az -= read(g, f[2], shift(c, a, +1)) + read(g, f[2], shift(c, a, -1));
          m += read_mag(g, f[2], shift(c, a, +1)) + read_mag(g, f[2], shift(c, a, -1));
        }
        const double res = read(g, f[1], c) - az;
        m += read_mag(g, f[1], c);
        Coord h{c[0] / 2, c[1] / 2, c[2] / 2};
        if (!rc) rc = atomic_add_m(g, f[0], h, P(0) * res, std::fabs(P(0)) * m, act_bit(activating, 0));
      });
      break;
    case OP_PROLONG:
      // fine z[c] += coarse z[c // 2]   (fields: f0 fine target, f1 coarse source)
      if (!need(2)) return fail(g, E_ARG, "PROLONG needs 2 fields");
      for_struct(g, t, [&](const Coord& c) {
        Coord h{c[0] / 2, c[1] / 2, c[2] / 2};
        const double v = read(g, f[0], c) + read(g, f[1], h);
        const double m = read_mag(g, f[0], c) + read_mag(g, f[1], h);
        if (!rc) rc = write(g, f[0], c, v, act_bit(activating, 0), m);
      });
      break;
    case OP_RESID_NORM2:
      // s[] += (r[c] - A z[c])^2   (fields: f0 0-D target, f1 r, f2 z)
      if (!need(3)) return fail(g, E_ARG, "RESID_NORM2 needs 3 fields");
      if (g->trees[g->fields[f[0]].tree].nd != 0) return fail(g, E_ARG, "RESID_NORM2 target must be 0-D");
      for_struct(g, t, [&](const Coord& c) {
        double az = 2.0 * D * read(g, f[2], c), m = 2.0 * D * read_mag(g, f[2], c);
        for (int a = 0; a < D; a++) {
          az -= read(g, f[2], shift(c, a, +1)) + read(g, f[2], shift(c, a, -1));
          m += read_mag(g, f[2], shift(c, a, +1)) + read_mag(g, f[2], shift(c, a, -1));
        }
        const double res = read(g, f[1], c) - az;
        m += read_mag(g, f[1], c);
        if (!rc) rc = atomic_add_m(g, f[0], Coord{0, 0, 0}, res * res, 2.0 * std::fabs(res) * m, false);
      });
      break;
    // --- conjugate gradients around the multigrid preconditioner (MGPCG, PAPER.md:438-441;
    // hu2019taichi): dot products into 0-D fields, updates scaled by a ratio of 0-D fields
    case OP_DOT:
      // f0[] += p0 * f1[c] * f2[c]
      if (!need(3)) return fail(g, E_ARG, "DOT needs 3 fields");
      if (g->trees[g->fields[f[0]].tree].nd != 0) return fail(g, E_ARG, "DOT target must be 0-D");
      for_struct(g, t, [&](const Coord& c) {
        const double a = read(g, f[1], c), b = read(g, f[2], c);
        const double m = std::fabs(P(0)) * read_mag(g, f[1], c) * read_mag(g, f[2], c);
        if (!rc) rc = atomic_add_m(g, f[0], Coord{0, 0, 0}, P(0) * a * b, m, false);
      });
      break;
    case OP_AXPY_RATIO:
    case OP_XPAY_RATIO: {
      // AXPY_RATIO: f0[c] += p0 * (f2[] / f3[]) * f1[c];  XPAY_RATIO: f0[c] = f1[c] + (f2[] / f3[]) * f0[c]
      if (!need(4)) return fail(g, E_ARG, "ratio updates need 4 fields");
      for (int k = 2; k < 4; k++)
        if (g->trees[g->fields[f[k]].tree].nd != 0) return fail(g, E_ARG, "ratio operands must be 0-D");
      const Coord z{0, 0, 0};
      const double num = read(g, f[2], z), den = read(g, f[3], z);
      const double ratio = num / den;
      const double rm = (read_mag(g, f[2], z) + std::fabs(ratio) * read_mag(g, f[3], z)) / std::fabs(den);
      for_struct(g, t, [&](const Coord& c) {
        const double a = read(g, f[1], c), am = read_mag(g, f[1], c);
        const double o = read(g, f[0], c), om = read_mag(g, f[0], c);
        double v, m;
        if (op == OP_AXPY_RATIO) {
          v = o + P(0) * ratio * a;
          m = om + std::fabs(P(0)) * (std::fabs(ratio) * am + rm * std::fabs(a));
        } else {
          v = a + ratio * o;
          m = am + std::fabs(ratio) * om + rm * std::fabs(o);
        }
        if (!rc) rc = write(g, f[0], c, v, act_bit(activating, 0), m);
      });
    } break;
    case OP_JITTER:
      // x[i] += x[i + 1] for even i along axis 0 (PAPER.md:505 deep_hierarchy)
      if (!need(1)) return fail(g, E_ARG, "JITTER needs 1 field");
      for_struct(g, t, [&](const Coord& c) {
        if (c[0] % 2 != 0) return;
        double x = read(g, f[0], shift(c, 0, 1));
        if (!rc) rc = atomic_add(g, f[0], c, x, act_bit(activating, 0));
      });
      break;
    case OP_GRID_OP:
      // MLS-MPM grid update (hu2018moving, cited at PAPER.md:444; mpm3d-like):
      // momentum -> velocity, gravity, sticky-free boundary.  p0 dt, p1 gravity,
      // p2 bound (cells), p3 n_grid.  Fields: f0..f2 velocity/momentum, f3 mass.
      if (!need(4)) return fail(g, E_ARG, "GRID_OP needs 4 fields");
      for_struct(g, t, [&](const Coord& c) {
        if (rc) return;
        double m = read(g, f[3], c), mm = read_mag(g, f[3], c);
        double v[3], mv[3];
        for (int a = 0; a < 3; a++) { v[a] = read(g, f[a], c); mv[a] = read_mag(g, f[a], c); }
        if (m > 0) {
          for (int a = 0; a < 3; a++) {
            double q = v[a] / m;
            // propagated bound of |v/m| under relative errors of v and m
            mv[a] = (mv[a] + std::fabs(v[a]) * (mm / m)) / m;
            v[a] = q;
          }
        }
        v[1] -= P(0) * P(1);
        mv[1] += std::fabs(P(0) * P(1));
        double bound = P(2), n = P(3);
        for (int a = 0; a < D; a++) {
          bool cond = ((double)c[a] < bound && v[a] < 0) || ((double)c[a] > n - bound && v[a] > 0);
          if (cond) { v[a] = 0; mv[a] = 0; }
        }
        for (int a = 0; a < 3 && !rc; a++) rc = write(g, f[a], c, v[a], false, mv[a]);
      });
      break;
    default:
      return fail(g, E_ARG, "unknown struct-for op");
  }
  if (rc) { g->touched.clear(); return rc; }
  return end_task(g);
}

// ---------------------------------------------------------------------------
// Range-for: MLS-MPM particle transfers (hu2018moving, cited at PAPER.md:444;
// the P2G scatter with atomic adds of PAPER.md:457).  Quadratic B-spline
// weights over the 3x3x3 neighbourhood.  The index decision (base cell) is
// made in f32 with the same operation order as the device (reading R16); the
// rest is f64.  Arrays: a0 x (3 comps), a1 v (3), a2 C (9, row-major), a3 J (1).
// ---------------------------------------------------------------------------
struct Kernel {
  int base[3];
  double fx[3], w[3][3], dw[3][3];
};

Kernel bspline(const float xp[3], float inv_dx, const double* x64 = nullptr) {
  Kernel k;
  for (int a = 0; a < 3; a++) {
    volatile float X = xp[a] * inv_dx;          // f32 rounding, no contraction
    volatile float Xm = X - 0.5f;
    k.base[a] = (int)std::floor((float)Xm);
    volatile float fx = X - (float)k.base[a];
    // exact mode (f64 storage, finite-difference pins): same base, f64 fraction
    k.fx[a] = x64 ? x64[a] * (double)inv_dx - (double)k.base[a] : (double)(float)fx;
    double q = k.fx[a];
    k.w[0][a] = 0.5 * (1.5 - q) * (1.5 - q);
    k.w[1][a] = 0.75 - (q - 1.0) * (q - 1.0);
    k.w[2][a] = 0.5 * (q - 0.5) * (q - 0.5);
    // d w / d fx
    k.dw[0][a] = q - 1.5;
    k.dw[1][a] = -2.0 * (q - 1.0);
    k.dw[2][a] = q - 0.5;
  }
  return k;
}

// Grid velocity after the grid update (mpm3d grid op, reading R28), from the
// pre-update momentum p and mass m of a node; mask[r] = 0 where the wall
// condition zeroed component r.
void grid_update(double p[3], double m, const int node[3], double dt, double grav, double bound, double ng, int D,
                 double u[3], double mask[3]) {
  for (int r = 0; r < 3; r++) u[r] = m > 0 ? p[r] / m : p[r];
  u[1] -= dt * grav;
  for (int r = 0; r < 3; r++) {
    mask[r] = 1.0;
    if (r < D && ((node[r] < bound && u[r] < 0) || (node[r] > ng - bound && u[r] > 0))) { u[r] = 0.0; mask[r] = 0.0; }
  }
}


double& A_(Grid* g, int arr, int comp, int64_t i) { Array& a = g->arrays[arr]; return a.val[comp * a.n + i]; }
double& M_(Grid* g, int arr, int comp, int64_t i) { Array& a = g->arrays[arr]; return a.mag[comp * a.n + i]; }

int range_for(Grid* g, int op, int64_t n, const int32_t* f, int nf, const int32_t* ar, int na, const float* p,
              int np, uint32_t activating) {
  auto P = [&](int i) { return i < np ? (double)p[i] : 0.0; };
  for (int i = 0; i < na; i++)
    if (ar[i] < 0 || ar[i] >= (int)g->arrays.size()) return fail(g, E_ARG, "bad array");
  for (int i = 0; i < nf; i++) if (f[i] >= 0 && !field_ok(g, f[i])) return fail(g, E_ARG, "bad field");
  for (int i = 0; i < na; i++)
    if (g->arrays[ar[i]].n < n) return fail(g, E_ARG, "array shorter than range");
  int rc = OK;
  const float inv_dx = (float)P(1);
  const double dx = 1.0 / (double)inv_dx, idx = (double)inv_dx, s4 = 4.0 * idx * idx;
  auto kernel_of = [&](int arr, int64_t i) {
    float xp[3] = {(float)A_(g, arr, 0, i), (float)A_(g, arr, 1, i), (float)A_(g, arr, 2, i)};
    double x64[3] = {A_(g, arr, 0, i), A_(g, arr, 1, i), A_(g, arr, 2, i)};
    return bspline(xp, inv_dx, g->exact ? x64 : nullptr);
  };
  // node weight, its gradient d W / d x, and dpos for offset (a, b, c)
  auto node_w = [&](const Kernel& k, int a, int b, int c, double& W, double gW[3], double dpos[3]) {
    int off[3] = {a, b, c};
    W = k.w[a][0] * k.w[b][1] * k.w[c][2];
    gW[0] = idx * k.dw[a][0] * k.w[b][1] * k.w[c][2];
    gW[1] = idx * k.w[a][0] * k.dw[b][1] * k.w[c][2];
    gW[2] = idx * k.w[a][0] * k.w[b][1] * k.dw[c][2];
    for (int d = 0; d < 3; d++) dpos[d] = ((double)off[d] - k.fx[d]) * dx;
  };
  auto round_arrays = [&](std::initializer_list<int> ids) {
    if (g->exact) return;
    for (int id : ids) for (double& v : g->arrays[id].val) v = (double)(float)v;
  };
  switch (op) {
    case OP_P2G: {
      // p0 dt, p1 inv_dx, p2 p_mass, p3 p_vol, p4 E
      if (nf < 4 || na < 4) return fail(g, E_ARG, "P2G needs 4 fields and 4 arrays");
      const double dt = P(0), pm = P(2), pv = P(3), E = P(4);
      for (int64_t i = 0; i < n && !rc; i++) {
        Kernel k = kernel_of(ar[0], i);
        double J = A_(g, ar[3], 0, i);
        double stress = -dt * 4.0 * E * pv * (J - 1.0) * idx * idx;
        // shadow magnitudes (reading R15: the sum of the absolute values of
        // every term the value is computed from, inputs at their own shadow
        // magnitude): |stress| counts |J| + 1, the momentum |p_mass v| +
        // sum_d |aff_rd dpos_d| term by term (they may cancel)
        const double stress_m = dt * 4.0 * E * pv * (M_(g, ar[3], 0, i) + 1.0) * idx * idx;
        double aff[3][3], affm[3][3], v[3], vm[3];
        for (int r = 0; r < 3; r++) {
          v[r] = A_(g, ar[1], r, i);
          vm[r] = M_(g, ar[1], r, i);
          for (int c = 0; c < 3; c++) {
            aff[r][c] = pm * A_(g, ar[2], 3 * r + c, i) + (r == c ? stress : 0.0);
            affm[r][c] = pm * M_(g, ar[2], 3 * r + c, i) + (r == c ? stress_m : 0.0);
          }
        }
        for (int a = 0; a < 3 && !rc; a++)
          for (int b = 0; b < 3 && !rc; b++)
            for (int c = 0; c < 3 && !rc; c++) {
              double W, gW[3], dpos[3];
              node_w(k, a, b, c, W, gW, dpos);
              Coord node{k.base[0] + a, k.base[1] + b, k.base[2] + c};
              for (int r = 0; r < 3 && !rc; r++) {
                double mom = pm * v[r], momm = pm * vm[r];
                for (int d = 0; d < 3; d++) {
                  mom += aff[r][d] * dpos[d];
                  momm += affm[r][d] * std::fabs(dpos[d]);
                }
                rc = atomic_add_m(g, f[r], node, W * mom, std::fabs(W) * momm, act_bit(activating, r));
              }
              if (!rc) rc = atomic_add(g, f[3], node, W * pm, act_bit(activating, 3));
            }
      }
    } break;
    case OP_G2P: {
      // p0 dt, p1 inv_dx.  Reads grid velocity f0..f2 at the particle state a0..a3
      // and writes the new state to a4..a7 (in place when a4 is absent).
      if (nf < 3 || na < 4) return fail(g, E_ARG, "G2P needs 3 fields and 4 arrays");
      const double dt = P(0);
      const int o0 = na >= 8 ? 4 : 0;
      for (int64_t i = 0; i < n; i++) {
        Kernel k = kernel_of(ar[0], i);
        double nv[3] = {0, 0, 0}, mv[3] = {0, 0, 0}, nC[3][3] = {{0}}, mC[3][3] = {{0}};
        for (int a = 0; a < 3; a++)
          for (int b = 0; b < 3; b++)
            for (int c = 0; c < 3; c++) {
              double W, gW[3], dpos[3];
              node_w(k, a, b, c, W, gW, dpos);
              Coord node{k.base[0] + a, k.base[1] + b, k.base[2] + c};
              for (int r = 0; r < 3; r++) {
                double gv = read(g, f[r], node), gm = read_mag(g, f[r], node) + std::fabs(gv);
                nv[r] += W * gv;
                mv[r] += std::fabs(W) * gm;
                for (int d = 0; d < 3; d++) {
                  double s = s4 * W * dpos[d];
                  nC[r][d] += s * gv;
                  mC[r][d] += std::fabs(s) * gm;
                }
              }
            }
        double tr = nC[0][0] + nC[1][1] + nC[2][2];
        double mtr = mC[0][0] + mC[1][1] + mC[2][2];
        const double J = A_(g, ar[3], 0, i);
        for (int r = 0; r < 3; r++) {
          double x = A_(g, ar[0], r, i);
          A_(g, ar[o0 + 1], r, i) = nv[r]; M_(g, ar[o0 + 1], r, i) = mv[r];
          A_(g, ar[o0 + 0], r, i) = x + dt * nv[r];
          M_(g, ar[o0 + 0], r, i) = std::fabs(x) + dt * mv[r];
          for (int d = 0; d < 3; d++) {
            A_(g, ar[o0 + 2], 3 * r + d, i) = nC[r][d]; M_(g, ar[o0 + 2], 3 * r + d, i) = mC[r][d];
          }
        }
        A_(g, ar[o0 + 3], 0, i) = J * (1.0 + dt * tr);
        M_(g, ar[o0 + 3], 0, i) = std::fabs(J) * (1.0 + dt * mtr);
      }
      round_arrays({ar[o0], ar[o0 + 1], ar[o0 + 2], ar[o0 + 3]});
    } break;
    case OP_LOSS_MEAN: {
      // f0 (0-D) += p1 * sum_i a0[p0][i]   (loss = mean x of the particles, C4)
      if (nf < 1 || na < 1) return fail(g, E_ARG, "LOSS_MEAN needs a field and an array");
      const int comp = (int)P(0);
      for (int64_t i = 0; i < n && !rc; i++)
        rc = atomic_add(g, f[0], Coord{0, 0, 0}, P(1) * A_(g, ar[0], comp, i), false);
    } break;
    case OP_PERMUTE: {
      // a2 = a1 in SOME order of the particles (the method fixes none; the
      // device uses its bin order).  The oracle takes the identity; parity
      // tests match particles by id.
      if (na < 3) return fail(g, E_ARG, "PERMUTE needs 3 arrays");
      Array &src = g->arrays[ar[1]], &dst = g->arrays[ar[2]];
      const int nc = std::min(src.ncomp, dst.ncomp);
      for (int c = 0; c < nc; c++)
        for (int64_t i = 0; i < n; i++) {
          dst.val[c * dst.n + i] = src.val[c * src.n + i];
          dst.mag[c * dst.n + i] = src.mag[c * src.n + i];
        }
    } break;
    case OP_ADJ_INIT: {
      // adjoint of the last state: a0[p0] = p1 (d loss / d x_T), everything else 0
      if (na < 4) return fail(g, E_ARG, "ADJ_INIT needs 4 arrays");
      for (int k = 0; k < 4; k++) {
        Array& a = g->arrays[ar[k]];
        for (int c = 0; c < a.ncomp; c++)
          for (int64_t i = 0; i < n; i++) {
            A_(g, ar[k], c, i) = (k == 0 && c == (int)P(0)) ? P(1) : 0.0;
            M_(g, ar[k], c, i) = std::fabs(A_(g, ar[k], c, i));
          }
      }
    } break;
    case OP_G2P_ADJ: {
      // Adjoint of GRID_OP (folded) and G2P for step s.  p0 dt, p1 inv_dx,
      // p2 gravity, p3 bound, p4 n_grid.  Fields: f0..f2 grid momentum p, f3
      // mass m (forward, read), f4..f6 adjoint of p, f7 adjoint of m (scattered,
      // activating).  Arrays: a0 x_s, a1 J_s, a2..a5 adjoints (x, v, C, J) of
      // state s+1, a6 adjoint of x_s (written), a7 adjoint of J_s (written).
      // The *m variables are the shadow magnitudes (reading R32): the sum of
      // |terms| each result is accumulated from, propagated through products
      // and quotients, so parity tolerances scale with them.
      if (nf < 8 || na < 8) return fail(g, E_ARG, "G2P_ADJ needs 8 fields and 8 arrays");
      const double dt = P(0), grav = P(2), bound = P(3), ng = P(4);
      const int D = 3;
      for (int64_t i = 0; i < n && !rc; i++) {
        Kernel k = kernel_of(ar[0], i);
        const double J = A_(g, ar[1], 0, i);
        double xb1[3], vb1[3], Cb1[3][3];
        for (int r = 0; r < 3; r++) {
          xb1[r] = A_(g, ar[2], r, i);
          vb1[r] = A_(g, ar[3], r, i);
          for (int d = 0; d < 3; d++) Cb1[r][d] = A_(g, ar[4], 3 * r + d, i);
        }
        const double Jb1 = A_(g, ar[5], 0, i);
        // input shadow magnitudes (adjoints of s+1 and J_s come from earlier tasks)
        const double Jm = M_(g, ar[1], 0, i), Jb1m = M_(g, ar[5], 0, i);
        double xb1m[3], vb1m[3], Cb1m[3][3];
        for (int r = 0; r < 3; r++) {
          xb1m[r] = M_(g, ar[2], r, i);
          vb1m[r] = M_(g, ar[3], r, i);
          for (int d = 0; d < 3; d++) Cb1m[r][d] = M_(g, ar[4], 3 * r + d, i);
        }
        // forward grid velocities of the 27 nodes and the new C (for tr C')
        double u[27][3], um[27][3], mask[27][3], pn[27][3], pm_[27][3], mn[27], mm[27];
        double trC = 0.0, trCm = 0.0;
        for (int a = 0, q = 0; a < 3; a++)
          for (int b = 0; b < 3; b++)
            for (int c = 0; c < 3; c++, q++) {
              double W, gW[3], dpos[3];
              node_w(k, a, b, c, W, gW, dpos);
              Coord node{k.base[0] + a, k.base[1] + b, k.base[2] + c};
              int nd[3] = {(int)node[0], (int)node[1], (int)node[2]};
              for (int r = 0; r < 3; r++) { pn[q][r] = read(g, f[r], node); pm_[q][r] = read_mag(g, f[r], node); }
              mn[q] = read(g, f[3], node);
              mm[q] = read_mag(g, f[3], node);
              grid_update(pn[q], mn[q], nd, dt, grav, bound, ng, D, u[q], mask[q]);
              for (int r = 0; r < 3; r++) {
                um[q][r] = mn[q] > 0 ? (pm_[q][r] + std::fabs(pn[q][r]) * mm[q] / mn[q]) / mn[q] : pm_[q][r];
                if (r == 1) um[q][r] += std::fabs(dt * grav);
                um[q][r] *= mask[q][r];
                trC += s4 * W * u[q][r] * dpos[r];
                trCm += s4 * std::fabs(W) * um[q][r] * std::fabs(dpos[r]);
              }
            }
        double vt[3], vtm[3], Ct[3][3], Ctm[3][3];
        for (int r = 0; r < 3; r++) {
          vt[r] = vb1[r] + dt * xb1[r];
          vtm[r] = vb1m[r] + dt * xb1m[r];
          for (int d = 0; d < 3; d++) {
            Ct[r][d] = Cb1[r][d] + (r == d ? Jb1 * J * dt : 0.0);
            Ctm[r][d] = Cb1m[r][d] + (r == d ? Jb1m * Jm * dt : 0.0);
          }
        }
        double Jb = Jb1 * (1.0 + dt * trC), mJ = Jb1m * (1.0 + dt * trCm);
        double xb[3] = {xb1[0], xb1[1], xb1[2]}, mx[3] = {xb1m[0], xb1m[1], xb1m[2]};
        for (int a = 0, q = 0; a < 3 && !rc; a++)
          for (int b = 0; b < 3 && !rc; b++)
            for (int c = 0; c < 3 && !rc; c++, q++) {
              double W, gW[3], dpos[3];
              node_w(k, a, b, c, W, gW, dpos);
              Coord node{k.base[0] + a, k.base[1] + b, k.base[2] + c};
              double gbar[3], gbm[3], Wbar = 0.0, Wbm = 0.0, dposbar[3] = {0, 0, 0}, dpbm[3] = {0, 0, 0};
              for (int r = 0; r < 3; r++) {
                double ct = 0.0, ctm = 0.0;
                for (int d = 0; d < 3; d++) { ct += Ct[r][d] * dpos[d]; ctm += Ctm[r][d] * std::fabs(dpos[d]); }
                gbar[r] = W * vt[r] + s4 * W * ct;
                gbm[r] = std::fabs(W) * (vtm[r] + s4 * ctm);
                Wbar += u[q][r] * vt[r] + s4 * u[q][r] * ct;
                Wbm += um[q][r] * (vtm[r] + s4 * ctm);
                for (int d = 0; d < 3; d++) {
                  dposbar[d] += s4 * W * Ct[r][d] * u[q][r];
                  dpbm[d] += s4 * std::fabs(W) * Ctm[r][d] * um[q][r];
                }
              }
              for (int d = 0; d < 3; d++) {
                xb[d] += Wbar * gW[d] - dposbar[d];
                mx[d] += Wbm * std::fabs(gW[d]) + dpbm[d];
              }
              // GRID_OP adjoint: u = mask * (p / m - dt g e_y)
              double pb[3], pbm[3], mb = 0.0, mbm = 0.0;
              for (int r = 0; r < 3; r++) {
                const double ub = gbar[r] * mask[q][r], ubm = gbm[r] * mask[q][r];
                if (mn[q] > 0) {
                  pb[r] = ub / mn[q];
                  pbm[r] = (ubm + std::fabs(ub) * mm[q] / mn[q]) / mn[q];
                  mb -= pb[r] * (pn[q][r] / mn[q]);
                  mbm += (ubm * std::fabs(pn[q][r]) + std::fabs(ub) * pm_[q][r] +
                          2.0 * std::fabs(ub * pn[q][r]) * mm[q] / mn[q]) / (mn[q] * mn[q]);
                } else {
                  pb[r] = ub;
                  pbm[r] = ubm;
                }
              }
              for (int r = 0; r < 3 && !rc; r++)
                rc = atomic_add_m(g, f[4 + r], node, pb[r], pbm[r], act_bit(activating, 4 + r));
              if (!rc) rc = atomic_add_m(g, f[7], node, mb, mbm, act_bit(activating, 7));
            }
        for (int d = 0; d < 3; d++) { A_(g, ar[6], d, i) = xb[d]; M_(g, ar[6], d, i) = mx[d]; }
        A_(g, ar[7], 0, i) = Jb;
        M_(g, ar[7], 0, i) = mJ;
      }
      round_arrays({ar[6], ar[7]});
    } break;
    case OP_P2G_ADJ: {
      // Adjoint of P2G for step s.  p0 dt, p1 inv_dx, p2 p_mass, p3 p_vol, p4 E.
      // Fields f0..f2 adjoint of grid momentum, f3 adjoint of mass (gathered).
      // Arrays a0..a3 state s (x, v, C, J); a4 adjoint x_s (+=), a5 adjoint v_s,
      // a6 adjoint C_s (written), a7 adjoint J_s (+=).  Magnitudes as in G2P_ADJ.
      if (nf < 4 || na < 8) return fail(g, E_ARG, "P2G_ADJ needs 4 fields and 8 arrays");
      const double dt = P(0), pm = P(2), pv = P(3), E = P(4);
      const double kJ = -dt * 4.0 * E * pv * idx * idx;
      for (int64_t i = 0; i < n; i++) {
        Kernel k = kernel_of(ar[0], i);
        const double J = A_(g, ar[3], 0, i);
        const double Jm = M_(g, ar[3], 0, i);
        double v[3], vm[3], A[3][3], Am[3][3];
        for (int r = 0; r < 3; r++) {
          v[r] = A_(g, ar[1], r, i);
          vm[r] = M_(g, ar[1], r, i);
          for (int c = 0; c < 3; c++) {
            A[r][c] = pm * A_(g, ar[2], 3 * r + c, i) + (r == c ? kJ * (J - 1.0) : 0.0);
            Am[r][c] = pm * M_(g, ar[2], 3 * r + c, i) + (r == c ? std::fabs(kJ) * (Jm + 1.0) : 0.0);
          }
        }
        double vb[3] = {0, 0, 0}, Ab[3][3] = {{0}}, Abm[3][3] = {{0}}, xb[3] = {0, 0, 0}, mx[3] = {0, 0, 0},
               mv[3] = {0, 0, 0};
        for (int a = 0; a < 3; a++)
          for (int b = 0; b < 3; b++)
            for (int c = 0; c < 3; c++) {
              double W, gW[3], dpos[3];
              node_w(k, a, b, c, W, gW, dpos);
              Coord node{k.base[0] + a, k.base[1] + b, k.base[2] + c};
              double pb[3], pbm[3];
              for (int r = 0; r < 3; r++) { pb[r] = read(g, f[r], node); pbm[r] = read_mag(g, f[r], node); }
              const double mb = read(g, f[3], node), mbm = read_mag(g, f[3], node);
              double Wbar = mb * pm, Wbm = mbm * pm, dposbar[3] = {0, 0, 0}, dpbm[3] = {0, 0, 0};
              for (int r = 0; r < 3; r++) {
                double mom = pm * v[r], momm = pm * vm[r];
                for (int d = 0; d < 3; d++) { mom += A[r][d] * dpos[d]; momm += Am[r][d] * std::fabs(dpos[d]); }
                Wbar += pb[r] * mom;
                Wbm += pbm[r] * momm;
                vb[r] += W * pm * pb[r];
                mv[r] += std::fabs(W) * pm * pbm[r];
                for (int d = 0; d < 3; d++) {
                  Ab[r][d] += W * pb[r] * dpos[d];
                  Abm[r][d] += std::fabs(W) * pbm[r] * std::fabs(dpos[d]);
                  dposbar[d] += W * pb[r] * A[r][d];
                  dpbm[d] += std::fabs(W) * pbm[r] * Am[r][d];
                }
              }
              for (int d = 0; d < 3; d++) {
                xb[d] += Wbar * gW[d] - dposbar[d];
                mx[d] += Wbm * std::fabs(gW[d]) + dpbm[d];
              }
            }
        for (int d = 0; d < 3; d++) {
          A_(g, ar[4], d, i) += xb[d];
          M_(g, ar[4], d, i) += mx[d];
          A_(g, ar[5], d, i) = vb[d];
          M_(g, ar[5], d, i) = mv[d];
          for (int c = 0; c < 3; c++) {
            A_(g, ar[6], 3 * d + c, i) = pm * Ab[d][c];
            M_(g, ar[6], 3 * d + c, i) = pm * Abm[d][c];
          }
        }
        const double trA = Ab[0][0] + Ab[1][1] + Ab[2][2];
        A_(g, ar[7], 0, i) += kJ * trA;
        M_(g, ar[7], 0, i) += std::fabs(kJ) * (Abm[0][0] + Abm[1][1] + Abm[2][2]);
      }
      round_arrays({ar[4], ar[5], ar[6], ar[7]});
    } break;
    default:
      return fail(g, E_ARG, "unknown range-for op");
  }
  if (rc) { g->touched.clear(); return rc; }
  return end_task(g);
}

int serial(Grid* g, int op, const int32_t* f, int nf, const float* p, int np) {
  (void)p; (void)np;
  switch (op) {
    case OP_CLEAR_SCALAR: {
      if (nf < 1 || !field_ok(g, f[0])) return fail(g, E_ARG, "CLEAR_SCALAR needs a field");
      if (g->trees[g->fields[f[0]].tree].nd != 0) return fail(g, E_ARG, "CLEAR_SCALAR target must be 0-D");
      int rc = write(g, f[0], Coord{0, 0, 0}, 0.0, false, 0.0);
      if (rc) { g->touched.clear(); return rc; }
      return end_task(g);
    }
    case OP_COPY_SCALAR: {
      // f0[] = f1[]  (MGPCG: zTr_old = zTr_new)
      if (nf < 2 || !field_ok(g, f[0]) || !field_ok(g, f[1])) return fail(g, E_ARG, "COPY_SCALAR needs 2 fields");
      if (g->trees[g->fields[f[0]].tree].nd != 0 || g->trees[g->fields[f[1]].tree].nd != 0)
        return fail(g, E_ARG, "COPY_SCALAR operands must be 0-D");
      const Coord z{0, 0, 0};
      int rc = write(g, f[0], z, read(g, f[1], z), false, read_mag(g, f[1], z));
      if (rc) { g->touched.clear(); return rc; }
      return end_task(g);
    }
    default:
      return fail(g, E_ARG, "unknown serial op");
  }
}

// DEACTIVATE(S): every cell of level S and below becomes inactive, their
// payload is dropped (reads 0) and pointer children are freed (reading R7).
int deactivate(Grid* g, int snode) {
  if (snode <= 0 || snode >= (int)g->nodes.size()) return fail(g, E_ARG, "bad snode");
  const Node& n = g->nodes[snode];
  if (!sparse(n.kind)) return fail(g, E_ARG, "deactivate needs a sparse level");
  const Tree& t = g->trees[n.tree];
  int k = chain_index(t, snode);
  for (size_t m = k; m < t.levels.size(); m++) {
    int l = t.levels[m];
    if (!sparse(g->nodes[l].kind)) continue;
    if (g->nodes[l].kind == K_POINTER) g->freed[l] += (int64_t)g->active[l].size();
    g->active[l].clear();
  }
  for (int pl : t.fields) {
    for (size_t fi = 0; fi < g->fields.size(); fi++)
      if (g->fields[fi].snode == pl) { g->fields[fi].val.clear(); g->fields[fi].mag.clear(); }
  }
  g->tasks++;
  return OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C API of the oracle (names distinct from the product's sg_*).
// ---------------------------------------------------------------------------
extern "C" {

void* orc_create(const int32_t* desc, int32_t n, char* err, int32_t errlen) {
  Grid* g = new Grid();
  int rc = build_layout(g, desc, n);
  if (rc) {
    if (err && errlen > 0) { std::snprintf(err, errlen, "%s", g->err.c_str()); }
    delete g;
    return nullptr;
  }
  return g;
}

void orc_destroy(void* h) { delete (Grid*)h; }

const char* orc_error(void* h) { return ((Grid*)h)->err.c_str(); }

int32_t orc_num_fields(void* h) { return (int32_t)((Grid*)h)->fields.size(); }

// f64 storage (no f32 rounding): for the finite-difference pins of the adjoints.
void orc_set_exact(void* h, int32_t on) { ((Grid*)h)->exact = on != 0; }

int32_t orc_activate(void* h, int32_t field, const int32_t* coords, int64_t n) {
  Grid* g = (Grid*)h;
  if (!field_ok(g, field)) return fail(g, E_ARG, "bad field");
  Tree& t = tree_of_field(g, field);
  for (int64_t i = 0; i < n; i++) {
    Coord c{0, 0, 0};
    for (int a = 0; a < t.nd; a++) c[a] = coords[i * t.nd + a];
    if (!in_range(g, t, c)) return fail(g, E_RANGE, "activate coordinate out of range");
  }
  for (int64_t i = 0; i < n; i++) {
    Coord c{0, 0, 0};
    for (int a = 0; a < t.nd; a++) c[a] = coords[i * t.nd + a];
    activate_cell(g, t, c);
  }
  g->tasks++;
  return OK;
}

int32_t orc_listgen(void* h, int32_t snode) { return listgen((Grid*)h, snode); }

int32_t orc_clear_list(void* h, int32_t snode) {
  Grid* g = (Grid*)h;
  if (snode <= 0 || snode >= (int)g->nodes.size()) return fail(g, E_ARG, "bad snode");
  g->lists[snode].clear();
  g->tasks++;
  return OK;
}

int32_t orc_struct_for(void* h, int32_t op, int32_t snode, const int32_t* fields, int32_t nf,
                       const float* params, int32_t np, uint32_t activating) {
  return struct_for((Grid*)h, op, snode, fields, nf, params, np, activating);
}

int32_t orc_serial(void* h, int32_t op, const int32_t* fields, int32_t nf, const float* params, int32_t np) {
  return serial((Grid*)h, op, fields, nf, params, np);
}

int32_t orc_deactivate(void* h, int32_t snode) { return deactivate((Grid*)h, snode); }

// Particle arrays: the oracle keeps its own copy (f32-rounded values in f64).
int32_t orc_register_array(void* h, const float* data, int64_t n, int32_t ncomp) {
  Grid* g = (Grid*)h;
  Array a;
  a.n = n; a.ncomp = ncomp;
  a.val.resize((size_t)n * ncomp);
  a.mag.resize((size_t)n * ncomp);
  for (size_t i = 0; i < a.val.size(); i++) { a.val[i] = data[i]; a.mag[i] = std::fabs((double)data[i]); }
  g->arrays.push_back(a);
  return (int32_t)g->arrays.size() - 1;
}

int32_t orc_read_array(void* h, int32_t id, double* out, double* mag, int64_t total) {
  Grid* g = (Grid*)h;
  if (id < 0 || id >= (int)g->arrays.size()) return fail(g, E_ARG, "bad array");
  Array& a = g->arrays[id];
  if (total != (int64_t)a.val.size()) return fail(g, E_ARG, "size mismatch");
  for (int64_t i = 0; i < total; i++) { out[i] = a.val[i]; if (mag) mag[i] = a.mag[i]; }
  return OK;
}

int32_t orc_load_array(void* h, int32_t id, const double* data, int64_t total) {
  Grid* g = (Grid*)h;
  if (id < 0 || id >= (int)g->arrays.size()) return fail(g, E_ARG, "bad array");
  Array& a = g->arrays[id];
  if (total != (int64_t)a.val.size()) return fail(g, E_ARG, "size mismatch");
  for (int64_t i = 0; i < total; i++) { a.val[i] = data[i]; a.mag[i] = std::fabs(data[i]); }
  return OK;
}

int32_t orc_range_for(void* h, int32_t op, int64_t n, const int32_t* fields, int32_t nf, const int32_t* arrays,
                      int32_t na, const float* params, int32_t np, uint32_t activating) {
  return range_for((Grid*)h, op, n, fields, nf, arrays, na, params, np, activating);
}

// Sorted set of active level-global cells of a sparse level.
int64_t orc_export_mask(void* h, int32_t snode, int32_t* out, int64_t cap) {
  Grid* g = (Grid*)h;
  if (snode <= 0 || snode >= (int)g->nodes.size() || !sparse(g->nodes[snode].kind))
    return fail(g, E_ARG, "bad snode");
  const std::set<Coord>& s = g->active[snode];
  int nd = g->nodes[snode].nd;
  int64_t i = 0;
  for (const Coord& c : s) {
    if (i < cap) for (int a = 0; a < nd; a++) out[i * nd + a] = (int32_t)c[a];
    i++;
  }
  return i;
}

// The level's current list, as stored.
int64_t orc_export_list(void* h, int32_t snode, int32_t* out, int64_t cap) {
  Grid* g = (Grid*)h;
  if (snode <= 0 || snode >= (int)g->nodes.size()) return fail(g, E_ARG, "bad snode");
  const std::vector<Coord>& s = g->lists[snode];
  int nd = g->nodes[snode].nd;
  int64_t i = 0;
  for (const Coord& c : s) {
    if (i < cap) for (int a = 0; a < nd; a++) out[i * nd + a] = (int32_t)c[a];
    i++;
  }
  return i;
}

// Dense bounding array of a field (row-major, last axis fastest), inactive -> 0,
// plus the shadow magnitude of each element.
int32_t orc_read_field(void* h, int32_t field, double* out, double* mag, int64_t n) {
  Grid* g = (Grid*)h;
  if (!field_ok(g, field)) return fail(g, E_ARG, "bad field");
  Tree& t = tree_of_field(g, field);
  const int64_t* r = leaf_res(g, t);
  int64_t total = 1;
  for (int a = 0; a < t.nd; a++) total *= r[a];
  if (n != total) return fail(g, E_ARG, "size mismatch");
  int64_t e[3] = {t.nd > 0 ? r[0] : 1, t.nd > 1 ? r[1] : 1, t.nd > 2 ? r[2] : 1};
  int64_t i = 0;
  for_box(Coord{0, 0, 0}, e, [&](const Coord& c) {
    out[i] = read(g, field, c);
    if (mag) mag[i] = read_mag(g, field, c);
    i++;
  });
  return OK;
}

// Load values of ACTIVE cells from a dense array (single-step state handoff).
int32_t orc_load_field(void* h, int32_t field, const double* dense, int64_t n) {
  Grid* g = (Grid*)h;
  if (!field_ok(g, field)) return fail(g, E_ARG, "bad field");
  Tree& t = tree_of_field(g, field);
  const int64_t* r = leaf_res(g, t);
  int64_t e[3] = {t.nd > 0 ? r[0] : 1, t.nd > 1 ? r[1] : 1, t.nd > 2 ? r[2] : 1};
  if (n != e[0] * e[1] * e[2]) return fail(g, E_ARG, "size mismatch");
  int64_t i = 0;
  Field& fl = g->fields[field];
  for_box(Coord{0, 0, 0}, e, [&](const Coord& c) {
    if (is_active(g, t, c)) { fl.val[c] = dense[i]; fl.mag[c] = std::fabs(dense[i]); }
    i++;
  });
  return OK;
}

// counters: [tasks, listgens, sum allocated, sum freed]
int32_t orc_counters(void* h, int64_t* out) {
  Grid* g = (Grid*)h;
  int64_t a = 0, f = 0;
  for (auto& kv : g->allocated) a += kv.second;
  for (auto& kv : g->freed) f += kv.second;
  out[0] = g->tasks; out[1] = g->listgens; out[2] = a; out[3] = f;
  return OK;
}

}  // extern "C"
