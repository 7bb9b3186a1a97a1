// planner.h -- the asynchronous engine's host side: lowering, state-flow graph,
// whole-program passes, plan cache (PAPER.md sections 4-7).
#ifndef SG_PLANNER_H_
#define SG_PLANNER_H_

#include <stdint.h>
#include <string>
#include <unordered_map>
#include <vector>
#include "sg_internal.h"

namespace sg {

// ---- layout facts the planner needs (derived once by sg_create) ------------
struct HTree {
  int nd = 0;
  std::vector<int> levels;   // snode ids root->leaf (empty: 0-D)
  std::vector<int> fields;   // field ids placed at the leaf
  int driving = -1;          // chain index of the driving level, -1 none
  bool leaf_bitmasked = false;
};

struct HLayout {
  std::vector<sg_snode_desc> nodes;
  std::vector<HTree> trees;
  std::vector<int> field_tree, field_slot, field_dtype, field_scalar;
  std::vector<int> snode_tree, snode_pos;   // tree id / chain index of each level snode
  int n_scalars = 0;
  // arrays whose writes are ordered against the exchange sequence (the
  // multi-GPU send buffers: on the peer transport they are the neighbours'
  // receive buffers, so a write must stay between the same exchanges)
  std::vector<char> seq_arrays;
  bool is_sparse(int snode) const {
    return nodes[snode].kind == SG_BITMASKED || nodes[snode].kind == SG_POINTER;
  }
  // sparse levels a struct-for over tree t needs a list for (reading R5)
  std::vector<int> listed_levels(int t) const;
  std::vector<int> sparse_levels(int t) const;
  // DEACTIVATE of the tree's first sparse level on a tree whose dense volume is
  // at most 64 MiB runs as a pool RESET (zero every allocated container, reset
  // the allocators): no list input, so its listgens fall to DSE (reading R33)
  bool deactivate_resets(int snode) const;
};

// ---- states ------------------------------------------------
enum StateKind { ST_VALUE = 0, ST_ARRAY = 1, ST_MASK = 2, ST_LIST = 3, ST_ALLOC = 4 };
inline int64_t skey(int kind, int id) { return ((int64_t)kind << 32) | (uint32_t)id; }
inline int skind(int64_t s) { return (int)(s >> 32); }
inline int sid(int64_t s) { return (int)(uint32_t)s; }

enum Access { AC_ID = 0, AC_NBR = 1, AC_DIV2 = 2, AC_CONST = 3, AC_DATA = 4, AC_NONE = 5 };

struct Use {
  int64_t state;
  int access;
  bool complete;   // outputs: the write fully determines the state
};

// A lowered task; after fusion a task may carry several member ops.
struct PTask {
  int type = 0;           // TT_*
  int call = -1;          // user call index inside the flush window
  int snode = -1;         // listgen / clear-list / deactivate level; struct-for leaf
  int tree = -1;
  int field = -1;         // activate target
  const int32_t* coords = nullptr;
  int64_t n = 0;
  int coords_class = -1;  // canonical id of (coords, n) inside the window
  sg_task t{};            // struct-for / range-for / serial op
  uint32_t act = 0;       // effective activating bits (after demotion)
  bool pinned = false;    // explicit listgen: never removed
  int pos = 0;            // index in the eager lowered sequence
  std::vector<int> members;   // eager positions of the fused member tasks (in order)
  std::vector<uint32_t> member_act;
  std::vector<int> phase_end; // SG_PASS_CHAIN: cumulative member counts at phase ends
  std::vector<Use> in, out;
};

struct PlanRecord { int group, type, call, snode; uint32_t act; int flags; };

struct PlanStats {
  int64_t listgens_removed = 0, demotions = 0, fused = 0, dead = 0, chained = 0;
};

struct Plan {
  std::vector<std::vector<int>> groups;        // eager positions per launch group
  std::vector<std::vector<uint32_t>> acts;     // effective act bits per member
  std::vector<std::vector<int>> phase_ends;    // per group: cumulative member counts (1 entry unless chained)
  PlanStats stats;
};

// Meta of a single (unfused) task: input / output states with access kinds.
void task_meta(const HLayout& L, PTask& t);
// Lowering of one user call into tasks (readings R3, R5).
struct UserCall {
  int kind;               // 0 activate, 1 listgen, 2 task, 3 clear
  int field = -1, snode = -1, mode = 0;
  const int32_t* coords = nullptr;
  int64_t n = 0;
  sg_task t{};
};
int lower_call(const HLayout& L, const UserCall& c, int call_index, bool faithful, std::vector<PTask>& out,
               std::string& err);

// The optimizer (PAPER.md sections 6.2-6.5) over an eager lowered sequence.
Plan optimize(const HLayout& L, const std::vector<PTask>& eager, uint32_t passes,
              const std::vector<char>& observed_fields);

uint64_t stream_hash(const std::vector<PTask>& eager, uint32_t passes, const std::vector<char>& observed);

// --- state-flow graph (exposed for tests through the plan) -------------------
struct Graph {
  int n = 0;
  std::vector<std::vector<int>> succ, pred;
  std::vector<std::unordered_map<int64_t, int>> in_ver;       // state -> producer (-1 initial)
  std::vector<std::unordered_map<int64_t, int>> next_writer;  // output state -> next writer (-1 none)
  std::vector<std::unordered_map<int64_t, int>> readers;      // output state -> # RAW readers
  std::vector<std::vector<std::pair<int, int64_t>>> edges_to; // (from, state) per destination
};
Graph build_graph(const std::vector<PTask>& seq);

// Bit i set: the op writes arrays[i] (from the planner's op-use table).
uint32_t task_array_writes(const sg_task& t);

}  // namespace sg
#endif
