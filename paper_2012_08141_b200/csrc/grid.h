// grid.h -- the library-side state of one sg_grid (shared by sg_api.cu and
// dist.cu; not part of the C-ABI: sg_grid is opaque to callers).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "planner.h"
#include "sg_internal.h"

namespace sg {
// Multi-GPU data plane (sg_dist_init).  Exchange kinds:
// 0 halo reduce, 1 halo fill, 2 particle migration; sides 0 = left (x-1),
// 1 = right (x+1).  The arena is one cudaMalloc allocation per grid (IPC
// shareable): control words (flags the neighbours store into, local epochs),
// then the receive buffers, each [count word, 3 pad words, payload].
enum { DIST_KINDS = 3, DIST_CTRL_WORDS = 64 };
enum { DIST_NONE = 0, DIST_PEER = 1, DIST_NCCL = 2 };
struct DistState {
  bool on = false;
  int rank = 0, world = 1, axis = 0;
  int transport = DIST_NONE;
  void* comm = nullptr;                  // ncclComm_t (NCCL transport / peer discovery)
  uint32_t* arena = nullptr;             // local arena (flags, epochs, receive buffers)
  size_t arena_words = 0;
  uint32_t* peer_arena[2] = {nullptr, nullptr};   // neighbours' arenas, mapped (peer transport)
  bool peer_ipc[2] = {false, false};     // mapped with cudaIpcOpenMemHandle (close on destroy)
  uint32_t* send_local[DIST_KINDS][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
  int64_t words[DIST_KINDS] = {0, 0, 0};   // words per buffer (4-word header + payload)
  size_t recv_off[DIST_KINDS][2] = {{0, 0}, {0, 0}, {0, 0}};
  int ids_send[DIST_KINDS][2] = {{-1, -1}, {-1, -1}, {-1, -1}};
  int ids_recv[DIST_KINDS][2] = {{-1, -1}, {-1, -1}, {-1, -1}};
  bool has_nb[2] = {false, false};
  int group = -1;                        // in-process group (virtual ranks), -1 none
};
}  // namespace sg

using namespace sg;   // internal header: the library's own translation units only

struct sg_grid {
  sg::DistState dist;
  sg_opts opts{};
  cudaStream_t stream = nullptr;
  bool plan_only = false;
  sg::HLayout L;
  std::vector<DTree> dtrees;
  std::vector<std::vector<DList>> lists;   // [tree][chain position]
  std::vector<DArray> arrays;
  std::vector<void*> allocs;
  DevCtx ctx{};
  DTree* d_trees = nullptr;
  DField* d_fields = nullptr;
  DArray* d_arrays = nullptr;
  int d_arrays_cap = 0;
  // flush window
  std::vector<PTask> eager;
  int ncalls = 0;
  std::vector<std::pair<const int32_t*, int64_t>> coords_seen;
  std::unordered_map<uint64_t, Plan> cache;
  std::vector<PlanRecord> last_plan;
  int64_t task_counter = 0;         // launch index inside the current flush (error reports)
  // CUDA graphs: a plan that already ran once is captured (on a private
  // stream), instantiated once per plan and updated in place afterwards, and
  // replayed with one cudaGraphLaunch on the user stream
  bool use_graphs = true;           // SG_NO_GRAPH=1 disables
  cudaStream_t user_stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  std::unordered_map<uint64_t, cudaGraphExec_t> gexec;
  std::unordered_map<uint64_t, int64_t> gaux;   // aux kernels captured in each plan's graph
  std::unordered_map<uint64_t, uint64_t> gsig;   // launch-argument signature of each exec's last capture
  std::unordered_map<uint64_t, int> plan_runs;
  std::unordered_map<uint64_t, char> jit_prefetched;   // plans whose groups were submitted to the JIT
  int num_sms = 148;
  uint64_t* mig_status = nullptr;   // G2P_MIGRATE look-back scratch
  uint64_t mig_tiles = 0;
  uint32_t* mig_ctl = nullptr;
  uint32_t* mig_holes = nullptr;    // MIGRATE_COMPACT hole list ([0] count) + tail marks
  uint32_t* mig_tail = nullptr;
  uint64_t mig_hole_cap = 0;
  // flag-chained JACOBI sweeps (kernels_flow.cu): per tree one completion flag
  // per half block of the leaf pool, one epoch / done counter pair per grid
  std::vector<uint32_t*> flow_flags;
  uint32_t* flow_ctl = nullptr;
  std::vector<sg::T2Buffers> t2_bufs;   // 2-sweep chain scratch per tree
  // particle bins (binned MPM kernels) + a one-entry cache keyed by the
  // position array, its write epoch, the tree and the range
  DBins bins{};
  int64_t bin_cap = 0;                 // per-particle scratch (rank, key) capacity
  uint32_t bin_keys_cap = 0;           // per-key scratch (hist, tsum) capacity
  // binnings of the current flush window, one slot each (perm, off, bins,
  // nbins), assigned in the order the window first needs them -- so a
  // replayed plan reuses the same slots (CUDA-graph arguments stay valid) --
  // and found again by (array, write epoch, range, geometry): C4's backward
  // pass reuses every substep's forward binning
  struct BinSlot {
    bool valid = false;
    int xa = -1, nb[3] = {0, 0, 0};
    uint64_t epoch = 0;
    int64_t n = 0, cap = 0;
    const int32_t* dcount = nullptr;
    float inv_dx = 0.0f;
    uint32_t kcap = 0;
    uint32_t *perm = nullptr, *off = nullptr, *bins = nullptr, *nbins = nullptr;
  };
  std::vector<BinSlot> bin_slots;
  int bin_next = 0;                    // next slot of this window
  uint64_t bin_gen = 0;                // bumped by every (re)allocation: CUDA-graph signature
  DBins bins_cur{};                    // the binning the current launch uses
  bool no_bin = false;                 // SG_NO_BIN=1: per-particle kernels (A/B measurements)
  std::vector<uint64_t> arr_epoch;     // bumped by every launched task that writes the array
  // launch profiling (benchmarks): event pairs per launch group
  bool profiling = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t get_event() {
    if (!event_pool.empty()) { cudaEvent_t e = event_pool.back(); event_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }

  void* dev_alloc(size_t bytes) {
    if (bytes == 0) bytes = 4;
    void* p = nullptr;
    if (opts.alloc) p = opts.alloc(opts.alloc_ctx, bytes, (void*)user_stream);
    else if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
    if (p) allocs.push_back(p);
    return p;
  }
  ~sg_grid() {
    for (auto& p : prof_pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
    for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
    for (void* p : allocs) {
      if (opts.free) opts.free(opts.alloc_ctx, p, (void*)stream);
      else cudaFree(p);
    }
  }
};


// dist.cu
int sg_dist_launch(sg_grid* g, int op, int kind, int task);
void sg_dist_destroy(sg_grid* g);
void sg_internal_set_error(const char* msg);
