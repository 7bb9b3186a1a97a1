/* sg.h -- C-ABI of the B200 sparse-grid task engine (libsg.so).
 *
 * The boundary of the hot path that AsyncTaichi (arXiv 2012.08141) optimizes:
 * sparse-grid task execution over an SNode hierarchy (root -> pointer ->
 * bitmasked -> dense -> place).  Calls follow the paper's statement of the
 * problem: tasks are queued and nothing runs until a synchronization point
 * (section 7.1 "We store all tasks into a queue until
 * synchronization"), where the whole queue is optimized by the state-flow-graph
 * passes (section 6) and launched.  The optimization is
 * transparent: results equal eager execution (PAPER.md:97, PAPER.md:250
 * "Order independency").
 *
 * Conventions (every entry point):
 *   - Return SG_OK (0) or a negative sg_status; sg_last_error() gives a
 *     thread-local message for the last failure on the calling thread.
 *   - sg_grid is opaque, single-owner and not thread-safe.
 *   - Device pointers passed in (coordinates, particle arrays) are BORROWED:
 *     they must stay valid and unmodified until the flush that consumes them
 *     has completed on the grid's stream (ordinary stream ordering).
 *   - Host pointers are only read/written during the call.
 *   - Enqueue calls (sg_activate, sg_listgen, sg_struct_for, sg_clear) do no
 *     device work.  sg_flush plans and enqueues kernels on the grid's stream and
 *     returns without synchronizing.  Exports flush, then synchronize.
 *   - Device-detected errors (pool exhausted, list overflow, demotion trap in
 *     debug builds) are latched in a device error word and reported by the next
 *     sg_sync / export; after one, the grid state is undefined until
 *     sg_destroy.
 *   - Layout: every field's payload is stored SoA in 4-byte elements (f32 or
 *     i32) inside leaf containers, each leaf block contiguous.
 */
#ifndef SG_H_
#define SG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t sg_status;
enum {
  SG_OK = 0,
  SG_ERR_ARG = -1,             /* bad argument / unknown id / wrong operand count */
  SG_ERR_LAYOUT = -2,          /* invalid SNode tree */
  SG_ERR_RANGE = -3,           /* coordinate outside the field's bounding shape */
  SG_ERR_CUDA = -4,            /* CUDA runtime failure */
  SG_ERR_NCCL = -5,            /* collective failure (multi-GPU) */
  SG_ERR_DEMOTION_TRAP = -6,   /* debug: non-activating write to an inactive cell */
  SG_ERR_OVERFLOW = -7,        /* reserved */
  SG_ERR_POOL_EXHAUSTED = -8,  /* device: pointer pool has no free container */
  SG_ERR_LIST_OVERFLOW = -9,   /* device: element list exceeded its capacity */
  SG_ERR_STATE = -10,          /* call not valid in this state (e.g. plan-only grid) */
  SG_ERR_TIMEOUT = -11         /* device: a neighbour rank's exchange signal never arrived */
};

/* --- SNode tree (Fig. 2 caption; section 4) ---------- */
enum { SG_ROOT = 0, SG_DENSE = 1, SG_BITMASKED = 2, SG_POINTER = 3, SG_PLACE = 4 };
enum { SG_F32 = 0, SG_I32 = 1 };

/* One row per node.  Row 0 is the root (parent -1).  Each structural child of
 * the root starts a chain ("tree") of levels; every level of a chain has the
 * same ndim (1..3) and power-of-two extents (1 on unused axes); places (fields)
 * hang only from the last level of a chain, which must be dense or bitmasked;
 * a place directly under the root is a 0-D scalar field.  Field ids are the
 * order of place rows.  snode ids are row indices. */
typedef struct {
  int32_t kind;       /* SG_ROOT / SG_DENSE / SG_BITMASKED / SG_POINTER / SG_PLACE */
  int32_t parent;     /* row index of the parent, -1 for the root */
  int32_t ndim;       /* number of axes of the chain (0 for 0-D places) */
  int32_t extent[3];  /* per-axis extent of this level (power of two) */
  int32_t dtype;      /* SG_PLACE only: SG_F32 or SG_I32 */
} sg_snode_desc;

/* Device memory callbacks (e.g. torch's caching allocator).  NULL -> cudaMalloc. */
typedef void* (*sg_alloc_fn)(void* ctx, size_t bytes, void* stream);
typedef void (*sg_free_fn)(void* ctx, void* ptr, void* stream);

typedef struct {
  int32_t device;          /* CUDA device ordinal */
  int32_t debug;           /* 1: device checks (demotion trap, range) */
  int32_t plan_only;       /* 1: no device at all; sg_flush plans and counts only */
  int32_t lowering;        /* 0: folded (no clear-list tasks); 1: paper-faithful
                              clear-list + listgen per sparse level */
  void* stream;            /* cudaStream_t the grid launches on (borrowed); NULL = default */
  sg_alloc_fn alloc;
  sg_free_fn free;
  void* alloc_ctx;
  int64_t pool_capacity;   /* max containers per pointer level; 0 = every pointer cell */
  int64_t list_capacity;   /* max entries of any element list; 0 = derived from pools */
  /* multi-GPU exchange buffers (sg_dist_init), in 4-byte words per buffer
   * including a 4-word header (word 0 = record count): halo buffers (kinds 0, 1)
   * and particle-migration buffers (kind 2); 0 = 4 + 1 Mi words */
  int64_t dist_halo_words;
  int64_t dist_part_words;
} sg_opts;

typedef struct sg_grid sg_grid;

/* Validates the tree (power-of-two extents, places only at
 * leaves, one ndim per chain), derives the container layout (PAPER.md:148
 * Fig. 2, "dense, bitmasked, pointer") and allocates: per pointer
 * level a pool of containers (zeroed: the zero-on-free reading of PAPER.md:157
 * "zero-fill the initial data"), per sparse level a list buffer with a
 * device-side count (PAPER.md:143 element lists), and the device error word.
 * The memory allocator is a state of the program ("Allocator").
 * nodes: n host rows (read during the call).  *out receives the grid; on error
 * *out = NULL and nothing is allocated.  Errors: SG_ERR_LAYOUT (invalid tree,
 * sg_last_error says which rule), SG_ERR_CUDA (allocation). */
sg_status sg_create(const sg_snode_desc* nodes, int32_t n, const sg_opts* opts, sg_grid** out);
/* Waits for the grid's stream and frees everything the grid allocated (pools,
 * lists, cached plans and CUDA graphs, exchange buffers; mapped peer buffers
 * are unmapped) -- the end of the program's lifetime of the SNode tree and its
 * allocator states.  Borrowed buffers are not touched.  NULL
 * is a no-op. */
sg_status sg_destroy(sg_grid* g);

/* Registers an external SoA particle array (ncomp components of n elements,
 * component c at dev_ptr + c*n, 4-byte elements, device memory, borrowed) as a
 * Value state usable by range-for ops ("Value" states of the
 * state-flow graph; particles are range-for operands, PAPER.md:444 MPM).
 * *id receives the array id.  Errors: SG_ERR_ARG. */
sg_status sg_register_array(sg_grid* g, void* dev_ptr, int64_t n, int32_t dtype, int32_t ncomp, int32_t* id);
/* Gives array `id` a device-resident element count (int32 at dev_count,
 * borrowed; <= the registered n, which becomes the capacity).  Range-for tasks
 * with range_n < 0 iterate [0, *dev_count of arrays[0]) read on the device, and
 * the migration / halo ops (below) update it on the device (a range-for over a
 * range known only on the device: "no host round trip until an
 * output is needed"). */
sg_status sg_set_array_count(sg_grid* g, int32_t id, int32_t* dev_count);

/* --- task vocabulary --------------------------------------------------------- */
enum { SG_TASK_STRUCT_FOR = 0, SG_TASK_RANGE_FOR = 1, SG_TASK_SERIAL = 2 };

/* Ops.  Operand roles by slot (fields[i]); params p[i].  Access patterns are
 * what the planner's fusion/demotion rules read.
 *   FILL        struct-for  f0[c] = p0                        f0 identity, complete
 *   ADD_CONST   struct-for  f0[c] = f1[c] + p0                 chain_copy
 *   INC         struct-for  f0[c] += p0                        increments
 *   AXPY        struct-for  f0[c] = p0*f1[c] + f2[c]           sparse_saxpy
 *   STENCIL     struct-for  f0[c] = sum_nbr f1 - 2D f1[c]      f1 neighbour access
 *   JACOBI      struct-for  f0[c] = (f2[c] + sum_nbr f1)/(2D)  f1 neighbour access
 *   REDUCE_SUM  struct-for  f0[] += f1[c]                      f0 0-D
 *   DOWNSAMPLE  struct-for  f0[c//2] += p0*f1[c] + p1          PAPER.md:350, Fig. 3
 *   JITTER      struct-for  f0[c] += f0[c+e0] for even c0      deep_hierarchy
 *   CLEAR_SCALAR serial     f0[] = 0
 *   P2G / GRID_OP / G2P     MLS-MPM transfer ops
 *   ARRAY_COUNT  serial     *count(a0) = p0
 *   HALO_PACK    struct-for blocks with origin x in [p0, p1) appended to buffer a0
 *                           (record: 4-word header {org0,org1,org2,0} + f0..f(nf-1) payload;
 *                           p2 = capacity in records; count = a0's device count)
 *   HALO_UNPACK  range-for  n = capacity*cells-per-block: record cells of a0 added
 *                           (p0 = 0) or stored (p0 = 1) into f0..; activating
 *   G2P_MIGRATE  range-for  G2P over a0..a3 (x,v,C,J) + a4 (id) with device count, then
 *                           stable in-place compaction of the particles whose cell x stays
 *                           in [p2, p3); leavers appended to a5 (x < p2) / a6 (x >= p3)
 *   MIGRATE_COMPACT range-for on a0..a3 (x,v,C,J) + a4 (id) with device count: the
 *                           particles whose cell x (p1 inv_dx) left [p2, p3) are packed
 *                           into a5 (x < p2) / a6 (x >= p3) and their slots refilled from
 *                           the tail (hole filling: the order changes, O(leavers) moves)
 *   MIGRATE_APPEND range-for particles of buffers a5, a6 appended to a0..a4
 *   G2P out of place with p2 != 0: the new state is written in the BIN ORDER of
 *                           the input positions (the particle the binned kernel visits
 *                           j-th goes to index j): a permutation of the particles (the
 *                           paper fixes no particle order), which keeps the next step's
 *                           binned kernels' particle reads sequential.  Pair it with:
 *   PERMUTE      range-for  a2[c][j] = a1[c][perm(j)] for every component, perm = the
 *                           bin order of positions a0 (the same binning as G2P), f0 any
 *                           field of the grid tree, p1 inv_dx (moves ids along)
 * Differentiable MPM (C4; "kernels and their gradients", the
 * global fields / particle states serve as checkpoints):
 *   G2P with arrays a4..a7 set: reads state a0..a3, writes the new state to
 *                           a4..a7 (x, v, C, J) instead of in place
 *   LOSS_MEAN    range-for  f0[] (0-D) += p1 * sum_i a0[comp p0][i]   (deterministic
 *                           f64 tree reduction; loss = mean x with p1 = 1/n)
 *   ADJ_INIT     range-for  a0[comp p0][i] = p1; every other entry of a0..a3 = 0
 *   G2P_ADJ      range-for  adjoint of GRID_OP (folded) + G2P of one substep.
 *                           f0..f3 grid momentum / mass from P2G (read), f4..f7 their
 *                           adjoints in a second tree (scattered with atomics,
 *                           activating); a0 x_s, a1 J_s, a2..a5 adjoint of state s+1
 *                           (x, v, C, J), writes a6 = adjoint x_s, a7 = adjoint J_s;
 *                           p0 dt, p1 inv_dx, p2 gravity, p3 bound, p4 n_grid
 *   P2G_ADJ      range-for  adjoint of P2G: gathers f0..f3 (grid adjoints); a0..a3
 *                           state s; a4 adjoint x_s (+=), a5 adjoint v_s (=), a6
 *                           adjoint C_s (=), a7 adjoint J_s (+=); p0 dt, p1 inv_dx,
 *                           p2 p_mass, p3 p_vol, p4 E
 * Multigrid (SURVEY N1; PAPER.md:348-361 restriction, :438-441 MGPCG), A = -Laplacian, h = 1:
 *   SMOOTH_RB    struct-for red-black Gauss-Seidel half sweep: cells with (sum c) % 2 == p0
 *                           get f0[c] = (f1[c] + sum_nbr f0) / (2D); f0 neighbour access
 *   RESTRICT     struct-for f0[c//2] += p0 * (f1[c] - A f2[c])   f0 on the half-resolution
 *                           tree (activating, demotable like DOWNSAMPLE); f2 neighbour access
 *   PROLONG      struct-for f0[c] += f1[c//2]                    f1 on the half-resolution tree
 *   RESID_NORM2  struct-for f0[] += (f1[c] - A f2[c])^2          f0 0-D (reduction)
 * Conjugate gradients around the V-cycle (MGPCG); scalars are 0-D
 * fields read on the device, so no host round trip:
 *   DOT          struct-for f0[] += p0 * f1[c] * f2[c]            f0 0-D (reduction)
 *   AXPY_RATIO   struct-for f0[c] += p0 * (f2[] / f3[]) * f1[c]  f2, f3 0-D
 *   XPAY_RATIO   struct-for f0[c] = f1[c] + (f2[] / f3[]) * f0[c]
 *   COPY_SCALAR  serial     f0[] = f1[]                            both 0-D
 * Inactive or out-of-bound reads give 0. */
enum {
  SG_OP_FILL = 1, SG_OP_ADD_CONST = 2, SG_OP_INC = 3, SG_OP_AXPY = 4, SG_OP_STENCIL = 5,
  SG_OP_JACOBI = 6, SG_OP_REDUCE_SUM = 7, SG_OP_DOWNSAMPLE = 8, SG_OP_JITTER = 9,
  SG_OP_CLEAR_SCALAR = 10, SG_OP_ARRAY_COUNT = 11,
  SG_OP_P2G = 20, SG_OP_GRID_OP = 21, SG_OP_G2P = 22,
  SG_OP_HALO_PACK = 23, SG_OP_HALO_UNPACK = 24, SG_OP_G2P_MIGRATE = 25, SG_OP_MIGRATE_APPEND = 26,
  SG_OP_LOSS_MEAN = 27, SG_OP_ADJ_INIT = 28, SG_OP_G2P_ADJ = 29, SG_OP_P2G_ADJ = 30,
  SG_OP_SMOOTH_RB = 31, SG_OP_RESTRICT = 32, SG_OP_PROLONG = 33, SG_OP_RESID_NORM2 = 34,
  SG_OP_DOT = 35, SG_OP_AXPY_RATIO = 36, SG_OP_XPAY_RATIO = 37, SG_OP_COPY_SCALAR = 38,
  SG_OP_DIST_SIGNAL = 40, SG_OP_DIST_WAIT = 41,  /* exchange tasks (sg_dist_init) */
  SG_OP_PERMUTE = 42, SG_OP_MIGRATE_COMPACT = 43
};

typedef struct {
  int32_t kind;         /* SG_TASK_* */
  int32_t op;           /* SG_OP_* */
  int32_t snode;        /* struct-for: the LEAF level of the iterated tree */
  int32_t pad_;
  int64_t range_n;      /* range-for: loop extent */
  int32_t fields[8];    /* operand field ids, -1 = unused */
  int32_t arrays[8];    /* operand array ids (range-for), -1 = unused */
  uint32_t activating;  /* bit i: fields[i] is written with activation-on-write */
  float params[8];
} sg_task;

/* Enqueue: activate the cells at `dev_coords` (n x ndim int32, row-major,
 * device memory, borrowed) of `field`'s tree: every sparse ancestor becomes
 * active; newly active cells read 0. */
sg_status sg_activate(sg_grid* g, int32_t field, const int32_t* dev_coords, int64_t n);
/* Enqueue: generate the element lists of every sparse level from the top of
 * snode's chain down to snode. */
sg_status sg_listgen(sg_grid* g, int32_t snode);
/* Enqueue one kernel-level task (PAPER.md:138-143 struct-for over the active
 * elements of a leaf; range-for and serial tasks, "kernels are
 * decomposed into tasks").  t is read during the call; operand device buffers
 * (registered arrays) are borrowed.  Validation errors (unknown op, operand
 * count, dtype or tree mismatch) return SG_ERR_ARG at enqueue time. */
sg_status sg_struct_for(sg_grid* g, const sg_task* t);
/* Enqueue n tasks (host array, borrowed for the call) in order: the same as n
 * sg_struct_for calls, one library call (a solver loop
 * re-submitted each step).  Errors as sg_struct_for, reported for the first
 * failing task; the tasks before it stay enqueued. */
sg_status sg_struct_for_batch(sg_grid* g, const sg_task* tasks, int32_t n);

enum { SG_CLEAR_VALUES = 0, SG_DEACTIVATE = 1 };
/* Enqueue: SG_CLEAR_VALUES: target = field id, store 0 on every active cell
 *          (a complete overwrite: earlier stores become dead).
 *          SG_DEACTIVATE:   target = sparse snode id, every cell of that level
 *          and below becomes inactive, payload zeroed, pointer children freed
 *          (PAPER.md:166 deactivation, PAPER.md:200 allocator state). */
sg_status sg_clear(sg_grid* g, int32_t target, int32_t mode);

/* Pass toggles.  sg_flush replays a cached plan as a CUDA
 * graph from its second run on; when the flush window and its device pointers
 * are identical to the graph's last capture, the graph is relaunched without
 * re-capturing (one cudaGraphLaunch). */
enum {
  SG_PASS_LISTGEN_REMOVAL = 1,   /* section 6.2 */
  SG_PASS_ACT_DEMOTION = 2,      /* section 6.3 */
  SG_PASS_FUSION = 4,            /* section 6.4 */
  SG_PASS_DSE = 8,               /* section 6.5 */
  SG_PASS_ALL = 15,
  /* Beyond the paper: after the four passes, adjacent
   * struct-for groups over the same list version (with independent tasks
   * hoisted out of the way) become the phases of ONE persistent cooperative
   * launch with a grid-wide barrier between phases -- legal for the dependent
   * stencil chains the paper's rule cannot fuse.  Reported
   * separately from SG_PASS_ALL. */
  SG_PASS_CHAIN = 16
};

typedef struct {
  int64_t tasks_lowered;        /* tasks in the eager lowering of this flush */
  int64_t launches;             /* task launches of this flush (one per launch group) */
  int64_t listgen_launched;
  int64_t clear_list_launched;
  int64_t listgens_removed;
  int64_t demotions;            /* activating operands demoted (incl. removed repeats) */
  int64_t tasks_fused;          /* tasks merged into another task */
  int64_t dead_removed;         /* tasks removed by DSE */
  int64_t plan_cache_hits;
  int64_t plan_cache_misses;
  double plan_us;               /* host planning time of this flush */
  int64_t tasks_chained;        /* SG_PASS_CHAIN: struct-for groups merged into chains */
  int64_t launches_chained;     /* SG_PASS_CHAIN: cooperative chain launches */
  int64_t aux_kernels;          /* extra kernels inside task launches: particle binning for the
                                   binned MPM ops (5 per binning; a binning is reused while the
                                   positions and the bin geometry are unchanged) */
} sg_stats;

/* Optimize and launch the queue (section 7.1: the queued
 * tasks form the state-flow graph, the passes of section 6 run, the plan is
 * cached by the stream's hash like the IR bank).  passes = 0 launches one
 * kernel per lowered task in program order (the eager baseline).  Returns
 * after enqueueing (no synchronization).  observed: field ids whose final
 * values the caller will read (NULL / n_observed < 0: every field and array);
 * masks are always observed.  out may be NULL. */
sg_status sg_flush(sg_grid* g, uint32_t passes, const int32_t* observed, int32_t n_observed, sg_stats* out);
/* Synchronization point ("until synchronization"): waits for the
 * grid's stream and reports a latched device error (SG_ERR_POOL_EXHAUSTED,
 * SG_ERR_LIST_OVERFLOW, SG_ERR_DEMOTION_TRAP, SG_ERR_RANGE, SG_ERR_TIMEOUT)
 * with the launch index of the task that raised it (sg_last_error). */
sg_status sg_sync(sg_grid* g);

/* Exports (flush + sync: "anything we need to output" is a sync point,
 * PAPER.md:390).  Coordinates are level-global (row-major n x ndim, host
 * memory of cap rows; *count = the full count even when it exceeds cap).
 * The mask export is the set of active cells of a sparse level (PAPER.md:152
 * activation), the list export the element list, both compared
 * as sorted sets (reading R1/R2). */
sg_status sg_export_mask(sg_grid* g, int32_t snode, int32_t* host_coords, int64_t cap, int64_t* count);
sg_status sg_export_list(sg_grid* g, int32_t snode, int32_t* host_coords, int64_t cap, int64_t* count);
/* Dense bounding array of a field (row-major, last axis fastest, bytes = 4 x
 * cells); inactive -> 0 (PAPER.md:195 reads of inactive cells return 0). */
sg_status sg_read_field(sg_grid* g, int32_t field, void* host_dense, int64_t bytes);
/* Enqueue (no flush, no sync) the device-to-host copy of a 0-D field's 4 bytes
 * into host_dst, ordered after everything flushed so far on the grid's stream
 * (an output read without forcing a sync: PAPER.md:390).  host_dst should be
 * pinned (else the copy is synchronous); it is valid once the stream reaches
 * this point (sg_sync, or an event the caller records).  Errors: SG_ERR_ARG
 * (not a 0-D field). */
sg_status sg_read_scalar_async(sg_grid* g, int32_t field, void* host_dst);
/* State handoff (SURVEY.md s8c reading 17, sg_load_state): overwrite the
 * values of the ACTIVE cells of a field from a dense host array (inactive
 * entries ignored; masks unchanged).  Flushes and synchronizes first. */
sg_status sg_load_field(sg_grid* g, int32_t field, const void* host_dense, int64_t bytes);

/* The launch plan of the last flush (the optimized SFG's launch order,
 * PAPER.md:212-254), for host-side tests: `count` records of
 * 6 int32 {group, task_type, call_index, snode, activating, op} (op: the
 * sg_task op of struct-for / range-for / serial tasks, else 0).  task_type:
 * 0 activate, 1 listgen, 2 clear_list, 3 struct_for, 4 range_for, 5 serial,
 * 6 deactivate.  call_index = index of the enqueue call within the flush window. */
sg_status sg_last_plan(sg_grid* g, int32_t* out, int64_t cap, int64_t* count);

/* Launch profiling for benchmarks (launch counts and times are the quantities
 * PAPER.md:411-424 Table 1 reports): when on, sg_flush records a CUDA event pair
 * on the grid's stream around every launch group.  sg_profile_read waits for
 * the stream and returns, per launch kind, the summed device time (ms) and the
 * number of launches since the last read (kinds: 0 activate, 1 listgen,
 * 2 clear_list, 3 struct_for, 4 range_for, 5 serial, 6 deactivate; struct-for
 * launches are also accumulated under 100 + op of their first member, listgens
 * under 200 + snode, range-for launches under 300 + op of their first member). */
sg_status sg_set_profiling(sg_grid* g, int32_t on);
sg_status sg_profile_read(sg_grid* g, double* ms, int64_t* count, int32_t n_kinds);

/* Device pointers of the leaf payload pools (the SNode layout of PAPER.md:148),
 * for benchmarks (read-only): out[0] = number of trees, then 4 values per tree
 * (pool base, stride words, capacity, payload offset words). */
sg_status sg_device_info(sg_grid* g, int64_t* out, int32_t n);

/* JIT-specialized fusion (PAPER.md:265-266 parallel
 * compilation, PAPER.md:394-396 the IR bank): every fused struct-for group is
 * hashed by its content (ops, operand slots, activation bits, parameters,
 * block geometry, value type); worker threads compile a kernel whose op table
 * is a compile-time constant with NVRTC for sm_100a and cache it by the hash;
 * launches of that content use it once ready (the op-table interpreter runs
 * meanwhile; CUDA graphs are recaptured).  Env SG_JIT: 0 off, 1
 * asynchronous (default), 2 synchronous (first launch waits: tests and
 * benchmarks).
 * out (n <= 7 int64): [mode, kernels ready, compiling, failed, hits, misses,
 * total compile time in microseconds]. */
sg_status sg_jit_info(int64_t* out, int32_t n);
/* Process-wide JIT mode (0, 1, 2 as SG_JIT; -1 = back to the environment) of
 * the parallel compilation of PAPER.md:265-266.  Errors: SG_ERR_ARG. */
sg_status sg_jit_set_mode(int32_t mode);
/* Stops the JIT (PAPER.md:265-266 compiler threads) for the rest of the
 * process: queued compilations are dropped,
 * in-flight ones are waited for (<= 60 s), later launches use the op-table
 * interpreter.  Call before process exit while compilations may be running:
 * NVRTC's exit-time teardown under a running compile crashes the process
 * (the Python binding calls it from an atexit hook).  Always SG_OK. */
sg_status sg_jit_shutdown(void);
/* Host-side check (no GPU needed) of the specialization of PAPER.md:394-396
 * (one compiled kernel per fused task content): NVRTC-compiles, without loading, the
 * specialized kernel of a group of `nops` op codes with placeholder operands
 * (nd / gl: quad-path dimensionality and constant block geometry, i32: value
 * type); the compile log is copied into log (cap bytes).  SG_ERR_STATE when
 * NVRTC is missing or the compile fails. */
sg_status sg_jit_selftest(int32_t nd, int32_t gl, int32_t i32, const int32_t* ops, int32_t nops, char* log,
                          int64_t cap);

/* Thread-local message of the last failing call on this thread (SPEC.md:50,
 * :59, :78 error conventions). */
const char* sg_last_error(void);

/* --- multi-GPU data plane (BASELINE north_star "partitioned
 * ... into spatial slabs ... with boundary-block halo exchange"; N3 peer
 * memory over NVLink).  The paper itself is single-device.
 *
 * sg_dist_init makes the grid rank `rank` of `world` ranks partitioned along
 * `axis` (0 = x); its neighbours are rank-1 (left) and rank+1 (right).  It
 * allocates the exchange arena (sizes from sg_opts.dist_*_words), registers 12
 * arrays (send and receive buffer per exchange kind x side, each with a device
 * count in its header word; ids from sg_dist_info) and connects the
 * neighbours:
 *   nccl_uid != NULL: a 128-byte ncclUniqueId shared by every rank (the caller
 *     broadcasts it, e.g. over torch.distributed).  The library creates the
 *     NCCL communicator, exchanges IPC handles of the arenas over it and maps
 *     each neighbour's arena when the devices can access each other (NVLink /
 *     NVSwitch): the PEER transport -- packing kernels store their records and
 *     counts straight into the neighbour's receive buffer, so exactly the
 *     packed bytes move and no host ever sees a count.  Otherwise (or with
 *     SG_DIST_TRANSPORT=nccl) the NCCL transport: ncclSend/ncclRecv of whole
 *     buffers on the grid's stream.
 *   nccl_uid == NULL: no NCCL.  Either an in-process group (virtual ranks,
 *     e.g. several grids on one GPU): grids calling sg_dist_init with ranks
 *     0..world-1 in order form a group and map each other's arenas directly
 *     (peer transport) -- or, one rank per process, the caller exchanges the
 *     256-byte sg_dist_peer_info blobs over any process group (e.g. gloo) and
 *     passes all of them to sg_dist_connect (peer transport through CUDA IPC).
 * Exchange tasks (serial ops, never fused or removed by the passes):
 *   SG_OP_DIST_SIGNAL  p0 = kind: release the neighbours (their receive buffer
 *     of that kind is complete); arrays [sendL, sendR, recvL, recvR].
 *   SG_OP_DIST_WAIT    p0 = kind: wait until both neighbours signalled that kind
 *     (device-side spin, SG_ERR_TIMEOUT after 30 s); NCCL transport: the
 *     send/recv of that kind.  Same arrays.
 * Every rank must enqueue the same exchange sequence (SPMD).  Virtual ranks on
 * one stream must flush after each SIGNAL and enqueue every rank's SIGNAL of a
 * kind before any rank's WAIT of it.  Errors: SG_ERR_ARG, SG_ERR_STATE (called
 * twice), SG_ERR_NCCL, SG_ERR_CUDA. */
sg_status sg_dist_init(sg_grid* g, int32_t rank, int32_t world, const void* nccl_uid, int32_t axis);
/* The data plane of sg_dist_init.  out (n >= 16 int32):
 * [0] transport (0 none, 1 peer, 2 nccl), [1] rank,
 * [2] world, [3] axis, [4 + 2k + s] send array id of kind k side s,
 * [10 + 2k + s] receive array id (on a side without a neighbour the arrays
 * exist but nothing arrives: counts stay 0). */
sg_status sg_dist_info(sg_grid* g, int32_t* out, int32_t n);
/* ncclGetUniqueId into out (128 bytes), for rank 0 to broadcast (the NCCL
 * halo exchange of the north star).  SG_ERR_NCCL when NCCL
 * cannot be loaded. */
sg_status sg_nccl_unique_id(void* out);
/* This rank's 256-byte connection blob (IPC handle of its exchange arena,
 * PCI bus id, host, pid) after sg_dist_init(nccl_uid = NULL): the N3 peer
 * transport.  Errors: SG_ERR_STATE before sg_dist_init. */
sg_status sg_dist_peer_info(sg_grid* g, void* out);
/* Connects the neighbours from every rank's blob (world x 256 bytes, rank
 * order): maps their arenas (peer transport).  SG_ERR_CUDA
 * when a neighbour cannot be mapped (other host, same process, no peer
 * access). */
sg_status sg_dist_connect(sg_grid* g, const void* all_infos);

#ifdef __cplusplus
}
#endif
#endif /* SG_H_ */
