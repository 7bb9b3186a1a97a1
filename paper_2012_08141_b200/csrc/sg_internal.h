// sg_internal.h -- descriptors shared by the host runtime and the sm_100a kernels.
//
// Memory layout:
//   A chain of levels is cut into *segments* after every pointer level.  The
//   cells of segment 0 live in the single root container; the cells of segment
//   s>0 live in containers allocated from the pool of the pointer level that
//   ends segment s-1 ("memory allocator will automatically manage
//   sparse data structure nodes").  A container is
//       [bitmask words of every bitmasked level of the segment]
//       [u32 child slots of the pointer level ending the segment (0 = NULL,
//        0xFFFFFFFF = BUSY, else container index + 1)]
//       [leaf segment only: per-field SoA payload, 4-byte elements]
//   Within a container, level-l cells are numbered hierarchically
//   (idx_l = idx_{l-1} * |E_l| + row-major local index), so the leaf cells below
//   any cell form one contiguous run: each leaf block is contiguous per field.
//   Pools are zeroed at creation and every freed container is zeroed before
//   it is pushed back (zero-on-free): an inactive cell's payload is always 0,
//   so reads never need a mask test ("the inactive voxel has
//   value 0").
//   Element-list entries are u32 (container index << log2 cells-per-container)
//   | cell index; the container's owning pointer cell is kept in origin[].
#ifndef SG_INTERNAL_H_
#define SG_INTERNAL_H_

#include <stdint.h>
#include "../../include/sg.h"

#define SG_MAXL 6         // levels per chain
#define SG_MAXOPS 16      // ops in one fused group
#define SG_SLOT_NULL 0u
#define SG_SLOT_BUSY 0xFFFFFFFFu

struct DLevel {
  int32_t kind;        // SG_DENSE / SG_BITMASKED / SG_POINTER
  int32_t seg;         // segment holding this level's cells
  int32_t le[3];       // log2 extents
  int32_t lE;          // log2 cells per parent cell (= le0+le1+le2)
  int32_t lbelow[3];   // log2 leaf cells per cell of this level, per axis
  int32_t ln;          // log2 cells of this level per container
  uint32_t mask_off;   // bitmasked: u32-word offset of its bits in the container
  uint32_t slot_off;   // pointer: u32-word offset of its child slots
  int32_t lres[3];     // log2 level-global resolution
};

struct DSeg {
  uint32_t* base;      // container array
  uint64_t stride;     // u32 words per container
  uint32_t capacity;   // containers
  int32_t first, last; // chain positions of the first / last level in the segment
  int32_t* origin;     // [capacity*3] level-global coords of the owning pointer cell
  int32_t* alloc;      // [0] bump counter, [1] free-list top
  uint32_t* free_list; // [capacity]
  uint32_t header_words; // masks + slots (zeroed on free)
};

struct DTree {
  int32_t nd, nlev, nseg;
  int32_t driving;        // chain index of the level whose list drives struct-fors, -1: none
  int32_t lblk;           // log2 leaf cells per driving entry (a "block")
  int32_t leaf_bitmasked; // leaf level is bitmasked: bits tested per cell
  int32_t payload_off;    // u32-word offset of the payload in leaf containers
  int32_t ln_leaf;        // log2 leaf cells per leaf container
  int32_t nfields;
  uint32_t zero_blk;      // word offset (leaf pool) of a never-written all-zero container's
                          // payload: absent neighbour blocks point here, so loads need no branch
  DLevel lev[SG_MAXL];
  DSeg seg[SG_MAXL];
};

struct DField {
  int32_t tree;     // -1 for 0-D fields
  int32_t slot;     // field slot within the tree's payload
  int32_t dtype;    // SG_F32 / SG_I32
  int32_t scalar;   // 0-D: index into the scalar array
};

struct DArray {
  void* ptr;
  int64_t n;            // capacity (elements per component)
  int32_t ncomp, dtype;
  int32_t* dcount;      // device-side element count, or null (= n)
};

// Per-entry block table written by the listgen of a tree's driving level: the
// resolved leaf block and its 2*nd face neighbours, so struct-for tiles start
// with one coalesced load instead of a chain of tree walks.  Valid exactly as
// long as the list is (any mask change regenerates both).
// Offsets are u32 word offsets from the leaf segment's pool base (SG_NO_BLOCK =
// absent), so the kernels address global memory as base + offset.
#define SG_NO_BLOCK 0xFFFFFFFFu
struct BlockRow {
  uint32_t blk;        // payload of field slot 0, first cell of the block
  uint32_t maskw;      // bitmasked leaf: word offset of the block's first mask word
  uint32_t first;      // first leaf index of the block in its container
  int32_t org[3];      // leaf coords of the block origin
  uint32_t nbr[6];     // face-neighbour blocks (field slot 0, first cell)
};

// Element list of one level.
struct DList {
  uint32_t* entries;
  uint32_t* count;     // device-side count
  uint64_t* status;    // look-back tile descriptors
  uint32_t* ctl;       // [0] tile counter, [1] done counter, [2] epoch, [3] table-row ticket,
                       // [4] table_ok: rows of the current list version are built
  BlockRow* table;     // driving level only, else null (rows built by the first struct-for)
  uint32_t capacity;
  uint32_t max_tiles;
};

// One op inside a fused struct-for / range-for / serial launch.
struct DOp {
  int32_t op;
  int32_t nf;
  int32_t f[8];        // field ids
  int32_t slot[8];     // payload slot of f[i] in the loop tree (-1: other tree / 0-D)
  int32_t a[8];        // array ids
  uint32_t act;        // activating operand bits (after demotion)
  int32_t dt;          // SG_F32 / SG_I32 (uniform over the op's fields)
  int32_t scalar;      // 0-D target: index into the scalar array, else -1
  int32_t pad_;
  float p[8];
};

// Particle bins (csrc/mpm_bin.cuh): counting sort of particle ids by leaf block.
struct DBins {
  uint32_t* hist;     // [nkeys_pad] counts, zero between uses
  uint32_t* rank;     // [cap] rank of particle i within its bin
  uint32_t* key;      // [cap] bin of particle i
  uint32_t* off;      // [nkeys + 1] exclusive prefix of the counts (off[nkeys] = n)
  uint32_t* tsum;     // [2 * ntiles] per-tile (count, non-empty) sums -> prefixes
  uint32_t* bins;     // [nkeys] non-empty keys, ascending
  uint32_t* nbins;    // [1]
  uint32_t* perm;     // [cap] particle ids sorted by bin (stable within a bin: no)
  uint32_t nkeys;     // blocks in the domain + 1 (overflow)
  int nb[3];          // blocks per axis
};

struct DevCtx {
  DTree* trees;        // device array
  DField* fields;      // device array
  DArray* arrays;      // device array
  uint32_t* scalars;   // 0-D field storage
  uint32_t* err;       // [0] code (negative sg_status as u32), [1] task id
  double* partials;    // [SG_MAXOPS][max_grid] per-CTA reduction partials
  uint32_t* red_done;  // CTA ticket for the last-block reduction
  int32_t max_grid;
  int32_t debug;
};

enum { TT_ACTIVATE = 0, TT_LISTGEN = 1, TT_CLEAR_LIST = 2, TT_STRUCT_FOR = 3, TT_RANGE_FOR = 4,
       TT_SERIAL = 5, TT_DEACTIVATE = 6 };

// Host-side launchers (kernels.cu).
struct cudaStreamLaunchInfo;
namespace sg {
struct HostTree;  // forward
int launch_activate(const DevCtx& c, const DTree& t, int tree_id, int field, const int32_t* coords, int64_t n,
                    int task_id, void* stream);
int launch_listgen(const DevCtx& c, const DTree& t, int tree_id, int level, int parent_level,
                   const DList* parent, const DList& out, int task_id, void* stream, int grid_hint);
int launch_clear_list(const DList& l, void* stream);
// nphases > 1: a chain (SG_PASS_CHAIN) -- `ops` are the LAST phase's ops (reductions),
// the whole op table and the phase ends are in device memory.
int launch_struct_for(const DevCtx& c, const DTree& t, int tree_id, const DList* drive, const DOp* ops, int nops,
                      int task_id, void* stream, int grid_hint, const DOp* chain_ops, const int* chain_phase_end,
                      int nphases, int chain_needs_nbr);
// The tail of a chain (SG_PASS_CHAIN) whose phases are lone f32 JACOBI sweeps
// on 8^3 dense blocks (the last may be fused with the reduction of its
// output) runs as ONE persistent launch with per-half-block completion flags
// (kernels_flow.cu).  jacobi_flow_start: the first phase of that tail (>= 2
// phases), or -1.  flags: 2 * (leaf pool words / 512 + 1) zeroed u32; ctl: 3
// zeroed u32.
int jacobi_flow_start(const DTree& t, const DList* drive, const DOp* ops, const int* phase_end, int nph);
// Scratch of the 2-sweep (temporal) chain kernels (kernels_flow.cu): inv
// [leaf pool words / 512 + 1] u64, rows [list capacity * 54] u32, tmp [list
// capacity * 512] f32, ctl 2 zeroed u32.
struct T2Buffers {
  uint64_t* inv;
  uint32_t* rows;
  float* tmp;
  uint32_t* ctl;
};
// The chain tail [first, nph) ping-pongs between two fields with one rhs and
// has >= 4 sweeps; the launches it takes two sweeps per launch.
bool jacobi_t2_applies(const DOp* ops, const int* phase_end, int first, int nph);
int jacobi_t2_launches(int first, int nph);
// Launches the chain tail [first, nph) two sweeps per launch; returns the
// launch count, 0 when the chain does not have the ping-pong shape, or a
// negative sg_status.
int launch_jacobi_t2(const DevCtx& c, const DTree& t, const DList* drive, const DOp* ops, const int* phase_end,
                     int first, int nph, const T2Buffers& bf, int task_id, void* stream);
int launch_jacobi_flow(const DevCtx& c, const DTree& t, const DList* drive, const DOp* ops, const int* phase_end,
                       int first, int nph, uint32_t* flags, uint32_t* ctl, int task_id, void* stream);
struct RangeScratch {
  uint64_t* status;   // look-back descriptors for G2P_MIGRATE tiles
  uint32_t* ctl;      // [0..3] migrate tile/done/epoch/count, [5] append ticket
  uint32_t* holes;    // MIGRATE_COMPACT: [0] hole count, then hole indices
  uint32_t* tail;     // MIGRATE_COMPACT: per-tail-position hole marks
  uint64_t hole_cap;  // capacity of holes / tail (entries)
};
int launch_range_for(const DevCtx& c, int64_t n, const int32_t* dcount, const DOp* ops, int nops, int task_id,
                     void* stream, const RangeScratch* rs, const DTree* grid_tree, const DTree* tree2,
                     const DBins* bins);
// Bin the particles of position array x (3 comps, component stride xs) by the
// leaf blocks of a tree with 4^3 blocks (nb blocks per axis).
constexpr int BIN_KERNELS = 5;   // kernels one launch_bin issues (count, tiles, top, apply, scatter)
int launch_bin(const DBins& b, const float* x, int64_t xs, int64_t n, const int32_t* dcount, float inv_dx,
               void* stream);
uint32_t bin_ntiles(uint32_t nkeys);
int launch_serial(const DevCtx& c, const DOp* ops, int nops, int task_id, void* stream);
int launch_deactivate(const DevCtx& c, const DTree& t, int tree_id, int level, const DList* lists,
                      int task_id, void* stream);
int launch_deactivate_reset(const DTree& t, void* stream);
int launch_read_field(const DevCtx& c, const DTree& t, int tree_id, int slot, uint32_t* dense, void* stream);
int launch_load_field(const DevCtx& c, const DTree& t, int tree_id, int slot, const uint32_t* dense, void* stream);
int launch_mask_scan(const DevCtx& c, const DTree& t, int tree_id, int level, uint8_t* flags, void* stream);
int launch_list_decode(const DTree& t, int level, const DList& l, int32_t* coords, void* stream);
int launch_pool_init(uint32_t* base, uint64_t words, void* stream);
}  // namespace sg

#endif  // SG_INTERNAL_H_
