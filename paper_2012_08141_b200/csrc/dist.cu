// dist.cu -- the multi-GPU data plane of libsg (sg_dist_init; SURVEY.md s8e,
// N3 "NVLink-native halo").
//
// Every rank owns an x-slab of the grid (the partition arithmetic is the
// caller's; the library moves the bytes).  An exchange of kind k (0 halo
// reduce, 1 halo fill, 2 particle migration) goes from each rank's send
// buffers to its neighbours' receive buffers.  Two transports:
//
//   PEER  the send arrays ARE the neighbours' receive buffers, mapped into this
//         process (CUDA IPC of the neighbour's arena over NVLink / NVSwitch, or
//         the same allocation for virtual ranks in one process).  The packing
//         kernels (HALO_PACK, G2P_MIGRATE) store records and bump counts
//         straight into the neighbour's memory: exactly the packed bytes move
//         and no count ever reaches a host.  SG_OP_DIST_SIGNAL publishes an
//         epoch into each neighbour's flag word (release, system scope);
//         SG_OP_DIST_WAIT spins on its own flags (acquire) -- both device-side,
//         so a flush with exchanges is one CUDA-graph launch.
//   NCCL  send arrays are local; SG_OP_DIST_WAIT runs ncclSend / ncclRecv of the
//         whole buffers (header word = count) on the grid's stream.
//
// Buffer reuse needs no double-buffering: the three kinds use separate
// buffers, and a rank repacks a kind only after it waited for the neighbour's
// signal of a LATER kind, which the neighbour sends after consuming this one
// (stream order on the neighbour).  Epochs live on the device (graph replay
// safe); flags only grow.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "grid.h"

// --- NCCL, loaded lazily (libsg must load on hosts without a GPU or NCCL) -----
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
enum { NCCL_INT8 = 0, NCCL_UINT8 = 1, NCCL_INT32 = 2, NCCL_UINT32 = 3 };
enum { NCCL_MIN = 3 };

struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  int (*getUniqueId)(nccl_uid_t*) = nullptr;
  int (*commInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  int (*commDestroy)(nccl_comm_t) = nullptr;
  int (*send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*allGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*errStr)(int) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi A;
  if (A.tried) return A;
  A.tried = true;
  // the NCCL torch loaded (same soname) when present, else the loader's search path
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { A.why = std::string("dlopen libnccl.so.2: ") + dlerror(); return A; }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  A.getUniqueId = (int (*)(nccl_uid_t*))sym("ncclGetUniqueId");
  A.commInitRank = (int (*)(nccl_comm_t*, int, nccl_uid_t, int))sym("ncclCommInitRank");
  A.commDestroy = (int (*)(nccl_comm_t))sym("ncclCommDestroy");
  A.send = (int (*)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclSend");
  A.recv = (int (*)(void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclRecv");
  A.groupStart = (int (*)())sym("ncclGroupStart");
  A.groupEnd = (int (*)())sym("ncclGroupEnd");
  A.allGather = (int (*)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t))sym("ncclAllGather");
  A.allReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclAllReduce");
  A.errStr = (const char* (*)(int))sym("ncclGetErrorString");
  A.ok = A.getUniqueId && A.commInitRank && A.commDestroy && A.send && A.recv && A.groupStart && A.groupEnd &&
         A.allGather && A.allReduce;
  if (!A.ok) A.why = "libnccl.so.2 lacks a needed symbol";
  return A;
}

// sg_api.cu owns the thread-local error slot behind sg_last_error
void sg_internal_set_error(const char* msg);
static sg_status dfail(sg_status code, const std::string& msg) {
  sg_internal_set_error(msg.c_str());
  return code;
}

#define DCUDA(x)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return dfail(SG_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

// --- device side ---------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bumps the local epoch of this kind and publishes it to the neighbours.
__global__ void k_dist_signal(uint64_t* epoch, uint64_t* peer_flag0, uint64_t* peer_flag1) {
  if (threadIdx.x != 0) return;
  const uint64_t e = *epoch + 1;
  *epoch = e;
  __threadfence_system();   // every earlier write of this stream (the packing kernels') before the flags
  if (peer_flag0) st_release_sys(peer_flag0, e);
  if (peer_flag1) st_release_sys(peer_flag1, e);
}

// Waits until the neighbours published this kind's current epoch.
__global__ void k_dist_wait(const uint64_t* epoch, const uint64_t* flag0, const uint64_t* flag1, uint32_t* err,
                            int task) {
  if (threadIdx.x != 0) return;
  const uint64_t e = *epoch;
  const uint64_t t0 = globaltimer();
  const uint64_t* f[2] = {flag0, flag1};
  for (int s = 0; s < 2; s++) {
    if (!f[s]) continue;
    while (ld_acquire_sys(f[s]) < e) {
      if (globaltimer() - t0 > 30ull * 1000 * 1000 * 1000) {
        if (atomicCAS(err, 0u, (uint32_t)SG_ERR_TIMEOUT) == 0u) err[1] = (uint32_t)task;
        return;
      }
      __nanosleep(200);
    }
  }
  __threadfence_system();
}

// --- host side -------------------------------------------------------------------
namespace {
enum { CTRL_FLAG = 0, CTRL_EPOCH = 16 };
inline uint64_t* flag_ptr(uint32_t* arena, int kind, int side) { return (uint64_t*)(arena + CTRL_FLAG) + 2 * kind + side; }
inline uint64_t* epoch_ptr(uint32_t* arena, int kind) { return (uint64_t*)(arena + CTRL_EPOCH) + kind; }

struct PeerInfo {
  cudaIpcMemHandle_t handle;
  char busid[32];
  uint64_t host;
  int32_t pid;
  int32_t ok;
  char pad[256 - sizeof(cudaIpcMemHandle_t) - 32 - 8 - 8];
};
static_assert(sizeof(PeerInfo) == 256, "PeerInfo is 256 bytes");

uint64_t host_hash() {
  char h[256] = {0};
  gethostname(h, sizeof(h) - 1);
  uint64_t v = 1469598103934665603ull;
  for (const char* p = h; *p; p++) { v ^= (uint8_t)*p; v *= 1099511628211ull; }
  return v;
}

std::vector<sg_grid*>& pending_group() {
  static std::vector<sg_grid*> v;
  return v;
}
int next_group_id() {
  static int n = 0;
  return ++n;
}
}  // namespace

extern "C" sg_status sg_register_array(sg_grid* g, void* ptr, int64_t n, int32_t dtype, int32_t ncomp, int32_t* id);
extern "C" sg_status sg_set_array_count(sg_grid* g, int32_t id, int32_t* dev_count);

// Allocates the arena and the local send buffers, registers the receive arrays.
static sg_status dist_alloc(sg_grid* g) {
  DistState& D = g->dist;
  const int64_t hw = g->opts.dist_halo_words > 4 ? g->opts.dist_halo_words : 4 + (1ll << 20);
  const int64_t pw = g->opts.dist_part_words > 4 ? g->opts.dist_part_words : 4 + (1ll << 20);
  D.words[0] = D.words[1] = (hw + 31) & ~31ll;
  D.words[2] = (pw + 31) & ~31ll;
  size_t off = DIST_CTRL_WORDS;
  for (int k = 0; k < DIST_KINDS; k++)
    for (int s = 0; s < 2; s++) { D.recv_off[k][s] = off; off += (size_t)D.words[k]; }
  D.arena_words = off;
  if (!g->plan_only) {
    DCUDA(cudaMalloc(&D.arena, D.arena_words * 4));   // not the caching allocator: IPC-shareable
    DCUDA(cudaMemsetAsync(D.arena, 0, D.arena_words * 4, g->stream));
    for (int k = 0; k < DIST_KINDS; k++)
      for (int s = 0; s < 2; s++) {
        D.send_local[k][s] = (uint32_t*)g->dev_alloc((size_t)D.words[k] * 4);
        if (!D.send_local[k][s]) return dfail(SG_ERR_CUDA, "exchange buffer allocation failed");
        DCUDA(cudaMemsetAsync(D.send_local[k][s], 0, (size_t)D.words[k] * 4, g->stream));
      }
  }
  for (int k = 0; k < DIST_KINDS; k++)
    for (int s = 0; s < 2; s++) {
      int32_t id = -1;
      uint32_t* base = D.arena ? D.arena + D.recv_off[k][s] : nullptr;
      sg_status rc = sg_register_array(g, base ? base + 4 : nullptr, D.words[k] - 4, SG_I32, 1, &id);
      if (rc) return rc;
      if (base && (rc = sg_set_array_count(g, id, (int32_t*)base))) return rc;
      D.ids_recv[k][s] = id;
    }
  return SG_OK;
}

// Registers the send arrays once the neighbours are known.  Peer transport:
// a send array is the neighbour's receive buffer of the opposite side.
static sg_status dist_register_sends(sg_grid* g) {
  DistState& D = g->dist;
  for (int k = 0; k < DIST_KINDS; k++)
    for (int s = 0; s < 2; s++) {
      uint32_t* base = D.send_local[k][s];
      if (D.transport == DIST_PEER && D.has_nb[s] && D.peer_arena[s]) base = D.peer_arena[s] + D.recv_off[k][1 - s];
      int32_t id = -1;
      sg_status rc = sg_register_array(g, base ? base + 4 : nullptr, D.words[k] - 4, SG_I32, 1, &id);
      if (rc) return rc;
      if (base && (rc = sg_set_array_count(g, id, (int32_t*)base))) return rc;
      D.ids_send[k][s] = id;
      if ((int)g->L.seq_arrays.size() <= id) g->L.seq_arrays.resize(id + 1, 0);
      g->L.seq_arrays[id] = 1;
    }
  return SG_OK;
}

// Maps the arenas of the neighbours (peer transport) from their 256-byte
// PeerInfo blobs.  Returns false (nothing mapped) when a neighbour is on
// another host, in this process, or on a device this one cannot access.
static bool map_neighbours(sg_grid* g, const PeerInfo* all, const PeerInfo& mine) {
  DistState& D = g->dist;
  for (int s = 0; s < 2; s++) {
    if (!D.has_nb[s]) continue;
    const PeerInfo& p = all[s == 0 ? D.rank - 1 : D.rank + 1];
    int dev = -1, can = 0;
    bool ok = p.host == mine.host && p.pid != mine.pid && cudaDeviceGetByPCIBusId(&dev, p.busid) == cudaSuccess;
    if (ok && dev != g->opts.device) ok = cudaDeviceCanAccessPeer(&can, g->opts.device, dev) == cudaSuccess && can;
    void* ptr = nullptr;
    if (ok) ok = cudaIpcOpenMemHandle(&ptr, p.handle, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      for (int t = 0; t < s; t++)
        if (D.peer_ipc[t]) { cudaIpcCloseMemHandle(D.peer_arena[t]); D.peer_ipc[t] = false; D.peer_arena[t] = nullptr; }
      return false;
    }
    D.peer_arena[s] = (uint32_t*)ptr;
    D.peer_ipc[s] = true;
  }
  return true;
}

static sg_status local_info(sg_grid* g, PeerInfo& mine) {
  std::memset(&mine, 0, sizeof(mine));
  DCUDA(cudaIpcGetMemHandle(&mine.handle, g->dist.arena));
  DCUDA(cudaDeviceGetPCIBusId(mine.busid, sizeof(mine.busid), g->opts.device));
  mine.host = host_hash();
  mine.pid = (int32_t)getpid();
  return SG_OK;
}

static sg_status dist_connect_nccl(sg_grid* g, const void* uid) {
  DistState& D = g->dist;
  NcclApi& N = nccl();
  if (!N.ok) return dfail(SG_ERR_NCCL, "NCCL unavailable: " + N.why);
  nccl_uid_t id;
  std::memcpy(&id, uid, sizeof(id));
  nccl_comm_t comm = nullptr;
  int r = N.commInitRank(&comm, D.world, id, D.rank);
  if (r) return dfail(SG_ERR_NCCL, std::string("ncclCommInitRank: ") + (N.errStr ? N.errStr(r) : "error"));
  D.comm = comm;
  // peer discovery: every rank's arena handle, device and host, over NCCL
  PeerInfo mine;
  sg_status rc = local_info(g, mine);
  if (rc) return rc;
  std::vector<PeerInfo> all(D.world);
  void* dbuf = nullptr;
  DCUDA(cudaMalloc(&dbuf, sizeof(PeerInfo) * (D.world + 1) + 8));
  char* dall = (char*)dbuf + sizeof(PeerInfo);
  DCUDA(cudaMemcpyAsync(dbuf, &mine, sizeof(mine), cudaMemcpyHostToDevice, g->stream));
  r = N.allGather(dbuf, dall, sizeof(PeerInfo), NCCL_UINT8, comm, g->stream);
  if (!r) {
    cudaMemcpyAsync(all.data(), dall, sizeof(PeerInfo) * D.world, cudaMemcpyDeviceToHost, g->stream);
    cudaStreamSynchronize(g->stream);
  }
  const char* force = std::getenv("SG_DIST_TRANSPORT");
  const bool want_peer = !(force && std::strcmp(force, "nccl") == 0);
  int ok = !r && want_peer && map_neighbours(g, all.data(), mine) ? 1 : 0;
  // one transport for every rank: peer only if every rank mapped its neighbours
  int32_t* dok = (int32_t*)((char*)dbuf + sizeof(PeerInfo) * (D.world + 1));
  int32_t all_ok = 0;
  DCUDA(cudaMemcpyAsync(dok, &ok, 4, cudaMemcpyHostToDevice, g->stream));
  r = N.allReduce(dok, dok, 1, NCCL_INT32, NCCL_MIN, comm, g->stream);
  DCUDA(cudaMemcpyAsync(&all_ok, dok, 4, cudaMemcpyDeviceToHost, g->stream));
  DCUDA(cudaStreamSynchronize(g->stream));
  cudaFree(dbuf);
  if (r) return dfail(SG_ERR_NCCL, "ncclAllReduce (transport agreement) failed");
  D.transport = all_ok ? DIST_PEER : DIST_NCCL;
  if (D.transport == DIST_NCCL)
    for (int s = 0; s < 2; s++)
      if (D.peer_ipc[s]) { cudaIpcCloseMemHandle(D.peer_arena[s]); D.peer_ipc[s] = false; D.peer_arena[s] = nullptr; }
  return dist_register_sends(g);
}

// In-process group: once the grids of ranks 0..world-1 have all called
// sg_dist_init (nccl_uid = NULL) in this process, they map each other's arenas.
static sg_status dist_join_local(sg_grid* g) {
  std::vector<sg_grid*>& P = pending_group();
  DistState& D = g->dist;
  if (D.rank == 0 || P.empty() || P[0]->dist.world != D.world || (int)P.size() != D.rank) P.clear();
  if ((int)P.size() != D.rank) return SG_OK;   // not (yet) an in-process group: sg_dist_connect may follow
  D.group = D.rank == 0 ? next_group_id() : P[0]->dist.group;
  P.push_back(g);
  if ((int)P.size() < D.world) return SG_OK;
  for (int r = 0; r < D.world; r++) {
    sg_grid* h = P[r];
    DistState& H = h->dist;
    H.transport = DIST_PEER;
    for (int s = 0; s < 2; s++) {
      if (!H.has_nb[s]) continue;
      sg_grid* nb = P[s == 0 ? r - 1 : r + 1];
      if (nb->dist.words[0] != H.words[0] || nb->dist.words[2] != H.words[2])
        return dfail(SG_ERR_ARG, "in-process group: exchange buffer sizes differ between ranks");
      H.peer_arena[s] = nb->dist.arena;
      if (!h->plan_only && nb->opts.device != h->opts.device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, h->opts.device, nb->opts.device);
        if (!can) return dfail(SG_ERR_CUDA, "in-process group: devices cannot access each other");
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(h->opts.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(nb->opts.device, 0);
        cudaGetLastError();
        cudaSetDevice(prev);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return dfail(SG_ERR_CUDA, "cudaDeviceEnablePeerAccess failed");
      }
    }
    sg_status rc = dist_register_sends(h);
    if (rc) return rc;
  }
  P.clear();
  return SG_OK;
}

extern "C" sg_status sg_dist_peer_info(sg_grid* g, void* out) {
  if (!g || !out) return dfail(SG_ERR_ARG, "null argument");
  if (!g->dist.on || g->plan_only) return dfail(SG_ERR_STATE, "sg_dist_peer_info needs sg_dist_init on a device grid");
  PeerInfo mine;
  sg_status rc = local_info(g, mine);
  if (rc) return rc;
  std::memcpy(out, &mine, sizeof(mine));
  return SG_OK;
}

extern "C" sg_status sg_dist_connect(sg_grid* g, const void* infos) {
  if (!g || !infos) return dfail(SG_ERR_ARG, "null argument");
  DistState& D = g->dist;
  if (!D.on || g->plan_only) return dfail(SG_ERR_STATE, "sg_dist_connect needs sg_dist_init on a device grid");
  if (D.transport != DIST_NONE) return dfail(SG_ERR_STATE, "grid already connected");
  std::vector<sg_grid*>& P = pending_group();
  for (size_t i = 0; i < P.size(); i++)
    if (P[i] == g) { P.clear(); break; }
  PeerInfo mine;
  sg_status rc = local_info(g, mine);
  if (rc) return rc;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(g->opts.device);
  const bool ok = map_neighbours(g, (const PeerInfo*)infos, mine);
  cudaSetDevice(prev);
  if (!ok) return dfail(SG_ERR_CUDA, "sg_dist_connect: a neighbour's exchange arena cannot be mapped "
                                     "(other host, same process, or no peer access): use the NCCL transport");
  D.transport = DIST_PEER;
  return dist_register_sends(g);
}

extern "C" sg_status sg_dist_init(sg_grid* g, int32_t rank, int32_t world, const void* nccl_uid, int32_t axis) {
  if (!g) return dfail(SG_ERR_ARG, "null grid");
  if (g->dist.on) return dfail(SG_ERR_STATE, "sg_dist_init called twice");
  if (world < 1 || rank < 0 || rank >= world || axis < 0 || axis > 2) return dfail(SG_ERR_ARG, "bad rank / world / axis");
  DistState& D = g->dist;
  D.on = true;
  D.rank = rank; D.world = world; D.axis = axis;
  D.has_nb[0] = rank > 0;
  D.has_nb[1] = rank < world - 1;
  int prev = -1;
  if (!g->plan_only) { cudaGetDevice(&prev); cudaSetDevice(g->opts.device); }
  sg_status rc = dist_alloc(g);
  if (!rc) {
    if (world == 1) { D.transport = DIST_PEER; rc = dist_register_sends(g); }
    else if (nccl_uid && !g->plan_only) rc = dist_connect_nccl(g, nccl_uid);
    else if (nccl_uid) { D.transport = DIST_NCCL; rc = dist_register_sends(g); }   // plan-only: ids only
    else rc = dist_join_local(g);
  }
  if (!g->plan_only && !rc) {
    cudaError_t e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) rc = dfail(SG_ERR_CUDA, std::string("sg_dist_init: ") + cudaGetErrorString(e));
  }
  if (prev >= 0) cudaSetDevice(prev);
  return rc;
}

extern "C" sg_status sg_dist_info(sg_grid* g, int32_t* out, int32_t n) {
  if (!g || !out || n < 16) return dfail(SG_ERR_ARG, "sg_dist_info needs 16 ints");
  const DistState& D = g->dist;
  out[0] = D.transport; out[1] = D.rank; out[2] = D.world; out[3] = D.axis;
  for (int k = 0; k < DIST_KINDS; k++)
    for (int s = 0; s < 2; s++) {
      out[4 + 2 * k + s] = D.ids_send[k][s];
      out[10 + 2 * k + s] = D.ids_recv[k][s];
    }
  return SG_OK;
}

extern "C" sg_status sg_nccl_unique_id(void* out) {
  if (!out) return dfail(SG_ERR_ARG, "null output");
  NcclApi& N = nccl();
  if (!N.ok) return dfail(SG_ERR_NCCL, "NCCL unavailable: " + N.why);
  nccl_uid_t id;
  int r = N.getUniqueId(&id);
  if (r) return dfail(SG_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out, &id, sizeof(id));
  return SG_OK;
}

// Launch of an exchange task (called by sg_flush's launch_group).
int sg_dist_launch(sg_grid* g, int op, int kind, int task) {
  DistState& D = g->dist;
  if (!D.on) { dfail(SG_ERR_STATE, "exchange task on a grid without sg_dist_init"); return SG_ERR_STATE; }
  if (kind < 0 || kind >= DIST_KINDS) { dfail(SG_ERR_ARG, "bad exchange kind"); return SG_ERR_ARG; }
  if (D.world == 1) return SG_OK;
  if (D.transport == DIST_PEER) {
    if (op == SG_OP_DIST_SIGNAL) {
      uint64_t* f0 = D.has_nb[0] ? flag_ptr(D.peer_arena[0], kind, 1) : nullptr;
      uint64_t* f1 = D.has_nb[1] ? flag_ptr(D.peer_arena[1], kind, 0) : nullptr;
      k_dist_signal<<<1, 32, 0, g->stream>>>(epoch_ptr(D.arena, kind), f0, f1);
    } else {
      const uint64_t* f0 = D.has_nb[0] ? flag_ptr(D.arena, kind, 0) : nullptr;
      const uint64_t* f1 = D.has_nb[1] ? flag_ptr(D.arena, kind, 1) : nullptr;
      k_dist_wait<<<1, 32, 0, g->stream>>>(epoch_ptr(D.arena, kind), f0, f1, g->ctx.err, task);
    }
    return cudaGetLastError() == cudaSuccess ? SG_OK : SG_ERR_CUDA;
  }
  if (op == SG_OP_DIST_SIGNAL) return SG_OK;   // NCCL: the wait moves the data
  NcclApi& N = nccl();
  nccl_comm_t comm = (nccl_comm_t)D.comm;
  int r = N.groupStart();
  for (int s = 0; s < 2 && !r; s++) {
    if (!D.has_nb[s]) continue;
    const int peer = s == 0 ? D.rank - 1 : D.rank + 1;
    r = N.send(D.send_local[kind][s], (size_t)D.words[kind], NCCL_UINT32, peer, comm, g->stream);
    if (!r) r = N.recv(D.arena + D.recv_off[kind][s], (size_t)D.words[kind], NCCL_UINT32, peer, comm, g->stream);
  }
  int r2 = N.groupEnd();
  if (r || r2) { dfail(SG_ERR_NCCL, "ncclSend/ncclRecv failed"); return SG_ERR_NCCL; }
  return SG_OK;
}

void sg_dist_destroy(sg_grid* g) {
  DistState& D = g->dist;
  std::vector<sg_grid*>& P = pending_group();
  for (size_t i = 0; i < P.size(); i++)
    if (P[i] == g) { P.clear(); break; }
  if (!D.on) return;
  for (int s = 0; s < 2; s++)
    if (D.peer_ipc[s] && D.peer_arena[s]) cudaIpcCloseMemHandle(D.peer_arena[s]);
  if (D.comm && nccl().ok) nccl().commDestroy((nccl_comm_t)D.comm);
  if (D.arena) cudaFree(D.arena);
  D = DistState();
}

// Diagnostics: SG_SEGV_TRACE=1 installs a SIGSEGV handler at library load that
// prints the faulting thread's native backtrace to stderr (Python's
// faulthandler is off by the time C exit handlers run).
namespace {
void sg_segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "libsg: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof(msg) - 1);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvTrace {
  SegvTrace() {
    const char* e = std::getenv("SG_SEGV_TRACE");
    if (e && std::atoi(e)) signal(SIGSEGV, sg_segv_handler);
  }
} g_segv_trace;
}  // namespace
