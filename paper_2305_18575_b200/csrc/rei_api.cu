// rei_api.cu -- the C ABI (include/rei.h): context, level scheduler, memory, and
// regex reconstruction of the B200 REI hot path.
//
// Host side of Algorithm 1: for each cost level c the host plans the
// operand blocks -- Q = lvl(c - c2), S = lvl(c - c3), C = lvl(L) x lvl(R) for all
// L + R = c - c4 (ordered, reading A7), U = lvl(L) x lvl(R) for L <= R, L + R = c - c5
// (i < j when L = R, reading A8) -- flattens them into one rank space (Q, S, C by L
// ascending, U by L ascending, row-major; reading A9 counts candidates from it),
// launches the level kernels (levels.cu) and reads back one 64-byte control line.
// The language cache, dedup set and transposed slabs never leave the device.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rei.h"
#include "rei_common.cuh"
#include "rei_host.h"

namespace rei {
namespace {
// NCCL is resolved at run time (dlopen), only when a multi-GPU context is made:
// the library itself does not depend on libnccl, so loading it can never shadow the
// NCCL build torch ships (callers import torch first, then its libnccl is reused).
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = nullptr;
  if (const char* path = getenv("REI_NCCL_LIB")) {  // the binding points at torch's copy
    h = dlopen(path, RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  }
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) return a;
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
  a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(h, "ncclBroadcast"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
  a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.Broadcast && a.GroupStart &&
         a.GroupEnd && a.Send && a.Recv;
  return a;
}
}  // namespace
}  // namespace rei

namespace rei {
namespace {

std::string g_init_error;

struct PlanBlock {
  uint32_t kind;
  int L, R;
  uint64_t na, nb;
  uint64_t cand_off, cand_count;
  bool tri;
  uint64_t a_off = 0, b_off = 0;  // sharded cache: level index of the operand shards' first entries
};

struct LevelInfo {
  int cost = 0;
  uint64_t begin = 0;   // arena index
  uint64_t size = 0;
  uint64_t slab = 0;    // tarena slab index
  std::vector<PlanBlock> plan;
  bool seeds = false;
  // sharded cache (f3): owner o's shard = its arena entries [sbegin[o], +ssize[o]),
  // slabs from sslab[o]; level index soff[o] + i (rank-order concatenation)
  std::vector<uint64_t> sbegin, ssize, sslab, soff;
};

struct EventPair {
  cudaEvent_t a, b;
  int cls;
  cudaStream_t s;
};

struct Ctx {
  int device = 0;
  int sms = 148;  // multiprocessors of `device` (work-item sizing)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string alphabet;
  std::vector<std::vector<uint8_t>> P, N;
  rei_costs costs{};
  uint32_t err_num = 0, err_den = 1;
  uint32_t flags = 0;
  uint64_t budget = 0;       // user budget, or (sharded) the driver's free memory once queried
  bool budget_user = false;  // rei_options.mem_budget_bytes was given
  uint64_t budget_used = 0;  // bytes allocated before the budget was first queried
  uint64_t entry_limit = 0;  // rei_options.max_entries (0 = budget only)
  int otf_level = 0;         // first level checked in OnTheFly mode (0 = none)

  DeviceTables tab;
  int W32 = 1;
  int mode = DEDUP_BITMAP;

  // device buffers
  uint32_t* arena = nullptr;
  unsigned long long* bp = nullptr;
  uint32_t* tarena = nullptr;
  uint64_t cap = 0;        // entries
  uint64_t slab_cap = 0;   // slabs
  uint32_t* bitmap = nullptr;
  uint64_t bitmap_words = 0;
  unsigned long long* table = nullptr;
  uint64_t slots = 0;
  uint64_t table_slot_bytes = 0;  // slot size the dedup table was allocated with
  unsigned int* special = nullptr;
  LevelCtl* ctl = nullptr;       // the current level's control line (in ctl_base)
  LevelCtl* ctl_base = nullptr;  // [2]: sharded mode alternates by level parity
  LevelCtl* h_ctl = nullptr;  // pinned
  unsigned long long* h_rb = nullptr;  // pinned: back-pointer reads of the reconstruction
  Block* d_blocks = nullptr;  // [3][kMaxBlocks]: concat (B sliced), concat (A sliced), union
  Block* h_blocks = nullptr;  // pinned
  static constexpr int kMaxBlocks = 4096;

  // search state
  std::map<int, LevelInfo> levels;
  uint64_t arena_used = 0, slabs_used = 0;
  std::vector<rei_level_stat> stats;
  std::string regex;
  std::string err;
  rei_result result{};

  // concurrent level kernels: 0 = one stream; 1 = ? / * on an auxiliary stream;
  // 2 = also union on a second one; 3 = as 2 with concat on a high-priority
  // stream and union on a low-priority one, so union only fills SMs concat
  // leaves idle (REI_CONCURRENT; the kernels of a level are independent: they
  // read lower levels and insert through atomics)
  // sharded cache (f3): every rank's buffers as mapped in this process (self included)
  bool sharded = false;
  rei_allgather_fn allgather = nullptr;
  void* allgather_user = nullptr;
  struct PeerBuf {
    uint32_t* arena;
    unsigned long long* bp;
    uint32_t* tarena;
    LevelCtl* ctl_base;
    uint32_t* bitmap;
    unsigned long long* table;
    unsigned int* special;
    uint64_t cap, slots;
  };
  std::vector<PeerBuf> peers;
  std::vector<void*> ipc_opened;
  static constexpr int kMaxShards = 64;
  Peer* d_peers = nullptr;  // [kMaxShards]
  Peer* h_peers = nullptr;  // pinned
  std::vector<uint64_t> sh_used, sh_slabs;  // every owner's arena / slab fill

  int concurrency = 0;
  bool sort_levels = false;
  bool union_first = false;  // launch a level's union kernel before its concat kernels
  cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[3] = {nullptr, nullptr, nullptr};
  // post-level work (the finished level's sort + transpose) on its own stream, so that
  // the next level's concatenation / union kernels -- which never read the level just
  // finished -- start without waiting for it; anything that reads that level waits
  cudaStream_t post = nullptr;
  cudaEvent_t ev_level_done = nullptr, ev_post = nullptr;
  bool post_pending = false;
  int post_level = 0;
  std::vector<int> post_levels;  // every level whose sort / transpose is still on `post`
  void wait_post(cudaStream_t s) {
    if (post_pending) cudaStreamWaitEvent(s, ev_post, 0);
  }
  void join_post() {  // the context's stream (and everything after it) sees the post work
    wait_post(stream);
    post_pending = false;
    post_levels.clear();
  }
  // lagged levels (solve_lagged): device base of the level being launched, the previous
  // (unread) level's control line and first arena index
  static constexpr int kLag = 4;              // control-line slots: up to kLag - 1 levels in flight
  unsigned long long* d_lag_base = nullptr;  // [kLag] device arena base of each slot's level
  unsigned long long* h_lag_base = nullptr;  // pinned [kLag]: host-known bases copied to the device
  const LevelCtl* lag_prev_ctl = nullptr;
  int lag_prev_par = 0;
  int lag_par = 0;
  LevelCtl* h_lag = nullptr;  // pinned [kLag]: control lines read back without a stream sync
  // pinned block tables [kLag][3][kMaxBlocks]: a lagged level's H2D copy of its plan may
  // run after the host has planned the next level, so each slot has its own staging
  Block* h_blocks_ring = nullptr;
  bool lag_active = false;
  // split levels: part 1 = the binary kernels only (no join), part 2 = the unary kernel only
  int lag_part = 0;
  uint32_t lag_unary_reads = 0;          // how many of the level's ? / * sources are the level in flight
  unsigned long long* d_rank_off = nullptr;  // [kLag]
  cudaEvent_t ev_lag[kLag] = {nullptr, nullptr, nullptr, nullptr};

  // multi-rank
  int world = 1, rank = 0;
  bool exchange_self = false;        // REI_FLAG_EXCHANGE_SELF: one rank, full exchange over NCCL
  void* nccl = nullptr;              // ncclComm_t (one process per GPU)
  bool host_xport = false;           // exchange through the caller's allgather callback
  LevelCtl* d_ctl_all = nullptr;     // [world] gathered control lines
  unsigned long long* d_small = nullptr;      // [64] small all-gather send (NCCL)
  unsigned long long* d_small_all = nullptr;  // [world * 64]
  uint32_t* st_cs = nullptr;         // staging list of an exchanged level (this rank's new CSs)
  unsigned long long* st_bp = nullptr;
  uint64_t st_cap = 0;
  XScratch xs;
  MergeScratch merge;

  // device level loop (DevLoop): device arrays + pinned mirror, same layout
  void* d_loop = nullptr;
  void* h_loop = nullptr;
  size_t loop_bytes = 0;

  // profiling
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  uint64_t launches = 0;
  uint64_t k_launches[REI_K_COUNT] = {0};
  double k_ms[REI_K_COUNT] = {0};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  std::vector<EventPair> pending;

  // device buffers come from the process-wide pool (devmem.cu) unless they are
  // exported through CUDA IPC (sharded-cache contexts); pinned host blocks are cached
  cudaError_t dmalloc(void** p, size_t bytes) {
    if (sharded) return cudaMalloc(p, bytes);
    return dev_alloc(p, bytes, stream);
  }
  template <class T>
  cudaError_t dmalloc(T** p, size_t bytes) { return dmalloc(reinterpret_cast<void**>(p), bytes); }
  void dfree(void* p) {
    if (!p) return;
    if (sharded) cudaFree(p); else dev_free(p, stream);
  }

  ~Ctx() {
    if (post) cudaStreamSynchronize(post);
    if (stream) cudaStreamSynchronize(stream);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    for (void* q : {(void*)arena, (void*)bp, (void*)tarena, (void*)bitmap, (void*)table, (void*)special,
                    (void*)ctl_base, (void*)d_blocks, (void*)d_peers, (void*)tab.split, (void*)tab.nsplit,
                    (void*)tab.word_len, (void*)tab.seeds, (void*)d_ctl_all, (void*)st_cs, (void*)st_bp,
                    (void*)d_small, (void*)d_small_all, d_loop, (void*)d_lag_base, (void*)d_rank_off})
      dfree(q);
    host_free(h_loop);
    host_free(h_rb);
    host_free(h_lag);
    host_free(h_lag_base);
    host_free(h_blocks_ring);
    for (auto e : ev_lag)
      if (e) cudaEventDestroy(e);
    host_free(h_peers);
    host_free(h_ctl);
    host_free(h_blocks);
    for (auto e : ev_pool) cudaEventDestroy(e);
    free_merge_scratch(merge);
    free_xscratch(xs);
    if (nccl) nccl_api().CommDestroy((ncclComm_t)nccl);
    if (stream) cudaStreamSynchronize(stream);  // the pooled frees above are stream-ordered
    for (int i = 0; i < 3; ++i) {
      if (aux[i]) cudaStreamDestroy(aux[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (post) cudaStreamDestroy(post);
    if (ev_level_done) cudaEventDestroy(ev_level_done);
    if (ev_post) cudaEventDestroy(ev_post);
    for (auto& pr : lvl_ev_p)
      for (auto e : pr)
        if (e) cudaEventDestroy(e);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  cudaEvent_t next_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  // per-kernel CUDA events (rei_kernel_stats); off (REI_KERNEL_EVENTS=0): one event
  // pair per level on the context's stream gives the level time
  bool kernel_events = false;  // on after rei_reset_kernel_stats (or REI_KERNEL_EVENTS=1)
  cudaEvent_t lvl_ev_p[4][2] = {};
  bool lvl_open_p[4] = {false, false, false, false};
  int ev_par = 0;  // which pair level_mark / collect_events use (lagged levels alternate)
  void begin_kernel(int cls, EventPair& ep, cudaStream_t s = nullptr) {
    ep.cls = cls;
    ep.s = s ? s : stream;
    if (!kernel_events) return;
    ep.a = next_event();
    ep.b = next_event();
    cudaEventRecord(ep.a, ep.s);
  }
  void end_kernel(EventPair& ep, int n) {
    launches += n;
    k_launches[ep.cls] += n;
    if (!kernel_events) return;
    cudaEventRecord(ep.b, ep.s);
    pending.push_back(ep);
  }
  void level_mark(int i) {  // 0 before a level's first launch, 1 after its join
    if (kernel_events) return;
    cudaEvent_t& e = lvl_ev_p[ev_par][i];
    if (!e) cudaEventCreate(&e);
    cudaEventRecord(e, stream);
    lvl_open_p[ev_par] = true;
  }
  // after a stream sync: fold the pending event pairs into the per-class totals
  // level_ms = the wall span of the pending launches (first start to last end): a
  // level's kernels may overlap on the auxiliary streams, so their sum would overcount
  void collect_events(double* level_ms) {
    if (!kernel_events) {
      float ms = 0;
      cudaEvent_t* e = lvl_ev_p[ev_par];
      if (lvl_open_p[ev_par] && e[0] && e[1]) cudaEventElapsedTime(&ms, e[0], e[1]);
      lvl_open_p[ev_par] = false;
      if (level_ms) *level_ms = ms;
      return;
    }
    float lo = 0, hi = 0;
    for (auto& ep : pending) {
      float ms = 0, a = 0, b = 0;
      cudaEventElapsedTime(&ms, ep.a, ep.b);
      k_ms[ep.cls] += ms;
      cudaEventElapsedTime(&a, pending[0].a, ep.a);
      cudaEventElapsedTime(&b, pending[0].a, ep.b);
      lo = std::min(lo, a);
      hi = std::max(hi, b);
    }
    pending.clear();
    ev_next = 0;
    if (level_ms) *level_ms = hi - lo;
  }
};

#define CUDA_OK(c, x)                                                        \
  do {                                                                       \
    cudaError_t e__ = (x);                                                   \
    if (e__ != cudaSuccess) {                                                \
      (c)->err = std::string(#x ": ") + cudaGetErrorString(e__);             \
      return REI_ECUDA;                                                      \
    }                                                                        \
  } while (0)

int next_pow2_words(int n) {
  int w = (n + 31) / 32;
  int p = 1;
  while (p < w) p <<= 1;
  return p;
}

// bytes per dedup-set slot: an 8-byte key / index word, or the whole CS (inline keys)
uint64_t slot_bytes(const Ctx* c) { return c->mode == DEDUP_HASHIN ? 4ull * c->W32 : 8ull; }

uint64_t bytes_per_entry(const Ctx* c) {
  // CS + back-pointer + transposed copy (+ hash slots at load <= 1/2)
  uint64_t b = 4ull * c->W32 + 8 + 4ull * c->W32;
  if (c->mode != DEDUP_BITMAP) b += 2 * slot_bytes(c);
  return b;
}

// (Re)allocate arena, bp, tarena (and the dedup table) for `cap` entries, preserving the
// first `keep` entries.  Out of device memory: REI_OUT_OF_MEMORY with the previous
// buffers unchanged (or, if only the new table failed, a table of the previous size and
// the previous capacity), so the caller can fall back to OnTheFly mode.
rei_status alloc_arena(Ctx* c, uint64_t new_cap, uint64_t keep, uint64_t keep_slabs) {
  const uint64_t new_slab_cap = new_cap / 32 + 4096;
  uint32_t* a = nullptr;
  unsigned long long* b = nullptr;
  uint32_t* t = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  auto oom = [&](cudaError_t e, const char* what) {
    c->dfree(a); c->dfree(b); c->dfree(t);
    cudaGetLastError();
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? REI_OUT_OF_MEMORY : REI_ECUDA;
  };
  cudaError_t e;
  if ((e = c->dmalloc(&a, new_cap * 4ull * c->W32)) != cudaSuccess) return oom(e, "arena allocation");
  if ((e = c->dmalloc(&b, new_cap * 8ull)) != cudaSuccess) return oom(e, "back-pointer allocation");
  if ((e = c->dmalloc(&t, new_slab_cap * 32ull * c->W32 * 4ull)) != cudaSuccess) return oom(e, "slab allocation");
  if (getenv("REI_TRACE")) {
    cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[rei_alloc] arena %llu entries: %.3f ms\n", (unsigned long long)new_cap,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  if (keep) {
    CUDA_OK(c, cudaMemcpyAsync(a, c->arena, keep * 4ull * c->W32, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_OK(c, cudaMemcpyAsync(b, c->bp, keep * 8ull, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (keep_slabs)
    CUDA_OK(c, cudaMemcpyAsync(t, c->tarena, keep_slabs * 32ull * c->W32 * 4ull, cudaMemcpyDeviceToDevice,
                               c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  const uint64_t old_cap = c->cap, old_slots = c->slots;
  c->dfree(c->arena); c->dfree(c->bp); c->dfree(c->tarena);
  c->arena = a; c->bp = b; c->tarena = t;
  c->cap = new_cap;
  c->slab_cap = new_slab_cap;
  if (c->mode != DEDUP_BITMAP) {
    uint64_t want = 1;
    while (want < 2 * new_cap) want <<= 1;
    if (want != c->slots || c->table_slot_bytes != slot_bytes(c)) {
      // the table's contents are rebuilt from the arena after a growth: release first
      c->dfree(c->table);
      c->table = nullptr;
      e = c->dmalloc(&c->table, want * slot_bytes(c));
      if (e != cudaSuccess) {
        cudaGetLastError();
        c->err = std::string("dedup table allocation: ") + cudaGetErrorString(e);
        if (old_slots && c->table_slot_bytes == slot_bytes(c) &&
            c->dmalloc(&c->table, old_slots * slot_bytes(c)) == cudaSuccess) {
          c->cap = std::min(old_cap, new_cap);  // entries the previous table was sized for
          return REI_OUT_OF_MEMORY;
        }
        c->slots = 0;
        return REI_ECUDA;
      }
      c->slots = want;
      c->table_slot_bytes = slot_bytes(c);
    }
  }
  return REI_OK;
}

void fill_params(Ctx* c, LevelParams& p) {
  memset(&p, 0, sizeof(p));
  p.arena = c->arena;
  p.arena_out = c->arena;
  p.tarena = c->tarena;
  p.bp = c->bp;
  p.n = (uint32_t)c->tab.n;
  p.maxk = (uint32_t)c->tab.maxk;
  p.exact = c->err_num == 0 ? 1 : 0;
  const uint64_t total = c->P.size() + c->N.size();
  p.max_errors = c->err_num ? (uint32_t)((uint64_t)c->err_num * total / c->err_den) : 0;
  p.early_exit = (c->flags & REI_FLAG_COMPLETE_FINAL_LEVEL) ? 0 : 1;
  p.cap = c->entry_limit ? std::min<uint64_t>(c->cap, c->entry_limit) : c->cap;
  p.split = c->tab.split;
  p.nsplit = c->tab.nsplit;
  p.word_len = c->tab.word_len;
  p.ctl = c->ctl;
  p.dedup.mode = c->mode;
  p.dedup.bitmap = c->bitmap;
  p.dedup.table = c->table;
  p.dedup.mask = c->slots ? c->slots - 1 : 0;
  p.dedup.special = c->special;
  p.out_base_dev = (c->lag_prev_ctl || c->lag_part == 2) ? c->d_lag_base + c->lag_par : nullptr;
  p.rank_off_dev = (c->lag_part == 1 && c->lag_unary_reads) ? c->d_rank_off + c->lag_par : nullptr;
  for (int q = 0; q < kMaxW32; ++q) { p.pos[q] = c->tab.pos[q]; p.neg[q] = c->tab.neg[q]; }
}

rei_status clear_dedup(Ctx* c) {
  if (c->mode == DEDUP_BITMAP) {
    CUDA_OK(c, cudaMemsetAsync(c->bitmap, 0, c->bitmap_words * 4, c->stream));
  } else {
    CUDA_OK(c, cudaMemsetAsync(c->table, c->mode == DEDUP_HASHIDX ? 0x00 : 0xff, c->slots * slot_bytes(c), c->stream));
    CUDA_OK(c, cudaMemsetAsync(c->special, 0, sizeof(unsigned int), c->stream));
  }
  return REI_OK;
}

rei_status reset_ctl(Ctx* c) {
  LevelCtl z;
  memset(&z, 0, sizeof(z));
  z.found_rank = ~0ull;
  *c->h_ctl = z;
  CUDA_OK(c, cudaMemcpyAsync(c->ctl, c->h_ctl, sizeof(LevelCtl), cudaMemcpyHostToDevice, c->stream));
  c->h2d_bytes += sizeof(LevelCtl);
  return REI_OK;
}

rei_status read_ctl(Ctx* c) {
  CUDA_OK(c, cudaMemcpyAsync(c->h_ctl, c->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->d2h_bytes += sizeof(LevelCtl);
  return REI_OK;
}

uint64_t level_size(const Ctx* c, int cost) {
  auto it = c->levels.find(cost);
  return it == c->levels.end() ? 0 : it->second.size;
}

// Decode a rank of level `cost` into (kind, L, i, R, j) (inverse of the flattening).
struct Node {
  uint32_t kind;  // 0..3 = Q S C U, 4 = symbol
  int L, R;
  uint64_t i, j;
};

Node decode_rank(const Ctx* c, int cost, uint64_t rank) {
  const LevelInfo& lv = c->levels.at(cost);
  Node nd{};
  if (lv.seeds) { nd.kind = 4; nd.i = rank; return nd; }
  for (const PlanBlock& b : lv.plan) {
    if (rank < b.cand_off || rank >= b.cand_off + b.cand_count) continue;
    const uint64_t t = rank - b.cand_off;
    nd.kind = b.kind;
    nd.L = b.L;
    nd.R = b.R;
    if (b.kind == BK_Q || b.kind == BK_S) { nd.i = b.a_off + t; return nd; }
    if (!b.tri) { nd.i = b.a_off + t / b.nb; nd.j = b.b_off + t % b.nb; return nd; }
    // triangular: start(i) = i*m - i(i+1)/2; largest i with start(i) <= t
    const uint64_t m = b.na;
    uint64_t lo = 0, hi = m - 1;
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) / 2;
      const uint64_t start = mid * m - mid * (mid + 1) / 2;
      if (start <= t) lo = mid; else hi = mid - 1;
    }
    nd.i = b.a_off + lo;
    nd.j = b.b_off + t - (lo * m - lo * (lo + 1) / 2) + lo + 1;
    return nd;
  }
  nd.kind = 99;
  return nd;
}

// Printer (paper syntax): postfix > concatenation > union; a postfix operator wraps
// any operand that is not a single symbol; concatenation wraps union operands.
enum { PR_UNION = 0, PR_CAT = 1, PR_ATOM = 2 };

bool rebuild(Ctx* c, int cost, uint64_t rank, std::string& out, int& prec, int depth);

// device address of the back-pointer of entry idx of level `cost`
const unsigned long long* bp_src(const Ctx* c, int cost, uint64_t idx) {
  const LevelInfo& lv = c->levels.at(cost);
  if (!lv.ssize.empty()) {  // sharded cache: the entry lives in its owner's shard
    size_t o = 0;
    while (o + 1 < lv.ssize.size() && idx >= lv.soff[o] + lv.ssize[o]) ++o;
    return c->peers[o].bp + lv.sbegin[o] + (idx - lv.soff[o]);
  }
  return c->bp + lv.begin + idx;
}

bool rebuild_entry(Ctx* c, int cost, uint64_t idx, std::string& out, int& prec, int depth) {
  if (!c->h_rb && host_alloc(reinterpret_cast<void**>(&c->h_rb), 8 * 4096) != cudaSuccess) return false;
  unsigned long long r = 0;
  const unsigned long long* src = bp_src(c, cost, idx);
  // one pinned 8-byte read on the context's stream (a pageable cudaMemcpy stages
  // through a driver buffer: ~2x the round trip per node of the regex tree)
  if (cudaMemcpyAsync(c->h_rb, src, 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return false;
  r = *c->h_rb;
  c->d2h_bytes += 8;
  return rebuild(c, cost, r, out, prec, depth + 1);
}

bool rebuild(Ctx* c, int cost, uint64_t rank, std::string& out, int& prec, int depth) {
  if (depth > 100000) return false;
  Node nd = decode_rank(c, cost, rank);
  const rei_costs& k = c->costs;
  switch (nd.kind) {
    case 4:
      out = std::string(1, c->alphabet[nd.i]);
      prec = PR_ATOM;
      return true;
    case BK_Q:
    case BK_S: {
      const int L = (nd.kind == BK_Q) ? cost - (int)k.opt : cost - (int)k.star;
      std::string s;
      int ps;
      if (!rebuild_entry(c, L, nd.i, s, ps, depth)) return false;
      if (!(ps == PR_ATOM && s.size() == 1)) s = "(" + s + ")";
      out = s + (nd.kind == BK_Q ? "?" : "*");
      prec = PR_ATOM;
      return true;
    }
    case BK_C:
    case BK_U: {
      std::string l, r;
      int pl, pr;
      if (!rebuild_entry(c, nd.L, nd.i, l, pl, depth)) return false;
      if (!rebuild_entry(c, nd.R, nd.j, r, pr, depth)) return false;
      if (nd.kind == BK_C) {
        if (pl == PR_UNION) l = "(" + l + ")";
        if (pr == PR_UNION) r = "(" + r + ")";
        out = l + r;
        prec = PR_CAT;
      } else {
        out = l + "+" + r;
        prec = PR_UNION;
      }
      return true;
    }
  }
  return false;
}

// Build the level plan for cost c from the sizes of lower levels.
void plan_level(Ctx* c, int cost, LevelInfo& lv, std::vector<Block>& cat, std::vector<Block>& uni,
                uint64_t& nq, uint64_t& ns, uint64_t& ncat, uint64_t& nuni) {
  const rei_costs& k = c->costs;
  const int c1 = (int)k.sym;
  uint64_t off = 0;
  lv.plan.clear();
  cat.clear();
  uni.clear();
  nq = level_size(c, cost - (int)k.opt);
  if (cost - (int)k.opt < c1) nq = 0;
  if (nq) { lv.plan.push_back({BK_Q, cost - (int)k.opt, 0, nq, 0, off, nq, false}); off += nq; }
  ns = level_size(c, cost - (int)k.star);
  if (cost - (int)k.star < c1) ns = 0;
  if (ns) { lv.plan.push_back({BK_S, cost - (int)k.star, 0, ns, 0, off, ns, false}); off += ns; }
  ncat = 0;
  // candidates per work item: large items amortise the per-slab set-up at deep
  // levels; small levels get small items so that ~4 items per resident warp
  // (SMs x 24 warps) keep every SM busy instead of a few warps running serially
  uint64_t pairs = 0;
  for (int L = c1; L <= cost - (int)k.cat - c1; ++L) pairs += level_size(c, L) * level_size(c, cost - (int)k.cat - L);
  for (int L = c1; L <= cost - (int)k.alt - L; ++L) pairs += level_size(c, L) * level_size(c, cost - (int)k.alt - L);
  const uint64_t target = std::min<uint64_t>(8192, std::max<uint64_t>(128, pairs / ((uint64_t)c->sms * 24 * 4)));
  auto tile_u = [&](uint64_t nu) { return std::max<uint64_t>(1, std::min<uint64_t>({64, nu, target / 32})); };
  uint64_t item_off = 0;
  for (int L = c1; L <= cost - (int)k.cat - c1; ++L) {
    const int R = cost - (int)k.cat - L;
    const uint64_t na = level_size(c, L), nb = level_size(c, R);
    if (!na || !nb) continue;
    PlanBlock pb{BK_C, L, R, na, nb, off, na * nb, false};
    lv.plan.push_back(pb);
    Block b{};
    b.kind = BK_C;
    b.slice_a = (na > nb) ? 1 : 0;  // slice the larger side, the smaller is uniform
    const LevelInfo& A = c->levels.at(L);
    const LevelInfo& B = c->levels.at(R);
    b.a_base = A.begin; b.b_base = B.begin; b.a_slab = A.slab; b.b_slab = B.slab;
    b.na = na; b.nb = nb;
    b.cand_off = off; b.cand_count = na * nb;
    const uint64_t nu = b.slice_a ? nb : na, nsl = b.slice_a ? na : nb;
    const uint64_t slabs = (nsl + 31) / 32;
    b.tu = tile_u(nu);
    b.ts = std::max<uint64_t>(1, std::min<uint64_t>(slabs, target / (32 * b.tu)));
    b.u_tiles = (nu + b.tu - 1) / b.tu;
    b.s_tiles = (slabs + b.ts - 1) / b.ts;
    b.item_off = item_off;
    item_off += b.u_tiles * b.s_tiles;
    cat.push_back(b);
    off += na * nb;
    ncat += na * nb;
  }
  nuni = 0;
  item_off = 0;
  for (int L = c1; L <= cost - (int)k.alt - L; ++L) {
    const int R = cost - (int)k.alt - L;
    const uint64_t na = level_size(c, L), nb = level_size(c, R);
    if (!na || !nb) continue;
    const bool tri = (L == R);
    const uint64_t cnt = tri ? na * (na - 1) / 2 : na * nb;
    if (!cnt) continue;
    lv.plan.push_back({BK_U, L, R, na, nb, off, cnt, tri});
    Block b{};
    b.kind = BK_U;
    b.tri = tri ? 1 : 0;
    b.slice_a = (!tri && na > nb) ? 1 : 0;
    const LevelInfo& A = c->levels.at(L);
    const LevelInfo& B = c->levels.at(R);
    b.a_base = A.begin; b.b_base = B.begin; b.a_slab = A.slab; b.b_slab = B.slab;
    b.na = na; b.nb = nb;
    b.cand_off = off; b.cand_count = cnt;
    const uint64_t nu = b.slice_a ? nb : na, nsl = b.slice_a ? na : nb;
    const uint64_t slabs = (nsl + 31) / 32;
    b.tu = tile_u(nu);
    b.ts = std::max<uint64_t>(1, std::min<uint64_t>(slabs, target / (32 * b.tu)));
    b.u_tiles = (nu + b.tu - 1) / b.tu;
    b.s_tiles = (slabs + b.ts - 1) / b.ts;
    b.item_off = item_off;
    item_off += b.u_tiles * b.s_tiles;
    uni.push_back(b);
    off += cnt;
    nuni += cnt;
  }
}

uint64_t items_of(const std::vector<Block>& v) {
  if (v.empty()) return 0;
  return v.back().item_off + v.back().u_tiles * v.back().s_tiles;
}

void renumber_items(std::vector<Block>& v) {
  uint64_t off = 0;
  for (Block& b : v) {
    b.item_off = off;
    off += b.u_tiles * b.s_tiles;
  }
}

rei_status rebuild_dedup(Ctx* c, uint64_t entries) {
  c->join_post();
  rei_status s = clear_dedup(c);
  if (s != REI_OK) return s;
  if ((s = reset_ctl(c)) != REI_OK) return s;  // a stale overflow flag would stop the inserts
  if (!entries) return REI_OK;
  LevelParams p;
  fill_params(c, p);
  EventPair ep;
  c->begin_kernel(REI_K_OTHER, ep);
  int n = launch_rehash(c->W32, p, 0, entries, c->stream);
  c->end_kernel(ep, n);
  CUDA_OK(c, cudaGetLastError());
  return REI_OK;
}

// Device memory the context's cache may use: rei_options.mem_budget_bytes (a fixed total),
// else 80 % of the free HBM as the process-wide pool estimates it (dev_free_estimate:
// one cudaMemGetInfo per process -- 0.3-70 ms on B200 -- then the pool's own traffic).
// Sharded-cache contexts allocate outside the pool and query the driver once.
uint64_t budget_of(Ctx* c) {
  if (c->budget_user) return c->budget;
  if (c->sharded) {
    if (!c->budget) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      c->budget = (uint64_t)(0.8 * (double)fr);
    }
    return c->budget;
  }
  return (uint64_t)(0.8 * (double)dev_free_estimate(c->device));
}

// Bytes of the cache buffers for `cap` entries: arena + back-pointers + transposed
// slabs (abt) and the dedup table (power-of-two slots, load <= 1/2).
uint64_t abt_bytes(const Ctx* c, uint64_t cap) {
  return cap * (4ull * c->W32 + 8ull) + (cap / 32 + 4096) * 32ull * c->W32 * 4ull;
}
uint64_t table_bytes(const Ctx* c, uint64_t cap) {
  if (c->mode == DEDUP_BITMAP) return 0;
  uint64_t want = 1;
  while (want < 2 * cap) want <<= 1;
  return want * slot_bytes(c);
}

// Total HBM of the current device, queried once per process and device.
uint64_t device_total_bytes(int dev) {
  static std::mutex mu;
  static std::map<int, uint64_t> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  return cache[dev] = tot;
}

rei_status grow(Ctx* c, uint64_t need_entries) {
  if (c->sharded) return REI_OUT_OF_MEMORY;  // peers map the buffers: fixed at rei_init
  c->join_post();  // the copy below must see the last level's sort and transpose
  // the bitmap-mode cache already holds every one of the 2^n possible CSs: nothing to
  // grow, and no cudaMemGetInfo (0.3-70 ms on B200) for the budget (it was the 8-15 ms
  // tail of fresh-context solves of Table 1 row 1 at level 28)
  if (c->mode == DEDUP_BITMAP && c->cap >= (1ull << c->tab.n) + 64) return REI_OUT_OF_MEMORY;
  if (c->entry_limit && c->cap >= c->entry_limit) return REI_OUT_OF_MEMORY;
  // x8 per growth: every growth rehashes the whole cache, so grow rarely
  uint64_t nc = std::max<uint64_t>(c->cap * 8, need_entries);
  if (c->mode == DEDUP_BITMAP) nc = std::min<uint64_t>(nc, (1ull << c->tab.n) + 64);
  if (c->entry_limit) nc = std::min<uint64_t>(nc, c->entry_limit);
  // memory: with a user budget the new buffers must fit it; otherwise the new arena /
  // back-pointer / slab buffers must fit next to the old ones (they are copied), and the
  // new buffers with the new table must fit once the old ones are released
  const uint64_t B = budget_of(c), held = abt_bytes(c, c->cap) + table_bytes(c, c->cap);
  auto fits = [&](uint64_t cap) {
    if (c->budget_user) return abt_bytes(c, cap) + table_bytes(c, cap) <= B;
    return abt_bytes(c, cap) <= B && abt_bytes(c, cap) + table_bytes(c, cap) <= B + held;
  };
  if (!fits(nc) && c->mode == DEDUP_HASHIN) {
    // inline wide keys cost 2 x 16-32 bytes of table per entry: when they no longer fit,
    // continue with fingerprint + index slots (8 bytes; the table is rebuilt from the
    // arena after every growth anyway, so the switch costs nothing extra)
    c->mode = DEDUP_HASHIDX;
    if (!fits(nc)) c->mode = DEDUP_HASHIN;
  }
  if (!fits(nc)) {  // the largest capacity in (cap, nc) that fits
    uint64_t lo = c->cap, hi = nc;
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      (fits(mid) ? lo : hi) = mid;
    }
    nc = lo;
  }
  if (nc <= c->cap) return REI_OUT_OF_MEMORY;
  const bool trace = getenv("REI_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  rei_status s = alloc_arena(c, nc, c->arena_used, c->slabs_used);
  if (s != REI_OK && c->table && c->table_slot_bytes != slot_bytes(c)) c->mode = DEDUP_HASHIN;  // switch undone
  if (s == REI_OUT_OF_MEMORY && c->mode != DEDUP_BITMAP && c->table) {
    // the previous buffers are in place (the table may have been re-allocated empty)
    rei_status r = rebuild_dedup(c, c->arena_used);
    return r != REI_OK ? r : s;
  }
  if (s != REI_OK) return s;
  const auto t1 = std::chrono::steady_clock::now();
  s = rebuild_dedup(c, c->arena_used);
  if (trace) {
    cudaStreamSynchronize(c->stream);
    const auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[rei_grow] %llu -> %llu entries: realloc+copy %.3f ms, rehash %llu %.3f ms\n",
            (unsigned long long)c->cap, (unsigned long long)nc,
            std::chrono::duration<double, std::milli>(t1 - t0).count(), (unsigned long long)c->arena_used,
            std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  return s;
}

// The same printer over the whole tree, expanded breadth first: the children of every
// node of one tree depth are cache entries whose back-pointers are read with one
// stream synchronisation per depth (the recursive walk pays one per node).
constexpr size_t kRebuildBatch = 4096;  // pinned back-pointer slots (c->h_rb)
bool rebuild_batched(Ctx* c, int cost, uint64_t rank, std::string& out) {
  struct TNode {
    int cost;
    uint64_t rank;
    Node nd;
    int child[2];
    std::string s;
    int prec;
  };
  std::vector<TNode> t;
  t.push_back({cost, rank, Node{}, {-1, -1}, {}, 0});
  std::vector<int> frontier = {0};
  const rei_costs& k = c->costs;
  while (!frontier.empty()) {
    std::vector<int> next;
    std::vector<const unsigned long long*> src;
    for (int id : frontier) {
      t[id].nd = decode_rank(c, t[id].cost, t[id].rank);
      const Node& nd = t[id].nd;
      if (nd.kind == 4) continue;
      if (nd.kind > BK_U) return false;
      int ncost[2], nch = 1;
      uint64_t nidx[2];
      if (nd.kind == BK_Q || nd.kind == BK_S) {
        ncost[0] = (nd.kind == BK_Q) ? t[id].cost - (int)k.opt : t[id].cost - (int)k.star;
        nidx[0] = nd.i;
      } else {
        ncost[0] = nd.L; nidx[0] = nd.i;
        ncost[1] = nd.R; nidx[1] = nd.j;
        nch = 2;
      }
      for (int q = 0; q < nch; ++q) {
        if (t.size() > 100000) return false;
        t[id].child[q] = (int)t.size();
        t.push_back({ncost[q], 0, Node{}, {-1, -1}, {}, 0});
        next.push_back(t[id].child[q]);
        src.push_back(bp_src(c, ncost[q], nidx[q]));
      }
    }
    if (next.size() > kRebuildBatch) return false;
    for (size_t q = 0; q < src.size(); ++q)
      if (cudaMemcpyAsync(c->h_rb + q, src[q], 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) return false;
    if (!src.empty() && cudaStreamSynchronize(c->stream) != cudaSuccess) return false;
    c->d2h_bytes += 8 * src.size();
    for (size_t q = 0; q < next.size(); ++q) t[next[q]].rank = c->h_rb[q];
    frontier.swap(next);
  }
  for (int id = (int)t.size() - 1; id >= 0; --id) {  // children were created after parents
    TNode& n = t[id];
    switch (n.nd.kind) {
      case 4:
        n.s = std::string(1, c->alphabet[n.nd.i]);
        n.prec = PR_ATOM;
        break;
      case BK_Q:
      case BK_S: {
        std::string a = t[n.child[0]].s;
        if (!(t[n.child[0]].prec == PR_ATOM && a.size() == 1)) a = "(" + a + ")";
        n.s = a + (n.nd.kind == BK_Q ? "?" : "*");
        n.prec = PR_ATOM;
        break;
      }
      default: {
        std::string l = t[n.child[0]].s, r = t[n.child[1]].s;
        if (n.nd.kind == BK_C) {
          if (t[n.child[0]].prec == PR_UNION) l = "(" + l + ")";
          if (t[n.child[1]].prec == PR_UNION) r = "(" + r + ")";
          n.s = l + r;
          n.prec = PR_CAT;
        } else {
          n.s = l + "+" + r;
          n.prec = PR_UNION;
        }
      }
    }
    if (id) t[id].s.shrink_to_fit();
  }
  out = t[0].s;
  return true;
}

rei_status finish_found(Ctx* c, int cost, uint64_t rank) {
  c->join_post();  // reconstruction reads back-pointers of the last sorted level
  std::string rx;
  int pr;
  const auto t0 = std::chrono::steady_clock::now();
  if (!c->h_rb && host_alloc(reinterpret_cast<void**>(&c->h_rb), 8 * kRebuildBatch) != cudaSuccess) {
    c->err = "pinned allocation failed";
    return REI_ECUDA;
  }
  if (!rebuild_batched(c, cost, rank, rx) && !rebuild(c, cost, rank, rx, pr, 0)) {
    c->err = "regex reconstruction failed";
    return REI_ECUDA;
  }
  if (getenv("REI_TRACE"))
    fprintf(stderr, "[rei_solve] regex reconstruction: %.3f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  c->regex = rx;
  c->result.cost = (uint32_t)cost;
  return REI_OK;
}

// Device level loop (k_level_loop): levels c1 + 1 .. while they are
// small run inside one cooperative kernel with no host round trip per level.  On
// return the finished levels are in c->levels / c->stats exactly as the host loop
// would have left them (plans recomputed by plan_level from the level sizes, so
// back-pointer ranks decode identically); *next = the level the host loop continues
// with; *done = the search ended (a precise candidate).
bool device_loop_ok(const Ctx* c, uint32_t max_cost) {
  return !c->sharded && !c->otf_level && c->world == 1 && !c->exchange_self && (c->mode == DEDUP_BITMAP || c->mode == DEDUP_HASH64) &&
         c->W32 <= 2 && max_cost <= 65535 && getenv("REI_NO_DEVICE_LOOP") == nullptr;
}

rei_status device_levels(Ctx* c, uint32_t max_cost, int from_cost, int* next, uint64_t* cand, bool* done) {
  *done = false;
  const rei_costs& k = c->costs;
  const int c1 = (int)k.sym;
  *next = from_cost;
  if ((int)max_cost < from_cost) return REI_OK;
  c->join_post();  // the loop reads every finished level (sorted, transposed)
  const size_t L = (size_t)max_cost + 1;
  const size_t arr = L * 8;
  const size_t off_blocks = 5 * arr;
  const size_t off_state = off_blocks + sizeof(Block) * kLoopMaxBlocks;
  const size_t off_bar = off_state + sizeof(LoopState);
  const size_t off_hist = off_bar + 64;
  const size_t bytes = off_hist + 4 * kLoopSortBuckets;
  if (c->loop_bytes < bytes) {
    c->dfree(c->d_loop);
    host_free(c->h_loop);
    c->d_loop = nullptr;
    c->h_loop = nullptr;
    c->loop_bytes = 0;
    if (c->dmalloc(&c->d_loop, bytes) != cudaSuccess || host_alloc(&c->h_loop, bytes) != cudaSuccess) {
      cudaGetLastError();
      return REI_OK;  // the host loop runs every level instead
    }
    c->loop_bytes = bytes;
  }
  auto* h = static_cast<uint8_t*>(c->h_loop);
  auto* dv = static_cast<uint8_t*>(c->d_loop);
  auto* h_size = reinterpret_cast<unsigned long long*>(h);
  auto* h_begin = h_size + L;
  auto* h_slab = h_begin + L;
  auto* h_eval = h_slab + L;
  auto* h_ns = reinterpret_cast<long long*>(h_eval + L);
  auto* h_st = reinterpret_cast<LoopState*>(h + off_state);
  memset(h, 0, bytes);
  for (const auto& kv : c->levels) {  // every finished level (the loop may resume mid-search)
    if (kv.first >= from_cost || kv.first > (int)max_cost) continue;
    h_size[kv.first] = kv.second.size;
    h_begin[kv.first] = kv.second.begin;
    h_slab[kv.first] = kv.second.slab;
  }
  h_st->arena_used = c->arena_used;
  h_st->slabs_used = c->slabs_used;
  h_st->found_rank = ~0ull;
  CUDA_OK(c, cudaMemcpyAsync(dv, h, bytes, cudaMemcpyHostToDevice, c->stream));
  c->h2d_bytes += bytes;
  rei_status s;
  if ((s = reset_ctl(c)) != REI_OK) return s;
  LevelParams p;
  fill_params(c, p);
  DevLoop d{};
  d.lvl_size = reinterpret_cast<unsigned long long*>(dv);
  d.lvl_begin = d.lvl_size + L;
  d.lvl_slab = d.lvl_begin + L;
  d.lvl_eval = d.lvl_slab + L;
  d.lvl_ns = reinterpret_cast<long long*>(d.lvl_eval + L);
  d.blocks = reinterpret_cast<Block*>(dv + off_blocks);
  d.st = reinterpret_cast<LoopState*>(dv + off_state);
  d.bar = reinterpret_cast<unsigned int*>(dv + off_bar);
  d.hist = reinterpret_cast<unsigned int*>(dv + off_hist);
  const char* ev = getenv("REI_DEVICE_LOOP_CAND");
  d.cand_limit = ev ? strtoull(ev, nullptr, 10) : (1ull << 22);  // A/B: profiles/r02_sweep_loop.txt
  d.entry_limit = p.cap;
  d.slab_limit = c->slab_cap;
  d.sort_min = c->sort_levels ? (1ull << 14) : 0;
  d.c1 = (uint32_t)c1;
  d.first_cost = (uint32_t)from_cost;
  d.max_cost = max_cost;
  d.k_opt = k.opt;
  d.k_star = k.star;
  d.k_cat = k.cat;
  d.k_alt = k.alt;
  d.rows = getenv("REI_LOOP_ROWS") ? (uint32_t)atoi(getenv("REI_LOOP_ROWS")) : 1u;
  EventPair ep;
  c->begin_kernel(REI_K_OTHER, ep);
  const int n = launch_level_loop(c->W32, p, d, c->stream);
  c->end_kernel(ep, n);
  if (!n) {  // not co-resident / not supported: the host loop runs every level
    double ms;
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    c->collect_events(&ms);
    return REI_OK;
  }
  CUDA_OK(c, cudaMemcpyAsync(h, dv, off_state + sizeof(LoopState), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->d2h_bytes += off_state + sizeof(LoopState);
  double loop_ms = 0;
  c->collect_events(&loop_ms);
  const LoopState S = *h_st;
  if (getenv("REI_TRACE"))
    fprintf(stderr, "[rei_solve] device loop levels %d..%u stop %u next %u: %.3f ms\n", from_cost, S.last_cost, S.stop,
            S.next_cost, loop_ms);
  std::vector<Block> cat, uni;
  for (int cost = from_cost; cost <= (int)S.last_cost; ++cost) {
    LevelInfo lv;
    lv.cost = cost;
    uint64_t nq, ns, ncat, nuni;
    plan_level(c, cost, lv, cat, uni, nq, ns, ncat, nuni);
    if (lv.plan.empty()) continue;
    lv.begin = h_begin[cost];
    lv.size = h_size[cost];
    lv.slab = h_slab[cost];
    const bool found_here = S.stop == LOOP_FOUND && cost == (int)S.last_cost;
    const uint64_t total = nq + ns + ncat + nuni;
    rei_level_stat st{};
    st.cost = (uint32_t)cost;
    st.cand_q = nq; st.cand_s = ns; st.cand_c = ncat; st.cand_u = nuni;
    st.unique = lv.size;
    st.ms = h_ns[cost] * 1e-6;
    const bool complete = !found_here || (c->flags & REI_FLAG_COMPLETE_FINAL_LEVEL);
    st.complete = complete ? 1 : 0;
    st.evaluated = complete ? total : h_eval[cost];
    st.eval_c = complete ? ncat : 0;
    st.eval_u = complete ? nuni : 0;
    c->levels[cost] = lv;
    c->stats.push_back(st);
    if (found_here) {
      c->arena_used = lv.begin + lv.size;
      c->result.candidates = *cand + st.evaluated;
      if (complete) {
        c->result.last_complete_cost = (uint32_t)cost;
        c->result.cand_complete = *cand + st.evaluated;
      }
      *done = true;
      return finish_found(c, cost, S.found_rank);
    }
    *cand += total;
    c->result.cand_complete = *cand;
    c->result.candidates = *cand;
    c->result.last_complete_cost = (uint32_t)cost;
  }
  c->arena_used = S.arena_used;
  c->slabs_used = S.slabs_used;
  *next = (int)S.next_cost;
  if (S.stop == LOOP_OVERFLOW) return rebuild_dedup(c, c->arena_used);  // drop the partial level
  if (S.stop == LOOP_SORT) {  // the host orders the last level, then transposes it
    LevelInfo& lv = c->levels.at((int)S.last_cost);
    std::string err;
    if (!sort_level((uint32_t)c->tab.n, c->arena + lv.begin, c->bp + lv.begin, lv.size, c->merge, c->stream, err,
                    &c->launches, true)) {
      c->err = err;
      return REI_ECUDA;
    }
    lv.slab = c->slabs_used;
    EventPair et;
    c->begin_kernel(REI_K_TRANSPOSE, et);
    const int nt = launch_transpose(c->W32, c->arena, lv.begin, lv.size, c->tarena, lv.slab, c->stream);
    c->end_kernel(et, nt);
    c->slabs_used += (lv.size + 31) / 32;
  }
  return REI_OK;
}

// Multi-rank transport of the sharded level.  `m` holds the ranks
// driven by this process: all `world` ranks (virtual ranks, rei_solve_group: device /
// peer copies) or exactly one (one process per GPU: NCCL, or -- host_xport -- the
// caller's host all-gather callback, e.g. torch.distributed gloo).
struct Comm {
  int world = 1;
  int rank0 = 0;
  std::vector<Ctx*> m;
  void* nccl = nullptr;  // ncclComm_t of m[0] when each process holds one rank
  bool host = false;     // one rank per process, exchanging through m[0]->allgather
};

void reset_search(Ctx* c) {
  c->otf_level = 0;
  c->levels.clear();
  c->stats.clear();
  c->regex.clear();
  c->arena_used = 0;
  c->slabs_used = 0;
  memset(&c->result, 0, sizeof(c->result));
  c->result.n_ic = (uint32_t)c->tab.n;
  c->result.cs_words = (uint32_t)c->W32;
}

rei_status host_allgather(Ctx* c, const void* send, void* recv, size_t bytes, const char* what) {
  if (c->allgather(c->allgather_user, send, recv, bytes) != 0) {
    c->err = std::string("allgather callback failed (") + what + ")";
    return REI_ENCCL;
  }
  return REI_OK;
}

// Every rank's control line, in rank order, on every member.
rei_status gather_ctl(Comm& g, std::vector<LevelCtl>& all) {
  all.assign(g.world, LevelCtl{});
  if (!g.nccl && !g.host) {
    for (size_t i = 0; i < g.m.size(); ++i) all[g.rank0 + i] = *g.m[i]->h_ctl;
    return REI_OK;
  }
  Ctx* c = g.m[0];
  if (g.host) return host_allgather(c, c->h_ctl, all.data(), sizeof(LevelCtl), "level control");
  if (nccl_api().AllGather(c->ctl, c->d_ctl_all, sizeof(LevelCtl), ncclUint8, (ncclComm_t)g.nccl, c->stream) !=
      ncclSuccess) {
    c->err = "ncclAllGather(level control) failed";
    return REI_ENCCL;
  }
  CUDA_OK(c, cudaMemcpyAsync(all.data(), c->d_ctl_all, sizeof(LevelCtl) * g.world, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->d2h_bytes += sizeof(LevelCtl) * g.world;
  return REI_OK;
}

// All-gather of k host u64 per rank: out[r * k + j] = rank r's value j.
rei_status x_gather_u64(Comm& g, const std::vector<std::vector<uint64_t>>& mine, size_t k,
                        std::vector<uint64_t>& out) {
  out.assign((size_t)g.world * k, 0);
  if (!g.nccl && !g.host) {
    for (size_t i = 0; i < g.m.size(); ++i)
      std::copy(mine[i].begin(), mine[i].begin() + k, out.begin() + (g.rank0 + i) * k);
    return REI_OK;
  }
  Ctx* c = g.m[0];
  if (g.host) return host_allgather(c, mine[0].data(), out.data(), k * 8, "counts");
  if (k > 64) { c->err = "x_gather_u64: k > 64"; return REI_EINVAL; }
  CUDA_OK(c, cudaMemcpyAsync(c->d_small, mine[0].data(), k * 8, cudaMemcpyHostToDevice, c->stream));
  if (nccl_api().AllGather(c->d_small, c->d_small_all, k * 8, ncclUint8, (ncclComm_t)g.nccl, c->stream) !=
      ncclSuccess) {
    c->err = "ncclAllGather(counts) failed";
    return REI_ENCCL;
  }
  CUDA_OK(c, cudaMemcpyAsync(out.data(), c->d_small_all, (size_t)g.world * k * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->h2d_bytes += k * 8;
  c->d2h_bytes += (size_t)g.world * k * 8;
  return REI_OK;
}

// All-to-all of variable-size record buckets: rank r sends cnt[r][o] records from
// send[r] + soff(r, o) to rank o, which receives them at recv[o] + roff(o, r)
// (sources in rank order).  send / recv are indexed by member.
rei_status x_alltoallv(Comm& g, const std::vector<const uint8_t*>& send, const std::vector<uint8_t*>& recv,
                       const std::vector<uint64_t>& cnt, size_t rec) {
  const int W = g.world;
  // offsets of bucket o in rank r's send list / of source r in rank o's receive list
  std::vector<uint64_t> so((size_t)W * (W + 1)), ro((size_t)W * (W + 1));
  for (int r = 0; r < W; ++r) {
    rei_exchange_offsets(W, cnt.data(), r, &so[(size_t)r * (W + 1)], &ro[(size_t)r * (W + 1)]);
    so[(size_t)r * (W + 1) + W] = so[(size_t)r * (W + 1) + W - 1] + cnt[(size_t)r * W + W - 1];
    ro[(size_t)r * (W + 1) + W] = ro[(size_t)r * (W + 1) + W - 1] + cnt[(size_t)(W - 1) * W + r];
  }
  auto soff = [&](int r, int o) { return so[(size_t)r * (W + 1) + o]; };
  auto roff = [&](int o, int r) { return ro[(size_t)o * (W + 1) + r]; };
  if (!g.nccl && !g.host) {
    for (Ctx* c : g.m) CUDA_OK(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < g.m.size(); ++i) {        // destination
      Ctx* d = g.m[i];
      const int o = g.rank0 + (int)i;
      for (size_t j = 0; j < g.m.size(); ++j) {      // source
        const int r = g.rank0 + (int)j;
        const uint64_t n = cnt[(size_t)r * W + o];
        if (!n) continue;
        CUDA_OK(d, cudaMemcpyPeerAsync(recv[i] + roff(o, r) * rec, d->device, send[j] + soff(r, o) * rec,
                                       g.m[j]->device, n * rec, d->stream));
      }
    }
    for (Ctx* c : g.m) CUDA_OK(c, cudaStreamSynchronize(c->stream));
    return REI_OK;
  }
  Ctx* c = g.m[0];
  const int me = g.rank0;
  if (g.host) {
    uint64_t maxb = 0;
    for (int r = 0; r < W; ++r) maxb = std::max<uint64_t>(maxb, soff(r, W) * rec);
    maxb = std::max<uint64_t>(maxb, 8);
    std::vector<uint8_t> mine(maxb, 0), all((size_t)W * maxb);
    if (soff(me, W))
      CUDA_OK(c, cudaMemcpyAsync(mine.data(), send[0], soff(me, W) * rec, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    rei_status s = host_allgather(c, mine.data(), all.data(), maxb, "level records");
    if (s != REI_OK) return s;
    for (int r = 0; r < W; ++r) {
      const uint64_t n = cnt[(size_t)r * W + me];
      if (n)
        CUDA_OK(c, cudaMemcpyAsync(recv[0] + roff(me, r) * rec, all.data() + (size_t)r * maxb + soff(r, me) * rec,
                                   n * rec, cudaMemcpyHostToDevice, c->stream));
    }
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    c->d2h_bytes += soff(me, W) * rec;
    c->h2d_bytes += roff(me, W) * rec;
    return REI_OK;
  }
  // NCCL: grouped point-to-point sends / receives (the self bucket is a local copy)
  const uint64_t self = cnt[(size_t)me * W + me];
  if (self)
    CUDA_OK(c, cudaMemcpyAsync(recv[0] + roff(me, me) * rec, send[0] + soff(me, me) * rec, self * rec,
                               cudaMemcpyDeviceToDevice, c->stream));
  nccl_api().GroupStart();
  for (int o = 0; o < W; ++o) {
    if (o == me) continue;
    const uint64_t ns = cnt[(size_t)me * W + o], nr = cnt[(size_t)o * W + me];
    if (ns) nccl_api().Send(send[0] + soff(me, o) * rec, ns * rec, ncclUint8, o, (ncclComm_t)g.nccl, c->stream);
    if (nr) nccl_api().Recv(recv[0] + roff(me, o) * rec, nr * rec, ncclUint8, o, (ncclComm_t)g.nccl, c->stream);
  }
  if (nccl_api().GroupEnd() != ncclSuccess) {
    c->err = "NCCL all-to-all of the level records failed";
    return REI_ENCCL;
  }
  return REI_OK;
}

// All-gather of variable-size record lists: rank r's u[r] records from send[r] land at
// recv + uoff(r) on every rank (rank order).
rei_status x_allgatherv(Comm& g, const std::vector<const uint8_t*>& send, const std::vector<uint8_t*>& recv,
                        const std::vector<uint64_t>& u, size_t rec) {
  const int W = g.world;
  std::vector<uint64_t> uoff(W + 1, 0);
  for (int r = 0; r < W; ++r) uoff[r + 1] = uoff[r] + u[r];
  if (!g.nccl && !g.host) {
    for (Ctx* c : g.m) CUDA_OK(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < g.m.size(); ++i)
      for (size_t j = 0; j < g.m.size(); ++j) {
        const int r = g.rank0 + (int)j;
        if (!u[r]) continue;
        CUDA_OK(g.m[i], cudaMemcpyPeerAsync(recv[i] + uoff[r] * rec, g.m[i]->device, send[j], g.m[j]->device,
                                            u[r] * rec, g.m[i]->stream));
      }
    for (Ctx* c : g.m) CUDA_OK(c, cudaStreamSynchronize(c->stream));
    return REI_OK;
  }
  Ctx* c = g.m[0];
  const int me = g.rank0;
  if (g.host) {
    uint64_t maxb = 8;
    for (int r = 0; r < W; ++r) maxb = std::max<uint64_t>(maxb, u[r] * rec);
    std::vector<uint8_t> mine(maxb, 0), all((size_t)W * maxb);
    if (u[me]) CUDA_OK(c, cudaMemcpyAsync(mine.data(), send[0], u[me] * rec, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    rei_status s = host_allgather(c, mine.data(), all.data(), maxb, "level uniques");
    if (s != REI_OK) return s;
    for (int r = 0; r < W; ++r)
      if (u[r])
        CUDA_OK(c, cudaMemcpyAsync(recv[0] + uoff[r] * rec, all.data() + (size_t)r * maxb, u[r] * rec,
                                   cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    c->d2h_bytes += u[me] * rec;
    c->h2d_bytes += uoff[W] * rec;
    return REI_OK;
  }
  nccl_api().GroupStart();
  for (int r = 0; r < W; ++r) {
    if (!u[r]) continue;
    nccl_api().Broadcast(r == me ? (const void*)send[0] : nullptr, recv[0] + uoff[r] * rec, u[r] * rec, ncclUint8, r,
                         (ncclComm_t)g.nccl, c->stream);
  }
  if (nccl_api().GroupEnd() != ncclSuccess) {
    c->err = "NCCL all-gather of the level uniques failed";
    return REI_ENCCL;
  }
  return REI_OK;
}

// Staging list of a multi-rank level (this rank's locally new CSs), >= n entries.
rei_status ensure_stage(Ctx* c, uint64_t n) {
  if (c->st_cap >= n) return REI_OK;
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->dfree(c->st_cs);
  c->dfree(c->st_bp);
  c->st_cs = nullptr;
  c->st_bp = nullptr;
  const uint64_t cap = std::max<uint64_t>(n, 2 * c->st_cap);
  c->st_cap = 0;
  CUDA_OK(c, c->dmalloc(&c->st_cs, cap * 4ull * c->W32));
  CUDA_OK(c, c->dmalloc(&c->st_bp, cap * 8ull));
  c->st_cap = cap;
  return REI_OK;
}

rei_status grow(Ctx* c, uint64_t need_entries);

// The level exchange of north_star / SURVEY 8(e): every rank buckets its locally new
// CSs (staging list) by hash owner; an all-to-all sends each bucket to its owner; the
// owner keeps one copy of each CS; the owners' unique lists are all-gathered (owner
// order) into every rank's arena at `begin` and inserted into its dedup set.  Every
// rank then holds the same level, byte for byte.  Returns its size.
rei_status exchange_level(Comm& g, uint64_t begin, const std::vector<LevelCtl>& all, uint64_t* out_count) {
  const int W = g.world;
  const size_t nm = g.m.size();
  rei_status s;
  Ctx* c0 = g.m[0];
  const size_t rec = 4ull * (c0->W32 + 2);
  // 1) bucket the staged entries by owner
  std::vector<std::vector<uint64_t>> rows(nm, std::vector<uint64_t>(W, 0));
  for (size_t i = 0; i < nm; ++i) {
    Ctx* c = g.m[i];
    std::string err;
    if (!owner_bucket(c->W32, c->st_cs, c->st_bp, all[g.rank0 + i].count, W, c->xs, c->stream, rows[i].data(), err,
                      &c->launches)) {
      c->err = err;
      return REI_ECUDA;
    }
  }
  // 2) the G x G count matrix on every rank
  std::vector<uint64_t> cnt;
  if ((s = x_gather_u64(g, rows, W, cnt)) != REI_OK) return s;
  // 3) all-to-all of the buckets
  std::vector<const uint8_t*> sp(nm);
  std::vector<uint8_t*> rp(nm);
  std::vector<uint64_t> mo(nm, 0);
  for (size_t i = 0; i < nm; ++i) {
    Ctx* c = g.m[i];
    const int o = g.rank0 + (int)i;
    for (int r = 0; r < W; ++r) mo[i] += cnt[(size_t)r * W + o];
    if (!ensure_recv(c->W32, mo[i], c->xs, c->stream)) { c->err = "exchange receive buffer allocation failed"; return REI_OUT_OF_MEMORY; }
    sp[i] = static_cast<const uint8_t*>(c->xs.send);
    rp[i] = static_cast<uint8_t*>(c->xs.recv);
  }
  if ((s = x_alltoallv(g, sp, rp, cnt, rec)) != REI_OK) return s;
  // 4) owner dedup
  std::vector<std::vector<uint64_t>> un(nm, std::vector<uint64_t>(1, 0));
  for (size_t i = 0; i < nm; ++i) {
    Ctx* c = g.m[i];
    std::string err;
    if (!owner_dedup(c->W32, mo[i], c->xs, c->stream, &un[i][0], err, &c->launches)) {
      c->err = err;
      return REI_ECUDA;
    }
  }
  // 5) owner counts, then the unique lists all-gathered in owner order
  std::vector<uint64_t> u;
  if ((s = x_gather_u64(g, un, 1, u)) != REI_OK) return s;
  uint64_t U = 0;
  for (int r = 0; r < W; ++r) U += u[r];
  for (size_t i = 0; i < nm; ++i) {
    Ctx* c = g.m[i];
    if (!ensure_gather_recs(c->W32, U, c->xs, c->stream)) { c->err = "exchange gather buffer allocation failed"; return REI_OUT_OF_MEMORY; }
    sp[i] = static_cast<const uint8_t*>(c->xs.uniq);
    rp[i] = static_cast<uint8_t*>(c->xs.gath);
  }
  if ((s = x_allgatherv(g, sp, rp, u, rec)) != REI_OK) return s;
  // 6) the level into the arena, and into the dedup set (tentative slots re-pointed)
  for (Ctx* c : g.m) {
    if (begin + U > c->cap && (s = grow(c, begin + U)) != REI_OK) return s;
    if (!unpack_records(c->W32, static_cast<const uint32_t*>(c->xs.gath), U, c->arena + begin * c->W32, c->bp + begin,
                        c->stream, &c->launches)) {
      c->err = "unpack of the exchanged level failed";
      return REI_ECUDA;
    }
    LevelParams p;
    fill_params(c, p);
    p.stage_cs = c->st_cs;
    EventPair ep;
    c->begin_kernel(REI_K_OTHER, ep);
    int n = launch_rehash(c->W32, p, begin, U, c->stream);
    c->end_kernel(ep, n);
    CUDA_OK(c, cudaGetLastError());
  }
  *out_count = U;
  return REI_OK;
}

// staged = a multi-rank level that is exchanged afterwards: new CSs go to the staging
// list (and indexed-hash slots are marked tentative) instead of the arena.
rei_status launch_level(Ctx* c, int rank, int world, int cost, uint64_t begin, uint64_t nq, uint64_t ns,
                        const std::vector<Block>& cat, const std::vector<Block>& uni, bool staged = false) {
  const rei_costs& k = c->costs;
  rei_status s;
  LevelParams p;
  fill_params(c, p);
  p.out_base = begin;
  p.otf = c->otf_level ? 1 : 0;
  if (staged) {
    p.arena_out = c->st_cs;
    p.bp = c->st_bp;
    p.out_base = 0;
    p.cap = c->st_cap;
    p.stage_cs = c->st_cs;
    p.tent = c->mode == DEDUP_HASHIDX ? 0x80000000u : 0u;
  }
  const int part = c->lag_part;  // 0 whole level, 1 binary kernels only, 2 unary kernel only
  if (part != 2 && (s = reset_ctl(c)) != REI_OK) return s;
  if (part != 2 && c->lag_prev_ctl) {  // lagged: this level's arena base from the previous level's count
    launch_next_base(c->lag_prev_ctl, c->d_lag_base + c->lag_prev_par, c->d_lag_base + c->lag_par, c->ctl,
                     part == 1 && c->lag_unary_reads ? c->d_rank_off + c->lag_par : nullptr, c->lag_unary_reads,
                     c->stream);
    ++c->launches;
  }
  // operand blocks -> device (one small H2D per level).  Concatenation blocks are
  // split by orientation (left or right operand sliced): one launch each.
  std::vector<Block> catv[2];
  for (const Block& b : cat) catv[b.slice_a ? 1 : 0].push_back(b);
  for (auto& v : catv) renumber_items(v);
  const std::vector<Block>* lists[3] = {&catv[0], &catv[1], &uni};
  {
    // the pair kernels stage a launch's block table in shared memory next to <= 64 KB
    // of split tables and append stages: refuse a level whose table cannot fit
    static int optin = 0;
    if (!optin && cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device) != cudaSuccess)
      optin = 227 * 1024;
    for (int r = 0; r < 3; ++r)
      if (lists[r]->size() * sizeof(Block) + 64 * 1024 > (size_t)optin) {
        c->err = "level " + std::to_string(cost) + " has " + std::to_string(lists[r]->size()) +
                 " operand blocks in one launch; their table exceeds the shared memory of a CTA";
        return REI_EINVAL;
      }
  }
  Block* hb = (c->lag_active && c->h_blocks_ring) ? c->h_blocks_ring + (size_t)c->lag_par * 3 * Ctx::kMaxBlocks
                                                  : c->h_blocks;
  for (int r = 0; r < 3; ++r) {
    if (lists[r]->empty()) continue;
    std::copy(lists[r]->begin(), lists[r]->end(), hb + r * Ctx::kMaxBlocks);
    CUDA_OK(c, cudaMemcpyAsync(c->d_blocks + r * Ctx::kMaxBlocks, hb + r * Ctx::kMaxBlocks,
                               lists[r]->size() * sizeof(Block), cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += lists[r]->size() * sizeof(Block);
  }
  // this rank's share of every work list (SURVEY 8(e) partition)
  auto share = [&](uint64_t total, LevelParams& q) {
    uint64_t b = 0, e = total;
    rei_partition(total, world, rank, &b, &e);
    q.item_begin = b;
    q.total_items = e;
    return e > b;
  };
  // fork: the level's kernels are independent (they read lower levels and insert
  // through atomics), so ? / * (and union) may run on auxiliary streams
  // small levels run on one stream: their kernels are launch-latency bound and the
  // fork / join events would cost more than the overlap gains
  uint64_t level_cand = nq + ns;
  for (const Block& b : cat) level_cand += b.cand_count;
  for (const Block& b : uni) level_cand += b.cand_count;
  const uint64_t small = getenv("REI_SMALL_LEVEL") ? strtoull(getenv("REI_SMALL_LEVEL"), nullptr, 10) : 0;
  const int conc = level_cand < small ? 0 : std::min(3, c->concurrency);
  cudaStream_t su = conc >= 1 ? c->aux[0] : c->stream;
  cudaStream_t sn = conc >= 2 ? c->aux[1] : c->stream;
  cudaStream_t sc = conc >= 3 ? c->aux[2] : c->stream;
  if ((c->concurrency == 5 || c->concurrency == 6) && conc >= 3) {
    // union on the context's stream (no event wait: it reaches the SMs first), concat on
    // an auxiliary stream: the persistent union grid runs ahead of concat, whose CTAs
    // fill the SMs as union CTAs retire (an early exit at c* is met in union first)
    sn = c->stream;
  }
  // the previous level's sort + transpose (post stream): the unary kernel reads that
  // level (Q / S blocks); concatenation / union blocks wait only if one of them does
  if (c->post_pending) {
    bool binary_reads = conc < 1;
    for (int pl : c->post_levels) {
      const uint64_t pb = c->levels.at(pl).begin;
      for (const Block& b : cat) binary_reads |= b.a_base == pb || b.b_base == pb;
      for (const Block& b : uni) binary_reads |= b.a_base == pb || b.b_base == pb;
    }
    if (binary_reads) c->join_post();
  }
  if (part != 2) c->level_mark(0);
  if (conc >= 1) {
    if (part != 2) {  // part 2 runs on the streams part 1 forked
      CUDA_OK(c, cudaEventRecord(c->ev_fork, c->stream));
      for (int i = 0; i < conc; ++i) CUDA_OK(c, cudaStreamWaitEvent(c->aux[i], c->ev_fork, 0));
    }
    if (part != 1) {
      c->wait_post(su);  // su = aux[0]: the unary kernel
      c->post_pending = false;  // the join below makes the context's stream wait for su
      c->post_levels.clear();
    }
  }
  if (part != 1 && nq + ns) {
    const uint64_t bq = nq ? c->levels.at(cost - (int)k.opt).begin : 0;
    const uint64_t bs = ns ? c->levels.at(cost - (int)k.star).begin : 0;
    const uint64_t slab_s = ns ? c->levels.at(cost - (int)k.star).slab : 0;
    LevelParams pq = p;
    if (share(nq + ns, pq)) {
      EventPair ep;
      c->begin_kernel(REI_K_UNARY, ep, su);
      int n = launch_unary(c->W32, pq, nq, ns, bq, bs, nq, slab_s, su);
      c->end_kernel(ep, n);
    }
  }
  auto launch_cat = [&]() -> rei_status {
    for (int r = 0; r < 2; ++r) {
      if (catv[r].empty()) continue;
      LevelParams pc = p;
      pc.blocks = c->d_blocks + r * Ctx::kMaxBlocks;
      pc.nblocks = (uint32_t)catv[r].size();
      if (!share(items_of(catv[r]), pc)) continue;
      EventPair ep;
      c->begin_kernel(REI_K_CONCAT, ep, sc);
      int n = launch_concat(c->W32, pc, r == 1, sc);
      c->end_kernel(ep, n);
    }
    return REI_OK;
  };
  auto launch_uni = [&]() -> rei_status {
    if (uni.empty()) return REI_OK;
    LevelParams pu = p;
    pu.blocks = c->d_blocks + 2 * Ctx::kMaxBlocks;
    pu.nblocks = (uint32_t)uni.size();
    if (share(items_of(uni), pu)) {
      EventPair ep;
      c->begin_kernel(REI_K_UNION, ep, sn);
      int n = launch_union(c->W32, pu, sn);
      c->end_kernel(ep, n);
    }
    return REI_OK;
  };
  // union first (bitmap dedup default, REI_UNION_FIRST): the union kernel takes the SMs
  // first, so a precise union is met early at c* (see rei_init)
  if (part != 2) {
    if (c->union_first) { launch_uni(); launch_cat(); } else { launch_cat(); launch_uni(); }
  }
  if (part == 1) {  // split level: the unary part (part 2) joins the streams
    CUDA_OK(c, cudaGetLastError());
    return REI_OK;
  }
  if (conc >= 1) {  // join
    for (int i = 0; i < conc; ++i) {
      CUDA_OK(c, cudaEventRecord(c->ev_join[i], c->aux[i]));
      CUDA_OK(c, cudaStreamWaitEvent(c->stream, c->ev_join[i], 0));
    }
  }
  c->level_mark(1);
  CUDA_OK(c, cudaGetLastError());
  return REI_OK;
}

// Does level `cost` need a level that OnTheFly mode checked but did not cache?  A
// block with an uncached operand level is needed unless its other operand level is
// known to be empty.
bool needs_uncached(const Ctx* c, int cost) {
  const rei_costs& k = c->costs;
  const int c1 = (int)k.sym;
  auto unk = [&](int L) { return c->otf_level && L >= c->otf_level; };
  auto maybe = [&](int L) { return L >= c1 && (unk(L) || level_size(c, L) > 0); };
  if (unk(cost - (int)k.opt) || unk(cost - (int)k.star)) return true;
  for (int L = c1; L <= cost - (int)k.cat - c1; ++L) {
    const int R = cost - (int)k.cat - L;
    if ((unk(L) && maybe(R)) || (unk(R) && maybe(L))) return true;
  }
  for (int L = c1; L <= cost - (int)k.alt - L; ++L) {
    const int R = cost - (int)k.alt - L;
    if ((unk(L) && maybe(R)) || (unk(R) && maybe(L))) return true;
  }
  return false;
}

// Algorithm 1 over all ranks of `g` (world = 1: the single-GPU path, no exchange).
// ============================================================================
// Lagged level loop (single rank).  A level that does not read the level launched just
// before it -- its unary operands are levels c - c_opt, c - c_star and its binary
// operands sum to c - c_cat / c - c_alt, so with unary costs > 1 (Table 1 row 8:
// (10,10,10,1,10)) it never reads level c - 1 -- is planned and launched before that
// level's count has come back: its arena base is computed on the device from the
// previous level's count (k_next_base) and its control line alternates with the
// previous one's.  At most two levels are in flight; a level is finalised (count,
// precision, statistics, sort / transpose on the post stream) when a later level needs
// it, or one level later.  The capacity for both is reserved up front (every candidate
// new at worst); an overflow, a growth the budget refuses or an OnTheFly switch hands
// the search back to the synchronous loop at that level.  A precise candidate in the
// older level makes the younger one exit at once (k_next_base marks it) and the result
// is the older level's.  REI_NO_LAG=1 turns it off.
bool lag_ok(const Ctx* c) {
  return !c->sharded && !c->otf_level && c->world == 1 && !c->exchange_self && !c->kernel_events &&
         (c->mode == DEDUP_BITMAP || c->mode == DEDUP_HASH64) && c->W32 <= 2 &&
         !(c->flags & REI_FLAG_COMPLETE_FINAL_LEVEL) && getenv("REI_NO_LAG") == nullptr;
}

rei_status solve_lagged(Ctx* c, uint32_t max_cost, int* first_cost, uint64_t* cand, bool* done) {
  *done = false;
  const rei_costs& k = c->costs;
  const int c1 = (int)k.sym;
  rei_status s;
  constexpr int K = Ctx::kLag;
  if (!c->d_lag_base && c->dmalloc(&c->d_lag_base, K * sizeof(unsigned long long)) != cudaSuccess) return REI_OK;
  if (!c->h_lag && host_alloc(reinterpret_cast<void**>(&c->h_lag), K * sizeof(LevelCtl)) != cudaSuccess) return REI_OK;
  if (!c->h_lag_base && host_alloc(reinterpret_cast<void**>(&c->h_lag_base), K * 8) != cudaSuccess) return REI_OK;
  if (!c->h_blocks_ring && host_alloc(reinterpret_cast<void**>(&c->h_blocks_ring),
                                      sizeof(Block) * K * 3 * Ctx::kMaxBlocks) != cudaSuccess)
    return REI_OK;
  if (!c->d_rank_off && c->dmalloc(&c->d_rank_off, K * sizeof(unsigned long long)) != cudaSuccess) return REI_OK;
  const bool split_ok = getenv("REI_NO_SPLIT") == nullptr;
  for (auto& e : c->ev_lag)
    if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return REI_OK;
  struct Fly {
    int cost;
    LevelInfo lv;
    uint64_t nq, ns, ncat, nuni;
    int par;
  };
  std::deque<Fly> fly;
  std::vector<Block> cat, uni;
  const bool trace = getenv("REI_TRACE") != nullptr;
  auto reads = [&](int cost, int x) {
    return cost - (int)k.opt == x || cost - (int)k.star == x || cost - (int)k.cat - x >= c1 ||
           cost - (int)k.alt - x >= c1;
  };
  auto total = [](const Fly& f) { return f.nq + f.ns + f.ncat + f.nuni; };
  // finalise the oldest level in flight; *stop: the search ended (found) or goes back
  // to the synchronous loop (*first_cost set)
  auto finalize = [&](bool* stop) -> rei_status {
    Fly f = fly.front();
    fly.pop_front();
    CUDA_OK(c, cudaEventSynchronize(c->ev_lag[f.par]));
    const LevelCtl ctl = c->h_lag[f.par];
    c->d2h_bytes += sizeof(LevelCtl);
    c->ev_par = f.par;
    double ms = 0;
    c->collect_events(&ms);
    if (ctl.overflow) {  // redo from this level in the synchronous loop (younger levels exit at once)
      CUDA_OK(c, cudaStreamSynchronize(c->stream));
      fly.clear();
      rei_status r = rebuild_dedup(c, c->arena_used);
      *first_cost = f.cost;
      *stop = true;
      return r;
    }
    const bool found = ctl.found_rank != ~0ull;
    f.lv.begin = c->arena_used;
    f.lv.size = ctl.count;
    f.lv.slab = c->slabs_used;
    rei_level_stat st{};
    st.cost = (uint32_t)f.cost;
    st.cand_q = f.nq; st.cand_s = f.ns; st.cand_c = f.ncat; st.cand_u = f.nuni;
    st.unique = f.lv.size;
    st.ms = ms;
    st.complete = found ? 0 : 1;
    st.evaluated = found ? ctl.evaluated : total(f);
    st.eval_c = found ? ctl.eval_c : f.ncat;
    st.eval_u = found ? ctl.eval_u : f.nuni;
    if (trace) fprintf(stderr, "[rei_solve] level %3d (lagged) device %8.3f ms\n", f.cost, ms);
    c->levels[f.cost] = f.lv;
    c->stats.push_back(st);
    if (found) {
      CUDA_OK(c, cudaStreamSynchronize(c->stream));  // the younger level saw the mark and exited
      fly.clear();
      c->arena_used = f.lv.begin + f.lv.size;
      c->result.candidates = *cand + st.evaluated;
      *stop = true;
      *done = true;
      return finish_found(c, f.cost, ctl.found_rank);
    }
    *cand += total(f);
    c->result.cand_complete = *cand;
    c->result.candidates = *cand;
    c->result.last_complete_cost = (uint32_t)f.cost;
    c->arena_used += f.lv.size;
    // sort + transpose after this level's kernels only (younger levels never read it)
    cudaStream_t ps = c->post ? c->post : c->stream;
    if (c->post) CUDA_OK(c, cudaStreamWaitEvent(c->post, c->ev_lag[f.par], 0));
    if (c->sort_levels && f.lv.size >= (1u << 14)) {
      std::string err;
      if (!sort_level((uint32_t)c->tab.n, c->arena + f.lv.begin, c->bp + f.lv.begin, f.lv.size, c->merge, ps, err,
                      &c->launches, true)) {
        c->err = err;
        return REI_ECUDA;
      }
    }
    EventPair et;
    c->begin_kernel(REI_K_TRANSPOSE, et, ps);
    const int n = launch_transpose(c->W32, c->arena, f.lv.begin, f.lv.size, c->tarena, f.lv.slab, ps);
    c->end_kernel(et, n);
    c->slabs_used += (f.lv.size + 31) / 32;
    if (c->post) {
      CUDA_OK(c, cudaEventRecord(c->ev_post, c->post));
      c->post_pending = true;
      c->post_level = f.cost;
      c->post_levels.push_back(f.cost);
    }
    *stop = false;
    return REI_OK;
  };
  auto drain = [&](bool* stop) -> rei_status {
    *stop = false;
    while (!fly.empty() && !*stop)
      if ((s = finalize(stop)) != REI_OK) return s;
    return REI_OK;
  };
  for (int cost = *first_cost; cost <= (int)max_cost; ++cost) {
    bool stop = false;
    // split level: when the only level in flight is read by this level's ? / * blocks
    // alone, its binary kernels go first (they never read it) and the unary kernel
    // follows once that level is final
    auto binary_reads = [&](int x) { return cost - (int)k.cat - x >= c1 || cost - (int)k.alt - x >= c1; };
    const bool split = split_ok && fly.size() == 1 && !binary_reads(fly.back().cost) &&
                       (cost - (int)k.opt == fly.back().cost || cost - (int)k.star == fly.back().cost);
    // finalise what this level reads (and everything older), and keep at most K - 2
    // levels in flight under it
    while (!split && !fly.empty()) {
      bool need = fly.size() >= (size_t)(K - 1);
      for (const Fly& f : fly) need |= reads(cost, f.cost);
      if (!need) break;
      if ((s = finalize(&stop)) != REI_OK) return s;
      if (stop) return REI_OK;
    }
    LevelInfo lv;
    lv.cost = cost;
    uint64_t nq, ns, ncat, nuni;
    plan_level(c, cost, lv, cat, uni, nq, ns, ncat, nuni);
    if (lv.plan.empty() && !split) continue;  // (split: the ? / * blocks of the level in flight)
    uint64_t tot = nq + ns + ncat + nuni;
    uint64_t infl = 0;
    for (const Fly& f : fly) infl += total(f);
    // a split level also has the ? / * candidates of the level in flight (<= 2 x its candidates)
    const uint64_t need = tot + (split ? 2 * infl : 0);
    const uint64_t cap = c->entry_limit ? std::min<uint64_t>(c->cap, c->entry_limit) : c->cap;
    if (!fly.empty() && (c->arena_used + infl + need > cap || c->slabs_used + (infl + need) / 32 + 4 > c->slab_cap)) {
      if ((s = drain(&stop)) != REI_OK) return s;
      if (stop) return REI_OK;
      if (split) {  // the level in flight is final now: plan the whole level
        plan_level(c, cost, lv, cat, uni, nq, ns, ncat, nuni);
        tot = nq + ns + ncat + nuni;
        if (lv.plan.empty()) continue;
      }
    }
    if (fly.empty()) {  // as the synchronous loop: grow ahead when the level may not fit
      const uint64_t prev = c->stats.empty() ? 0 : c->stats.back().unique;
      const uint64_t expect = std::min<uint64_t>(tot, 4 * prev + 1024);
      if (c->arena_used + expect > c->cap || c->slabs_used + expect / 32 + 2 > c->slab_cap) {
        if ((s = grow(c, c->arena_used + expect)) != REI_OK) {
          if (s != REI_OUT_OF_MEMORY) return s;
          *first_cost = cost;  // the synchronous loop handles OnTheFly
          return REI_OK;
        }
      }
    }
    const int par = (c->lag_par + 1) % K;  // round robin: in-order finalisation frees slots in order
    c->ctl = c->ctl_base + par;
    c->ev_par = par;
    if (!fly.empty()) {
      c->lag_prev_ctl = c->ctl_base + fly.back().par;
      c->lag_prev_par = fly.back().par;
    } else {  // a host-known base, on the device for the next level to chain from
      c->h_lag_base[par] = c->arena_used;
      CUDA_OK(c, cudaMemcpyAsync(c->d_lag_base + par, c->h_lag_base + par, 8, cudaMemcpyHostToDevice, c->stream));
    }
    c->lag_par = par;
    lv.begin = c->arena_used;  // final only when nothing is in flight
    c->lag_active = true;
    if (split && !fly.empty()) {
      const int x = fly.back().cost;
      c->lag_unary_reads = (cost - (int)k.opt == x ? 1u : 0u) + (cost - (int)k.star == x ? 1u : 0u);
      c->lag_part = 1;  // binary kernels now (nq, ns of the level in flight counted on the device)
      s = launch_level(c, 0, 1, cost, lv.begin, 0, 0, cat, uni, false);
      c->lag_part = 0;
      c->lag_prev_ctl = nullptr;
      c->lag_active = false;
      if (s != REI_OK) return s;
      if ((s = finalize(&stop)) != REI_OK) return s;  // the level the unary blocks read
      if (stop) return REI_OK;
      plan_level(c, cost, lv, cat, uni, nq, ns, ncat, nuni);  // the full plan (ranks as the device's)
      if (lv.plan.empty()) {  // the level in flight came back empty: no level at this cost
        c->lag_unary_reads = 0;
        continue;
      }
      lv.begin = c->arena_used;
      c->ctl = c->ctl_base + par;
      c->ev_par = par;
      c->lag_par = par;
      c->lag_part = 2;  // the unary kernel; appends from the device base of this level
      c->lag_active = true;
      std::vector<Block> none;
      s = launch_level(c, 0, 1, cost, lv.begin, nq, ns, none, none, false);
      c->lag_part = 0;
      c->lag_unary_reads = 0;
    } else {
      s = launch_level(c, 0, 1, cost, lv.begin, nq, ns, cat, uni, false);
    }
    c->lag_active = false;
    c->lag_prev_ctl = nullptr;
    if (s != REI_OK) return s;
    CUDA_OK(c, cudaMemcpyAsync(c->h_lag + par, c->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(c, cudaEventRecord(c->ev_lag[par], c->stream));
    fly.push_back({cost, lv, nq, ns, ncat, nuni, par});
  }
  bool stop = false;
  if ((s = drain(&stop)) != REI_OK) return s;
  if (!stop) *first_cost = (int)max_cost + 1;
  c->ctl = c->ctl_base;
  c->ev_par = 0;
  return REI_OK;
}

rei_status solve_group(Comm& g, uint32_t max_cost) {
  Ctx* c0 = g.m[0];
  const rei_costs& k = c0->costs;
  const int c1 = (int)k.sym;
  const bool multi = g.world > 1 || c0->exchange_self;
  rei_status s;
  for (Ctx* c : g.m) reset_search(c);
  uint64_t cand = 1;  // Alg. 1 line 1: the empty regex is the first candidate (A9)

  const uint64_t total_ex = c0->P.size() + c0->N.size();
  const bool empty_ok = c0->P.empty() ||
                        (c0->err_num && (uint64_t)c0->P.size() * c0->err_den <= (uint64_t)c0->err_num * total_ex);
  const bool eps_ok = c0->P.size() == 1 && c0->P[0].empty();  // Alg. 1 line 2
  if (empty_ok || eps_ok) {
    for (Ctx* c : g.m) {
      c->regex = empty_ok ? "empty" : "eps";
      c->result.cost = k.sym;
      c->result.candidates = cand;
    }
    return REI_OK;
  }
  // levels with fewer candidates than this run on every rank (no exchange; SURVEY
  // 8(e) "early levels"), then sorted into a rank-independent order (|IC| <= 64)
  const uint64_t redundant_below =
      getenv("REI_REDUNDANT_CAND") ? strtoull(getenv("REI_REDUNDANT_CAND"), nullptr, 10) : 50000000ull;

  // ---- level c1: the alphabet symbols (Alg. 1 line 3), identical on every rank
  uint64_t found_seed = ~0ull;
  for (Ctx* c : g.m) {
    if ((s = clear_dedup(c)) != REI_OK) return s;
    LevelInfo lv;
    lv.cost = c1;
    lv.seeds = true;
    LevelParams p;
    fill_params(c, p);
    p.out_base = 0;
    if ((s = reset_ctl(c)) != REI_OK) return s;
    EventPair ep;
    c->begin_kernel(REI_K_OTHER, ep);
    int n = launch_seeds(c->W32, p, c->tab.seeds, (int)c->alphabet.size(), c->stream);
    c->end_kernel(ep, n);
    CUDA_OK(c, cudaGetLastError());
    if ((s = read_ctl(c)) != REI_OK) return s;
    double ms;
    c->collect_events(&ms);
    lv.size = c->h_ctl->count;
    c->levels[c1] = lv;
    c->arena_used = lv.size;
    rei_level_stat st{};
    st.cost = c1;
    st.unique = lv.size;
    st.ms = ms;
    found_seed = c->h_ctl->found_rank;
    st.complete = found_seed == ~0ull ? 1 : 0;
    c->stats.push_back(st);
  }
  if (found_seed != ~0ull) {
    for (Ctx* c : g.m) {
      c->result.candidates = 1 + found_seed + 1;
      if ((s = finish_found(c, c1, found_seed)) != REI_OK) return s;
    }
    return REI_OK;
  }
  cand += c0->alphabet.size();
  for (Ctx* c : g.m) {
    EventPair et;
    c->begin_kernel(REI_K_TRANSPOSE, et);
    int n = launch_transpose(c->W32, c->arena, 0, c->arena_used, c->tarena, 0, c->stream);
    c->end_kernel(et, n);
    c->slabs_used = (c->arena_used + 31) / 32;
    c->result.last_complete_cost = c1;
    c->result.cand_complete = cand;
  }

  int first_cost = c1 + 1;
  const bool loop_ok = !multi && g.m.size() == 1 && device_loop_ok(c0, max_cost);
  if (loop_ok) {
    bool done = false;
    if ((s = device_levels(c0, max_cost, c1 + 1, &first_cost, &cand, &done)) != REI_OK) return s;
    if (done) return REI_OK;
  }
  if (!multi && g.m.size() == 1 && lag_ok(c0)) {
    bool done = false;
    if ((s = solve_lagged(c0, max_cost, &first_cost, &cand, &done)) != REI_OK) return s;
    c0->ctl = c0->ctl_base;
    c0->ev_par = 0;
    if (done) return REI_OK;
  }
  // REI_LOOP_RESUME=1: after a big level on the host, a run of small levels goes back to
  // the device loop (A/B on B200: Table 1 row 8, whose big levels alternate with runs
  // of small ones, 45.0 ms either way -- a resumed launch costs about what the host
  // round trips of the small levels it takes over do; off by default)
  const char* lce = getenv("REI_DEVICE_LOOP_CAND");
  const uint64_t loop_limit = lce ? strtoull(lce, nullptr, 10) : (1ull << 22);
  const bool loop_resume = loop_ok && getenv("REI_LOOP_RESUME") != nullptr;

  std::vector<Block> cat, uni;
  std::vector<LevelCtl> all;
  const bool trace = getenv("REI_TRACE") != nullptr;
  auto t_level = std::chrono::steady_clock::now();
  for (int cost = first_cost; cost <= (int)max_cost; ++cost) {
    if (c0->otf_level && needs_uncached(c0, cost)) {
      // OnTheFly mode needs a level it did not cache: stop
      for (Ctx* c : g.m) c->result.candidates = c->result.cand_complete;
      return REI_OUT_OF_MEMORY;
    }
    const bool otf = c0->otf_level != 0;
    LevelInfo lv;
    lv.cost = cost;
    uint64_t nq, ns, ncat, nuni;
    plan_level(c0, cost, lv, cat, uni, nq, ns, ncat, nuni);  // identical on every rank
    if (lv.plan.empty()) continue;
    if (loop_resume && !otf && cost > first_cost && nq + ns + ncat + nuni <= loop_limit) {
      bool done = false;
      int next = cost;
      if ((s = device_levels(c0, max_cost, cost, &next, &cand, &done)) != REI_OK) return s;
      if (done) return REI_OK;
      if (next > cost) {  // the loop finished levels cost .. next - 1
        cost = next - 1;
        continue;
      }
    }
    if ((int)(cat.size() + uni.size()) > Ctx::kMaxBlocks) {
      c0->err = "too many operand blocks in one level";
      return REI_EINVAL;
    }
    // grow ahead of the level when its new CSs may not fit (a level rarely has more
    // than ~4x the previous level's new CSs; an overflow still triggers a retry).  In
    // multi-rank mode a rank also stages its own list there, hence the factor 2.
    const uint64_t prev = c0->stats.empty() ? 0 : c0->stats.back().unique;
    const uint64_t expect = std::min<uint64_t>(nq + ns + ncat + nuni, 4 * prev + 1024);
    // multi-rank: a small level runs whole on every rank; a large one is split by
    // rei_partition and exchanged by hash owner
    const uint64_t level_cand = nq + ns + ncat + nuni;
    const bool redundant = multi && !otf && c0->W32 <= 2 && level_cand < redundant_below;
    const bool staged = multi && !otf && !redundant;
    for (Ctx* c : g.m) {
      if (otf) break;
      if (c->arena_used + expect > c->cap || c->slabs_used + expect / 32 + 2 > c->slab_cap) {
        if ((s = grow(c, c->arena_used + expect)) != REI_OK && s != REI_OUT_OF_MEMORY) return s;
      }
      if (staged && (s = ensure_stage(c, expect)) != REI_OK) return s;
    }
    lv.begin = c0->arena_used;
    lv.slab = c0->slabs_used;
    rei_level_stat st{};
    st.cost = (uint32_t)cost;
    st.cand_q = nq; st.cand_s = ns; st.cand_c = ncat; st.cand_u = nuni;
    double level_ms = 0;
    for (int attempt = 0;; ++attempt) {
      for (size_t i = 0; i < g.m.size(); ++i)
        if ((s = launch_level(g.m[i], redundant ? 0 : g.rank0 + (int)i, redundant ? 1 : g.world, cost, lv.begin, nq,
                              ns, cat, uni, staged)) != REI_OK)
          return s;
      for (Ctx* c : g.m) {
        if ((s = read_ctl(c)) != REI_OK) return s;
        double ms;
        c->collect_events(&ms);
        if (c == c0) level_ms += ms;
      }
      if ((s = gather_ctl(g, all)) != REI_OK) return s;
      bool overflow = false;
      uint64_t need = 0, need_stage = 0;
      for (auto& l : all) {
        overflow |= l.overflow != 0;
        need = std::max<uint64_t>(need, lv.begin + l.count + 1);
        need_stage = std::max<uint64_t>(need_stage, l.count + 1);
      }
      if (!overflow) break;
      if (staged) {
        // the staging list (or the dedup set) overflowed: a larger list, a clean dedup
        // set (drops this attempt's tentative inserts), and the arena if it is short
        bool grew = false;
        for (Ctx* c : g.m) {
          if ((s = ensure_stage(c, std::max<uint64_t>(2 * c->st_cap, need_stage))) != REI_OK) return s;
          if (lv.begin + need_stage > c->cap || attempt >= 1) {
            if ((s = grow(c, std::max<uint64_t>(lv.begin + need_stage, c->cap + 1))) != REI_OK) return s;
            grew = true;
          } else if ((s = rebuild_dedup(c, c->arena_used)) != REI_OK) {
            return s;
          }
        }
        if (attempt > 8 && !grew) {
          c0->err = "multi-rank level keeps overflowing";
          return REI_OUT_OF_MEMORY;
        }
        continue;
      }
      // capacity exceeded: grow the cache / dedup set and redo the level; when the
      // budget is exhausted, switch to OnTheFly mode and re-check the level
      bool to_otf = false;
      for (Ctx* c : g.m) {
        if ((s = grow(c, need)) != REI_OK) {
          if (s == REI_OUT_OF_MEMORY && !(c0->flags & REI_FLAG_NO_ONTHEFLY) && !c0->otf_level) {
            to_otf = true;
            break;
          }
          for (Ctx* d : g.m) d->result.candidates = d->result.cand_complete;
          return s;
        }
      }
      if (to_otf) {
        for (Ctx* c : g.m) {
          c->otf_level = cost;
          if ((s = rebuild_dedup(c, c->arena_used)) != REI_OK) return s;  // drop partial inserts
        }
      }
    }
    if (trace) {
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[rei_solve] level %3d host %8.3f ms device %8.3f ms\n", cost,
              std::chrono::duration<double, std::milli>(now - t_level).count(), level_ms);
      t_level = now;
    }
    const bool otf_now = c0->otf_level != 0;
    uint64_t found_rank = ~0ull, evaluated = 0, eval_c = 0, eval_u = 0;
    for (auto& l : all) {
      found_rank = std::min<uint64_t>(found_rank, l.found_rank);
      evaluated += l.evaluated;
      eval_c += l.eval_c;
      eval_u += l.eval_u;
    }
    const bool found = found_rank != ~0ull;
    const bool complete = !found || (c0->flags & REI_FLAG_COMPLETE_FINAL_LEVEL);
    uint64_t size = otf_now ? 0 : all[g.rank0].count;
    if (staged && complete && !otf_now) {
      if ((s = exchange_level(g, lv.begin, all, &size)) != REI_OK) return s;
    }
    if (redundant && complete && !otf_now) {
      for (Ctx* c : g.m) {
        if (c->h_ctl->count != size) {
          c->err = "ranks disagree on the size of a redundantly computed level";
          return REI_ECUDA;
        }
        std::string err;
        if (!canon_sort_level(c->W32, (uint32_t)c->tab.n, c->arena + lv.begin * c->W32, c->bp + lv.begin, size,
                              c->merge, c->stream, err, &c->launches)) {
          c->err = err;
          return REI_ECUDA;
        }
      }
    }
    lv.size = size;
    st.unique = size;
    st.ms = level_ms;
    st.complete = complete ? (otf_now ? 2 : 1) : 0;
    st.evaluated = complete ? (nq + ns + ncat + nuni) : evaluated;
    st.eval_c = complete ? ncat : eval_c;
    st.eval_u = complete ? nuni : eval_u;
    for (Ctx* c : g.m) {
      c->arena_used = lv.begin + lv.size;
      c->levels[cost] = lv;
      c->stats.push_back(st);
    }
    if (found) {
      for (Ctx* c : g.m) {
        c->result.candidates = cand + st.evaluated;
        if (complete) {
          c->result.last_complete_cost = (uint32_t)cost;
          c->result.cand_complete = cand + st.evaluated;
        }
        if ((s = finish_found(c, cost, found_rank)) != REI_OK) return s;
      }
      return REI_OK;
    }
    cand += nq + ns + ncat + nuni;
    for (Ctx* c : g.m) {
      c->result.cand_complete = cand;
      c->result.candidates = cand;
      c->result.last_complete_cost = (uint32_t)cost;
      if (otf_now) continue;  // nothing cached at this level
      if (c->slabs_used + (lv.size + 31) / 32 > c->slab_cap) {
        if ((s = grow(c, c->cap + 1)) != REI_OK) return s;
      }
      // the level's sort and transpose run on the post stream when this context has one
      // (single rank): the next level's binary kernels start meanwhile (launch_level)
      const bool overlap = c->post && !multi;
      cudaStream_t ps = overlap ? c->post : c->stream;
      if (overlap) {
        CUDA_OK(c, cudaEventRecord(c->ev_level_done, c->stream));
        CUDA_OK(c, cudaStreamWaitEvent(c->post, c->ev_level_done, 0));
      }
      if (c->sort_levels && lv.size >= (1u << 14) && !redundant) {  // bitmap mode: order by bitmap position
        std::string err;
        if (!sort_level((uint32_t)c->tab.n, c->arena + lv.begin, c->bp + lv.begin, lv.size, c->merge, ps, err,
                        &c->launches, g.world == 1)) {
          c->err = err;
          return REI_ECUDA;
        }
      }
      // transposed copy of level c (the sliced-operand layout for later levels)
      EventPair et;
      c->begin_kernel(REI_K_TRANSPOSE, et, ps);
      int n = launch_transpose(c->W32, c->arena, lv.begin, lv.size, c->tarena, lv.slab, ps);
      c->end_kernel(et, n);
      c->slabs_used += (lv.size + 31) / 32;
      if (overlap) {
        CUDA_OK(c, cudaEventRecord(c->ev_post, c->post));
        c->post_pending = true;
        c->post_level = cost;
        c->post_levels.push_back(cost);
      }
    }
  }
  return REI_NOT_FOUND;
}

// ============================================================================
// Sharded cache: capacity over G ranks.  Rank o owns the CSs whose
// hash is o mod G; level L's list is the rank-order concatenation of the owners'
// shards.  Operand blocks are shard pairs read through peer mappings; kernels insert
// every candidate into its owner's dedup set and shard (levels.cu sharded_new).

// Peer buffer views: virtual ranks (one process) use the group's own pointers.
void link_local(std::vector<Ctx*>& m) {
  for (Ctx* c : m) {
    c->peers.clear();
    for (Ctx* o : m)
      c->peers.push_back({o->arena, o->bp, o->tarena, o->ctl_base, o->bitmap, o->table, o->special, o->cap,
                          o->slots});
  }
}

// One process per rank: export every buffer with CUDA IPC, all-gather the handles
// through the caller's callback, open the other ranks' (collective, at rei_init).
rei_status link_ipc(Ctx* c) {
  struct Rec {
    cudaIpcMemHandle_t h[6];
    uint64_t cap, slots;
  };
  Rec mine{};
  void* bufs[6] = {c->arena, c->bp, c->tarena, c->ctl_base,
                   c->mode == DEDUP_BITMAP ? (void*)c->bitmap : (void*)c->table, c->special};
  for (int i = 0; i < 6; ++i) CUDA_OK(c, cudaIpcGetMemHandle(&mine.h[i], bufs[i]));
  mine.cap = c->cap;
  mine.slots = c->slots;
  std::vector<Rec> all(c->world);
  if (c->allgather(c->allgather_user, &mine, all.data(), sizeof(Rec)) != 0) {
    c->err = "allgather callback failed (IPC handle exchange)";
    return REI_ENCCL;
  }
  c->peers.assign(c->world, {});
  for (int r = 0; r < c->world; ++r) {
    void* q[6];
    if (r == c->rank) {
      for (int i = 0; i < 6; ++i) q[i] = bufs[i];
    } else {
      for (int i = 0; i < 6; ++i) {
        CUDA_OK(c, cudaIpcOpenMemHandle(&q[i], all[r].h[i], cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(q[i]);
      }
    }
    Ctx::PeerBuf& b = c->peers[r];
    b.arena = (uint32_t*)q[0];
    b.bp = (unsigned long long*)q[1];
    b.tarena = (uint32_t*)q[2];
    b.ctl_base = (LevelCtl*)q[3];
    b.bitmap = c->mode == DEDUP_BITMAP ? (uint32_t*)q[4] : nullptr;
    b.table = c->mode == DEDUP_BITMAP ? nullptr : (unsigned long long*)q[4];
    b.special = (unsigned int*)q[5];
    b.cap = all[r].cap;
    b.slots = all[r].slots;
  }
  return REI_OK;
}

// The kernels address a peer's level through the member's own arena / tarena base
// (flat 64-bit addresses: offset = byte distance / element size, wrapping), so the
// operand blocks need no per-block pointer.  Buffers are 2 MB-granular allocations.
bool peer_offsets_ok(const Ctx* c) {
  for (const auto& b : c->peers) {
    const int64_t da = (int64_t)((intptr_t)b.arena - (intptr_t)c->arena);
    const int64_t dt = (int64_t)((intptr_t)b.tarena - (intptr_t)c->tarena);
    if (da % (4 * c->W32) || dt % (128 * c->W32)) return false;
  }
  return true;
}
uint64_t rel_entry(const Ctx* c, int o, uint64_t begin) {
  return (uint64_t)((int64_t)((intptr_t)c->peers[o].arena - (intptr_t)c->arena) / (4 * c->W32)) + begin;
}
uint64_t rel_slab(const Ctx* c, int o, uint64_t slab) {
  return (uint64_t)((int64_t)((intptr_t)c->peers[o].tarena - (intptr_t)c->tarena) / (128 * c->W32)) + slab;
}

// Barrier of the ranks of `g` (no-op for virtual ranks: one host thread drives all).
rei_status group_barrier(Comm& g) {
  if ((int)g.m.size() == g.world) return REI_OK;
  Ctx* c = g.m[0];
  char x = 0;
  std::vector<char> r(g.world);
  if (c->allgather(c->allgather_user, &x, r.data(), 1) != 0) {
    c->err = "allgather callback failed (barrier)";
    return REI_ENCCL;
  }
  return REI_OK;
}

// Every rank's control line of this level (after the barrier that follows the kernels).
rei_status read_all_ctl(Comm& g, int parity, std::vector<LevelCtl>& all) {
  Ctx* c = g.m[0];
  all.assign(g.world, LevelCtl{});
  for (int r = 0; r < g.world; ++r)
    CUDA_OK(c, cudaMemcpy(&all[r], c->peers[r].ctl_base + parity, sizeof(LevelCtl), cudaMemcpyDeviceToHost));
  c->d2h_bytes += sizeof(LevelCtl) * g.world;
  return REI_OK;
}

rei_status upload_peers(Ctx* c, int parity) {
  const int G = (int)c->peers.size();
  for (int o = 0; o < G; ++o) {
    const Ctx::PeerBuf& b = c->peers[o];
    Peer& q = c->h_peers[o];
    q.arena_out = b.arena;
    q.bp = b.bp;
    q.ctl = b.ctl_base + parity;
    q.dedup.mode = c->mode;
    q.dedup.bitmap = b.bitmap;
    q.dedup.table = b.table;
    q.dedup.mask = b.slots ? b.slots - 1 : 0;
    q.dedup.special = b.special;
    q.out_base = c->sh_used[o];
    q.cap = c->entry_limit ? std::min<uint64_t>(b.cap, c->entry_limit) : b.cap;
  }
  CUDA_OK(c, cudaMemcpyAsync(c->d_peers, c->h_peers, sizeof(Peer) * G, cudaMemcpyHostToDevice, c->stream));
  c->h2d_bytes += sizeof(Peer) * G;
  return REI_OK;
}

struct Shard {
  int o;
  uint64_t n, begin, slab, off;
};
std::vector<Shard> shards_of(const Ctx* c, int L) {
  std::vector<Shard> v;
  auto it = c->levels.find(L);
  if (it == c->levels.end()) return v;
  const LevelInfo& lv = it->second;
  for (size_t o = 0; o < lv.ssize.size(); ++o)
    if (lv.ssize[o]) v.push_back({(int)o, lv.ssize[o], lv.sbegin[o], lv.sslab[o], lv.soff[o]});
  return v;
}

struct UnaryWork {
  bool star;
  uint64_t n, base, slab, rank_base;
};

// The level plan over shard pairs (same candidate multiset as plan_level; the rank
// space is flattened Q, S, C, U with each operand level taken shard by shard).
void plan_sharded(Ctx* c, int cost, LevelInfo& lv, std::vector<Block>& cat, std::vector<Block>& uni,
                  std::vector<UnaryWork>& un, uint64_t& nq, uint64_t& ns, uint64_t& ncat, uint64_t& nuni) {
  const rei_costs& k = c->costs;
  const int c1 = (int)k.sym;
  uint64_t off = 0;
  lv.plan.clear();
  cat.clear();
  uni.clear();
  un.clear();
  nq = ns = ncat = nuni = 0;
  for (int star = 0; star < 2; ++star) {
    const int L = cost - (int)(star ? k.star : k.opt);
    if (L < c1) continue;
    for (const Shard& a : shards_of(c, L)) {
      PlanBlock pb{star ? (uint32_t)BK_S : (uint32_t)BK_Q, L, 0, a.n, 0, off, a.n, false};
      pb.a_off = a.off;
      lv.plan.push_back(pb);
      un.push_back({star != 0, a.n, rel_entry(c, a.o, a.begin), rel_slab(c, a.o, a.slab), off});
      off += a.n;
      (star ? ns : nq) += a.n;
    }
  }
  uint64_t pairs = 0;
  for (int L = c1; L <= cost - (int)k.cat - c1; ++L) pairs += level_size(c, L) * level_size(c, cost - (int)k.cat - L);
  for (int L = c1; L <= cost - (int)k.alt - L; ++L) pairs += level_size(c, L) * level_size(c, cost - (int)k.alt - L);
  const uint64_t target = std::min<uint64_t>(8192, std::max<uint64_t>(128, pairs / ((uint64_t)c->sms * 24 * 4)));
  auto tile_u = [&](uint64_t nu) { return std::max<uint64_t>(1, std::min<uint64_t>({64, nu, target / 32})); };
  auto add = [&](std::vector<Block>& v, uint32_t kind, int L, int R, const Shard& a, const Shard& b, bool tri,
                 uint64_t cnt, uint64_t& item_off) {
    PlanBlock pb{kind, L, R, a.n, b.n, off, cnt, tri};
    pb.a_off = a.off;
    pb.b_off = b.off;
    lv.plan.push_back(pb);
    Block x{};
    x.kind = kind;
    x.tri = tri ? 1 : 0;
    x.slice_a = (!tri && a.n > b.n) ? 1 : 0;
    x.a_base = rel_entry(c, a.o, a.begin);
    x.b_base = rel_entry(c, b.o, b.begin);
    x.a_slab = rel_slab(c, a.o, a.slab);
    x.b_slab = rel_slab(c, b.o, b.slab);
    x.na = a.n;
    x.nb = b.n;
    x.cand_off = off;
    x.cand_count = cnt;
    const uint64_t nu = x.slice_a ? b.n : a.n, nsl = x.slice_a ? a.n : b.n;
    const uint64_t slabs = (nsl + 31) / 32;
    x.tu = tile_u(nu);
    x.ts = std::max<uint64_t>(1, std::min<uint64_t>(slabs, target / (32 * x.tu)));
    x.u_tiles = (nu + x.tu - 1) / x.tu;
    x.s_tiles = (slabs + x.ts - 1) / x.ts;
    x.item_off = item_off;
    item_off += x.u_tiles * x.s_tiles;
    v.push_back(x);
    off += cnt;
  };
  uint64_t item_off = 0;
  for (int L = c1; L <= cost - (int)k.cat - c1; ++L) {
    const int R = cost - (int)k.cat - L;
    const auto A = shards_of(c, L), B = shards_of(c, R);
    for (const Shard& a : A)
      for (const Shard& b : B) {
        add(cat, BK_C, L, R, a, b, false, a.n * b.n, item_off);
        ncat += a.n * b.n;
      }
  }
  item_off = 0;
  for (int L = c1; L <= cost - (int)k.alt - L; ++L) {
    const int R = cost - (int)k.alt - L;
    const auto A = shards_of(c, L), B = shards_of(c, R);
    for (const Shard& a : A)
      for (const Shard& b : B) {
        if (L == R && a.o > b.o) continue;  // i < j over the level (A8): shard a before shard b
        const bool tri = (L == R && a.o == b.o);
        const uint64_t cnt = tri ? a.n * (a.n - 1) / 2 : a.n * b.n;
        if (!cnt) continue;
        add(uni, BK_U, L, R, a, b, tri, cnt, item_off);
        nuni += cnt;
      }
  }
}

rei_status launch_sharded(Ctx* c, int rank, int world, const std::vector<UnaryWork>& un,
                          const std::vector<Block>& cat, const std::vector<Block>& uni) {
  LevelParams p;
  fill_params(c, p);
  p.otf = c->otf_level ? 1 : 0;
  p.shards = (uint32_t)world;
  p.peers = c->d_peers;
  std::vector<Block> catv[2];
  for (const Block& b : cat) catv[b.slice_a ? 1 : 0].push_back(b);
  for (auto& v : catv) renumber_items(v);
  const std::vector<Block>* lists[3] = {&catv[0], &catv[1], &uni};
  {
    // the pair kernels stage a launch's block table in shared memory next to <= 64 KB
    // of split tables and append stages: refuse a level whose table cannot fit
    static int optin = 0;
    if (!optin && cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device) != cudaSuccess)
      optin = 227 * 1024;
    for (int r = 0; r < 3; ++r)
      if (lists[r]->size() * sizeof(Block) + 64 * 1024 > (size_t)optin) {
        c->err = "a sharded level has " + std::to_string(lists[r]->size()) +
                 " operand blocks in one launch; their table exceeds the shared memory of a CTA";
        return REI_EINVAL;
      }
  }
  Block* hb = (c->lag_active && c->h_blocks_ring) ? c->h_blocks_ring + (size_t)c->lag_par * 3 * Ctx::kMaxBlocks
                                                  : c->h_blocks;
  for (int r = 0; r < 3; ++r) {
    if (lists[r]->empty()) continue;
    std::copy(lists[r]->begin(), lists[r]->end(), hb + r * Ctx::kMaxBlocks);
    CUDA_OK(c, cudaMemcpyAsync(c->d_blocks + r * Ctx::kMaxBlocks, hb + r * Ctx::kMaxBlocks,
                               lists[r]->size() * sizeof(Block), cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += lists[r]->size() * sizeof(Block);
  }
  auto share = [&](uint64_t total, LevelParams& q) {
    uint64_t b = 0, e = total;
    rei_partition(total, world, rank, &b, &e);
    q.item_begin = b;
    q.total_items = e;
    return e > b;
  };
  for (const UnaryWork& u : un) {
    LevelParams pq = p;
    pq.rank_base = u.rank_base;
    if (!share(u.n, pq)) continue;
    EventPair ep;
    c->begin_kernel(REI_K_UNARY, ep);
    int n = u.star ? launch_unary(c->W32, pq, 0, u.n, 0, u.base, 0, u.slab, c->stream)
                   : launch_unary(c->W32, pq, u.n, 0, u.base, 0, 0, 0, c->stream);
    c->end_kernel(ep, n);
  }
  for (int r = 0; r < 2; ++r) {
    if (catv[r].empty()) continue;
    LevelParams pc = p;
    pc.blocks = c->d_blocks + r * Ctx::kMaxBlocks;
    pc.nblocks = (uint32_t)catv[r].size();
    if (!share(items_of(catv[r]), pc)) continue;
    EventPair ep;
    c->begin_kernel(REI_K_CONCAT, ep);
    int n = launch_concat(c->W32, pc, r == 1, c->stream);
    c->end_kernel(ep, n);
  }
  if (!uni.empty()) {
    LevelParams pu = p;
    pu.blocks = c->d_blocks + 2 * Ctx::kMaxBlocks;
    pu.nblocks = (uint32_t)uni.size();
    if (share(items_of(uni), pu)) {
      EventPair ep;
      c->begin_kernel(REI_K_UNION, ep);
      int n = launch_union(c->W32, pu, c->stream);
      c->end_kernel(ep, n);
    }
  }
  CUDA_OK(c, cudaGetLastError());
  return REI_OK;
}

// Start of a level: every member resets its control line of this parity, then the
// ranks meet (nobody inserts into an owner's line before the owner reset it).
rei_status begin_sharded_level(Comm& g, int cost) {
  rei_status s;
  for (Ctx* c : g.m) {
    c->ctl = c->ctl_base + (cost & 1);
    if ((s = reset_ctl(c)) != REI_OK) return s;
    if ((s = upload_peers(c, cost & 1)) != REI_OK) return s;
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
  }
  return group_barrier(g);
}

// End of a level: kernels done everywhere, then every rank's control line.
rei_status end_sharded_level(Comm& g, int cost, std::vector<LevelCtl>& all, double* ms) {
  rei_status s;
  for (Ctx* c : g.m) {
    CUDA_OK(c, cudaStreamSynchronize(c->stream));
    double t;
    c->collect_events(&t);
    if (c == g.m[0] && ms) *ms += t;
  }
  if ((s = group_barrier(g)) != REI_OK) return s;
  return read_all_ctl(g, cost & 1, all);
}

// Record the shards of a finished level and transpose each member's own shard.
rei_status commit_shards(Comm& g, LevelInfo& lv, const std::vector<LevelCtl>& all, bool transpose) {
  const int G = g.world;
  lv.sbegin.assign(G, 0); lv.ssize.assign(G, 0); lv.sslab.assign(G, 0); lv.soff.assign(G, 0);
  uint64_t off = 0;
  for (int o = 0; o < G; ++o) {
    lv.sbegin[o] = g.m[0]->sh_used[o];
    lv.sslab[o] = g.m[0]->sh_slabs[o];
    lv.ssize[o] = all[o].count;
    lv.soff[o] = off;
    off += all[o].count;
  }
  lv.size = off;
  for (size_t i = 0; i < g.m.size(); ++i) {
    Ctx* c = g.m[i];
    const int me = g.rank0 + (int)i;
    if (transpose && lv.ssize[me]) {
      if (lv.sslab[me] + (lv.ssize[me] + 31) / 32 > c->slab_cap) return REI_OUT_OF_MEMORY;
      EventPair et;
      c->begin_kernel(REI_K_TRANSPOSE, et);
      int n = launch_transpose(c->W32, c->arena, lv.sbegin[me], lv.ssize[me], c->tarena, lv.sslab[me], c->stream);
      c->end_kernel(et, n);
      CUDA_OK(c, cudaGetLastError());
    }
    for (int o = 0; o < G; ++o) {
      c->sh_used[o] += lv.ssize[o];
      c->sh_slabs[o] += (lv.ssize[o] + 31) / 32;
    }
    c->arena_used = c->sh_used[me];
    c->slabs_used = c->sh_slabs[me];
    c->levels[lv.cost] = lv;
  }
  return REI_OK;
}

// Algorithm 1 over a sharded cache (the members of `g` are sharded contexts).
rei_status solve_sharded(Comm& g, uint32_t max_cost) {
  Ctx* c0 = g.m[0];
  const rei_costs& k = c0->costs;
  const int c1 = (int)k.sym;
  const int G = g.world;
  rei_status s;
  for (Ctx* c : g.m) {
    reset_search(c);
    c->sh_used.assign(G, 0);
    c->sh_slabs.assign(G, 0);
    if (!peer_offsets_ok(c)) {
      c->err = "peer buffers are not aligned for flat addressing";
      return REI_ECUDA;
    }
  }
  uint64_t cand = 1;  // the empty regex (A9)
  const uint64_t total_ex = c0->P.size() + c0->N.size();
  const bool empty_ok = c0->P.empty() ||
                        (c0->err_num && (uint64_t)c0->P.size() * c0->err_den <= (uint64_t)c0->err_num * total_ex);
  const bool eps_ok = c0->P.size() == 1 && c0->P[0].empty();
  if (empty_ok || eps_ok) {
    for (Ctx* c : g.m) {
      c->regex = empty_ok ? "empty" : "eps";
      c->result.cost = k.sym;
      c->result.candidates = cand;
    }
    return REI_OK;
  }
  // ---- level c1: the symbols (rank 0 inserts them into their owners)
  for (Ctx* c : g.m) {
    if ((s = clear_dedup(c)) != REI_OK) return s;
  }
  if ((s = begin_sharded_level(g, c1)) != REI_OK) return s;
  if (g.rank0 == 0) {
    Ctx* c = g.m[0];
    LevelParams p;
    fill_params(c, p);
    p.shards = (uint32_t)G;
    p.peers = c->d_peers;
    EventPair ep;
    c->begin_kernel(REI_K_OTHER, ep);
    int n = launch_seeds(c->W32, p, c->tab.seeds, (int)c->alphabet.size(), c->stream);
    c->end_kernel(ep, n);
    CUDA_OK(c, cudaGetLastError());
  }
  std::vector<LevelCtl> all;
  double ms0 = 0;
  if ((s = end_sharded_level(g, c1, all, &ms0)) != REI_OK) return s;
  {
    LevelInfo lv;
    lv.cost = c1;
    lv.seeds = true;
    const uint64_t found_seed = all[0].found_rank;
    if ((s = commit_shards(g, lv, all, found_seed == ~0ull)) != REI_OK) return s;
    rei_level_stat st{};
    st.cost = c1;
    st.unique = lv.size;
    st.ms = ms0;
    st.complete = found_seed == ~0ull ? 1 : 0;
    for (Ctx* c : g.m) c->stats.push_back(st);
    if (found_seed != ~0ull) {
      for (Ctx* c : g.m) {
        c->result.candidates = 1 + found_seed + 1;
        if ((s = finish_found(c, c1, found_seed)) != REI_OK) return s;
      }
      return REI_OK;
    }
  }
  cand += c0->alphabet.size();
  for (Ctx* c : g.m) {
    c->result.last_complete_cost = c1;
    c->result.cand_complete = cand;
  }
  std::vector<Block> cat, uni;
  std::vector<UnaryWork> un;
  for (int cost = c1 + 1; cost <= (int)max_cost; ++cost) {
    if (c0->otf_level && needs_uncached(c0, cost)) {
      for (Ctx* c : g.m) c->result.candidates = c->result.cand_complete;
      return REI_OUT_OF_MEMORY;
    }
    LevelInfo lv;
    lv.cost = cost;
    uint64_t nq = 0, ns = 0, ncat = 0, nuni = 0;
    std::vector<std::vector<Block>> cats(g.m.size()), unis(g.m.size());
    std::vector<std::vector<UnaryWork>> uns(g.m.size());
    for (size_t i = 0; i < g.m.size(); ++i)  // same plan on every member; bases are member-relative
      plan_sharded(g.m[i], cost, lv, cats[i], unis[i], uns[i], nq, ns, ncat, nuni);
    if (lv.plan.empty()) continue;
    if ((int)(cats[0].size() + unis[0].size()) > Ctx::kMaxBlocks) {
      c0->err = "too many operand blocks in one level";
      return REI_EINVAL;
    }
    rei_level_stat st{};
    st.cost = (uint32_t)cost;
    st.cand_q = nq; st.cand_s = ns; st.cand_c = ncat; st.cand_u = nuni;
    double level_ms = 0;
    for (;;) {
      if ((s = begin_sharded_level(g, cost)) != REI_OK) return s;
      for (size_t i = 0; i < g.m.size(); ++i)
        if ((s = launch_sharded(g.m[i], g.rank0 + (int)i, G, uns[i], cats[i], unis[i])) != REI_OK) return s;
      if ((s = end_sharded_level(g, cost, all, &level_ms)) != REI_OK) return s;
      bool overflow = false;
      for (auto& l : all) overflow |= l.overflow != 0;
      if (!overflow) break;
      // an owner's shard is full: OnTheFly -- drop the partial inserts
      // (each owner rebuilds its dedup set from its cached shards) and re-check the level
      if ((c0->flags & REI_FLAG_NO_ONTHEFLY) || c0->otf_level) {
        for (Ctx* c : g.m) c->result.candidates = c->result.cand_complete;
        return REI_OUT_OF_MEMORY;
      }
      for (Ctx* c : g.m) {
        c->otf_level = cost;
        if ((s = rebuild_dedup(c, c->arena_used)) != REI_OK) return s;
        CUDA_OK(c, cudaStreamSynchronize(c->stream));
      }
    }
    const bool otf_now = c0->otf_level != 0;
    uint64_t found_rank = ~0ull, evaluated = 0, eval_c = 0, eval_u = 0;
    for (auto& l : all) {
      found_rank = std::min<uint64_t>(found_rank, l.found_rank);
      evaluated += l.evaluated;
      eval_c += l.eval_c;
      eval_u += l.eval_u;
    }
    const bool found = found_rank != ~0ull;
    const bool complete = !found || (c0->flags & REI_FLAG_COMPLETE_FINAL_LEVEL);
    if (otf_now)
      for (auto& l : all) l.count = 0;  // nothing cached at an OnTheFly level
    if ((s = commit_shards(g, lv, all, !found && !otf_now)) != REI_OK) return s;
    st.unique = lv.size;
    st.ms = level_ms;
    st.complete = complete ? (otf_now ? 2 : 1) : 0;
    st.evaluated = complete ? (nq + ns + ncat + nuni) : evaluated;
    st.eval_c = complete ? ncat : eval_c;
    st.eval_u = complete ? nuni : eval_u;
    for (Ctx* c : g.m) c->stats.push_back(st);
    if (found) {
      for (Ctx* c : g.m) {
        c->result.candidates = cand + st.evaluated;
        if (complete) {
          c->result.last_complete_cost = (uint32_t)cost;
          c->result.cand_complete = cand + st.evaluated;
        }
        if ((s = finish_found(c, cost, found_rank)) != REI_OK) return s;
      }
      return REI_OK;
    }
    cand += nq + ns + ncat + nuni;
    for (Ctx* c : g.m) {
      c->result.cand_complete = cand;
      c->result.candidates = cand;
      c->result.last_complete_cost = (uint32_t)cost;
    }
  }
  return REI_NOT_FOUND;
}

rei_status solve_impl(Ctx* c, uint32_t max_cost) {
  Comm g;
  g.m = {c};
  g.world = c->world > 1 ? c->world : 1;
  g.rank0 = c->world > 1 ? c->rank : 0;
  g.nccl = c->nccl;
  g.host = c->world > 1 && c->host_xport;
  if (c->sharded && c->world > 1) return solve_sharded(g, max_cost);
  const rei_status s = solve_group(g, max_cost);
  c->join_post();  // later calls (level reads, the next solve) see every level in place
  return s;
}

// ============================================================================
// Many small specifications in packed launches (the paper's suites
// of thousands of small runs).  Every active specification advances one
// non-empty cost level per step; a step runs each kernel class (?/*, union, concat of
// either orientation; per CS width and split-count class) as ONE launch whose CTA
// groups serve the specifications (Packed / packed_params in levels.cu), resets and
// gathers all control lines with one kernel each, and syncs once.  The arithmetic is
// the single-spec kernels' (same bodies).  A specification that needs anything else
// (wider CSs, > 15 proper splits, a level overflow, OnTheFly) leaves the packed loop
// and is solved alone afterwards.
struct PackSpec {
  Ctx* c = nullptr;
  int cost = 0;
  uint64_t cand = 1;
  bool active = false, fallback = false;
  rei_status st = REI_OK;
  LevelInfo lv;
  std::vector<Block> cat, uni, catv[2];
  uint64_t nq = 0, ns = 0, ncat = 0, nuni = 0;
  double done_s = 0;  // host seconds from the start of the call to this spec's result
};

struct PackBuf {  // device + pinned staging of one step
  LevelParams* d_params = nullptr;
  LevelParams* h_params = nullptr;
  uint32_t* d_cta = nullptr;
  uint32_t* h_cta = nullptr;
  Block* d_blocks = nullptr;
  Block* h_blocks = nullptr;
  LevelCtl* d_ctl = nullptr;
  LevelCtl* h_ctl = nullptr;
  size_t cap_params = 0, cap_cta = 0, cap_blocks = 0, cap_ctl = 0;
  ~PackBuf() {
    for (void* q : {(void*)d_params, (void*)d_cta, (void*)d_blocks, (void*)d_ctl}) if (q) cudaFree(q);
    for (void* q : {(void*)h_params, (void*)h_cta, (void*)h_blocks, (void*)h_ctl}) if (q) cudaFreeHost(q);
  }
  template <class T>
  static bool ensure(T*& d, T*& h, size_t& cap, size_t n) {
    if (n <= cap) return true;
    const size_t c2 = std::max<size_t>(n, 2 * cap);
    if (d) cudaFree(d);
    if (h) cudaFreeHost(h);
    d = nullptr; h = nullptr; cap = 0;
    if (cudaMalloc(&d, c2 * sizeof(T)) != cudaSuccess || cudaMallocHost(&h, c2 * sizeof(T)) != cudaSuccess) return false;
    cap = c2;
    return true;
  }
};

rei_status solve_packed(std::vector<Ctx*>& cs, uint32_t max_cost, std::vector<rei_status>& status,
                        std::vector<double>& done_s, const std::vector<cudaStream_t>& own_streams) {
  const size_t n = cs.size();
  const auto t0 = std::chrono::steady_clock::now();
  auto now_s = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  cudaStream_t st = cs[0]->stream;
  std::vector<PackSpec> sp(n);
  status.assign(n, REI_OK);
  done_s.assign(n, 0.0);
  PackBuf pb;
  rei_status s;
  // ---- level c1 (Alg. 1 line 3) and the trivial answers (lines 1-2), per spec
  for (size_t i = 0; i < n; ++i) {
    Ctx* c = cs[i];
    PackSpec& q = sp[i];
    q.c = c;
    reset_search(c);
    c->sort_levels = false;  // a level's order is free; packed steps skip the sort
    const rei_costs& k = c->costs;
    const uint64_t total_ex = c->P.size() + c->N.size();
    const bool empty_ok = c->P.empty() ||
                          (c->err_num && (uint64_t)c->P.size() * c->err_den <= (uint64_t)c->err_num * total_ex);
    const bool eps_ok = c->P.size() == 1 && c->P[0].empty();
    if (empty_ok || eps_ok) {
      c->regex = empty_ok ? "empty" : "eps";
      c->result.cost = k.sym;
      c->result.candidates = 1;
      continue;
    }
    if (c->tab.n == 0 || c->world > 1 || c->exchange_self || c->sharded || !packable(c->W32, c->tab.maxk) ||
        c->otf_level) {
      q.fallback = true;
      continue;
    }
    if ((s = clear_dedup(c)) != REI_OK || (s = reset_ctl(c)) != REI_OK) return s;
    LevelParams p;
    fill_params(c, p);
    p.out_base = 0;
    c->launches += launch_seeds(c->W32, p, c->tab.seeds, (int)c->alphabet.size(), st);
    q.active = true;
  }
  CUDA_OK(cs[0], cudaGetLastError());
  for (size_t i = 0; i < n; ++i)
    if (sp[i].active)
      CUDA_OK(sp[i].c, cudaMemcpyAsync(sp[i].c->h_ctl, sp[i].c->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, st));
  CUDA_OK(cs[0], cudaStreamSynchronize(st));
  for (size_t i = 0; i < n; ++i) {
    PackSpec& q = sp[i];
    if (!q.active) continue;
    Ctx* c = q.c;
    const int c1 = (int)c->costs.sym;
    LevelInfo lv;
    lv.cost = c1;
    lv.seeds = true;
    lv.size = c->h_ctl->count;
    c->levels[c1] = lv;
    c->arena_used = lv.size;
    rei_level_stat stt{};
    stt.cost = c1;
    stt.unique = lv.size;
    const uint64_t found_seed = c->h_ctl->found_rank;
    stt.complete = found_seed == ~0ull ? 1 : 0;
    c->stats.push_back(stt);
    if (found_seed != ~0ull) {
      c->result.candidates = 1 + found_seed + 1;
      if ((status[i] = finish_found(c, c1, found_seed)) != REI_OK) {}
      q.active = false;
      done_s[i] = now_s();
      continue;
    }
    q.cand = 1 + c->alphabet.size();
    q.cost = c1;
    c->launches += launch_transpose(c->W32, c->arena, 0, c->arena_used, c->tarena, 0, st);
    c->slabs_used = (c->arena_used + 31) / 32;
    c->result.last_complete_cost = c1;
    c->result.cand_complete = q.cand;
    c->result.candidates = q.cand;
  }

  struct Item { uint32_t spec; uint64_t work; LevelParams p; };
  for (;;) {
    // ---- plan: every active spec's next non-empty level
    std::vector<size_t> act;
    for (size_t i = 0; i < n; ++i) {
      PackSpec& q = sp[i];
      if (!q.active) continue;
      Ctx* c = q.c;
      const rei_costs& k = c->costs;
      bool planned = false;
      while (q.cost < (int)max_cost) {
        ++q.cost;
        q.lv = LevelInfo{};
        q.lv.cost = q.cost;
        plan_level(c, q.cost, q.lv, q.cat, q.uni, q.nq, q.ns, q.ncat, q.nuni);
        if (!q.lv.plan.empty()) { planned = true; break; }
      }
      if (!planned) {
        status[i] = REI_NOT_FOUND;
        q.active = false;
        done_s[i] = now_s();
        continue;
      }
      if ((int)(q.cat.size() + q.uni.size()) > Ctx::kMaxBlocks) { q.active = false; q.fallback = true; continue; }
      const uint64_t prev = c->stats.empty() ? 0 : c->stats.back().unique;
      const uint64_t expect = std::min<uint64_t>(q.nq + q.ns + q.ncat + q.nuni, 4 * prev + 1024);
      if (c->arena_used + expect > c->cap || c->slabs_used + expect / 32 + 2 > c->slab_cap) {
        if ((s = grow(c, c->arena_used + expect)) != REI_OK && s != REI_OUT_OF_MEMORY) return s;
      }
      q.lv.begin = c->arena_used;
      q.lv.slab = c->slabs_used;
      q.catv[0].clear();
      q.catv[1].clear();
      for (const Block& b : q.cat) q.catv[b.slice_a ? 1 : 0].push_back(b);
      for (auto& v : q.catv) renumber_items(v);
      act.push_back(i);
    }
    if (act.empty()) break;
    const auto step_t0 = std::chrono::steady_clock::now();
    // ---- work classes: (kind, W32, maxk class, orientation) -> items of the specs
    std::map<std::tuple<int, int, int, int>, std::vector<Item>> cls;
    std::vector<Block> blocks;
    std::vector<LevelParams> ctlp;  // one LevelParams per active spec (control-line reset / gather)
    std::vector<std::pair<size_t, size_t>> boff;  // (item list ref) -> block offset, patched below
    struct Patch { std::tuple<int, int, int, int> key; size_t idx; size_t off; };
    std::vector<Patch> patches;
    for (size_t a = 0; a < act.size(); ++a) {
      PackSpec& q = sp[act[a]];
      Ctx* c = q.c;
      const rei_costs& k = c->costs;
      LevelParams p;
      fill_params(c, p);
      p.out_base = q.lv.begin;
      ctlp.push_back(p);
      const int mk = maxk_class(c->tab.maxk);
      if (q.nq + q.ns) {
        LevelParams pu = p;
        pu.item_begin = 0;
        pu.total_items = q.nq + q.ns;
        pu.un_q = q.nq;
        pu.un_s = q.ns;
        pu.un_bq = q.nq ? c->levels.at(q.cost - (int)k.opt).begin : 0;
        pu.un_bs = q.ns ? c->levels.at(q.cost - (int)k.star).begin : 0;
        pu.un_slab = q.ns ? c->levels.at(q.cost - (int)k.star).slab : 0;
        cls[{0, c->W32, mk, 0}].push_back({(uint32_t)a, (q.nq + 31) / 32 + (q.ns + 31) / 32, pu});
      }
      auto add_pairs = [&](int kind, int orient, const std::vector<Block>& v) {
        if (v.empty()) return;
        LevelParams pc = p;
        pc.nblocks = (uint32_t)v.size();
        pc.item_begin = 0;
        pc.total_items = items_of(v);
        auto key = std::make_tuple(kind, c->W32, kind == 1 ? mk : 0, orient);
        patches.push_back({key, cls[key].size(), blocks.size()});
        blocks.insert(blocks.end(), v.begin(), v.end());
        cls[key].push_back({(uint32_t)a, pc.total_items, pc});
      };
      add_pairs(2, 0, q.uni);      // union
      add_pairs(1, 0, q.catv[0]);  // concat, uniform left operand
      add_pairs(1, 1, q.catv[1]);  // concat, sliced left operand
    }
    // ---- one upload: control params, every class's params and CTA groups, block tables
    size_t np = ctlp.size(), ncta = 0;
    for (auto& kv : cls) { np += kv.second.size(); ncta += kv.second.size() + 1; }
    if (!PackBuf::ensure(pb.d_params, pb.h_params, pb.cap_params, np) ||
        !PackBuf::ensure(pb.d_cta, pb.h_cta, pb.cap_cta, std::max<size_t>(1, ncta)) ||
        !PackBuf::ensure(pb.d_blocks, pb.h_blocks, pb.cap_blocks, std::max<size_t>(1, blocks.size())) ||
        !PackBuf::ensure(pb.d_ctl, pb.h_ctl, pb.cap_ctl, act.size())) {
      cs[0]->err = "packed staging allocation failed";
      return REI_OUT_OF_MEMORY;
    }
    for (auto& pt : patches) cls[pt.key][pt.idx].p.blocks = pb.d_blocks + pt.off;
    std::copy(blocks.begin(), blocks.end(), pb.h_blocks);
    std::copy(ctlp.begin(), ctlp.end(), pb.h_params);
    size_t po = ctlp.size(), co = 0;
    struct Launch { std::tuple<int, int, int, int> key; size_t params, cta, nspec; uint32_t ctas; size_t maxnb; };
    std::vector<Launch> launches;
    const uint32_t budget = (uint32_t)cs[0]->sms * 4u * 4u;  // CTAs per packed launch: ~4 resident per SM x 4 waves
    for (auto& kv : cls) {
      auto& items = kv.second;
      uint64_t tot = 0;
      size_t maxnb = 0;
      for (auto& it : items) { tot += it.work; maxnb = std::max<size_t>(maxnb, it.p.nblocks); }
      uint32_t* cta = pb.h_cta + co;
      uint32_t acc = 0;
      for (size_t j = 0; j < items.size(); ++j) {
        cta[j] = acc;
        const uint64_t per = std::get<0>(kv.first) == 0 ? 8 : 8;  // work units per CTA (warps)
        uint64_t want = std::max<uint64_t>(1, (items[j].work + per - 1) / per);
        const uint64_t share = std::max<uint64_t>(1, tot ? (uint64_t)((double)budget * items[j].work / tot) : 1);
        acc += (uint32_t)std::min(want, share);
        pb.h_params[po + j] = items[j].p;
      }
      cta[items.size()] = acc;
      launches.push_back({kv.first, po, co, items.size(), acc, maxnb});
      po += items.size();
      co += items.size() + 1;
    }
    Ctx* c0 = cs[0];
    CUDA_OK(c0, cudaMemcpyAsync(pb.d_blocks, pb.h_blocks, std::max<size_t>(1, blocks.size()) * sizeof(Block),
                                cudaMemcpyHostToDevice, st));
    CUDA_OK(c0, cudaMemcpyAsync(pb.d_params, pb.h_params, po * sizeof(LevelParams), cudaMemcpyHostToDevice, st));
    CUDA_OK(c0, cudaMemcpyAsync(pb.d_cta, pb.h_cta, std::max<size_t>(1, co) * sizeof(uint32_t),
                                cudaMemcpyHostToDevice, st));
    uint64_t nl = launch_ctl_reset_packed(pb.d_params, (uint32_t)ctlp.size(), st);
    // unary, union, then concat (union first: a precise union stops the concat CTAs)
    for (int kind : {0, 2, 1}) {
      for (auto& L : launches) {
        if (std::get<0>(L.key) != kind) continue;
        Packed pk{pb.d_params + L.params, pb.d_cta + L.cta, (uint32_t)L.nspec};
        const int W = std::get<1>(L.key), mk = std::get<2>(L.key);
        if (kind == 0) nl += launch_unary_packed(W, mk, pk, L.ctas, st);
        else if (kind == 2) nl += launch_union_packed(W, pk, L.ctas, L.maxnb, st);
        else nl += launch_concat_packed(W, mk, std::get<3>(L.key) == 1, pk, L.ctas, L.maxnb, st);
      }
    }
    nl += launch_ctl_gather_packed(pb.d_params, (uint32_t)ctlp.size(), pb.d_ctl, st);
    CUDA_OK(c0, cudaGetLastError());
    CUDA_OK(c0, cudaMemcpyAsync(pb.h_ctl, pb.d_ctl, act.size() * sizeof(LevelCtl), cudaMemcpyDeviceToHost, st));
    CUDA_OK(c0, cudaStreamSynchronize(st));
    c0->launches += nl;
    const double step_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - step_t0).count();
    // ---- per spec: found / overflow / next level; transposes of the new levels (packed)
    std::vector<LevelParams> tp;
    std::map<int, std::vector<LevelParams>> tpw;
    for (size_t a = 0; a < act.size(); ++a) {
      const size_t i = act[a];
      PackSpec& q = sp[i];
      Ctx* c = q.c;
      const LevelCtl& l = pb.h_ctl[a];
      if (l.overflow) {  // redo this spec alone (grows its cache, OnTheFly if needed)
        q.active = false;
        q.fallback = true;
        continue;
      }
      rei_level_stat stt{};
      stt.cost = (uint32_t)q.cost;
      stt.cand_q = q.nq; stt.cand_s = q.ns; stt.cand_c = q.ncat; stt.cand_u = q.nuni;
      stt.ms = step_ms;
      const bool found = l.found_rank != ~0ull;
      const bool complete = !found || (c->flags & REI_FLAG_COMPLETE_FINAL_LEVEL);
      stt.unique = l.count;
      stt.complete = complete ? 1 : 0;
      stt.evaluated = complete ? (q.nq + q.ns + q.ncat + q.nuni) : l.evaluated;
      stt.eval_c = complete ? q.ncat : l.eval_c;
      stt.eval_u = complete ? q.nuni : l.eval_u;
      q.lv.size = l.count;
      c->arena_used = q.lv.begin + q.lv.size;
      c->levels[q.cost] = q.lv;
      c->stats.push_back(stt);
      if (found) {
        c->result.candidates = q.cand + stt.evaluated;
        if (complete) {
          c->result.last_complete_cost = (uint32_t)q.cost;
          c->result.cand_complete = q.cand + stt.evaluated;
        }
        status[i] = finish_found(c, q.cost, l.found_rank);
        q.active = false;
        done_s[i] = now_s();
        continue;
      }
      q.cand += q.nq + q.ns + q.ncat + q.nuni;
      c->result.cand_complete = q.cand;
      c->result.candidates = q.cand;
      c->result.last_complete_cost = (uint32_t)q.cost;
      if (c->slabs_used + (q.lv.size + 31) / 32 > c->slab_cap) {
        if ((s = grow(c, c->cap + 1)) != REI_OK) { q.active = false; q.fallback = true; continue; }
      }
      LevelParams p;
      fill_params(c, p);
      p.un_q = q.lv.size;
      p.un_bq = q.lv.begin;
      p.un_slab = q.lv.slab;
      tpw[c->W32].push_back(p);
      c->slabs_used += (q.lv.size + 31) / 32;
    }
    // packed transposes: one launch per CS width
    size_t tpo = 0, tco = 0, tn = 0;
    for (auto& kv : tpw) tn += kv.second.size();
    if (tn) {
      if (!PackBuf::ensure(pb.d_params, pb.h_params, pb.cap_params, tn) ||
          !PackBuf::ensure(pb.d_cta, pb.h_cta, pb.cap_cta, tn + tpw.size())) {
        cs[0]->err = "packed staging allocation failed";
        return REI_OUT_OF_MEMORY;
      }
      std::vector<std::tuple<int, size_t, size_t, size_t, uint32_t>> tl;
      for (auto& kv : tpw) {
        uint32_t acc = 0;
        for (size_t j = 0; j < kv.second.size(); ++j) {
          pb.h_cta[tco + j] = acc;
          acc += (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(64, (kv.second[j].un_q + 255) / 256));
          pb.h_params[tpo + j] = kv.second[j];
        }
        pb.h_cta[tco + kv.second.size()] = acc;
        tl.emplace_back(kv.first, tpo, tco, kv.second.size(), acc);
        tpo += kv.second.size();
        tco += kv.second.size() + 1;
      }
      CUDA_OK(c0, cudaMemcpyAsync(pb.d_params, pb.h_params, tpo * sizeof(LevelParams), cudaMemcpyHostToDevice, st));
      CUDA_OK(c0, cudaMemcpyAsync(pb.d_cta, pb.h_cta, tco * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
      for (auto& t : tl) {
        Packed pk{pb.d_params + std::get<1>(t), pb.d_cta + std::get<2>(t), (uint32_t)std::get<3>(t)};
        c0->launches += launch_transpose_packed(std::get<0>(t), pk, std::get<4>(t), st);
      }
      CUDA_OK(c0, cudaGetLastError());
      // the pinned staging is rewritten by the next step only after its uploads: the
      // copies above are stream-ordered, but the host must not overwrite h_params early
      CUDA_OK(c0, cudaStreamSynchronize(st));
    }
  }
  // ---- specifications that left the packed loop: solved alone (same code as rei_solve)
  CUDA_OK(cs[0], cudaStreamSynchronize(st));
  for (size_t i = 0; i < n; ++i) {
    if (!sp[i].fallback) continue;
    Ctx* c = sp[i].c;
    c->stream = own_streams[i];
    c->sort_levels = c->mode == DEDUP_BITMAP && getenv("REI_NO_LEVEL_SORT") == nullptr;
    status[i] = solve_impl(c, max_cost);
    c->stream = st;
    done_s[i] = now_s();
  }
  for (size_t i = 0; i < n; ++i)  // sort_levels as rei_init set it (the packed steps skip it)
    sp[i].c->sort_levels = sp[i].c->mode == DEDUP_BITMAP && !sp[i].c->sharded && getenv("REI_NO_LEVEL_SORT") == nullptr;
  return REI_OK;
}

}  // namespace
}  // namespace rei

using rei::Ctx;

extern "C" {

rei_status rei_init(void** out, const char* alphabet, const char* const* P, size_t nP, const char* const* N,
                    size_t nN, rei_costs costs, const rei_options* opts) {
  using namespace rei;
  g_init_error.clear();
  if (!out || !alphabet) { g_init_error = "null argument"; return REI_EINVAL; }
  *out = nullptr;
  // REI_TRACE=1: host wall-clock of the init phases on stderr (diagnostics only)
  const bool trace = getenv("REI_TRACE") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (trace)
      fprintf(stderr, "[rei_init] %-28s %8.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };
  auto c = std::make_unique<Ctx>();
  c->alphabet = alphabet;
  const size_t k = c->alphabet.size();
  if (k == 0 || k > 255) { g_init_error = "alphabet must have 1..255 symbols"; return REI_EINVAL; }
  int rank_of[256];
  for (int i = 0; i < 256; ++i) rank_of[i] = -1;
  for (size_t i = 0; i < k; ++i) {
    const unsigned char ch = (unsigned char)c->alphabet[i];
    if (rank_of[ch] >= 0) { g_init_error = "duplicate alphabet symbol"; return REI_EINVAL; }
    rank_of[ch] = (int)i;
  }
  if (!costs.sym || !costs.opt || !costs.star || !costs.cat || !costs.alt) {
    g_init_error = "every constructor cost must be >= 1 (P:483)";
    return REI_EINVAL;
  }
  c->costs = costs;
  // longest word whose shortlex key (value < 2^58) is exact
  int max_len = 0;
  {
    long double v = 1;
    while (v * k < (long double)(1ull << 58) && max_len < 63) { v *= k; ++max_len; }
  }
  auto conv = [&](const char* const* S, size_t m, std::vector<std::vector<uint8_t>>& dst) -> bool {
    for (size_t i = 0; i < m; ++i) {
      if (!S[i]) { g_init_error = "null example string"; return false; }
      std::vector<uint8_t> w;
      for (const char* q = S[i]; *q; ++q) {
        const int r = rank_of[(unsigned char)*q];
        if (r < 0) { g_init_error = "example symbol not in the alphabet"; return false; }
        w.push_back((uint8_t)r);
      }
      if ((int)w.size() > max_len) { g_init_error = "example too long for the 58-bit shortlex key"; return false; }
      dst.push_back(w);
    }
    return true;
  };
  if (!conv(P, nP, c->P) || !conv(N, nN, c->N)) return REI_EINVAL;
  for (auto& p : c->P)
    for (auto& q : c->N)
      if (p == q) { g_init_error = "P and N intersect (P:472-477)"; return REI_EINVAL; }
  // dedup of repeated examples within P or N (sets)
  auto dedup_set = [](std::vector<std::vector<uint8_t>>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  dedup_set(c->P);
  dedup_set(c->N);
  if (opts) {
    c->err_num = opts->err_num;
    c->err_den = opts->err_den ? opts->err_den : 1;
    c->flags = opts->flags;
    c->budget = opts->mem_budget_bytes;
    c->budget_user = opts->mem_budget_bytes != 0;
    c->entry_limit = opts->max_entries;
    c->sharded = (opts->flags & REI_FLAG_SHARDED_CACHE) != 0;
    c->allgather = opts->allgather;
    c->allgather_user = opts->allgather_user;
    if (opts->world_size > 1 && c->sharded) {
      if (!opts->allgather || opts->rank < 0 || opts->rank >= opts->world_size ||
          opts->world_size > Ctx::kMaxShards) {
        g_init_error = "sharded-cache context needs rank in [0, world_size <= 64) and an allgather callback";
        return REI_EINVAL;
      }
      c->world = opts->world_size;
      c->rank = opts->rank;
    } else if (opts->world_size > 1) {
      if ((!opts->nccl_unique_id && !opts->allgather) || opts->rank < 0 || opts->rank >= opts->world_size ||
          opts->world_size > 64) {
        g_init_error = "multi-GPU context needs rank in [0, world_size <= 64) and an ncclUniqueId or an "
                       "allgather callback";
        return REI_EINVAL;
      }
      c->world = opts->world_size;
      c->rank = opts->rank;
      // no NCCL id: the level exchange goes through the host all-gather callback
      c->host_xport = opts->nccl_unique_id == nullptr;
    } else if (opts->flags & REI_FLAG_EXCHANGE_SELF) {
      if (!opts->nccl_unique_id || c->sharded) {
        g_init_error = "REI_FLAG_EXCHANGE_SELF needs an ncclUniqueId (and no sharded cache)";
        return REI_EINVAL;
      }
      c->exchange_self = true;
    }
  }
  if (opts && opts->device >= 0) {
    if (cudaSetDevice(opts->device) != cudaSuccess) { g_init_error = "cudaSetDevice failed"; return REI_ECUDA; }
    c->device = opts->device;
  } else {
    cudaGetDevice(&c->device);
  }
  {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) == cudaSuccess && sms > 0) c->sms = sms;
  }
  if (opts && opts->stream) {
    c->stream = (cudaStream_t)opts->stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      g_init_error = "no CUDA device / stream creation failed";
      return REI_ECUDA;
    }
    c->own_stream = true;
  }
  auto fail = [&](const std::string& m) { g_init_error = m; return REI_ECUDA; };
  phase("validate + stream");
  if (c->dmalloc(&c->tab.split, sizeof(uint32_t) * kMaxSplitRows * kMaxNW) != cudaSuccess ||
      c->dmalloc(&c->tab.nsplit, sizeof(uint32_t) * kMaxNW) != cudaSuccess ||
      c->dmalloc(&c->tab.word_len, sizeof(uint32_t) * kMaxNW) != cudaSuccess ||
      c->dmalloc(&c->tab.seeds, sizeof(uint32_t) * kMaxW32 * k) != cudaSuccess ||
      c->dmalloc(&c->ctl_base, Ctx::kLag * sizeof(LevelCtl)) != cudaSuccess ||
      c->dmalloc(&c->d_peers, sizeof(Peer) * Ctx::kMaxShards) != cudaSuccess ||
      host_alloc(reinterpret_cast<void**>(&c->h_peers), sizeof(Peer) * Ctx::kMaxShards) != cudaSuccess ||
      c->dmalloc(&c->special, sizeof(unsigned int)) != cudaSuccess ||
      c->dmalloc(&c->d_blocks, sizeof(Block) * 3 * Ctx::kMaxBlocks) != cudaSuccess ||
      host_alloc(reinterpret_cast<void**>(&c->h_ctl), sizeof(LevelCtl)) != cudaSuccess ||
      host_alloc(reinterpret_cast<void**>(&c->h_blocks), sizeof(Block) * 3 * Ctx::kMaxBlocks) != cudaSuccess)
    return fail(std::string("device allocation failed: ") + cudaGetErrorString(cudaGetLastError()));
  phase("aux streams + small buffers");
  c->ctl = c->ctl_base;
  cudaMemsetAsync(c->tab.split, 0, sizeof(uint32_t) * kMaxSplitRows * kMaxNW, c->stream);
  if ((c->world > 1 || c->exchange_self) && !c->sharded && !c->host_xport) {  // one process per GPU: NCCL
    ncclUniqueId id;
    memcpy(&id, opts->nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    if (!nccl_api().ok) {
      g_init_error = "NCCL not available";
      return REI_ENCCL;
    }
    // NCCL allocates its own device buffers: hand the pool's idle blocks back first (a
    // process that just ran a large search may hold tens of GB of them)
    release_cached_memory();
    if (nccl_api().CommInitRank(&comm, c->world, id, c->rank) != ncclSuccess) {
      g_init_error = "ncclCommInitRank failed";
      return REI_ENCCL;
    }
    c->nccl = comm;
    if (c->dmalloc(&c->d_ctl_all, sizeof(LevelCtl) * c->world) != cudaSuccess ||
        c->dmalloc(&c->d_small, 64 * 8) != cudaSuccess || c->dmalloc(&c->d_small_all, 64 * 8 * c->world) != cudaSuccess)
      return fail("device allocation failed (control lines)");
  }
  if (c->P.empty() && c->N.empty()) {
    // nothing to precompute: only the trivial case P = {} applies
    c->tab.n = 0;
    *out = c.release();
    return REI_OK;
  }
  std::string err;
  if (!run_precompute(c->P, c->N, (int)k, c->stream, c->tab, err, &c->launches)) {
    g_init_error = err;
    return err.find("|IC|") != std::string::npos || err.find("splits") != std::string::npos ? REI_EINVAL
                                                                                              : REI_ECUDA;
  }
  phase("device precompute");
  for (auto& w : c->P) c->h2d_bytes += w.size() + 4;
  for (auto& w : c->N) c->h2d_bytes += w.size() + 4;
  c->d2h_bytes += 64 + 8ull * c->tab.n;  // table summary + IC keys
  c->W32 = next_pow2_words(c->tab.n);
  // small-cache contexts (many alive at once, f4) keep the 2^|IC|-bit bitmap for
  // |IC| <= 20 only (<= 128 KB); wider one-word CSs use the two-word 64-bit-key hash set
  // (the storage width is invisible to results: reading A16)
  if ((c->flags & REI_FLAG_SMALL_CACHE) && c->W32 == 1 && c->tab.n > 20) c->W32 = 2;
  c->mode = (c->W32 == 1) ? DEDUP_BITMAP : (c->W32 == 2 ? DEDUP_HASH64 : DEDUP_HASHIDX);
  // wide CSs whose top bits are free keep the whole CS in the slot (one sector per probe,
  // no arena read on a fingerprint match); REI_INDEXED_KEYS=1 keeps fingerprint + index
  if (c->mode == DEDUP_HASHIDX && ((c->W32 == 4 && c->tab.n <= 127) || (c->W32 == 8 && c->tab.n <= 254)) &&
      getenv("REI_INDEXED_KEYS") == nullptr)
    c->mode = DEDUP_HASHIN;
  // Finished levels are reordered by the top 12 bits of their bitmap position (A/B on
  // B200, full final level: Table 1 row 1 67.5 -> 63.6 ms, row 8 neutral; a full 25-bit
  // sort cut the kernels as much but cost more).  REI_NO_LEVEL_SORT disables it.
  c->sort_levels = c->mode == DEDUP_BITMAP && !c->sharded && getenv("REI_NO_LEVEL_SORT") == nullptr;
  if (const char* ke = getenv("REI_KERNEL_EVENTS")) c->kernel_events = atoi(ke) != 0;
  // Launch order of a level's binary kernels (REI_UNION_FIRST=0/1 overrides).  With the
  // bitmap dedup the union kernel goes first: the early exit at c* then no longer waits
  // for the union CTAs to get SMs behind a full concat grid (A/B on B200, 15 interleaved
  // solves each: Table 1 row 1 median 30.7 ms both, p90 37.5 -> 30.9 ms, max 118 ->
  // 38 ms; row 8 equal).  The HBM hash sets keep concat first (C2 median 228 -> 296 ms
  // with union first).
  {
    const char* uf = getenv("REI_UNION_FIRST");
    c->union_first = uf ? atoi(uf) != 0 : c->mode == DEDUP_BITMAP;
  }
  {
    // A level's kernels run concurrently on auxiliary streams (REI_CONCURRENT):
    // 0 = one stream; 1 = ? / * on their own stream; 2 = also union on its own stream
    // (auxiliary streams at high priority, concat on the context's stream); 3 = concat on
    // a high-priority stream, union on a low-priority one; 4 = 3 with the priorities
    // swapped.  Default (A/B on B200): 2 for the bitmap dedup (L2-resident, ALU-bound
    // kernels: Table 1 row 1 37.7 -> 30.9 ms, row 8 -4 %, full levels within 2 %), 3 for
    // the HBM hash sets (two-word C2: 253 -> 212 ms -- the DRAM-bound kernels interfere
    // less when concat has priority).
    const char* ev = getenv("REI_CONCURRENT");
    c->concurrency = ev ? std::max(0, std::min(6, atoi(ev))) : (c->mode == DEDUP_BITMAP ? 2 : 3);
    // small-cache contexts (f4: hundreds alive at once, small levels) run one stream:
    // ~1000 priority streams in one process made stream creation fail on B200
    if ((c->flags & REI_FLAG_SMALL_CACHE) && !ev) c->concurrency = 0;
    const int nstreams = std::min(3, c->concurrency);
    if (nstreams >= 1) {
      int prio_lo = 0, prio_hi = 0;
      cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
      const int low = c->concurrency == 3 ? 1 : (c->concurrency == 4 || c->concurrency == 6) ? 2 : -1;
      for (int i = 0; i < nstreams; ++i)
        if (cudaStreamCreateWithPriority(&c->aux[i], cudaStreamNonBlocking, i == low ? prio_lo : prio_hi) !=
                cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) != cudaSuccess)
          return fail("auxiliary stream creation failed");
      if (cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess)
        return fail("event creation failed");
      // post-level stream (single-rank searches; REI_NO_POST_OVERLAP=1 keeps it inline)
      if (c->world == 1 && !c->exchange_self && !c->sharded && getenv("REI_NO_POST_OVERLAP") == nullptr &&
          (cudaStreamCreateWithPriority(&c->post, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
           cudaEventCreateWithFlags(&c->ev_level_done, cudaEventDisableTiming) != cudaSuccess ||
           cudaEventCreateWithFlags(&c->ev_post, cudaEventDisableTiming) != cudaSuccess))
        return fail("post-level stream creation failed");
    }
  }

  if (c->mode == DEDUP_BITMAP) {
    c->bitmap_words = std::max<uint64_t>(1, (1ull << c->tab.n) / 32);
    if (c->dmalloc(&c->bitmap, c->bitmap_words * 4) != cudaSuccess) return fail("bitmap allocation failed");
    if (c->budget_user) c->budget = c->budget > c->bitmap_words * 4 ? c->budget - c->bitmap_words * 4 : 0;
  }
  // bitmap mode: at most 2^n distinct CSs exist, so reserve them all up front (up to
  // 2^28 entries); hash modes start at 2^22 entries and grow ahead of each level.
  uint64_t cap0 = 1ull << 22;
  if (c->mode == DEDUP_BITMAP) cap0 = std::min<uint64_t>(1ull << 28, (1ull << c->tab.n) + 64);
  if (c->flags & REI_FLAG_SMALL_CACHE) cap0 = std::min<uint64_t>(cap0, 1ull << 16);
  // the free-memory query is skipped when the initial cache is < 1/8 of the HBM
  if (c->budget_user || c->sharded || cap0 * bytes_per_entry(c.get()) > device_total_bytes(c->device) / 8)
    cap0 = std::min<uint64_t>(cap0, std::max<uint64_t>(1024, budget_of(c.get()) / bytes_per_entry(c.get())));
  phase("budget");
  if (c->sharded) {  // sized once: peers map these buffers, so they never move
    cap0 = budget_of(c.get()) / bytes_per_entry(c.get());
    if (c->mode == DEDUP_BITMAP) cap0 = std::min<uint64_t>(cap0, (1ull << c->tab.n) + 64);
    if (c->entry_limit) cap0 = std::min<uint64_t>(cap0, c->entry_limit);
    cap0 = std::max<uint64_t>(cap0, 1024);
  }
  phase("bitmap");
  if (alloc_arena(c.get(), cap0, 0, 0) != REI_OK) return fail(c->err);
  phase("arena");
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return fail("init sync failed");
  phase("dedup set + language cache");
  if (c->sharded && c->world > 1) {  // collective: map every rank's buffers (CUDA IPC)
    rei_status st = link_ipc(c.get());
    if (st != REI_OK) { g_init_error = c->err; return st; }
  }
  *out = c.release();
  return REI_OK;
}

rei_status rei_solve(void* ctx, uint32_t max_cost, rei_result* out) {
  if (!ctx) return REI_EINVAL;
  Ctx* c = static_cast<Ctx*>(ctx);
  cudaSetDevice(c->device);
  c->err.clear();
  const auto t0 = std::chrono::steady_clock::now();
  rei_status s;
  if (c->tab.n == 0 && !c->P.empty()) {
    s = REI_EINVAL;
  } else {
    s = rei::solve_impl(c, max_cost);
  }
  c->result.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  c->result.regex = c->regex.c_str();
  uint64_t uniq = 0;
  for (auto& st : c->stats) uniq += st.unique;
  c->result.unique = uniq;
  if (out) *out = c->result;
  return s;
}

rei_status rei_level_stats(const void* ctx, rei_level_stat* buf, size_t cap, size_t* n_out) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (n_out) *n_out = c->stats.size();
  for (size_t i = 0; i < c->stats.size() && i < cap && buf; ++i) buf[i] = c->stats[i];
  return REI_OK;
}

rei_status rei_kernel_stats(const void* ctx, rei_kernel_class k, uint64_t* launches, double* ms) {
  if (!ctx || k < 0 || k >= REI_K_COUNT) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (launches) *launches = c->k_launches[k];
  if (ms) *ms = c->k_ms[k];
  return REI_OK;
}

rei_status rei_reset_kernel_stats(void* ctx) {
  if (!ctx) return REI_EINVAL;
  Ctx* c = static_cast<Ctx*>(ctx);
  c->kernel_events = true;  // per-kernel CUDA events from now on (a few us of host time per launch)
  for (int i = 0; i < REI_K_COUNT; ++i) { c->k_launches[i] = 0; c->k_ms[i] = 0; }
  c->launches = 0;
  return REI_OK;
}

uint64_t rei_launch_count(const void* ctx) { return ctx ? static_cast<const Ctx*>(ctx)->launches : 0; }

int rei_dedup_mode(const void* ctx) { return ctx ? static_cast<const Ctx*>(ctx)->mode : -1; }

rei_status rei_transfer_bytes(const void* ctx, uint64_t* h2d, uint64_t* d2h) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (h2d) *h2d = c->h2d_bytes;
  if (d2h) *d2h = c->d2h_bytes;
  return REI_OK;
}

const char* rei_last_error(const void* ctx) {
  return ctx ? static_cast<const Ctx*>(ctx)->err.c_str() : rei::g_init_error.c_str();
}
const char* rei_last_init_error(void) { return rei::g_init_error.c_str(); }

void rei_destroy(void* ctx) { delete static_cast<Ctx*>(ctx); }

void rei_release_cached_memory(void) { rei::release_cached_memory(); }

rei_status rei_ic(const void* ctx, uint32_t k, char* buf, size_t cap, uint32_t* n_ic) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (n_ic) *n_ic = (uint32_t)c->tab.n;
  if (!buf) return REI_OK;
  if (k >= (uint32_t)c->tab.n) return REI_EINVAL;
  const unsigned long long key = c->tab.ic_keys[k];
  const int len = (int)(key >> 58);
  unsigned long long v = key & ((1ull << 58) - 1);
  if ((size_t)len + 1 > cap) return REI_EINVAL;
  const size_t base = c->alphabet.size();
  for (int i = len - 1; i >= 0; --i) {
    buf[i] = c->alphabet[v % base];
    v /= base;
  }
  buf[len] = 0;
  return REI_OK;
}

rei_status rei_splits(const void* ctx, uint32_t w, uint32_t* pairs, size_t cap, uint32_t* count) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  if (w >= (uint32_t)c->tab.n) return REI_EINVAL;
  uint32_t m = 0;
  if (cudaMemcpy(&m, c->tab.nsplit + w, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return REI_ECUDA;
  if (count) *count = m;
  for (uint32_t kk = 0; kk < m && kk < cap && pairs; ++kk) {
    uint32_t sp = 0;
    if (cudaMemcpy(&sp, c->tab.split + (size_t)kk * rei::kMaxNW + w, 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      return REI_ECUDA;
    pairs[2 * kk] = sp >> 16;
    pairs[2 * kk + 1] = sp & 0xffff;
  }
  return REI_OK;
}

rei_status rei_masks(const void* ctx, uint32_t* pos, uint32_t* neg) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  for (int q = 0; q < c->W32; ++q) {
    if (pos) pos[q] = c->tab.pos[q];
    if (neg) neg[q] = c->tab.neg[q];
  }
  return REI_OK;
}

rei_status rei_level_cs(const void* ctx, uint32_t cost, uint32_t* out, size_t cap, size_t* count) {
  if (!ctx) return REI_EINVAL;
  const Ctx* c = static_cast<const Ctx*>(ctx);
  auto it = c->levels.find((int)cost);
  const uint64_t m = it == c->levels.end() ? 0 : it->second.size;
  if (count) *count = m;
  if (!out || !m) return REI_OK;
  const uint64_t take = std::min<uint64_t>(m, cap);
  const rei::LevelInfo& lv = it->second;
  if (!lv.ssize.empty()) {  // sharded cache: the owners' shards in rank order
    for (size_t o = 0; o < lv.ssize.size(); ++o) {
      if (lv.soff[o] >= take || !lv.ssize[o]) continue;
      const uint64_t n = std::min<uint64_t>(lv.ssize[o], take - lv.soff[o]);
      if (cudaMemcpy(out + lv.soff[o] * c->W32, c->peers[o].arena + lv.sbegin[o] * c->W32, n * 4ull * c->W32,
                     cudaMemcpyDeviceToHost) != cudaSuccess)
        return REI_ECUDA;
    }
    return REI_OK;
  }
  if (cudaMemcpy(out, c->arena + lv.begin * c->W32, take * 4ull * c->W32, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    return REI_ECUDA;
  return REI_OK;
}

rei_status rei_entry_regex(const void* ctx, uint32_t cost, uint64_t i, char* buf, size_t cap) {
  if (!ctx) return REI_EINVAL;
  Ctx* c = const_cast<Ctx*>(static_cast<const Ctx*>(ctx));
  auto it = c->levels.find((int)cost);
  if (it == c->levels.end() || i >= it->second.size) return REI_EINVAL;
  std::string s;
  int pr;
  if (!rei::rebuild_entry(c, (int)cost, i, s, pr, 0)) return REI_ECUDA;
  if (s.size() + 1 > cap) return REI_EINVAL;
  memcpy(buf, s.c_str(), s.size() + 1);
  return REI_OK;
}

rei_status rei_cs_ops(void* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out, size_t count) {
  if (!ctx || !a || !out) return REI_EINVAL;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!count) return REI_OK;
  const size_t bytes = count * 4ull * c->W32;
  uint32_t *da = nullptr, *db = nullptr, *dout = nullptr;
  CUDA_OK(c, cudaMalloc(&da, bytes));
  CUDA_OK(c, cudaMalloc(&db, bytes));
  CUDA_OK(c, cudaMalloc(&dout, bytes));
  CUDA_OK(c, cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, c->stream));
  if (b) CUDA_OK(c, cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, c->stream));
  rei::LevelParams p;
  rei::fill_params(c, p);
  rei::EventPair ep;
  c->begin_kernel(REI_K_OTHER, ep);
  int n = rei::launch_ops(c->W32, p, op, da, b ? db : nullptr, dout, count, c->stream);
  c->end_kernel(ep, n);
  CUDA_OK(c, cudaGetLastError());
  CUDA_OK(c, cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(c, cudaStreamSynchronize(c->stream));
  c->collect_events(nullptr);
  cudaFree(da); cudaFree(db); cudaFree(dout);
  return REI_OK;
}

rei_status rei_nccl_unique_id(void* out, size_t cap) {
  if (!out || cap < sizeof(ncclUniqueId)) return REI_EINVAL;
  ncclUniqueId id;
  if (!rei::nccl_api().ok || rei::nccl_api().GetUniqueId(&id) != ncclSuccess) return REI_ENCCL;
  memcpy(out, &id, sizeof(id));
  return REI_OK;
}

rei_status rei_solve_group(void* const* ctxs, int G, uint32_t max_cost, rei_result* out) {
  if (!ctxs || G < 1) return REI_EINVAL;
  rei::Comm g;
  g.world = G;
  g.rank0 = 0;
  for (int i = 0; i < G; ++i) {
    Ctx* c = static_cast<Ctx*>(ctxs[i]);
    if (!c || c->world > 1) return REI_EINVAL;
    if (i > 0 && (c->tab.n != g.m[0]->tab.n || c->W32 != g.m[0]->W32 || c->mode != g.m[0]->mode))
      return REI_EINVAL;
    c->err.clear();
    g.m.push_back(c);
  }
  const auto t0 = std::chrono::steady_clock::now();
  int n_sharded = 0;
  for (Ctx* c : g.m) n_sharded += c->sharded ? 1 : 0;
  if (n_sharded && n_sharded != G) return REI_EINVAL;
  if (n_sharded && G > Ctx::kMaxShards) return REI_EINVAL;
  if (n_sharded) rei::link_local(g.m);
  rei_status s = n_sharded && G > 1 ? rei::solve_sharded(g, max_cost) : rei::solve_group(g, max_cost);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::string first_err;
  for (Ctx* c : g.m)
    if (first_err.empty()) first_err = c->err;
  for (Ctx* c : g.m) {
    c->result.seconds = secs;
    c->result.regex = c->regex.c_str();
    uint64_t uniq = 0;
    for (auto& st : c->stats) uniq += st.unique;
    c->result.unique = uniq;
    if (s != REI_OK && s != REI_NOT_FOUND && s != REI_OUT_OF_MEMORY && c->err.empty()) c->err = first_err;
  }
  if (out) *out = g.m[0]->result;
  return s;
}

rei_status rei_solve_packed(void* const* ctxs, size_t n, uint32_t max_cost, rei_result* out, rei_status* status,
                            double* done_seconds) {
  if (!ctxs || n == 0) return REI_EINVAL;
  std::vector<Ctx*> cs(n);
  for (size_t i = 0; i < n; ++i) {
    cs[i] = static_cast<Ctx*>(ctxs[i]);
    if (!cs[i] || cs[i]->device != cs[0]->device) return REI_EINVAL;
  }
  cudaSetDevice(cs[0]->device);
  // every context's pending work (rei_init) is done before the shared stream runs
  for (Ctx* c : cs) cudaStreamSynchronize(c->stream);
  std::vector<rei_status> st;
  std::vector<double> done;
  const auto t0 = std::chrono::steady_clock::now();
  // every context's work (packed launches, growth, reconstruction) on one stream for
  // the packed steps; each context's own stream again for a spec solved alone
  std::vector<cudaStream_t> own(n);
  for (size_t i = 0; i < n; ++i) { own[i] = cs[i]->stream; cs[i]->stream = cs[0]->stream; }
  rei_status s = rei::solve_packed(cs, max_cost, st, done, own);
  for (size_t i = 0; i < n; ++i) cs[i]->stream = own[i];
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (size_t i = 0; i < n; ++i) {
    Ctx* c = cs[i];
    c->result.seconds = i < done.size() ? done[i] : secs;
    c->result.regex = c->regex.c_str();
    uint64_t uniq = 0;
    for (auto& l : c->stats) uniq += l.unique;
    c->result.unique = uniq;
    if (out) out[i] = c->result;
    if (status) status[i] = i < st.size() ? st[i] : s;
    if (done_seconds) done_seconds[i] = c->result.seconds;
  }
  return s;
}

rei_status rei_solve_batch(void* const* ctxs, size_t n, uint32_t max_cost, int threads, rei_result* out,
                           rei_status* status) {
  if (!ctxs) return REI_EINVAL;
  if (threads < 1) threads = 1;
  std::atomic<size_t> next{0};
  auto worker = [&]() {
    for (size_t i = next++; i < n; i = next++) {
      rei_result r{};
      const rei_status s = rei_solve(ctxs[i], max_cost, &r);
      if (out) out[i] = r;
      if (status) status[i] = s;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads && (size_t)t < n; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return REI_OK;
}

int rei_cs_owner(const uint32_t* cs, uint32_t cs_words, int world) {
  if (world <= 1 || !cs) return 0;
  switch (cs_words) {
#define REI_OWNER_CASE(W)                                          \
  case W: {                                                        \
    uint32_t x[W];                                                 \
    for (int q = 0; q < W; ++q) x[q] = cs[q];                      \
    return (int)rei::owner_of_hash(rei::hash_cs<W>(x), (uint32_t)world); \
  }
    REI_OWNER_CASE(1)
    REI_OWNER_CASE(2)
    REI_OWNER_CASE(4)
    REI_OWNER_CASE(8)
    REI_OWNER_CASE(16)
#undef REI_OWNER_CASE
    default:
      return -1;
  }
}

void rei_exchange_offsets(int world, const uint64_t* counts, int rank, uint64_t* send_off, uint64_t* recv_off) {
  for (int o = 0; o < world; ++o) {
    uint64_t x = 0;
    for (int q = 0; q < o; ++q) x += counts[(size_t)rank * world + q];
    if (send_off) send_off[o] = x;
  }
  for (int r = 0; r < world; ++r) {
    uint64_t x = 0;
    for (int q = 0; q < r; ++q) x += counts[(size_t)q * world + rank];
    if (recv_off) recv_off[r] = x;
  }
}

void rei_partition(uint64_t total, int G, int g, uint64_t* begin, uint64_t* end) {
  if (G <= 0) G = 1;
  const uint64_t b = total / (uint64_t)G * (uint64_t)g + std::min<uint64_t>((uint64_t)g, total % (uint64_t)G);
  const uint64_t len = total / (uint64_t)G + ((uint64_t)g < total % (uint64_t)G ? 1 : 0);
  if (begin) *begin = b;
  if (end) *end = b + len;
}

}  // extern "C"
