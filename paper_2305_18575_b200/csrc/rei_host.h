// rei_host.h -- host-side declarations shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "rei_common.cuh"

namespace rei {

// Device-resident staged precompute (owned by the context).
struct DeviceTables {
  int n = 0;        // |IC|
  int maxk = 0;     // max proper splits of one word
  int maxlen = 0;   // longest IC word
  uint32_t* split = nullptr;     // [kMaxSplitRows][kMaxNW]
  uint32_t* nsplit = nullptr;    // [kMaxNW]
  uint32_t* word_len = nullptr;  // [kMaxNW]
  uint32_t* seeds = nullptr;     // [k][kMaxW32]
  uint32_t pos[kMaxW32] = {0};
  uint32_t neg[kMaxW32] = {0};
  std::vector<unsigned long long> ic_keys;  // host copy for introspection / printing
};

bool run_precompute(const std::vector<std::vector<uint8_t>>& P, const std::vector<std::vector<uint8_t>>& N,
                    int k, cudaStream_t st, DeviceTables& t, std::string& err, uint64_t* launches);

// Kernel launchers (levels.cu).  Each returns the number of kernels launched.
int launch_seeds(int W32, const LevelParams& p, const uint32_t* seeds, int nsym, cudaStream_t st);
int launch_unary(int W32, const LevelParams& p, uint64_t n_q, uint64_t n_s, uint64_t a_base_q,
                 uint64_t a_base_s, uint64_t off_s, uint64_t slab_s, cudaStream_t st);
int launch_concat(int W32, const LevelParams& p, bool slice_a, cudaStream_t st);
int launch_union(int W32, const LevelParams& p, cudaStream_t st);
int launch_transpose(int W32, const uint32_t* arena, uint64_t base, uint64_t count, uint32_t* tarena,
                     uint64_t slab_base, cudaStream_t st);
int launch_rehash(int W32, const LevelParams& p, uint64_t base, uint64_t count, cudaStream_t st);
// Device-resident loop over the small levels (DevLoop); 0 = not launched.
int launch_level_loop(int W32, const LevelParams& p, const DevLoop& d, cudaStream_t st);
// Lagged levels: next level's arena base from the previous level's count (k_next_base).
int launch_next_base(const LevelCtl* prev, const unsigned long long* prev_base, unsigned long long* base,
                     LevelCtl* next, unsigned long long* rank_off, uint32_t unary_reads_prev, cudaStream_t st);
// Packed launches (f4, rei_solve_packed): one grid, CTA group i runs pk.params[i]
// (W32 in {1, 2} and <= 15 proper splits per word; maxk_class = 1, 3, 7 or 15).
int packable(int W32, int maxk);
int maxk_class(int maxk);
int launch_ctl_reset_packed(const LevelParams* params, uint32_t n, cudaStream_t st);
int launch_ctl_gather_packed(const LevelParams* params, uint32_t n, LevelCtl* out, cudaStream_t st);
int launch_concat_packed(int W32, int maxk, bool slice_a, const Packed& pk, uint32_t ctas, size_t max_nblocks,
                         cudaStream_t st);
int launch_union_packed(int W32, const Packed& pk, uint32_t ctas, size_t max_nblocks, cudaStream_t st);
int launch_unary_packed(int W32, int maxk, const Packed& pk, uint32_t ctas, cudaStream_t st);
int launch_transpose_packed(int W32, const Packed& pk, uint32_t ctas, cudaStream_t st);

// Canonical first-occurrence merge of an all-gathered level list (exchange.cu).
struct MergeScratch {
  void *keys = nullptr, *keys2 = nullptr, *pos = nullptr, *pos2 = nullptr, *flags = nullptr, *scan = nullptr,
       *temp = nullptr;
  size_t keys_cap = 0, keys2_cap = 0, pos_cap = 0, pos2_cap = 0, flags_cap = 0, scan_cap = 0, temp_cap = 0;
};
bool merge_level(int W32, const uint32_t* g_cs, const unsigned long long* g_bp, uint64_t m, uint32_t* out_cs,
                 unsigned long long* out_bp, uint64_t* out_count, MergeScratch& s, cudaStream_t st,
                 std::string& err, uint64_t* launches);
void free_merge_scratch(MergeScratch& s);
// Reorder a finished one-word (bitmap-mode) level by bitmap position, in place.
bool sort_level(uint32_t n, uint32_t* cs, unsigned long long* bp, uint64_t m, MergeScratch& s, cudaStream_t st,
                std::string& err, uint64_t* launches, bool may_skip);
// Hash-owner exchange of a multi-rank level (exchange.cu).  Records are
// (CS words, back-pointer as 2 words), 4 * (W32 + 2) bytes each.
struct XScratch {
  void *owner = nullptr, *send = nullptr, *recv = nullptr, *uniq = nullptr, *gath = nullptr, *table = nullptr,
       *ctr = nullptr;
  size_t owner_cap = 0, send_cap = 0, recv_cap = 0, uniq_cap = 0, gath_cap = 0, table_cap = 0, ctr_cap = 0;
};
// Bucket the m staged entries by hash owner into x.send (owner-contiguous records);
// counts[o] (host) = records owned by rank o.
bool owner_bucket(int W32, const uint32_t* cs, const unsigned long long* bp, uint64_t m, int world, XScratch& x,
                  cudaStream_t st, uint64_t* counts, std::string& err, uint64_t* launches);
bool ensure_recv(int W32, uint64_t m, XScratch& x, cudaStream_t st);
// Dedup the m records of x.recv into x.uniq (first insert of each CS wins); *out_count.
bool owner_dedup(int W32, uint64_t m, XScratch& x, cudaStream_t st, uint64_t* out_count, std::string& err,
                 uint64_t* launches);
bool ensure_gather_recs(int W32, uint64_t m, XScratch& x, cudaStream_t st);
bool unpack_records(int W32, const uint32_t* rec, uint64_t m, uint32_t* cs, unsigned long long* bp, cudaStream_t st,
                    uint64_t* launches);
// Sort a level computed redundantly on every rank into a rank-independent order (by CS).
bool canon_sort_level(int W32, uint32_t n, uint32_t* cs, unsigned long long* bp, uint64_t m, MergeScratch& s,
                      cudaStream_t st, std::string& err, uint64_t* launches);
void free_xscratch(XScratch& x);
int launch_ops(int W32, const LevelParams& p, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
               uint64_t count, cudaStream_t st);

// Process-wide caching allocators (devmem.cu): size-keyed free lists of device blocks
// and of pinned host blocks.
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st);
void dev_free(void* p, cudaStream_t st);
uint64_t dev_pool_idle_bytes(int dev);
// Free device memory as this process sees it: one cudaMemGetInfo per device, then the
// pool's own cudaMalloc / cudaFree traffic, plus its idle blocks (releasable on demand).
uint64_t dev_free_estimate(int dev);
void dev_free_estimate_reset(int dev);  // re-query on the next estimate (after an OOM)
cudaError_t host_alloc(void** p, size_t bytes);
void host_free(void* p);
void release_cached_memory();

// Work-item tiling of the pair kernels (uniform operands x slabs of 32).
constexpr int kTileU = 64;    // uniform operands per work item
constexpr int kTileS = 4;     // slabs (of 32 sliced operands) per work item

}  // namespace rei
