// rei_common.cuh -- device/host structures of the B200 REI hot path.
//
// Layout in HBM:
//   arena   : the language cache: one CS per entry,
//             W32 32-bit words, entries of one cost level contiguous, levels in
//             increasing cost, write-once.
//   bp      : one u64 back-pointer per entry = the candidate's rank in its level's
//             flattened block space (Q, S, C by L ascending, U by L ascending,
//             row-major); the host decodes it with the level plan.
//   tarena  : the same levels bit-transposed in slabs of 32 CSs: slab word v has
//             bit t = CS_t[v] (the "sliced" operand layout of the concat kernel).
//   dedup   : bitmap over all 2^n CSs (n <= 32) or an open-addressing hash set.
#pragma once
#include <cstdint>

namespace rei {

constexpr int kMaxW32 = 16;        // CS words: |IC| <= 512 bits
constexpr int kMaxNW = 32 * kMaxW32;
constexpr int kMaxSplitRows = 64;  // max proper splits of one IC word (|w| - 1)

enum BlockKind : uint32_t { BK_Q = 0, BK_S = 1, BK_C = 2, BK_U = 3 };

// One operand block of a cost level (Alg. 1 lines 5-8, Alg. 2 line 2).
struct Block {
  uint32_t kind;      // BlockKind
  uint32_t slice_a;   // C/U: 1 => the A (left) operand is the sliced side, B uniform
  uint32_t tri;       // U with L == R: only i < j
  uint32_t pad;
  uint64_t a_base, b_base;  // arena index of the first entry of level L / R
  uint64_t a_slab, b_slab;  // tarena slab index of level L / R
  uint64_t na, nb;          // |lvl(L)|, |lvl(R)|
  uint64_t cand_off;        // rank of the first candidate of this block within the level
  uint64_t cand_count;
  uint64_t item_off;        // first work item of this block (pair kernels)
  uint64_t u_tiles, s_tiles;  // work-item grid: uniform tiles x slab tiles
  uint64_t tu, ts;            // uniform operands / slabs (of 32) per work item
};

// Per-level control block, reset before each level.  The flags every warp polls
// (found_rank per work item, overflow every 16th probe step) sit on their own 128-byte
// line, away from the counters the warps update atomically (count per append flush,
// evaluated per work item): on one line the polls and the atomics serialise in the
// same L2 slice.
struct LevelCtl {
  unsigned long long found_rank;  // min rank of a precise candidate; ~0 = none
  unsigned int overflow;          // arena / hash capacity exceeded
  unsigned int special_seen;      // hash64 mode: the sentinel key was inserted
  unsigned long long pad0[14];
  unsigned long long count;       // new CSs appended to the level
  unsigned long long evaluated;   // candidates evaluated (items finished)
  unsigned long long eval_c;      // of which by the concat kernel
  unsigned long long eval_u;      // of which by the union kernel
  unsigned long long pad1[12];
};
static_assert(sizeof(LevelCtl) == 256, "two 128-byte lines");

// DEDUP_HASHIN: the CS itself is the slot (16 B for W32 = 4, 32 B for W32 = 8), so a
// probe that hits costs one random 32-byte sector; used when the top CS bit(s) are
// never set (|IC| <= 127 / 254), which frees the all-ones pattern as the empty slot.
enum DedupMode : int { DEDUP_BITMAP = 0, DEDUP_HASH64 = 1, DEDUP_HASHIDX = 2, DEDUP_HASHIN = 3 };

struct Dedup {
  int mode;
  int pad;
  uint32_t* bitmap;                 // DEDUP_BITMAP: 2^n bits
  unsigned long long* table;        // DEDUP_HASH64 / DEDUP_HASHIDX / DEDUP_HASHIN (W32 / 2 u64 per slot)
  unsigned long long mask;          // slots - 1
  unsigned int* special;            // DEDUP_HASH64: persistent "all-ones key present" flag
};

// One rank's cache as every rank sees it in sharded-cache mode:
// the owner of a CS (a hash of its bits) holds its dedup slot, arena entry and
// back-pointer; other ranks insert through peer mappings of these buffers (NVLink
// P2P, or CUDA IPC across processes).  Field names match LevelParams, so the insert
// routines take either.
struct Peer {
  uint32_t* arena_out;
  unsigned long long* bp;
  LevelCtl* ctl;
  Dedup dedup;
  unsigned long long out_base;  // owner's arena index of its shard of level c
  unsigned long long cap;       // owner's arena capacity
};

struct LevelParams {
  const uint32_t* arena;      // CS arena (read: operand levels)
  uint32_t* arena_out;        // same buffer (write: level c)
  const uint32_t* tarena;     // transposed slabs
  unsigned long long* bp;     // back-pointers
  const Block* blocks;
  uint32_t nblocks;
  uint32_t n;                 // |IC|
  uint32_t maxk;              // max proper splits per word
  uint32_t max_errors;        // allowed-error budget (misclassified examples)
  uint32_t exact;             // 1 = precise test, 0 = allowed-error test
  uint32_t early_exit;        // 1 = stop at the first precise candidate
  uint32_t otf;               // OnTheFly level: test every candidate, no dedup / append
  uint64_t item_begin;        // this rank's share [item_begin, total_items) of the work items
  uint64_t total_items;
  uint64_t out_base;          // arena index of the first entry of level c
  uint64_t cap;               // arena capacity in entries
  const uint32_t* split;      // [k][kMaxNW] packed (u << 16) | v proper splits
  const uint32_t* nsplit;     // [kMaxNW] number of proper splits per word
  const uint32_t* word_len;   // [kMaxNW] length of each IC word
  LevelCtl* ctl;
  Dedup dedup;
  uint32_t shards;            // sharded-cache mode: number of owners (0/1 = local cache)
  uint32_t pad_s;
  const Peer* peers;          // [shards], device memory of this rank
  uint64_t rank_base;         // unary kernels: rank of their first candidate
  const uint32_t* stage_cs;   // multi-rank levels: the staging list (== arena_out while the
                              // level runs) that tentative indexed-hash slots point into
  uint32_t tent;              // kTent in multi-rank levels with the indexed hash set, else 0
  uint32_t pad_t;
  // packed launches (f4, rei_solve_packed): the per-spec operands of the unary kernel
  // (? count / arena base, * count / arena base / first slab) and of the transpose
  // (level count in un_q, arena base in un_bq, first slab in un_slab)
  uint64_t un_q, un_s, un_bq, un_bs, un_slab;
  // lagged levels (rei_api.cu solve_group): the level's first arena index is computed on
  // the device from the previous level's count (k_next_base) and read from here; null
  // = out_base above
  const unsigned long long* out_base_dev;
  // split levels (solve_lagged): the binary kernels start before the count of the level
  // their unary blocks read is back; that count (the ? / * candidates ranked first) is
  // added to every block's cand_off on the device.  null = none
  const unsigned long long* rank_off_dev;
  uint32_t pos[kMaxW32];
  uint32_t neg[kMaxW32];
};

// Device-resident level loop (k_level_loop): the launch-bound small levels of a search
// run inside ONE persistent kernel -- plan (Alg. 1 lines 5-8), candidates, dedup,
// precision, append, transpose -- with grid barriers between levels instead of a host
// round trip per level.  Thread (0, 0) plans every level exactly as the host's
// plan_level flattens it (Q | S | C by L | U by L), so back-pointer ranks decode the
// same way.  State shared by the CTAs lives in `LoopState` (device memory).
struct LoopState {
  unsigned long long arena_used, slabs_used;  // cache fill (entries, slabs)
  unsigned long long out_base;                // arena index of the level being built
  unsigned long long items;                   // work items of that level
  unsigned long long tr_base, tr_count, tr_slab;  // level to transpose this round (count 0 = none)
  unsigned long long found_rank;              // copy of the level's ctl found_rank at stop
  long long t_level;                          // %globaltimer at the level's start
  uint32_t cost;                              // level being built (0 = none yet)
  uint32_t next_cost;                         // where the host continues
  uint32_t stop;                              // LoopStop
  uint32_t nblocks;
  uint32_t last_cost;                         // last level finished (complete or found)
  uint32_t sorting;                           // 1: order level [tr_base, +tr_count) this round
};
enum LoopStop : uint32_t {
  LOOP_RUN = 0, LOOP_FOUND = 1, LOOP_BIG = 2, LOOP_CAPACITY = 3, LOOP_SORT = 4, LOOP_MAXCOST = 5,
  LOOP_BLOCKS = 6, LOOP_OVERFLOW = 7
};
constexpr int kLoopMaxBlocks = 96;
constexpr int kLoopSortBuckets = 4096;  // top 12 bits of the bitmap position
struct DevLoop {
  unsigned long long* lvl_size;   // [max_cost + 1] entries of each level (0 = none)
  unsigned long long* lvl_begin;  // [max_cost + 1]
  unsigned long long* lvl_slab;   // [max_cost + 1]
  unsigned long long* lvl_eval;   // [max_cost + 1] candidates evaluated
  long long* lvl_ns;              // [max_cost + 1] level time (ns, %globaltimer)
  Block* blocks;                  // [kLoopMaxBlocks] the current level's plan
  LoopState* st;
  unsigned int* bar;              // [2] grid barrier: arrivals, generation
  unsigned long long cand_limit;  // a level with more candidates goes back to the host
  unsigned long long entry_limit; // cache entries the loop may fill (arena / hash load)
  unsigned long long sort_min;    // stop after a level of >= sort_min entries (0 = never)
  unsigned long long slab_limit;  // transposed slabs the loop may fill
  unsigned int* hist;             // [kLoopSortBuckets] bucket counts / cursors of the level sort
  uint32_t c1, first_cost, max_cost;
  uint32_t k_opt, k_star, k_cat, k_alt;
  uint32_t rows;                  // 1: bit-sliced concatenation rows (REI_LOOP_ROWS=0 turns off)
};

// One packed launch serving many specifications: CTA group i =
// blocks [cta_start[i], cta_start[i+1]) runs specification i with params[i].
struct Packed {
  const LevelParams* params;
  const uint32_t* cta_start;  // [nspec + 1]
  uint32_t nspec;
};

#ifdef __CUDACC__
// 64-bit hash of a CS (W 32-bit words): slot bits of the dedup sets, and the owner
// rank (bits 40.., independent of the slot bits) of the multi-GPU exchange and of the
// sharded cache.  Host and device share it (rei_cs_owner).
template <int W>
__host__ __device__ __forceinline__ unsigned long long hash_cs(const uint32_t (&cs)[W]) {
  unsigned long long h = 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    h = (h ^ cs[q]) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
  h *= 0x94D049BB133111EBull;
  return h ^ (h >> 29);
}
__host__ __device__ __forceinline__ uint32_t owner_of_hash(unsigned long long h, uint32_t world) {
  return (uint32_t)(h >> 40) % world;
}
#endif

}  // namespace rei
