/* rei.h -- C ABI of the B200-native Paresy REI hot path (librei_b200.so).
 *
 * Precise-and-minimal regular expression inference (REI) by bottom-up,
 * cost-level-by-cost-level enumeration of characteristic sequences (CS) over
 * the infix closure IC(P u N), after Valizadeh & Berger, "Search-Based
 * Regular Expression Inference on a GPU" (arXiv 2305.18575).
 * Citations: P:n = line n of the paper text; S:n = SPEC.md.
 *
 * Conventions for every call:
 *  - Plain C types and host pointers only; no torch / CUDA types cross the ABI
 *    (streams and NCCL communicators are passed as opaque `void*`).
 *  - Every call returns rei_status; no exception crosses the ABI.  After a
 *    non-OK status, rei_last_error(ctx) describes it (ctx may be NULL for
 *    rei_init failures: use rei_last_init_error()).
 *  - A context is NOT thread-safe; use one context per host thread / GPU.
 *  - All device memory is owned by the context and freed by rei_destroy().
 *  - Inputs are copied during rei_init; the caller keeps ownership of them.
 */
#ifndef REI_B200_H
#define REI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; 0/1/2/3 mirror SPEC's exit codes. */
typedef enum {
  REI_OK = 0,             /* a minimal precise regex was found                        */
  REI_EINVAL = 1,         /* invalid input: P cap N != {}, symbol outside Sigma,
                             cost < 1, duplicate symbol, |IC| > 512, word too long */
  REI_NOT_FOUND = 2,      /* max_cost exhausted: Alg. 1 "not_found"     */
  REI_OUT_OF_MEMORY = 3,  /* the language cache / dedup set cannot hold the next level:
                             the paper's "out-of-memory error"             */
  REI_ECUDA = 4,          /* a CUDA runtime error (message in rei_last_error)         */
  REI_ENCCL = 5           /* a collective failed (multi-GPU)                          */
} rei_status;

/* Cost homomorphism (c1..c5) = (cost(a), cost(?), cost(*), cost(.), cost(+)),
 * every c_i >= 1.  cost(empty) = cost(eps) = cost(a) = c1. */
typedef struct {
  uint32_t sym, opt, star, cat, alt;
} rei_costs;

/* Option flags. */
#define REI_FLAG_COMPLETE_FINAL_LEVEL 1u /* finish level c* instead of stopping at the
                                            first precise CS (for full level counts)  */
#define REI_FLAG_NO_EARLY_EXIT REI_FLAG_COMPLETE_FINAL_LEVEL
#define REI_FLAG_NO_ONTHEFLY 2u          /* stop with REI_OUT_OF_MEMORY as soon as the cache
                                            is full instead of switching to OnTheFly mode
                                            (check candidates built from cached
                                            levels without caching them, until a level needs
                                            an uncached one)                              */
#define REI_FLAG_SHARDED_CACHE 4u        /* multi-GPU capacity mode (not in the
                                            paper; P:731-734 names memory as the limit): every
                                            rank holds only the CSs it owns (hash of the CS mod
                                            world_size) -- dedup slot, cache entry, back-pointer --
                                            and the level kernels read operands from, and insert
                                            candidates into, the owners' buffers through peer
                                            mappings (NVLink P2P / CUDA IPC).  The cache is sized
                                            once at rei_init (no growth); G ranks hold G x the
                                            entries of one.  Needs world_size > 1 with `allgather`
                                            (one process per rank) or rei_solve_group.          */
#define REI_FLAG_SMALL_CACHE 8u          /* start the language cache at 2^16 entries and grow
                                            x8 on demand, also in bitmap mode (which otherwise
                                            reserves all 2^|IC| entries at rei_init): many
                                            small contexts alive at once (f4)              */
#define REI_FLAG_EXCHANGE_SELF 16u       /* a one-rank world (world_size 1 + nccl_unique_id)
                                            that still runs every step of the multi-GPU level
                                            exchange of SURVEY 8(e): redundant small levels with
                                            their canonical sort, staged levels bucketed by hash
                                            owner, grouped ncclSend/ncclRecv to itself, owner
                                            dedup, ncclBroadcast all-gather of the uniques and
                                            the control-line ncclAllGather -- the NCCL data
                                            plane on one GPU (results equal a plain solve)  */

/* Host all-gather supplied by the caller for REI_FLAG_SHARDED_CACHE across processes
 * (the binding builds it on torch.distributed): every rank passes `bytes` bytes in
 * `send`; `recv` receives world_size * bytes, rank order.  Returns 0 on success.  It is
 * also the per-level barrier of that mode. */
typedef int (*rei_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);

typedef struct {
  int device;                /* CUDA device ordinal; -1 = the current device             */
  void* stream;              /* cudaStream_t to run on; NULL = a context-owned stream   */
  uint64_t mem_budget_bytes; /* device bytes for cache + dedup set; 0 = 80% of free memory */
  uint32_t err_num, err_den; /* allowed error e = err_num/err_den; 0/x = exact */
  uint32_t flags;            /* REI_FLAG_*                                                */
  /* multi-GPU (one context per rank; rei_solve is then collective, S 8(e)) */
  int world_size;            /* 0 or 1 = single GPU                                       */
  int rank;
  const void* nccl_unique_id;/* 128-byte ncclUniqueId, broadcast by the caller (rank 0's);
                                NULL with `allgather` set: host-staged level exchange      */
  uint64_t max_entries;      /* cap on cached CSs (the language cache size); 0 = set by the
                                memory budget only.  With REI_FLAG_SHARDED_CACHE: per rank  */
  rei_allgather_fn allgather;/* one process per rank: the host all-gather used by
                                REI_FLAG_SHARDED_CACHE, and by the replicated multi-rank
                                search when nccl_unique_id is NULL (NULL otherwise)        */
  void* allgather_user;      /* passed back to `allgather`                                */
} rei_options;

/* Result of rei_solve.  `regex` is owned by the context and valid until the next
 * rei_solve or rei_destroy.  Regex syntax is the paper's: union '+', concatenation
 * by juxtaposition, postfix '?' and '*'; "empty" / "eps" for the trivial answers
 * (Alg. 1 lines 1-2). */
typedef struct {
  const char* regex;
  uint32_t cost;                /* c*, the minimal cost (valid when status == REI_OK)    */
  uint32_t last_complete_cost;  /* highest cost level fully enumerated                    */
  uint64_t candidates;          /* candidates through the last complete level (reading A9)
                                   plus those evaluated in the final level                 */
  uint64_t cand_complete;       /* candidates through the last complete level only        */
  uint64_t unique;              /* CSs in the language cache                              */
  double seconds;               /* wall time of rei_solve (host clock, device-synchronised) */
  uint32_t n_ic;                /* |IC(P u N)|, the CS length in bits        */
  uint32_t cs_words;            /* CS width in 32-bit words (power of two)                */
} rei_result;

/* Per-cost-level statistics (one entry per non-empty level, ascending cost). */
typedef struct {
  uint32_t cost;
  uint32_t complete;           /* 1 if the level was fully enumerated and cached; 2 if it
                                  was fully checked in OnTheFly mode (not cached, unique = 0);
                                  0 if the search stopped inside it                       */
  uint64_t cand_q, cand_s, cand_c, cand_u; /* candidates by outermost constructor (A9)  */
  uint64_t unique;             /* new unique CSs appended at this level                 */
  uint64_t evaluated;          /* candidates actually evaluated (== sum of cand_* when complete) */
  uint64_t eval_c, eval_u;     /* of which by the concatenation / union kernels        */
  double ms;                   /* device time of the level (CUDA events)                */
} rei_level_stat;

/* Kernel classes for rei_kernel_stats. */
typedef enum {
  REI_K_PRECOMPUTE = 0, REI_K_UNARY = 1, REI_K_CONCAT = 2, REI_K_UNION = 3,
  REI_K_TRANSPOSE = 4, REI_K_OTHER = 5, REI_K_COUNT = 6
} rei_kernel_class;

/* rei_init: validate the specification, copy it to the device and run the staged
 * precompute ON THE DEVICE: IC enumeration in shortlex
 * order (epsilon = bit 0, LSB first per Alg. 2 line 5/13),
 * the guide table of proper splits, the P/N masks and the seed CSs.
 *   alphabet : NUL-terminated string of distinct 1-byte symbols, in Sigma order.
 *   P, N     : arrays of nP / nN NUL-terminated strings over the alphabet; "" = eps.
 *   costs    : the cost homomorphism (all >= 1).
 *   opts     : may be NULL (defaults: current device, own stream, exact, budget 80%).
 * On success *out receives a new context (free with rei_destroy). */
rei_status rei_init(void** out, const char* alphabet, const char* const* P, size_t nP,
                    const char* const* N, size_t nN, rei_costs costs, const rei_options* opts);

/* rei_solve: Algorithm 1 for c = c1 .. max_cost on the device:
 * per level, ? (x | 1), * (guide-table fixpoint), concatenation (Algorithm 2,
 * P:1009-1049) and union (bitwise OR) over all operand levels whose costs sum to
 * the level; every candidate is tested against the P/N masks and
 * inserted into the dedup set; new CSs are appended to the language
 * cache with a back-pointer.  Stops at the first level holding a
 * precise CS and reconstructs its regex.  Returns REI_OK, REI_NOT_FOUND,
 * REI_OUT_OF_MEMORY (out->last_complete_cost set) or an error. `out` may be NULL. */
rei_status rei_solve(void* ctx, uint32_t max_cost, rei_result* out);

/* Per-level statistics of the last rei_solve; *n_out = number available. */
rei_status rei_level_stats(const void* ctx, rei_level_stat* buf, size_t cap, size_t* n_out);

/* Accumulated launches and device milliseconds (CUDA events on the launching stream)
 * of one kernel class since the last rei_reset_kernel_stats.  Per-kernel events cost
 * host time on every launch, so a context records them only after its first
 * rei_reset_kernel_stats (or with REI_KERNEL_EVENTS=1); before that, `ms` stays 0 and
 * the per-level times come from one event pair per level.  Launch counts always. */
rei_status rei_kernel_stats(const void* ctx, rei_kernel_class k, uint64_t* launches, double* ms);
rei_status rei_reset_kernel_stats(void* ctx);
/* Total kernel launches issued by this context (all classes). */
uint64_t rei_launch_count(const void* ctx);
/* The dedup set rei_init chose for this specification:
 * 0 = bitmap over all 2^|IC| CSs (|IC| <= 32), 1 = 8-byte inline keys (|IC| <= 64),
 * 2 = 32-bit fingerprint + arena index per 8-byte slot, 3 = the whole CS inline in a
 * 16- or 32-byte slot (|IC| 65..127 and 129..254).  -1 for a NULL context. */
int rei_dedup_mode(const void* ctx);
/* Host<->device bytes copied by this context since creation (inputs, level plans,
 * control lines, results). */
rei_status rei_transfer_bytes(const void* ctx, uint64_t* h2d, uint64_t* d2h);

const char* rei_last_error(const void* ctx);
const char* rei_last_init_error(void);
/* rei_destroy frees the context.  Its device buffers return to a process-wide cache
 * (per device, size-keyed free lists of cudaMalloc blocks, kept mapped) and its pinned
 * host blocks to a free list, so the next rei_init / growth in the process reuses them
 * instead of paying cudaMalloc / cudaMallocHost again (sharded-cache contexts use plain
 * cudaMalloc: their buffers are exported through CUDA IPC).  Idle cached blocks count
 * as free memory in the default budget and are released when an allocation fails. */
void rei_destroy(void* ctx);
/* Return every cached (idle) device and pinned host block to the driver.  Safe at
 * any time; live contexts are unaffected. */
void rei_release_cached_memory(void);

/* ---- introspection (tests / parity; device data copied back to the host) ---- */

/* |IC| and word k of IC (shortlex index k) copied to buf (NUL-terminated). */
rei_status rei_ic(const void* ctx, uint32_t k, char* buf, size_t cap, uint32_t* n_ic);
/* Proper splits (u, v), both non-empty, u v = word w, as pairs of IC
 * indices written to pairs[2*i], pairs[2*i+1]; *count = number of splits. */
rei_status rei_splits(const void* ctx, uint32_t w, uint32_t* pairs, size_t cap, uint32_t* count);
/* P and N masks, cs_words 32-bit words each. */
rei_status rei_masks(const void* ctx, uint32_t* pos, uint32_t* neg);
/* The CSs of cost level `cost` of the last solve (cs_words words each, in cache order). */
rei_status rei_level_cs(const void* ctx, uint32_t cost, uint32_t* out, size_t cap, size_t* count);
/* Regex reconstructed from cache entry i of level `cost`. */
rei_status rei_entry_regex(const void* ctx, uint32_t cost, uint64_t i, char* buf, size_t cap);
/* Apply a CS operation on the device to `count` operand pairs (cs_words words each):
 * op 0 union, 1 concatenation, 2 star(a), 3 question(a), 4 precise(a) (out word 0 = 0/1). */
rei_status rei_cs_ops(void* ctx, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                      size_t count);

/* ---- multi-GPU: the sharded level (north_star "Multi-GPU partition") ----
 * Every rank holds the full language cache (replicated: speed, not capacity).  A
 * level with fewer than REI_REDUNDANT_CAND candidates (default 5e7; |IC| <= 64) runs
 * whole on every rank and is then sorted by CS into a rank-independent order.  A
 * larger level is split: each of its work lists (? and * operands, concatenation and
 * union work items, the paper's pair space P:977-978) is cut into contiguous rank
 * shares (rei_partition); a rank probes its full replica for every candidate of its
 * share and stages the CSs new to it.  The exchange then (1) buckets the staged CSs
 * by hash owner (rei_cs_owner), (2) sends each bucket to its owner (NCCL grouped
 * send/recv all-to-all), (3) the owner keeps one copy of each CS, (4) the owners'
 * unique lists are all-gathered in owner order into every rank's arena and inserted
 * into its dedup set; the precise-candidate rank is min-reduced with the level's
 * control lines.  Every rank ends each level with byte-identical caches, so later
 * candidate ranks name the same operands everywhere.  Any |IC| <= 512.
 * Transports: NCCL (one process per GPU, rei_options.nccl_unique_id), the caller's
 * host all-gather callback (rei_options.allgather with nccl_unique_id NULL: a
 * host-staged exchange, e.g. torch.distributed gloo), or device peer copies
 * (virtual ranks, rei_solve_group). */
/* One process per GPU: rank 0 creates the id, the caller broadcasts it (e.g. with
 * torch.distributed) and passes it in rei_options.nccl_unique_id with world_size and
 * rank; rei_init and rei_solve are then collective over the world. out: 128 bytes. */
rei_status rei_nccl_unique_id(void* out, size_t cap);

/* Virtual ranks in one process: `ctxs` are G contexts created with world_size <= 1
 * (any devices, the same specification); rei_solve_group runs them as ranks
 * 0..G-1 of one sharded search, exchanging through device (peer) copies.  Every
 * context ends with the same result and identical cache; `out` receives rank 0's. */
rei_status rei_solve_group(void* const* ctxs, int G, uint32_t max_cost, rei_result* out);

/* ---- multi-GPU capacity: the sharded cache ----
 * Contexts created with REI_FLAG_SHARDED_CACHE.  Rank r owns the CSs whose hash
 * (bits 40.. of the 64-bit CS hash) is r mod G; level c's list is the rank-order
 * concatenation of the owners' shards.  Every rank enumerates its rei_partition share
 * of the level's work items (operand blocks = shard pairs, read through peer
 * mappings), inserts each candidate into its owner's dedup set and appends new CSs
 * to the owner's shard (remote atomics over NVLink / IPC); there is no list
 * exchange.  Per level the ranks meet twice (after resetting their control lines and
 * after their kernels) through the allgather callback, or not at all for virtual
 * ranks (rei_solve_group), which share one host thread.  Results: the level sizes
 * and the level CS sets equal the single-GPU search's; the regex and candidate
 * counts follow the same readings (A9, A11).  rei_level_cs / rei_entry_regex read
 * across the shards.  Any |IC| <= 512. */

/* ---- many small specifications ----
 * Solves n independent contexts (each created by rei_init, any devices) with
 * `threads` host threads; each context runs on its own stream, so the latency-bound
 * small searches overlap on the GPU.  out[i] / status[i] receive context i's
 * result and status (the call returns REI_OK once every context was attempted). */
rei_status rei_solve_batch(void* const* ctxs, size_t n, uint32_t max_cost, int threads, rei_result* out,
                           rei_status* status);
/* Packed solve of n contexts on ONE device (the paper's suites of many
 * small runs): all specifications advance one non-empty cost level per
 * step, and each step runs every kernel class (?/*, union, concatenation of either
 * orientation, per CS width and split-count class) as one launch whose CTA groups
 * serve the specifications, with one control-line gather and one sync per step.
 * Same arithmetic and results as rei_solve.  Contexts with |IC| > 64,
 * words of more than 16 symbols, a level overflow or a multi-GPU / sharded setup
 * are solved alone after the packed steps.  out[i] / status[i] as rei_solve;
 * done_seconds[i] (may be NULL) = host seconds from the call to context i's result. */
rei_status rei_solve_packed(void* const* ctxs, size_t n, uint32_t max_cost, rei_result* out, rei_status* status,
                            double* done_seconds);

/* ---- multi-GPU host logic (pure functions, usable without a GPU) ---- */

/* Hash owner of a CS (cs_words 32-bit words, LSB-first as everywhere) among `world`
 * ranks: the rank that deduplicates it in the level exchange (and owns it in the
 * sharded cache).  The level kernels use the same function.  -1 for a bad width. */
int rei_cs_owner(const uint32_t* cs, uint32_t cs_words, int world);
/* Offsets of the level exchange's all-to-all for `rank`, given the world x world
 * matrix counts[src * world + dst] of records rank src sends to rank dst:
 * send_off[o] = first record of the bucket for o in rank's send list (buckets in
 * owner order); recv_off[r] = first record from source r in rank's receive list
 * (sources in rank order).  Either output may be NULL. */
void rei_exchange_offsets(int world, const uint64_t* counts, int rank, uint64_t* send_off, uint64_t* recv_off);
/* Contiguous share of a flattened candidate / work-item space of size `total` for
 * rank g of G: [*begin, *end) (S 8(e) "Partition"). */
void rei_partition(uint64_t total, int G, int g, uint64_t* begin, uint64_t* end);

#ifdef __cplusplus
}
#endif
#endif /* REI_B200_H */
