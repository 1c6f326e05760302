// levels.cu -- sm_100a level kernels of the REI search (Algorithm 1).
//
// Work decomposition:
//   A *group* = one uniform operand x (warp-uniform) x one slab of 32 consecutive
//   operands of the other level (one per lane).  A warp evaluates a group of 32
//   candidates at once:
//     concat (Alg. 2; IPS product P:637):
//       lane w computes the bit-slice  acc[w] (bit t = candidate t's bit w)  as
//         acc[w] = (x[eps] ? T[w] : 0) | (x[w] ? T[eps] : 0)
//                | OR over proper splits (u, v) of word w with x[u] : T[v]
//       (x uniform on the left; mirrored when the left side is the sliced one),
//       where T is the slab in transposed form (T[v] bit t = operand_t[v]) fetched
//       with warp shuffles; the two epsilon splits of gt(w) are factored out.
//       A 5-stage shuffle transpose turns the 32 slices into 32 candidate CSs, one
//       per lane.
//     union: lane t holds operand_t, candidate = x | operand_t.
//   Every candidate is then tested for precision and, unless it equals
//   an operand (guaranteed duplicate), probed in the dedup set;
//   G groups are batched per lane so each lane keeps G independent probes in
//   flight.  New CSs are appended with a warp-aggregated atomic.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include <unordered_map>

#include "rei_common.cuh"
#include "rei_host.h"

namespace cg = cooperative_groups;

namespace rei {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 8;  // warps per CTA of the pair kernels
// groups per lane batch (independent probes in flight); wide CSs trade MLP for registers
#ifndef REI_BATCH8
#define REI_BATCH8 1
#endif
template <int W> struct Batch { static constexpr int G = (W <= 2) ? 8 : (W == 4 ? 2 : (W == 8 ? REI_BATCH8 : 1)); };
constexpr unsigned long long kEmpty64 = ~0ull;
constexpr uint32_t kLocked = 0xffffffffu;
constexpr int kMaxProbe = 1 << 12;  // at load <= 1/2 a longer chain means the table is full

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// 32x32 bit-matrix transpose across the warp: in lane r, bit c = M[r][c];
// out lane c, bit r = M[r][c].  Five shuffle stages (block-swap recursion).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, uint32_t lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t m = (j == 16) ? 0x0000FFFFu : (j == 8) ? 0x00FF00FFu
                     : (j == 4) ? 0x0F0F0F0Fu : (j == 2) ? 0x33333333u : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
  }
  return x;
}

template <int W>
__device__ __forceinline__ uint32_t get_bit(const uint32_t (&x)[W], uint32_t i) {
  if (W == 1) return (x[0] >> (i & 31)) & 1u;
  uint32_t word = x[0];
#pragma unroll
  for (int q = 1; q < W; ++q) word = ((i >> 5) == (uint32_t)q) ? x[q] : word;
  return (word >> (i & 31)) & 1u;
}

template <int W>
__device__ __forceinline__ bool satisfies(const uint32_t (&cs)[W], const LevelParams& p) {
  if (p.exact) {
    uint32_t bad = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) bad |= ((cs[q] & p.pos[q]) ^ p.pos[q]) | (cs[q] & p.neg[q]);
    return bad == 0;
  }
  uint32_t errs = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) errs += __popc(p.pos[q] & ~cs[q]) + __popc(p.neg[q] & cs[q]);
  return errs <= p.max_errors;
}

template <int W>
__device__ __forceinline__ bool cs_equal(const uint32_t (&a)[W], const uint32_t (&b)[W]) {
  uint32_t d = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) d |= a[q] ^ b[q];
  return d == 0;
}


template <int W>
__device__ __forceinline__ void load_cs(const uint32_t* __restrict__ arena, uint64_t idx, uint32_t (&x)[W]) {
  const uint32_t* src = arena + idx * W;
  if (W == 1) {
    x[0] = src[0];
  } else if (W == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(src);
    x[0] = v.x; x[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < W; q += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + q);
      x[q] = v.x; x[q + 1] = v.y; x[q + 2] = v.z; x[q + 3] = v.w;
    }
  }
}

// the same through L2 only (ld.global.cg): data written earlier in the same launch by
// other SMs (the device level loop) must not come from a stale L1 line
template <int W>
__device__ __forceinline__ void load_cs_cg(const uint32_t* __restrict__ arena, uint64_t idx, uint32_t (&x)[W]) {
  const uint32_t* src = arena + idx * W;
  if (W == 1) {
    x[0] = __ldcg(src);
  } else if (W == 2) {
    const uint2 v = __ldcg(reinterpret_cast<const uint2*>(src));
    x[0] = v.x; x[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < W; q += 4) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src + q));
      x[q] = v.x; x[q + 1] = v.y; x[q + 2] = v.z; x[q + 3] = v.w;
    }
  }
}

template <int W>
__device__ __forceinline__ void store_cs(uint32_t* __restrict__ arena, uint64_t idx, const uint32_t (&x)[W]) {
  uint32_t* dst = arena + idx * W;
  if (W == 1) {
    dst[0] = x[0];
  } else if (W == 2) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(x[0], x[1]);
  } else {
#pragma unroll
    for (int q = 0; q < W; q += 4)
      *reinterpret_cast<uint4*>(dst + q) = make_uint4(x[q], x[q + 1], x[q + 2], x[q + 3]);
  }
}

// first arena index of the level being built (device-resident for lagged levels)
__device__ __forceinline__ unsigned long long out_base_of(const LevelParams& p) {
  return p.out_base_dev ? __ldg(p.out_base_dev) : p.out_base;
}

// Warp-aggregated append of a new CS + back-pointer to level c.
template <int W>
__device__ __forceinline__ void append(const LevelParams& p, const uint32_t (&cs)[W], unsigned long long rank) {
  // the lanes that reach this point together share one atomicAdd
  const unsigned mask = __activemask();
  const int leader = __ffs(mask) - 1;
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(&p.ctl->count, (unsigned long long)__popc(mask));
  base = __shfl_sync(mask, base, leader) + __popc(mask & ((1u << lane) - 1u));
  const unsigned long long idx = out_base_of(p) + base;
  if (idx >= p.cap) {
    p.ctl->overflow = 1;
    return;
  }
  store_cs<W>(p.arena_out, idx, cs);
  p.bp[idx] = rank;
}

// ---- dedup: indexed hash set for wide CSs (fingerprint + arena index).
// Slot = (fp << 32) | idx, 0 = empty, idx == kLocked while the owner writes the CS.
// Multi-rank levels (p.tent = kTent) append to a staging list instead of the arena:
// their slots carry idx = kTent | staging index ("tentative"), and the CS is compared
// from p.stage_cs.  After the level exchange, k_rehash (do_append = false) re-points
// each tentative slot whose key is in the exchanged level to its arena index.
// `S` is LevelParams (the local cache) or Peer (the owner's cache, sharded mode).
constexpr uint32_t kTent = 0x80000000u;
constexpr uint32_t kDead = 0xfffffffeu;
template <class S>
__device__ __forceinline__ const uint32_t* stage_of(const S& p) { return nullptr; }
template <>
__device__ __forceinline__ const uint32_t* stage_of<LevelParams>(const LevelParams& p) { return p.stage_cs; }
template <class S>
__device__ __forceinline__ const uint32_t* arena_of(const S& p) { return p.arena_out; }
template <>
__device__ __forceinline__ const uint32_t* arena_of<LevelParams>(const LevelParams& p) { return p.arena; }
template <class S>
__device__ __forceinline__ uint32_t tent_of(const S& p) { return 0u; }
template <>
__device__ __forceinline__ uint32_t tent_of<LevelParams>(const LevelParams& p) { return p.tent; }

template <int W, class S>
__device__ bool insert_indexed(const S& p, const uint32_t (&cs)[W], unsigned long long rank,
                               bool do_append, unsigned long long known_idx) {
  const unsigned long long h = hash_cs<W>(cs);
  const uint32_t fp = (uint32_t)(h >> 32) | 1u;
  const uint32_t tent = do_append ? tent_of(p) : 0u;
  unsigned long long s = h & p.dedup.mask;
  for (int probe = 0; probe < kMaxProbe; ++probe) {
    // the level already overflowed: it will be redone after growth -- stop inserting.
    // Checked every 16th probe only: the control line is one L2 round trip that would
    // otherwise sit on every probe step's critical path
    if (do_append && (probe & 15) == 15 && *(volatile unsigned int*)&p.ctl->overflow) return false;
    unsigned long long v = *(volatile unsigned long long*)&p.dedup.table[s];
    if (v == 0) {
      const unsigned long long lock = ((unsigned long long)fp << 32) | kLocked;
      const unsigned long long old = atomicCAS(&p.dedup.table[s], 0ull, lock);
      if (old == 0) {
        unsigned long long idx = known_idx;
        if (do_append) {
          idx = p.out_base + atomicAdd(&p.ctl->count, 1ull);
          if (idx >= p.cap || idx >= (tent ? 0x7ffffff0ull : 0xfffffff0ull)) {
            p.ctl->overflow = 1;
            atomicExch(&p.dedup.table[s], ((unsigned long long)fp << 32) | kDead);  // dead
            return false;
          }
          store_cs<W>(p.arena_out, idx, cs);
          p.bp[idx] = rank;
          __threadfence();
        }
        atomicExch(&p.dedup.table[s], ((unsigned long long)fp << 32) | ((uint32_t)idx | tent));
        return true;
      }
      v = old;
    }
    if ((uint32_t)(v >> 32) == fp) {
      uint32_t idx = (uint32_t)v;
      while (idx == kLocked) {
        __nanosleep(32);
        idx = (uint32_t)(*(volatile unsigned long long*)&p.dedup.table[s]);
      }
      if (idx != kDead) {
        const bool tentative = (idx & kTent) != 0;
        const uint32_t* base = tentative ? stage_of(p) : arena_of(p);
        uint32_t other[W];
        const volatile uint32_t* src = base + (unsigned long long)(idx & ~(tentative ? kTent : 0u)) * W;
#pragma unroll
        for (int q = 0; q < W; ++q) other[q] = src[q];
        if (cs_equal<W>(cs, other)) {
          // the exchanged level's arena entry takes over a tentative (staged) slot
          if (!do_append && tentative)
            atomicExch(&p.dedup.table[s], ((unsigned long long)fp << 32) | (uint32_t)known_idx);
          return false;
        }
      }
    }
    s = (s + 1) & p.dedup.mask;
  }
  p.ctl->overflow = 1;
  return false;
}

// Resolve the insert of a hash64 key whose first slot value is already loaded.
template <class S>
__device__ __forceinline__ bool insert_hash64(const S& p, unsigned long long key,
                                              unsigned long long s, unsigned long long v) {
  if (key == kEmpty64) return atomicExch(p.dedup.special, 1u) == 0u;
  for (int probe = 0; probe < kMaxProbe; ++probe) {
    if (v == key) return false;
    // the level already overflowed: it will be redone after growth -- stop inserting
    // (every 16th probe: see insert_indexed)
    if ((probe & 15) == 15 && *(volatile unsigned int*)&p.ctl->overflow) return false;
    if (v == kEmpty64) {
      const unsigned long long old = atomicCAS(&p.dedup.table[s], kEmpty64, key);
      if (old == kEmpty64) return true;
      if (old == key) return false;
    }
    s = (s + 1) & p.dedup.mask;
    v = p.dedup.table[s];
  }
  p.ctl->overflow = 1;
  return false;
}

// ---- dedup: inline wide keys (DEDUP_HASHIN, W32 = 4 or 8).  A slot is the CS itself
// as W/2 u64 words; empty = all ones.  W32 = 4 (|IC| <= 127): one 16-byte CAS claims
// the slot with the whole key.  W32 = 8 (|IC| <= 254): the slot's first 16 bytes hold
// the key's HIGH half (u64 words 2, 3), claimed by a 16-byte CAS with bit 62 of word 3
// set ("second half pending"; bits 254/255 of a CS are never set, so a claimed slot is
// never all ones); the owner then stores the low half and clears the pending bit.
// Readers that match the high half wait for the pending bit, then compare the low half.
constexpr unsigned long long kPend = 1ull << 62;
// (A/B on B200, profiles/r02_ab_w8_probe.txt: reading the low half with the head for a
// plain-load hit test cost more than the ordered read it saves -- c4-big concat 886 ->
// 967 ms -- and a second batch group per lane doubled the eight-word concat time)
#ifndef REI_LOW_HINT
#define REI_LOW_HINT 0
#endif

__device__ __forceinline__ void ld16(const unsigned long long* a, unsigned long long& x, unsigned long long& y) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(a);
  x = v.x;
  y = v.y;
}
__device__ __forceinline__ void ld16v(const unsigned long long* a, unsigned long long& x, unsigned long long& y) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(a) : "memory");
}
__device__ __forceinline__ void st16v(unsigned long long* a, unsigned long long x, unsigned long long y) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(a), "l"(x), "l"(y) : "memory");
}
// 16-byte compare-and-swap (sm_90+ atom.cas.b128); returns the old value
__device__ __forceinline__ void cas16(unsigned long long* a, unsigned long long c0, unsigned long long c1,
                                      unsigned long long v0, unsigned long long v1, unsigned long long& o0,
                                      unsigned long long& o1) {
  asm volatile(
      "{\n\t.reg .b128 c, v, o;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 v, {%4, %5};\n\t"
      "atom.global.cas.b128 o, [%6], c, v;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(o0), "=l"(o1)
      : "l"(c0), "l"(c1), "l"(v0), "l"(v1), "l"(a)
      : "memory");
}

// the inline key of a CS: the claimed half first (W32 = 8: high half)
template <int W>
__device__ __forceinline__ void inline_key(const uint32_t (&cs)[W], unsigned long long (&k)[W / 2]) {
  static_assert(W == 4 || W == 8, "inline keys are 16 or 32 bytes");
#pragma unroll
  for (int q = 0; q < W / 2; ++q) {
    const int src = (W == 8) ? ((q + 2) & 3) : q;  // W = 8: words 2, 3, 0, 1
    k[q] = ((unsigned long long)cs[2 * src + 1] << 32) | cs[2 * src];
  }
}

// Resolve the insert of an inline key whose slot `s` head (16 B) is already loaded.
// W32 = 8: (l0, l1) = the slot's low half read together with its head by a plain
// load (same 32-byte sector) when have_low; a low half only ever goes from empty to its
// final value within a launch, so an equal one proves a hit and anything else falls
// back to the ordered (volatile) read below.
template <int W, class S>
__device__ bool insert_inline(const S& p, const unsigned long long (&k)[W / 2], unsigned long long s,
                              unsigned long long v0, unsigned long long v1, unsigned long long l0 = 0,
                              unsigned long long l1 = 0, bool have_low = false) {
  constexpr int U = W / 2;  // u64 words per slot
  for (int probe = 0; probe < kMaxProbe; ++probe) {
    unsigned long long* slot = p.dedup.table + s * U;
    if ((probe & 15) == 15 && *(volatile unsigned int*)&p.ctl->overflow) return false;  // see insert_indexed
    if (v0 == ~0ull && v1 == ~0ull) {  // empty: claim it
      unsigned long long o0, o1;
      cas16(slot, ~0ull, ~0ull, k[0], (W == 8) ? (k[1] | kPend) : k[1], o0, o1);
      if (o0 == ~0ull && o1 == ~0ull) {
        if (W == 8) {
          st16v(slot + 2, k[U > 2 ? 2 : 0], k[U > 2 ? 3 : 1]);
          __threadfence();
          atomicAnd(slot + 1, ~kPend);
        }
        return true;
      }
      v0 = o0;
      v1 = o1;
      continue;  // re-examine the slot with the value that won
    }
    if (v0 == k[0] && (v1 & ~(W == 8 ? kPend : 0ull)) == k[1]) {
      if (W == 4) return false;
      // a low half equal to the key's is the key, whatever order the loads took (a slot
      // only ever goes from empty to its final value): the common hit needs no fence
      if (have_low && l0 == k[U > 2 ? 2 : 0] && l1 == k[U > 2 ? 3 : 1]) return false;
      unsigned long long w0, w1;
      ld16v(slot + 2, w0, w1);
      if (w0 == k[U > 2 ? 2 : 0] && w1 == k[U > 2 ? 3 : 1]) return false;
      // otherwise wait until the owner has published its low half, then read it in order
      while (v1 & kPend) {
        __nanosleep(20);
        v1 = *(volatile unsigned long long*)(slot + 1);
      }
      __threadfence();
      ld16v(slot + 2, w0, w1);
      if (w0 == k[U > 2 ? 2 : 0] && w1 == k[U > 2 ? 3 : 1]) return false;
    }
    s = (s + 1) & p.dedup.mask;
    ld16(p.dedup.table + s * U, v0, v1);
    if (W == 8 && REI_LOW_HINT) {
      ld16(p.dedup.table + s * U + 2, l0, l1);
      have_low = true;
    }
  }
  p.ctl->overflow = 1;
  return false;
}

// Bitmap position of a one-word CS (dedup over all 2^n languages, |IC| <= 32): the
// n-bit CS bit-reversed.  The bits of the long IC words (high CS bits) are the ones
// that vary most among the 32 candidates of a warp group (one uniform operand x 32
// consecutive cached operands), so reversed they select the bit within a 32-byte
// sector and the short-word bits select the sector: a group's probes touch fewer
// distinct sectors (Table 1 row 1, level-20 groups in the oracle's cache order: 17.3
// -> 12.7 sectors per 32 probes), and the concat kernel is bound by L1TEX tag lookups
// (A/B on B200: solve 46.6 -> 39.7 ms).  REI_BITMAP_IDENTITY restores plain order.
__device__ __forceinline__ uint32_t bm_pos(uint32_t cs, uint32_t n) {
#ifdef REI_BITMAP_IDENTITY
  (void)n;
  return cs;
#else
  return n ? __brev(cs) >> (32 - n) : 0u;
#endif
}

template <int W>
__device__ __forceinline__ unsigned long long key64(const uint32_t (&cs)[W]) {
  return W == 1 ? (unsigned long long)cs[0]
                : ((unsigned long long)cs[W > 1 ? 1 : 0] << 32) | (unsigned long long)cs[0];
}

// Batched candidate processing: precision test on every candidate (reading A11),
// guaranteed duplicates skipped, G probes issued before any is resolved.  The
// candidate's rank (its back-pointer) is computed only when it is needed.
// The dedup structure is a function of the CS width (rei_init): |IC| <= 32 -> bitmap,
// <= 64 -> 64-bit inline keys, wider -> fingerprint + arena index.
template <int W> struct DedupOf {
  static constexpr int mode = (W == 1) ? DEDUP_BITMAP : (W == 2 ? DEDUP_HASH64 : DEDUP_HASHIDX);
};

// Per-warp staging of new CSs in shared memory: lanes deposit new entries with a
// ballot prefix, and the warp reserves arena space with ONE atomicAdd per flush (the
// level counter is a single address; per-candidate appends serialised on it when
// 7-10 % of the candidates were new).
constexpr int kStage = 128;  // entries per warp
#ifdef REI_UNION_NOSTAGE
constexpr bool kUnionStaged = false;
#else
constexpr bool kUnionStaged = true;
#endif
template <int W>
struct WarpStage {
  uint32_t* cs;               // [kStage][W] (shared)
  unsigned long long* rank;   // [kStage] (shared)
  uint32_t n;                 // entries held (warp-uniform)
  unsigned long long* lc = nullptr;  // [kLocal] keys known to be in the dedup set (shared)
};

// Per-warp cache of 64-bit keys known to be in the HBM hash set (DEDUP_HASH64): the set
// only grows during a search, so a key found here is a duplicate for certain and its
// global probe (one random HBM sector) is skipped -- exact, like the operand-equality
// filter.  Direct-mapped by hash bits 20.. (the slot uses the low bits).  A warp's
// candidates share a uniform operand across slabs, and x.y repeats along a row
// (40-60 % within-row duplicates).  REI_LOCAL_CACHE = entries (0 = off).
#ifndef REI_LOCAL_CACHE
#define REI_LOCAL_CACHE 0
#endif
constexpr int kLocal = REI_LOCAL_CACHE;
template <int W>
__device__ __forceinline__ void stage_init_lc(WarpStage<W>& st, unsigned long long* base) {
  if (kLocal == 0 || W != 2) return;
  st.lc = base + (threadIdx.x >> 5) * kLocal;
  for (int i = threadIdx.x & 31; i < kLocal; i += 32) st.lc[i] = ~0ull;
  __syncwarp();
}
// shared bytes of the local caches of one CTA of `warps` warps
constexpr size_t local_cache_bytes(int W, int warps) { return (kLocal && W == 2) ? (size_t)warps * kLocal * 8 : 0; }

// Out of line: the flush is rare and must not bloat the probe loop's instruction stream.
template <int W>
__device__ __noinline__ void stage_flush_n(LevelCtl* ctl, uint32_t* arena_out, unsigned long long* bp,
                                           unsigned long long out_base, unsigned long long cap,
                                           const uint32_t* scs, const unsigned long long* srank, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->count, (unsigned long long)n);
  base = __shfl_sync(kFull, base, 0);
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) {
    const unsigned long long idx = out_base + base + i;
    if (idx >= cap) {
      ctl->overflow = 1;
      continue;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) arena_out[idx * W + q] = scs[i * W + q];
    bp[idx] = srank[i];
  }
  __syncwarp();
}

template <int W>
__device__ __forceinline__ void stage_flush(const LevelParams& p, WarpStage<W>& s) {
  if (s.n == 0) return;
  stage_flush_n<W>(p.ctl, p.arena_out, p.bp, out_base_of(p), p.cap, s.cs, s.rank, s.n);
  s.n = 0;
}

// Called by all 32 lanes together (converged).
template <int W>
__device__ __forceinline__ void stage_push(const LevelParams& p, WarpStage<W>& s, bool isnew,
                                           const uint32_t (&cs)[W], unsigned long long rank) {
  const unsigned mask = __ballot_sync(kFull, isnew);
  if (!mask) return;
  const uint32_t cnt = __popc(mask);
  if (s.n + cnt > (uint32_t)kStage) stage_flush<W>(p, s);
  if (isnew) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pos = s.n + __popc(mask & ((1u << lane) - 1u));
#pragma unroll
    for (int q = 0; q < W; ++q) s.cs[pos * W + q] = cs[q];
    s.rank[pos] = rank;
  }
  s.n += cnt;
  __syncwarp();
}

// Sharded-cache mode (f3): route one candidate to the rank that owns its CS (hash
// bits 40.. mod shards, independent of the slot bits) and insert it there through
// the peer mapping; a new entry is appended to the owner's shard of level c.
// Out of line and with by-value arguments only, so the local-cache kernels keep
// their hot loops (and their CS arrays in registers) unchanged.
template <int W>
struct CsVal {
  uint32_t w[W];
};

template <int W>
__device__ __noinline__ bool sharded_new(const Peer* __restrict__ peers, uint32_t shards, uint32_t n,
                                         CsVal<W> v, unsigned long long rank) {
  uint32_t cs[W];
#pragma unroll
  for (int q = 0; q < W; ++q) cs[q] = v.w[q];
  const unsigned long long h = hash_cs<W>(cs);
  const Peer& o = peers[(uint32_t)(h >> 40) % shards];
  constexpr int MODE = DedupOf<W>::mode;
  bool isnew;
  if constexpr (W == 4 || W == 8) {
    if (o.dedup.mode == DEDUP_HASHIN) {
      unsigned long long key[W / 2], v0, v1;
      inline_key<W>(cs, key);
      const unsigned long long slot = h & o.dedup.mask;
      ld16v(o.dedup.table + slot * (W / 2), v0, v1);
      isnew = insert_inline<W>(o, key, slot, v0, v1);
      goto appended;
    }
  }
  if (MODE == DEDUP_HASHIDX) return insert_indexed<W>(o, cs, rank, true, 0);
  if (MODE == DEDUP_BITMAP) {
    const uint32_t pos = bm_pos(cs[0], n);
    const uint32_t bit = 1u << (pos & 31);
    isnew = !(atomicOr(&o.dedup.bitmap[pos >> 5], bit) & bit);
  } else {
    const unsigned long long slot = h & o.dedup.mask;
    isnew = insert_hash64(o, key64<W>(cs), slot, *(volatile unsigned long long*)&o.dedup.table[slot]);
  }
appended:
  if (!isnew) return false;
  const unsigned long long idx = o.out_base + atomicAdd(&o.ctl->count, 1ull);
  if (idx >= o.cap) {
    o.ctl->overflow = 1;
    return false;
  }
  store_cs<W>(o.arena_out, idx, cs);
  o.bp[idx] = rank;
  return true;
}

// Precision is tested on the CSs that are new (Alg. 2 lines 16-17): a CS
// already cached at a lower level cannot be precise, or the search would have stopped
// there, and a within-level duplicate is tested by the candidate that inserted it.
template <int W, class RankF>
__device__ __forceinline__ void on_new(const LevelParams& p, const uint32_t (&cs)[W], RankF rank_of, int g) {
  const unsigned long long r = rank_of(g);
  if (satisfies<W>(cs, p)) atomicMin(&p.ctl->found_rank, r);
  append<W>(p, cs, r);
}

// stage != nullptr: called by the whole warp in converged code; new CSs go through the
// warp's shared-memory stage.  stage == nullptr: per-lane warp-aggregated append.
// REVCS (one-word CSs from the concat fast path): cs holds the CS bit-reversed in 32
// bits (its bitmap position is then cs >> (32 - n)); the rare paths reverse it back.
template <int W, int G, bool SH = false, bool REVCS = false, class RankF>
__device__ __forceinline__ void process_batch(const LevelParams& p, uint32_t (&cs)[G][W], const bool (&valid)[G],
                                              const bool (&skip)[G], RankF rank_of,
                                              WarpStage<W>* stage = nullptr) {
  static_assert(!REVCS || W == 1, "reversed CSs are one-word only");
  if (REVCS) {
    if (p.otf) {  // (rare mode) back to the plain layout, then the common code
#pragma unroll
      for (int g = 0; g < G; ++g) cs[g][0] = __brev(cs[g][0]);
      process_batch<W, G, SH, false>(p, cs, valid, skip, rank_of, stage);
      return;
    }
  }
  if (p.otf) {  // OnTheFly: the cache is full -- check only (a cached operand is never precise)
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (valid[g] && !skip[g] && satisfies<W>(cs[g], p)) atomicMin(&p.ctl->found_rank, rank_of(g));
    return;
  }
  // sharded cache (SH kernels only): every candidate goes to its owner (warp-uniform)
  if (SH && p.shards > 1) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (valid[g] && !skip[g]) {
        CsVal<W> v;
#pragma unroll
        for (int q = 0; q < W; ++q) v.w[q] = cs[g][q];
        const unsigned long long r = rank_of(g);
        if (sharded_new<W>(p.peers, p.shards, p.n, v, r) && satisfies<W>(cs[g], p)) atomicMin(&p.ctl->found_rank, r);
      }
    return;
  }
  constexpr int MODE = DedupOf<W>::mode;
  if (MODE == DEDUP_BITMAP || MODE == DEDUP_HASH64) {
    bool isnew[G];
    if (MODE == DEDUP_BITMAP) {
      uint32_t word[G], pos[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool need = valid[g] && !skip[g];
        pos[g] = REVCS ? cs[g][0] >> (32 - p.n) : bm_pos(cs[g][0], p.n);
#ifdef REI_PROBE_CG  // (A/B) probe through L2 only
        word[g] = need ? __ldcg(&p.dedup.bitmap[pos[g] >> 5]) : kFull;
#else
        word[g] = need ? p.dedup.bitmap[pos[g] >> 5] : kFull;
#endif
      }
      // deep levels: > 99.9 % of the probes hit; one warp vote skips the insert /
      // append code (and its per-candidate branches) for a batch with no miss at all
      bool anymiss = false;
#pragma unroll
      for (int g = 0; g < G; ++g) anymiss |= !(word[g] & (1u << (pos[g] & 31)));
      if (!__any_sync(__activemask(), anymiss)) return;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t bit = 1u << (pos[g] & 31);
        isnew[g] = false;
        if (!(word[g] & bit)) {
          const uint32_t old = atomicOr(&p.dedup.bitmap[pos[g] >> 5], bit);
          isnew[g] = !(old & bit);
          if (REVCS) cs[g][0] = __brev(cs[g][0]);  // plain layout for the test / append
          if (!stage && isnew[g]) on_new<W>(p, cs[g], rank_of, g);  // rare: direct append
        }
      }
      if (!stage) return;
    } else {
      unsigned long long slot[G], val[G], key[G], hh[G];
      bool need[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        need[g] = valid[g] && !skip[g];
        key[g] = key64<W>(cs[g]);
        hh[g] = hash_cs<W>(cs[g]);
        slot[g] = hh[g] & p.dedup.mask;
      }
#ifdef REI_WARP_MATCH
      // equal keys within a group of 32 candidates: only the lowest lane probes
      if (stage) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const unsigned m = __match_any_sync(kFull, key[g]) & __ballot_sync(kFull, need[g]);
          if (need[g] && (threadIdx.x & 31) != (uint32_t)(__ffs(m) - 1)) need[g] = false;
        }
      }
#endif
      uint32_t lci[G];
      if (kLocal && stage && stage->lc) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          lci[g] = (uint32_t)(hh[g] >> 20) & (uint32_t)(kLocal - 1);
          if (need[g] && key[g] != kEmpty64 && stage->lc[lci[g]] == key[g]) need[g] = false;
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) val[g] = need[g] ? p.dedup.table[slot[g]] : key[g];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        isnew[g] = false;
        if (val[g] != key[g] || key[g] == kEmpty64) isnew[g] = need[g] && insert_hash64(p, key[g], slot[g], val[g]);
        // the key is in the set now (found or inserted): remember it
        if (kLocal && stage && stage->lc && need[g] && key[g] != kEmpty64) stage->lc[lci[g]] = key[g];
      }
    }
    // precision on the new CSs, then append
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (stage) {
        unsigned long long r = 0;
        if (isnew[g]) {
          r = rank_of(g);
          if (satisfies<W>(cs[g], p)) atomicMin(&p.ctl->found_rank, r);
        }
        stage_push<W>(p, *stage, isnew[g], cs[g], r);
      } else if (isnew[g]) {
        on_new<W>(p, cs[g], rank_of, g);
      }
    }
  } else if (p.dedup.mode == DEDUP_HASHIN) {
    if constexpr (W == 4 || W == 8) {
      // inline wide keys: the G slot heads are loaded before any is resolved
      unsigned long long key[G][W / 2], slot[G], v0[G], v1[G], l0[G], l1[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        inline_key<W>(cs[g], key[g]);
        slot[g] = hash_cs<W>(cs[g]) & p.dedup.mask;
        v0[g] = key[g][0];
        v1[g] = key[g][1];
        l0[g] = l1[g] = 0;
        if (valid[g] && !skip[g]) {
          ld16(p.dedup.table + slot[g] * (W / 2), v0[g], v1[g]);
          if (W == 8 && REI_LOW_HINT) ld16(p.dedup.table + slot[g] * (W / 2) + 2, l0[g], l1[g]);  // same sector
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (!valid[g] || skip[g]) continue;
        // W32 = 4: a head equal to the key is a hit without leaving the register file
        if (W == 4 && v0[g] == key[g][0] && v1[g] == key[g][1]) continue;
        if (insert_inline<W>(p, key[g], slot[g], v0[g], v1[g], l0[g], l1[g], W == 8 && REI_LOW_HINT))
          on_new<W>(p, cs[g], rank_of, g);
      }
    }
  } else {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (valid[g] && !skip[g]) {
        const unsigned long long r = rank_of(g);
        if (insert_indexed<W>(p, cs[g], r, true, 0) && satisfies<W>(cs[g], p))
          atomicMin(&p.ctl->found_rank, r);
      }
    }
  }
}

// Rotation-based 32x32 transpose step constants for this lane: stage j rotates the
// partner word left by (lane & j ? 32 - j : j) and keeps the lane's own bits under km.
struct TransposeLane {
  uint32_t rot[5], km[5];
  __device__ __forceinline__ explicit TransposeLane(uint32_t lane) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const uint32_t j = 16u >> s;
      const uint32_t m = (j == 16) ? 0x0000FFFFu : (j == 8) ? 0x00FF00FFu
                       : (j == 4) ? 0x0F0F0F0Fu : (j == 2) ? 0x33333333u : 0x55555555u;
      const bool hi = (lane & j) != 0;
      rot[s] = hi ? 32u - j : j;
      km[s] = hi ? ~m : m;
    }
    // byte-permute selectors of the 16- and 8-bit stages ({partner:own}, own = bytes 0-3)
    rot[0] = (lane & 16) ? 0x3276u : 0x5410u;
    rot[1] = (lane & 8) ? 0x3715u : 0x6240u;
    // paired byte stages: {send, receive into b} selectors (receive into a = rot[])
    psel[0] = (lane & 16) ? 0x5410u : 0x3276u;
    psel[1] = (lane & 16) ? 0x3254u : 0x7610u;
    psel[2] = (lane & 8) ? 0x6240u : 0x3715u;
    psel[3] = (lane & 8) ? 0x3614u : 0x7250u;
  }
  uint32_t psel[4];
  // Same matrix transpose as transpose32(): the 16- and 8-bit stages move whole bytes
  // (one PRMT each, per-lane selector), the 4/2/1-bit stages rotate + merge (SHF, LOP3).
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    uint32_t y = __shfl_xor_sync(kFull, x, 16);
    x = __byte_perm(x, y, rot[0]);
    y = __shfl_xor_sync(kFull, x, 8);
    x = __byte_perm(x, y, rot[1]);
#pragma unroll
    for (int s = 2; s < 5; ++s) {
      const uint32_t j = 16u >> s;
      y = __shfl_xor_sync(kFull, x, j);
      const uint32_t yr = __funnelshift_l(y, y, rot[s]);  // rotate left
      x = (x & km[s]) | (yr & ~km[s]);
    }
    return x;
  }
  // Two transposes at once (a, b): every butterfly stage moves half of each word to
  // the partner lane, so the two outgoing halves share ONE shuffle (packed), trading
  // one SHFL (an L1TEX wavefront) for one ALU op per stage.
  __device__ __forceinline__ void pair(uint32_t& a, uint32_t& b) const {
    // 16- and 8-bit stages: byte permutes
    uint32_t y = __shfl_xor_sync(kFull, __byte_perm(a, b, psel[0]), 16);
    b = __byte_perm(b, y, psel[1]);
    a = __byte_perm(a, y, rot[0]);
    y = __shfl_xor_sync(kFull, __byte_perm(a, b, psel[2]), 8);
    b = __byte_perm(b, y, psel[3]);
    a = __byte_perm(a, y, rot[1]);
    // 4-, 2-, 1-bit stages: the lane keeps km, sends a's other bits in place and b's
    // rotated into the km positions
#pragma unroll
    for (int s = 2; s < 5; ++s) {
      const uint32_t pk = (a & ~km[s]) | (__funnelshift_r(b, b, rot[s]) & km[s]);
      y = __shfl_xor_sync(kFull, pk, 16u >> s);
      b = (b & km[s]) | (y & ~km[s]);
      a = (a & km[s]) | (__funnelshift_l(y, y, rot[s]) & ~km[s]);
    }
  }
};

// Skewed 32x32 bit-matrix transpose with warp-uniform masks (no per-lane constants
// but the shuffle sources).  Element (row w, column t) of the matrix (lane w holds row
// w) is first placed at bit k = (w - t) mod 32 of lane w by the pre-skew
// z_w = rotr(brev(row_w), 31 - w); stage i then moves every bit whose position has bit
// i set down by 2^i lanes (one SHFL + one LOP3 with an immediate mask), so the element
// ends in lane w - k = t at position k = w - t, and a rotate-left by t puts row w's bit
// at position w.  The pre-skew is a bit permutation, so it commutes with the AND/OR of
// the fold against all-ones / zero masks: it is applied to the slab terms once per
// slab, not per candidate.  Per transpose: 5 SHFL + 5 LOP3 + 1 SHF.
struct SkewTranspose {
  uint32_t src[5];  // lane + 16, 8, 4, 2, 1 (mod 32: SHFL wraps)
  uint32_t lane;
  __device__ __forceinline__ explicit SkewTranspose(uint32_t l) : lane(l) {
#pragma unroll
    for (int i = 0; i < 5; ++i) src[i] = (l + (16u >> i)) & 31u;
  }
  __device__ __forceinline__ uint32_t pre(uint32_t v) const {
    const uint32_t r = __brev(v);
    return __funnelshift_r(r, r, 31u - lane);
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t z) const {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const uint32_t j = 16u >> i;
      const uint32_t M = (j == 16) ? 0xFFFF0000u : (j == 8) ? 0xFF00FF00u
                       : (j == 4) ? 0xF0F0F0F0u : (j == 2) ? 0xCCCCCCCCu : 0xAAAAAAAAu;
      const uint32_t y = __shfl_sync(kFull, z, src[i]);
      // z = (z & ~M) | (y & M) as ONE lop3 (truth table 0xB8 for a=z, b=M, c=y; the
      // compiler otherwise splits it in two)
      asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(z) : "r"(z), "r"(M), "r"(y));
    }
    return __funnelshift_l(z, z, lane);
  }
  // Two transposes (a, b): the byte-granular stages (16, 8) carry both words' moving
  // bytes in ONE shuffle (byte permutes with warp-uniform selectors), trading one SHFL
  // for one ALU op each; the bit stages stay single.
  __device__ __forceinline__ void pair(uint32_t& a, uint32_t& b) const {
    uint32_t y = __shfl_sync(kFull, __byte_perm(a, b, 0x3276u), src[0]);
    a = __byte_perm(a, y, 0x7610u);
    b = __byte_perm(b, y, 0x5410u);
    y = __shfl_sync(kFull, __byte_perm(a, b, 0x3715u), src[1]);
    a = __byte_perm(a, y, 0x7250u);
    b = __byte_perm(b, y, 0x6240u);
#pragma unroll
    for (int i = 2; i < 5; ++i) {
      const uint32_t j = 16u >> i;
      const uint32_t M = (j == 4) ? 0xF0F0F0F0u : (j == 2) ? 0xCCCCCCCCu : 0xAAAAAAAAu;
      const uint32_t ya = __shfl_sync(kFull, a, src[i]);
      const uint32_t yb = __shfl_sync(kFull, b, src[i]);
      asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(a) : "r"(a), "r"(M), "r"(ya));
      asm("lop3.b32 %0, %1, %2, %3, 0xB8;" : "=r"(b) : "r"(b), "r"(M), "r"(yb));
    }
    a = __funnelshift_l(a, a, lane);
    b = __funnelshift_l(b, b, lane);
  }
};

// ---- work-item decode (blocks staged in shared memory)
__device__ __forceinline__ int find_block(const Block* blocks, int nb, unsigned long long item) {
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (blocks[mid].item_off <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Packed launches: this CTA's specification (binary search of its group), its
// parameters copied to shared memory, and its block index / count within the group.
__device__ __forceinline__ const LevelParams& packed_params(const Packed& pk, uint32_t& bid, uint32_t& nbid) {
  __shared__ LevelParams s_p;
  __shared__ uint32_t s_i;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = pk.nspec - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (pk.cta_start[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
    }
    s_i = lo;
  }
  __syncthreads();
  const uint32_t i = s_i;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(pk.params + i);
  uint32_t* dst = reinterpret_cast<uint32_t*>(&s_p);
  for (uint32_t k = threadIdx.x; k < sizeof(LevelParams) / 4; k += blockDim.x) dst[k] = src[k];
  bid = blockIdx.x - pk.cta_start[i];
  nbid = pk.cta_start[i + 1] - pk.cta_start[i];
  __syncthreads();
  return s_p;
}

__device__ __forceinline__ bool found_and_stop(const LevelParams& p) {
  return p.early_exit && *(volatile unsigned long long*)&p.ctl->found_rank != ~0ull;
}
// Early exit inside a work item, once per slab pass (REI_SLAB_EXIT: 0 off, 1 a blocking
// check at each pass, 2 the check of the value loaded one pass earlier).  A/B on B200
// (profiles/r02_ab_slab_exit.txt, solve ms off / blocking / deferred): Table 1 row 1
// 27.16 / 27.52 / 28.07, row 8 47.75 / 48.57 / 49.54, C2 145.0 / 148.2 / 151.2 -- the
// extra reads of the control line (the level's append counter lives in it) cost more
// than the shorter drain saves, so the check stays per work item
#ifndef REI_SLAB_EXIT
#define REI_SLAB_EXIT 0
#endif
#if REI_SLAB_EXIT == 0
#define SLAB_EXIT(p, notfirst) false
#elif REI_SLAB_EXIT == 1
#define SLAB_EXIT(p, notfirst) ((notfirst) && found_and_stop(p))
#else
struct SlabExit {
  unsigned long long seen = ~0ull;
  __device__ __forceinline__ bool operator()(const LevelParams& p, bool notfirst) {
    const bool stop = notfirst && p.early_exit && seen != ~0ull;
    seen = *(volatile unsigned long long*)&p.ctl->found_rank;
    return stop;
  }
};
#define SLAB_EXIT(p, notfirst) slab_exit(p, notfirst)
#endif
#if REI_SLAB_EXIT == 2
#define SLAB_EXIT_DECL SlabExit slab_exit;
#else
#define SLAB_EXIT_DECL
#endif

// ============================================================================
// Concatenation kernel.  Dynamic shared memory: split table [maxk][NW], nsplit[NW],
// blocks[nblocks], and (W > 2) one transposed slab per warp.
template <int W, bool SH = false>
__global__ void __launch_bounds__(kWarps * 32) k_concat(LevelParams p) {
  constexpr int NW = 32 * W;
  constexpr bool kShfl = (W <= 2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Block* s_blocks = reinterpret_cast<Block*>(smem_raw);
  uint32_t* s_split = reinterpret_cast<uint32_t*>(s_blocks + p.nblocks);
  uint32_t* s_nsplit = s_split + p.maxk * NW;
  uint32_t* s_T = s_nsplit + NW;  // [kWarps][NW] (W > 2 only)

  for (int i = threadIdx.x; i < (int)(p.nblocks * sizeof(Block) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_blocks)[i] = reinterpret_cast<const uint32_t*>(p.blocks)[i];
  if (p.rank_off_dev) {  // split level: the ? / * candidates (ranked first) counted on the device
    __syncthreads();
    const unsigned long long off = __ldg(p.rank_off_dev);
    for (int i = threadIdx.x; i < (int)p.nblocks; i += blockDim.x) s_blocks[i].cand_off += off;
  }
  for (int i = threadIdx.x; i < (int)(p.maxk * NW); i += blockDim.x)
    s_split[i] = p.split[(i / NW) * kMaxNW + (i % NW)];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s_nsplit[i] = p.nsplit[i];
  __syncthreads();

  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  const unsigned long long gwarp = (unsigned long long)blockIdx.x * kWarps + warp;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * kWarps;
  uint32_t* myT = s_T + warp * (NW + W);
  uint32_t* myX = myT + NW;  // the uniform operand (W > 2)
  constexpr int G = Batch<W>::G;

  uint32_t nspl[W], kq[W];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    nspl[q] = s_nsplit[q * 32 + lane];
    // row q = words 32q .. 32q + 31 (nearly equal lengths in shortlex order): the fold
    // runs to the row's longest split list, and rows past |IC| are all zero
    kq[q] = __reduce_max_sync(kFull, nspl[q]);
  }
  const uint32_t rows = (p.n + 31) / 32;  // live CS rows (warp-uniform)

  unsigned long long warp_eval = 0;
  for (unsigned long long item = p.item_begin + gwarp; item < p.total_items; item += nwarps) {
    if (found_and_stop(p)) break;
    const Block& blk = s_blocks[find_block(s_blocks, p.nblocks, item)];
    const unsigned long long local = item - blk.item_off;
    const unsigned long long ut = local / blk.s_tiles, st = local % blk.s_tiles;
    const bool slice_a = blk.slice_a != 0;
    const unsigned long long nu = slice_a ? blk.nb : blk.na;
    const unsigned long long ns = slice_a ? blk.na : blk.nb;
    const unsigned long long u_base = slice_a ? blk.b_base : blk.a_base;
    const unsigned long long slab_base = slice_a ? blk.a_slab : blk.b_slab;
    const unsigned long long u0 = ut * blk.tu, u1 = min(u0 + blk.tu, nu);
    const unsigned long long nslabs = (ns + 31) / 32;
    const unsigned long long s0 = st * blk.ts, s1 = min(s0 + blk.ts, nslabs);
    uint32_t evaluated = 0;

    SLAB_EXIT_DECL
    for (unsigned long long s = s0; s < s1; ++s) {
      if (SLAB_EXIT(p, s != s0)) break;  // early exit per slab pass, not only per work item
      // the slab in transposed form
      uint32_t T[W];
#pragma unroll
      for (int q = 0; q < W; ++q) T[q] = p.tarena[(slab_base + s) * NW + q * 32 + lane];
      if (!kShfl) {
#pragma unroll
        for (int q = 0; q < W; ++q) myT[q * 32 + lane] = T[q];
        __syncwarp();
      }
      const uint32_t Teps = __shfl_sync(kFull, T[0], 0);
      const unsigned long long sj = s * 32 + lane;  // this lane's sliced operand
      const bool lane_ok = sj < ns;

      for (unsigned long long u = u0; u < u1; u += G) {
        uint32_t cs[G][W];
        bool valid[G], skip[G];
        unsigned long long rank[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const unsigned long long ui = u + g;
          const bool active = ui < u1;
          uint32_t x[W];
          if (active) load_cs<W>(p.arena, u_base + ui, x);
          else {
#pragma unroll
            for (int q = 0; q < W; ++q) x[q] = 0;
          }
          const uint32_t xeps = x[0] & 1u;
          if (!kShfl) {
            __syncwarp();
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < W; ++q) myX[q] = x[q];
            }
            __syncwarp();
          }
          uint32_t acc[W];
#pragma unroll
          for (int q = 0; q < W; ++q) acc[q] = (xeps ? T[q] : 0u) | (((x[q] >> lane) & 1u) ? Teps : 0u);
#pragma unroll
          for (int q = 0; q < W; ++q) {
            if (kShfl || (uint32_t)q >= rows) continue;  // (W <= 2: the loop below)
            for (uint32_t k = 0; k < kq[q]; ++k) {
              const uint32_t sp = s_split[k * NW + q * 32 + lane];
              const uint32_t ufix = slice_a ? (sp & 0xffffu) : (sp >> 16);
              const uint32_t vsl = slice_a ? (sp >> 16) : (sp & 0xffffu);
              const uint32_t t = myT[vsl & (NW - 1)];
              const uint32_t xb = (myX[(ufix >> 5) & (W - 1)] >> (ufix & 31)) & 1u;
              if (k < nspl[q] && xb) acc[q] |= t;
            }
          }
          for (uint32_t k = 0; kShfl && k < p.maxk; ++k) {
#pragma unroll
            for (int q = 0; q < W; ++q) {
              const uint32_t sp = s_split[k * NW + q * 32 + lane];
              // x uniform on the left: test x[u], fetch T[v]; mirrored for slice_a.
              const uint32_t ufix = slice_a ? (sp & 0xffffu) : (sp >> 16);
              const uint32_t vsl = slice_a ? (sp >> 16) : (sp & 0xffffu);
              uint32_t t;
              if (kShfl) {
                const uint32_t t0 = __shfl_sync(kFull, T[0], vsl & 31);
                if (W == 2) {
                  const uint32_t t1 = __shfl_sync(kFull, T[W > 1 ? 1 : 0], vsl & 31);
                  t = (vsl >> 5) ? t1 : t0;
                } else {
                  t = t0;
                }
              } else {
                t = myT[vsl & (NW - 1)];
              }
              const uint32_t xb = kShfl ? get_bit<W>(x, ufix) : ((myX[(ufix >> 5) & (W - 1)] >> (ufix & 31)) & 1u);
              if (k < nspl[q] && xb) acc[q] |= t;
            }
          }
#pragma unroll
          for (int q = 0; q < W; ++q) cs[g][q] = (kShfl || (uint32_t)q < rows) ? transpose32(acc[q], lane) : 0u;
          valid[g] = active && lane_ok;
          skip[g] = cs_equal<W>(cs[g], x);  // equals a cached operand: old
          evaluated += valid[g] ? 1u : 0u;
        }
        const unsigned long long cand_off = blk.cand_off, nb = blk.nb;
        process_batch<W, G, SH>(p, cs, valid, skip, [&](int g) {
          const unsigned long long ui = u + g;
          return cand_off + (slice_a ? sj * nb + ui : ui * nb + sj);
        });
      }
      if (!kShfl) __syncwarp();
    }
    warp_eval += __reduce_add_sync(kFull, evaluated);  // one atomic per warp per launch (below)
  }
  if (lane_id() == 0 && warp_eval) {  // the control line's counters: once per warp, not per item
    atomicAdd(&p.ctl->evaluated, warp_eval);
    atomicAdd(&p.ctl->eval_c, warp_eval);
  }
}

// ============================================================================
// Wide concatenation (W32 = 4, 8; <= MAXK proper splits per word): the same Alg. 2
// arithmetic as k_concat, reorganised so that a candidate costs a few instructions
// per split instead of three dependent shared loads and a dozen ALU operations:
//   * per lane and split (q, k) of its word 32q + lane, the byte offset of the
//     uniform-side word u (prefix, or suffix when A is the sliced side) is fixed for
//     the kernel; W32 = 4 keeps them in registers, W32 = 8 in a shared table;
//   * per uniform operand x the warp writes x's bits as all-ones / zero masks to
//     shared memory once (M[u] = -x[u], plus a zero word that invalid splits read);
//   * per slab the sliced-side terms t_qk = T[v] are fetched once (W32 = 4: into
//     registers, reused by every uniform operand of the work item);
//   * the fold is then acc_q |= t_qk & M[u_qk]: one shared load + one LOP3 per split;
//   * G uniform operands per batch, so each lane keeps G probes in flight.
// Variant knobs (A/B on B200, profiles/r02_ab_wide_concat.txt, REI_CONCURRENT=0 solves):
// c3-big (W32 = 4) concat 860 ms (generic k_concat) -> 776 (hoisted constants, G = 2,
// 2 CTAs/SM) -> 750 (constants in shared memory, 4 CTAs/SM: the kernel waits on its
// probes -- long-scoreboard stalls 12 of 18.5 cycles per issue -- so occupancy beats
// fewer instructions); G = 4 slower (1005-1049).  W32 = 8: one operand per batch (two
// doubled the time: fewer resident warps) at 4 CTAs/SM.
#ifndef REI_WIDE_HOIST
#define REI_WIDE_HOIST 0
#endif
#ifndef REI_WIDE_G
#define REI_WIDE_G 2
#endif
#ifndef REI_WIDE_MINB
#define REI_WIDE_MINB 4
#endif
#ifndef REI_WIDE_G8
#define REI_WIDE_G8 1
#endif
// eight-word CSs (A/B, profiles/r02_ab_w8_wide.txt, c4-big concat): generic k_concat 887
// ms; this kernel with one operand per batch at 3 CTAs/SM 827, at 4 CTAs/SM 750 ms
#ifndef REI_WIDE_MINB8
#define REI_WIDE_MINB8 4
#endif
template <int W, int MAXK, bool SLICE_A>
__global__ void __launch_bounds__(kWarps * 32, W == 4 ? REI_WIDE_MINB : REI_WIDE_MINB8) k_concat_wide(LevelParams p) {
  static_assert(W == 4 || W == 8, "wide path: four- and eight-word CSs");
  constexpr int NW = 32 * W;
  // (MAXK 15: 120 registers of constants spill)
  constexpr bool HOIST = REI_WIDE_HOIST && (W == 4 && MAXK <= 9);
  constexpr int G = W == 4 ? REI_WIDE_G : REI_WIDE_G8;  // uniform operands (probes per lane) per batch
  constexpr int MW = NW + 1;         // mask words per operand (+ the zero word)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Block* s_blocks = reinterpret_cast<Block*>(smem_raw);
  uint32_t* s_cu = reinterpret_cast<uint32_t*>(s_blocks + p.nblocks);  // [MAXK][NW] uniform-side byte offsets
  uint32_t* s_cv = s_cu + MAXK * NW;                                    // [MAXK][NW] sliced-side word index
  uint32_t* s_warp = s_cv + MAXK * NW;                                  // [kWarps][NW + G * MW]
  for (int i = threadIdx.x; i < (int)(p.nblocks * sizeof(Block) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_blocks)[i] = reinterpret_cast<const uint32_t*>(p.blocks)[i];
  if (p.rank_off_dev) {  // split level: the ? / * candidates (ranked first) counted on the device
    __syncthreads();
    const unsigned long long off = __ldg(p.rank_off_dev);
    for (int i = threadIdx.x; i < (int)p.nblocks; i += blockDim.x) s_blocks[i].cand_off += off;
  }
  for (int i = threadIdx.x; i < MAXK * NW; i += blockDim.x) {
    const uint32_t k = i / NW, w = i % NW;
    const bool ok = w < p.n && k < p.nsplit[w];
    const uint32_t sp = ok ? p.split[(size_t)k * kMaxNW + w] : 0u;
    const uint32_t u = SLICE_A ? (sp & 0xffffu) : (sp >> 16);  // uniform side
    const uint32_t v = SLICE_A ? (sp >> 16) : (sp & 0xffffu);  // sliced side
    s_cu[i] = (ok ? u : (uint32_t)NW) * 4u;  // an invalid split reads the zero mask word
    s_cv[i] = ok ? v : 0u;
  }
  __syncthreads();

  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* myT = s_warp + warp * (NW + G * MW);
  uint32_t* myM = myT + NW;
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) myM[g * MW + NW] = 0u;
  }
  const uint32_t rows = (p.n + 31) / 32;  // live CS rows (warp-uniform)
  uint32_t kq[W];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const uint32_t w = q * 32 + lane;
    kq[q] = __reduce_max_sync(kFull, w < p.n ? p.nsplit[w] : 0u);
  }
  uint32_t cu[HOIST ? W : 1][HOIST ? MAXK : 1];
  if constexpr (HOIST) {
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int k = 0; k < MAXK; ++k) cu[q][k] = s_cu[k * NW + q * 32 + lane];
  }
  const unsigned char* mbytes = reinterpret_cast<const unsigned char*>(myM);
  auto ldm = [&](uint32_t off) {  // one mask word at byte offset `off` of the warp's masks
    return *reinterpret_cast<const uint32_t*>(mbytes + off);
  };

  const unsigned long long gwarp = (unsigned long long)blockIdx.x * kWarps + warp;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * kWarps;
  unsigned long long warp_eval = 0;
  for (unsigned long long item = p.item_begin + gwarp; item < p.total_items; item += nwarps) {
    if (found_and_stop(p)) break;
    const Block& blk = s_blocks[find_block(s_blocks, p.nblocks, item)];
    const unsigned long long local = item - blk.item_off;
    const unsigned long long ut = local / blk.s_tiles, st = local % blk.s_tiles;
    const unsigned long long nu = SLICE_A ? blk.nb : blk.na;
    const unsigned long long ns = SLICE_A ? blk.na : blk.nb;
    const unsigned long long u_base = SLICE_A ? blk.b_base : blk.a_base;
    const unsigned long long slab_base = SLICE_A ? blk.a_slab : blk.b_slab;
    const unsigned long long u0 = ut * blk.tu, u1 = min(u0 + blk.tu, nu);
    const unsigned long long nslabs = (ns + 31) / 32;
    const unsigned long long s0 = st * blk.ts, s1 = min(s0 + blk.ts, nslabs);
    const unsigned long long cand_off = blk.cand_off, nb = blk.nb;
    uint32_t evaluated = 0;

    SLAB_EXIT_DECL
    for (unsigned long long s = s0; s < s1; ++s) {
      if (SLAB_EXIT(p, s != s0)) break;  // early exit per slab pass, not only per work item
      uint32_t T[W];
#pragma unroll
      for (int q = 0; q < W; ++q) T[q] = (uint32_t)q < rows ? p.tarena[(slab_base + s) * NW + q * 32 + lane] : 0u;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < W; ++q) myT[q * 32 + lane] = T[q];
      __syncwarp();
      const uint32_t Teps = __shfl_sync(kFull, T[0], 0);
      uint32_t t[HOIST ? W : 1][HOIST ? MAXK : 1];
      if constexpr (HOIST) {
#pragma unroll
        for (int q = 0; q < W; ++q)
#pragma unroll
          for (int k = 0; k < MAXK; ++k)
            t[q][k] = ((uint32_t)q < rows && (uint32_t)k < kq[q]) ? myT[s_cv[k * NW + q * 32 + lane]] : 0u;
      }
      const unsigned long long sj = s * 32 + lane;  // this lane's sliced operand
      const bool lane_ok = sj < ns;

      for (unsigned long long u = u0; u < u1; u += G) {
        uint32_t cs[G][W], x[G][W];
        bool valid[G], skip[G];
        // the G operands' bits as masks in shared memory
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool active = u + g < u1;
          if (active) load_cs<W>(p.arena, u_base + u + g, x[g]);
          else {
#pragma unroll
            for (int q = 0; q < W; ++q) x[g][q] = 0u;
          }
#pragma unroll
          for (int q = 0; q < W; ++q)
            if ((uint32_t)q < rows) myM[g * MW + q * 32 + lane] = 0u - ((x[g][q] >> lane) & 1u);
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t xe = 0u - (x[g][0] & 1u);
          uint32_t acc[W];
#pragma unroll
          for (int q = 0; q < W; ++q) {
            if ((uint32_t)q >= rows) { acc[q] = 0u; continue; }
            const uint32_t xw = 0u - ((x[g][q] >> lane) & 1u);
            uint32_t a = (xe & T[q]) | (xw & Teps);
#pragma unroll
            for (int k = 0; k < MAXK; ++k) {
              if ((uint32_t)k >= kq[q]) break;  // warp-uniform
              if constexpr (HOIST) {
                a |= t[q][k] & ldm(cu[q][k] + g * MW * 4);
              } else {
                const uint32_t c_u = s_cu[k * NW + q * 32 + lane];
                const uint32_t tv = myT[s_cv[k * NW + q * 32 + lane]];
                a |= tv & ldm(c_u + g * MW * 4);
              }
            }
            acc[q] = a;
          }
#pragma unroll
          for (int q = 0; q < W; ++q) cs[g][q] = (uint32_t)q < rows ? transpose32(acc[q], lane) : 0u;
          valid[g] = (u + g < u1) && lane_ok;
          skip[g] = cs_equal<W>(cs[g], x[g]);  // equals a cached operand: old
          evaluated += valid[g] ? 1u : 0u;
        }
        process_batch<W, G>(p, cs, valid, skip, [&](int g) {
          const unsigned long long ui = u + g;
          return cand_off + (SLICE_A ? sj * nb + ui : ui * nb + sj);
        });
      }
    }
    warp_eval += __reduce_add_sync(kFull, evaluated);  // one atomic per warp per launch (below)
  }
  if (lane_id() == 0 && warp_eval) {  // the control line's counters: once per warp, not per item
    atomicAdd(&p.ctl->evaluated, warp_eval);
    atomicAdd(&p.ctl->eval_c, warp_eval);
  }
}

// ============================================================================
// Concatenation fast path for W32 <= 2 (|IC| <= 64) and words with <= MAXK proper
// splits.  Same arithmetic as k_concat, reorganised for instruction-level
// parallelism:
//   * per lane, the split table of its word(s) lives in registers as
//     (uniform-side bit mask, sliced-side source word) pairs, fixed per orientation
//     (SLICE_A: the left operand is the sliced one);
//   * per slab, the shuffled slab words t_k = T[src_k] are fetched once and reused
//     by every uniform operand of the work item (up to 64 of them);
//   * per group the fold is MAXK predicated ORs; the transpose is 3 instructions
//     per stage (SHFL, funnel rotate, LOP3); G groups are independent chains.
template <int W, int MAXK, bool SLICE_A>
// resident CTAs per SM the register budget is sized for (A/B on B200: one-word CSs run
// best at 3 CTAs x 8 warps with G = 4 probes per lane; two-word CSs at 2 CTAs)
#ifndef REI_CONCAT_MINB1
#define REI_CONCAT_MINB1 3
#endif
__device__ __forceinline__ void concat_fast_body(const LevelParams& p, uint32_t bid, uint32_t nbid) {
  static_assert(W <= 2, "fast path is for one- and two-word CSs");
  constexpr int NW = 32 * W;
#ifndef REI_CONCAT_G1
#define REI_CONCAT_G1 4
#endif
#ifndef REI_CONCAT_G2
#define REI_CONCAT_G2 4
#endif
  constexpr int G = (W == 1) ? REI_CONCAT_G1 : REI_CONCAT_G2;  // groups (probes per lane) in flight
  // slabs per pass: keep SB * W * MAXK shuffled slab words in registers (<= 16 + W * MAXK)
#ifdef REI_SB1  // (A/B) slabs per pass for one-word CSs
  constexpr int SB0 = (W == 1) ? REI_SB1 : ((W * MAXK <= 3) ? 4 : (W * MAXK <= 7 ? 2 : 1));
#else
  constexpr int SB0 = (W * MAXK <= 3) ? 4 : (W * MAXK <= 7 ? 2 : 1);
#endif
  constexpr int SB = SB0 < G ? SB0 : G;
  constexpr int GX = G / SB;  // uniform operands per batch
  static_assert(G % SB == 0 && 32 % GX == 0, "batch shape");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Block* s_blocks = reinterpret_cast<Block*>(smem_raw);
  uint32_t* s_src = reinterpret_cast<uint32_t*>(s_blocks + p.nblocks);  // [MAXK][NW]
  for (int i = threadIdx.x; i < (int)(p.nblocks * sizeof(Block) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_blocks)[i] = reinterpret_cast<const uint32_t*>(p.blocks)[i];
  if (p.rank_off_dev) {  // split level: the ? / * candidates (ranked first) counted on the device
    __syncthreads();
    const unsigned long long off = __ldg(p.rank_off_dev);
    for (int i = threadIdx.x; i < (int)p.nblocks; i += blockDim.x) s_blocks[i].cand_off += off;
  }
  // REVL (one-word CSs): lane l computes the slice of word 31 - l, so the transposed
  // candidate comes out bit-reversed -- its bitmap position is one shift away
#ifdef REI_NO_REVLANES
  constexpr bool REVL = false;
#else
  constexpr bool REVL = (W == 1);
#endif
  auto word_of = [](uint32_t l) { return REVL ? 31u - l : l; };  // word <-> lane (W = 1)
  for (int i = threadIdx.x; i < MAXK * NW; i += blockDim.x) {
    const uint32_t sp = p.split[(size_t)(i / NW) * kMaxNW + word_of(i % NW)];
    const uint32_t v = SLICE_A ? (sp >> 16) : (sp & 0xffffu);  // word of the sliced slab
    s_src[i] = REVL ? word_of(v) : v;                            // ... = the lane holding it
  }
  __syncthreads();

  const uint32_t lane = lane_id();
  const uint32_t wl = word_of(lane);  // this lane's word (W = 1; q * 32 + lane otherwise)
  const uint32_t lanebit = 1u << wl;
#ifdef REI_TRANSPOSE_BFLY  // (A/B) the butterfly with per-lane masks / rotations
  const TransposeLane tr(lane);
  auto pre = [](uint32_t v) { return v; };
#else
  const SkewTranspose tr(lane);
  auto pre = [&](uint32_t v) { return tr.pre(v); };
#endif
  // this warp's stage for new CSs (after the split table): [kWarps][kStage][W] + ranks
  WarpStage<W> stage;
  {
    uint32_t* st_cs = s_src + MAXK * NW;
    auto* st_rank = reinterpret_cast<unsigned long long*>(st_cs + kWarps * kStage * W);
    const uint32_t warp = threadIdx.x >> 5;
    stage.cs = st_cs + warp * kStage * W;
    stage.rank = st_rank + warp * kStage;
    stage.n = 0;
    stage_init_lc<W>(stage, st_rank + kWarps * kStage);
  }
  // split masks: bit of the uniform operand that enables split k of word q*32+lane
  uint32_t mlo[W][MAXK], mhi[W][MAXK];
#ifndef REI_FOLD_SEL
  uint32_t shk[MAXK];
  // bit `lane` of x as 0/1 = umulhi(x & 2^lane, 2^(32-lane)); lane 0 (word eps) needs no
  // x[w] ? T[eps] term: it equals the x[eps] ? T[w] term there
  const uint32_t shw = wl ? (1u << (32 - wl)) : 0u;
#endif
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const uint32_t w = q * 32 + wl;
    const uint32_t ns = p.nsplit[w];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const bool ok = (uint32_t)k < ns;
      const uint32_t sp = ok ? p.split[(size_t)k * kMaxNW + w] : 0u;
      const uint32_t fixed = SLICE_A ? (sp & 0xffffu) : (sp >> 16);
      mlo[q][k] = (ok && fixed < 32) ? (1u << fixed) : 0u;
      mhi[q][k] = (ok && fixed >= 32) ? (1u << (fixed & 31)) : 0u;
#ifndef REI_FOLD_SEL
      // 2^(32-u): umulhi(x & 2^u, 2^(32-u)) = bit u of x as 0/1 (u >= 1: a proper prefix)
      if (q == 0) shk[k] = (ok && fixed >= 1 && fixed < 32) ? (1u << (32 - fixed)) : 0u;
#endif
    }
  }
  const unsigned long long gwarp = (unsigned long long)bid * kWarps + (threadIdx.x >> 5);
  const unsigned long long nwarps = (unsigned long long)nbid * kWarps;

  unsigned long long warp_eval = 0;
  for (unsigned long long item = p.item_begin + gwarp; item < p.total_items; item += nwarps) {
    if (found_and_stop(p)) break;
    const Block& blk = s_blocks[find_block(s_blocks, p.nblocks, item)];
    const unsigned long long local = item - blk.item_off;
    const unsigned long long ut = local / blk.s_tiles, st = local % blk.s_tiles;
    const unsigned long long nu = SLICE_A ? blk.nb : blk.na;
    const unsigned long long ns = SLICE_A ? blk.na : blk.nb;
    const uint32_t* ubase = p.arena + (SLICE_A ? blk.b_base : blk.a_base) * W;
    const unsigned long long slab_base = SLICE_A ? blk.a_slab : blk.b_slab;
    const unsigned long long u0 = ut * blk.tu, u1 = min(u0 + blk.tu, nu);
    const unsigned long long nslabs = (ns + 31) / 32;
    const unsigned long long s0 = st * blk.ts, s1 = min(s0 + blk.ts, nslabs);
    const unsigned long long cand_off = blk.cand_off, nb = blk.nb;
    const uint32_t nu_item = (uint32_t)(u1 - u0);  // <= 64 (kTileU)
    uint32_t evaluated = 0;
    // the item's uniform operands, lane l holds u0 + l and u0 + 32 + l; broadcast by shuffle
    uint32_t xa[W], xb[W];
#pragma unroll
    for (int q = 0; q < W; ++q) { xa[q] = 0; xb[q] = 0; }
    if (lane < nu_item) load_cs<W>(ubase, u0 + lane, xa);
    if (lane + 32 < nu_item) load_cs<W>(ubase, u0 + 32 + lane, xb);

    // SB slabs per pass: their shuffled words stay in registers while every uniform
    // operand of the item is applied to them; a batch = GX uniform operands x SB slabs
    SLAB_EXIT_DECL
    for (unsigned long long s = s0; s < s1; s += SB) {
      if (SLAB_EXIT(p, s != s0)) break;  // early exit per slab pass, not only per work item
      uint32_t T[SB][W], Teps[SB], tk[SB][W][MAXK];
      bool lane_ok[SB];
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        const bool slab_ok = s + j < s1;  // warp-uniform
        lane_ok[j] = slab_ok && (s + j) * 32 + lane < ns;
#pragma unroll
        for (int q = 0; q < W; ++q) T[j][q] = slab_ok ? p.tarena[(slab_base + s + j) * NW + q * 32 + wl] : 0u;
        Teps[j] = __shfl_sync(kFull, T[j][0], word_of(0));
#pragma unroll
        for (int q = 0; q < W; ++q) {
#pragma unroll
          for (int k = 0; k < MAXK; ++k) {
            const uint32_t src = s_src[k * NW + q * 32 + lane];
            const uint32_t t0 = __shfl_sync(kFull, T[j][0], src & 31);
            if (W == 2) {
              const uint32_t t1 = __shfl_sync(kFull, T[j][W - 1], src & 31);
              tk[j][q][k] = (src >> 5) ? t1 : t0;
            } else {
              tk[j][q][k] = t0;
            }
          }
        }
      }
      // the slab terms in the transposer's input layout (a per-lane bit permutation)
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        Teps[j] = pre(Teps[j]);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          T[j][q] = pre(T[j][q]);
#pragma unroll
          for (int k = 0; k < MAXK; ++k) tk[j][q][k] = pre(tk[j][q][k]);
        }
      }

      // one batch of GX uniform operands x SB slabs; FULL batches need no operand bound test
      auto batch = [&](uint32_t ub, auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        uint32_t cs[G][W], xk[GX][W];
        bool valid[G], skip[G];
        uint32_t xs[W];  // GX divides 32: a batch never straddles the two halves
#pragma unroll
        for (int q = 0; q < W; ++q) xs[q] = ub >= 32 ? xb[q] : xa[q];
#pragma unroll
        for (int gx = 0; gx < GX; ++gx) {
          const uint32_t ui = ub + gx;
          uint32_t x[W];
#pragma unroll
          for (int q = 0; q < W; ++q) x[q] = __shfl_sync(kFull, xs[q], ui & 31);
#ifndef REI_FOLD_SEL
          if constexpr (W == 1) {
            // one-word CSs: the fold's selects as 0/1 multiplies on the otherwise idle
            // FMA pipe (b = a bit of x as 0/1 via umulhi, term = t * b), merged with
            // 3-input ORs on the ALU pipe (A/B on B200: -2.4..3.5 % solve time; the
            // concat kernel is ALU-bound once the probes hit L1)
            auto mul = [](uint32_t t, uint32_t b) {
              uint32_t r;
              asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(t), "r"(b));
              return r;
            };
            const uint32_t be = x[0] & 1u, bw = __umulhi(x[0] & lanebit, shw);
            uint32_t bk[MAXK];
#pragma unroll
            for (int k = 0; k < MAXK; ++k) bk[k] = __umulhi(x[0] & mlo[0][k], shk[k]);
#pragma unroll
            for (int j = 0; j < SB; ++j) {
              const int g = gx * SB + j;
              uint32_t acc = mul(T[j][0], be) | mul(Teps[j], bw);
#pragma unroll
              for (int k = 0; k < MAXK; ++k) acc |= mul(tk[j][0][k], bk[k]);
              cs[g][0] = acc;
              valid[g] = FULL ? lane_ok[j] : (lane_ok[j] && ui < nu_item);
            }
            xk[gx][0] = x[0];
            continue;
          }
#endif
          // enable masks of this operand (all-ones / zero), shared by the SB slabs:
          // epsilon splits (x[eps] -> T[w], x[w] -> T[eps]) and the proper splits
          const uint32_t me = (x[0] & 1u) ? kFull : 0u;
          uint32_t mw[W], mk[W][MAXK];
#pragma unroll
          for (int q = 0; q < W; ++q) {
            mw[q] = (x[q] & lanebit) ? kFull : 0u;
#pragma unroll
            for (int k = 0; k < MAXK; ++k)
              mk[q][k] = ((x[0] & mlo[q][k]) | (W == 2 ? (x[W - 1] & mhi[q][k]) : 0u)) ? kFull : 0u;
          }
#pragma unroll
          for (int j = 0; j < SB; ++j) {
            const int g = gx * SB + j;
#pragma unroll
            for (int q = 0; q < W; ++q) {
              uint32_t acc = (me & T[j][q]) | (mw[q] & Teps[j]);
#pragma unroll
              for (int k = 0; k < MAXK; ++k) acc |= mk[q][k] & tk[j][q][k];
              cs[g][q] = acc;  // bit-slice; transposed below
            }
            valid[g] = FULL ? lane_ok[j] : (lane_ok[j] && ui < nu_item);
          }
#pragma unroll
          for (int q = 0; q < W; ++q) xk[gx][q] = x[q];
        }
        // slices -> candidate CSs (one per lane)
        {
          uint32_t* v = &cs[0][0];
#if !defined(REI_TRANSPOSE_SINGLE)  // (A/B on B200: skew pairs 2 % faster than single; butterfly pairs were 5 % slower)
#pragma unroll
          for (int i = 0; i + 1 < G * W; i += 2) tr.pair(v[i], v[i + 1]);
          if ((G * W) & 1) v[G * W - 1] = tr(v[G * W - 1]);
#else
#pragma unroll
          for (int i = 0; i < G * W; ++i) v[i] = tr(v[i]);
#endif
        }
        // equals its uniform operand: cached, no probe needed (two-word CSs, whose probes
        // go to HBM; one-word probes hit L1, and the compare cost more than it saved:
        // A/B -1 %; an x.y == y filter measured slower too: DESIGN.md)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          uint32_t xc[W];
#pragma unroll
          for (int q = 0; q < W; ++q) xc[q] = REVL ? __brev(xk[g / SB][q]) : xk[g / SB][q];
          skip[g] = (W == 1) ? false : cs_equal<W>(cs[g], xc);
        }
        process_batch<W, G, false, REVL>(p, cs, valid, skip, [&](int g) {
          const unsigned long long ui = u0 + ub + g / SB;
          const unsigned long long sj = (s + g % SB) * 32 + lane;
          return cand_off + (SLICE_A ? sj * nb + ui : ui * nb + sj);
        }, W == 2 ? &stage : nullptr);
      };
      uint32_t ub = 0;
      for (; ub + GX <= nu_item; ub += GX) batch(ub, std::true_type{});
      if (ub < nu_item) batch(ub, std::false_type{});
#pragma unroll
      for (int j = 0; j < SB; ++j) evaluated += lane_ok[j] ? nu_item : 0u;  // every operand of the item
    }
    warp_eval += __reduce_add_sync(kFull, evaluated);  // one atomic per warp per launch (below)
  }
  if (lane_id() == 0 && warp_eval) {  // the control line's counters: once per warp, not per item
    atomicAdd(&p.ctl->evaluated, warp_eval);
    atomicAdd(&p.ctl->eval_c, warp_eval);
  }
  if (W == 2) stage_flush<W>(p, stage);
}

template <int W, int MAXK, bool SLICE_A>
// two-word CSs (A/B on B200, profiles/r02_ab_c2_concat.txt, concat ms c2-t1-s0 /
// c2-t2-s4): 2 CTAs/SM x 4 groups 77.8 / 333; 3 CTAs/SM (<= 85 registers) 94.2 / 436;
// 3 CTAs/SM x 2 groups 81.1 / 377; 2 CTAs/SM x 8 groups 120.9 / 552
#ifndef REI_CONCAT_MINB2
#define REI_CONCAT_MINB2 2
#endif
__global__ void __launch_bounds__(kWarps * 32, W == 1 ? REI_CONCAT_MINB1 : REI_CONCAT_MINB2) k_concat_fast(LevelParams p) {
  concat_fast_body<W, MAXK, SLICE_A>(p, blockIdx.x, gridDim.x);
}
template <int W, int MAXK, bool SLICE_A>
__global__ void __launch_bounds__(kWarps * 32, W == 1 ? REI_CONCAT_MINB1 : 2) k_concat_fast_packed(Packed pk) {
  uint32_t bid, nbid;
  const LevelParams& p = packed_params(pk, bid, nbid);
  concat_fast_body<W, MAXK, SLICE_A>(p, bid, nbid);
}

// ============================================================================
// Union kernel: uniform operand x, lane t holds operand_t of the sliced level.
template <int W, bool SH = false>
#ifndef REI_UNION_MINB1  // 4 CTAs/SM for one-word CSs (A/B on B200, scripts/ab_variants.py,
                         // 14 interleaved solves: Table 1 row 1 30.4 -> 29.7 ms, row 8 equal;
                         // 2 CTAs x 8 probes and 3 x 8 were slower)
#define REI_UNION_MINB1 4
#endif
#ifndef REI_UNION_G1
#define REI_UNION_G1 4
#endif
__device__ __forceinline__ void union_body(const LevelParams& p, uint32_t bid, uint32_t nbid) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Block* s_blocks = reinterpret_cast<Block*>(smem_raw);
  for (int i = threadIdx.x; i < (int)(p.nblocks * sizeof(Block) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_blocks)[i] = reinterpret_cast<const uint32_t*>(p.blocks)[i];
  if (p.rank_off_dev) {  // split level: the ? / * candidates (ranked first) counted on the device
    __syncthreads();
    const unsigned long long off = __ldg(p.rank_off_dev);
    for (int i = threadIdx.x; i < (int)p.nblocks; i += blockDim.x) s_blocks[i].cand_off += off;
  }
  __syncthreads();
  const uint32_t lane = lane_id();
  const unsigned long long gwarp = (unsigned long long)bid * kWarps + (threadIdx.x >> 5);
  const unsigned long long nwarps = (unsigned long long)nbid * kWarps;
  constexpr int G = W == 1 ? REI_UNION_G1 : Batch<W>::G;
  WarpStage<W> stage;  // (W <= 2) new CSs staged per warp after the block table
  {
    uint32_t* st_cs = reinterpret_cast<uint32_t*>(s_blocks + p.nblocks);
    auto* st_rank = reinterpret_cast<unsigned long long*>(st_cs + kWarps * kStage * W);
    const uint32_t warp = threadIdx.x >> 5;
    stage.cs = st_cs + warp * kStage * W;
    stage.rank = st_rank + warp * kStage;
    stage.n = 0;
    if (W <= 2) stage_init_lc<W>(stage, st_rank + kWarps * kStage);
  }

  unsigned long long warp_eval = 0;
  for (unsigned long long item = p.item_begin + gwarp; item < p.total_items; item += nwarps) {
    if (found_and_stop(p)) break;
    const Block& blk = s_blocks[find_block(s_blocks, p.nblocks, item)];
    const unsigned long long local = item - blk.item_off;
    const unsigned long long ut = local / blk.s_tiles, st = local % blk.s_tiles;
    const bool slice_a = blk.slice_a != 0;  // uniform = B, sliced = A
    const bool tri = blk.tri != 0;
    const unsigned long long nu = slice_a ? blk.nb : blk.na;
    const unsigned long long ns = slice_a ? blk.na : blk.nb;
    const unsigned long long u_base = slice_a ? blk.b_base : blk.a_base;
    const unsigned long long s_base = slice_a ? blk.a_base : blk.b_base;
    const unsigned long long u0 = ut * blk.tu, u1 = min(u0 + blk.tu, nu);
    const unsigned long long nslabs = (ns + 31) / 32;
    unsigned long long s0 = st * blk.ts;
    const unsigned long long s1 = min(s0 + blk.ts, nslabs);
    if (tri) s0 = max(s0, (u0 + 1) / 32);  // slabs entirely at or below the diagonal hold no j > i
    const uint32_t nu_item = (uint32_t)(u1 - u0);  // <= 64 (kTileU)
    uint32_t evaluated = 0;
    const unsigned long long cand_off = blk.cand_off, na = blk.na, nb = blk.nb;
    // narrow CSs: the item's uniform operands are held by the lanes and broadcast by shuffle
    uint32_t xa[W], xb[W];
#pragma unroll
    for (int q = 0; q < W; ++q) { xa[q] = 0; xb[q] = 0; }
    if (W <= 2) {
      if (lane < nu_item) load_cs<W>(p.arena, u_base + u0 + lane, xa);
      if (lane + 32 < nu_item) load_cs<W>(p.arena, u_base + u0 + 32 + lane, xb);
    }

    // G slabs per pass (one operand of the sliced level per lane and slab): each uniform
    // operand is broadcast once and applied to all G of them (a batch = G candidates)
    SLAB_EXIT_DECL
    for (unsigned long long s = s0; s < s1; s += G) {
      if (SLAB_EXIT(p, s != s0)) break;  // early exit per slab pass, not only per work item
      const unsigned long long s_last = min(s + G, s1) - 1;
      uint32_t y[G][W];
      bool lane_ok[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const unsigned long long sj = (s + j) * 32 + lane;
        lane_ok[j] = s + j < s1 && sj < ns;
        if (lane_ok[j]) load_cs<W>(p.arena, s_base + sj, y[j]);
        else {
#pragma unroll
          for (int q = 0; q < W; ++q) y[j][q] = 0;
        }
      }
      // operand ub pairs with this lane's slab-j operand iff ub < dlim[j] (triangular
      // blocks: j > i, i.e. (s + j) * 32 + lane > u0 + ub); 32-bit, set once per pass
      int dlim[G];
      uint32_t ub_end = nu_item;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const long long d = (long long)((s + j) * 32 + lane) - (long long)u0;
        dlim[j] = !lane_ok[j] ? 0 : (!tri ? 64 : (int)max(0LL, min(d, 64LL)));
        evaluated += (uint32_t)min(dlim[j], (int)nu_item);
      }
      if (tri) {  // no j > i left in these slabs past ub_end
        const long long e = (long long)(s_last * 32 + 31) - (long long)u0;
        ub_end = (uint32_t)max(0LL, min(e, (long long)nu_item));
      }
      for (uint32_t ub = 0; ub < ub_end; ++ub) {
        uint32_t x[W];
        if (W <= 2) {
#pragma unroll
          for (int q = 0; q < W; ++q) x[q] = __shfl_sync(kFull, ub >= 32 ? xb[q] : xa[q], ub & 31);
        } else {
          load_cs<W>(p.arena, u_base + u0 + ub, x);
        }
        uint32_t cs[G][W];
        bool valid[G], skip[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
#pragma unroll
          for (int q = 0; q < W; ++q) cs[j][q] = x[q] | y[j][q];
          valid[j] = (int)ub < dlim[j];
          skip[j] = cs_equal<W>(cs[j], x) || cs_equal<W>(cs[j], y[j]);
        }
        process_batch<W, G, SH>(p, cs, valid, skip, [&](int g) {
          const unsigned long long ui = u0 + ub;
          const unsigned long long sj = (s + g) * 32 + lane;
          const unsigned long long i = slice_a ? sj : ui;
          const unsigned long long j = slice_a ? ui : sj;
          return cand_off + (tri ? i * na - i * (i + 1) / 2 + (j - i - 1) : i * nb + j);
        }, kUnionStaged && W <= 2 ? &stage : nullptr);
      }
    }
    warp_eval += __reduce_add_sync(kFull, evaluated);  // one atomic per warp per launch (below)
  }
  if (lane_id() == 0 && warp_eval) {  // the control line's counters: once per warp, not per item
    atomicAdd(&p.ctl->evaluated, warp_eval);
    atomicAdd(&p.ctl->eval_u, warp_eval);
  }
  if (kUnionStaged && W <= 2) stage_flush<W>(p, stage);
}

// (minB: W = 2 keeps 2 CTAs per SM)
template <int W, bool SH = false>
#ifndef REI_UNION_MINBW
#define REI_UNION_MINBW 1
#endif
#ifndef REI_UNION_MINB2
#define REI_UNION_MINB2 2
#endif
__global__ void __launch_bounds__(kWarps * 32, W == 1 ? REI_UNION_MINB1 : (W == 2 ? REI_UNION_MINB2 : REI_UNION_MINBW)) k_union(LevelParams p) {
  union_body<W, SH>(p, blockIdx.x, gridDim.x);
}
template <int W>
__global__ void __launch_bounds__(kWarps * 32, W == 1 ? REI_UNION_MINB1 : (W == 2 ? 2 : 1)) k_union_packed(Packed pk) {
  uint32_t bid, nbid;
  const LevelParams& p = packed_params(pk, bid, nbid);
  union_body<W, false>(p, bid, nbid);
}

// ============================================================================
// Unary kernel: thread per operand; first n_q are question marks (x | eps),
// the rest stars: single shortlex pass  s[eps] = 1,
//   s[w] = x[w] | OR_{proper (u,v) of w} x[u] & s[v]   (v shorter than w: already final),
// the least fixpoint of s = 1 + x s (r* = (+)_n r^n).
template <int W>
__device__ void star_cs(const uint32_t (&x)[W], uint32_t (&s)[W], uint32_t n, const uint32_t* s_split,
                        const uint32_t* s_nsplit, int NW) {
#pragma unroll
  for (int q = 0; q < W; ++q) s[q] = 0;
  s[0] = 1u;
  for (uint32_t w = 1; w < n; ++w) {
    uint32_t b = get_bit<W>(x, w);
    const uint32_t m = s_nsplit[w];
    for (uint32_t k = 0; k < m && !b; ++k) {
      const uint32_t sp = s_split[k * NW + w];
      b = get_bit<W>(x, sp >> 16) & get_bit<W>(s, sp & 0xffffu);
    }
    if (b) {
#pragma unroll
      for (int q = 0; q < W; ++q)
        if ((w >> 5) == (uint32_t)q) s[q] |= 1u << (w & 31);
    }
  }
}

template <int W, bool SH = false>
__global__ void __launch_bounds__(256) k_unary(LevelParams p, unsigned long long n_q, unsigned long long n_s,
                                               unsigned long long base_q, unsigned long long base_s,
                                               unsigned long long off_s) {
  constexpr int NW = 32 * W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_split = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* s_nsplit = s_split + p.maxk * NW;
  for (int i = threadIdx.x; i < (int)(p.maxk * NW); i += blockDim.x)
    s_split[i] = p.split[(i / NW) * kMaxNW + (i % NW)];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s_nsplit[i] = p.nsplit[i];
  __syncthreads();
  const unsigned long long total = n_q + n_s;
  const unsigned long long tb = p.item_begin;  // this rank's share [tb, te)
  const unsigned long long te = total < (unsigned long long)p.total_items ? total : (unsigned long long)p.total_items;
  for (unsigned long long t = tb + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < te;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t x[W], cs[1][W];
    bool valid[1] = {true}, skip[1];
    unsigned long long rank[1];
    if (t < n_q) {
      load_cs<W>(p.arena, base_q + t, x);
#pragma unroll
      for (int q = 0; q < W; ++q) cs[0][q] = x[q];
      cs[0][0] |= 1u;  // x? = eps + x
      rank[0] = p.rank_base + t;
    } else {
      load_cs<W>(p.arena, base_s + (t - n_q), x);
      star_cs<W>(x, cs[0], p.n, s_split, s_nsplit, NW);
      rank[0] = p.rank_base + off_s + (t - n_q);
    }
    skip[0] = cs_equal<W>(cs[0], x);
    process_batch<W, 1, SH>(p, cs, valid, skip, [&](int) { return rank[0]; });
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && te > tb) atomicAdd(&p.ctl->evaluated, te - tb);
}

// Bit-sliced unary kernel (W32 <= 2): a warp takes a slab of 32 operands.  ? is
// x | eps per lane.  * runs on the transposed slab: lane w holds X[w] (bit t =
// operand t's bit w) and builds S[w] = X[w] | OR_{proper (u,v) of w} X[u] & S[v] one
// word length at a time (v is shorter than w, so S[v] is final when w's round comes),
// shuffling X[u] and S[v] from their lanes; a transpose turns the 32 slices into the
// 32 operands' stars (same fixpoint as star_cs).
template <int W, int MAXK>
__device__ __forceinline__ void unary_fast_body(const LevelParams& p, unsigned long long n_q, unsigned long long n_s,
                                                unsigned long long base_q, unsigned long long base_s,
                                                unsigned long long slab_s, uint32_t bid, uint32_t nbid) {
  static_assert(W <= 2, "sliced unary kernel is for one- and two-word CSs");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpStage<W> stage;  // new CSs staged per warp: [8 warps][kStage][W] + ranks
  {
    uint32_t* st_cs = reinterpret_cast<uint32_t*>(smem_raw);
    auto* st_rank = reinterpret_cast<unsigned long long*>(st_cs + 8 * kStage * W);
    const uint32_t warp = threadIdx.x >> 5;
    stage.cs = st_cs + warp * kStage * W;
    stage.rank = st_rank + warp * kStage;
    stage.n = 0;
    stage_init_lc<W>(stage, st_rank + 8 * kStage);
  }
  constexpr int NW = 32 * W;
  const uint32_t lane = lane_id();
  const TransposeLane tr(lane);
  uint32_t len[W], spl[W][MAXK];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const uint32_t w = q * 32 + lane;
    len[q] = w < p.n ? p.word_len[w] : 0u;
    const uint32_t ns = p.nsplit[w];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) spl[q][k] = (uint32_t)k < ns ? p.split[(size_t)k * kMaxNW + w] : 0xffffffffu;
  }
  uint32_t maxlen = 0;
#pragma unroll
  for (int q = 0; q < W; ++q) maxlen = max(maxlen, len[q]);
  maxlen = __reduce_max_sync(kFull, maxlen);

  const unsigned long long total = n_q + n_s;
  const unsigned long long tb = p.item_begin;  // this rank's operand share [tb, te)
  const unsigned long long te = total < (unsigned long long)p.total_items ? total : (unsigned long long)p.total_items;
  const unsigned long long slabs_q = (n_q + 31) / 32, slabs_s = (n_s + 31) / 32;
  const unsigned long long gwarp = ((unsigned long long)bid * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)nbid * blockDim.x) >> 5;
  uint32_t evaluated = 0;
#ifndef REI_UNARY_G
#define REI_UNARY_G 2  // A/B (profiles/r02_ab_unary_union.txt): C2 unary 31.5 (G = 4) -> 29.4 ms, G = 8 37.9
#endif
  constexpr int G = REI_UNARY_G;  // slabs per batch: G independent probes per lane in flight
  const unsigned long long nslab = slabs_q + slabs_s;
  for (unsigned long long it0 = gwarp * G; it0 < nslab; it0 += nwarps * G) {
   uint32_t cs[G][W];
   bool vv[G], skip[G];
   unsigned long long rk[G];
#pragma unroll
   for (int g = 0; g < G; ++g) {
    const unsigned long long it = it0 + g;
    const bool star = it >= slabs_q;
    const unsigned long long s = star ? it - slabs_q : it;
    const unsigned long long cnt = star ? n_s : n_q;
    const unsigned long long first = (star ? n_q : 0) + s * 32;  // unary rank of lane 0
    rk[g] = p.rank_base + first + lane;
    vv[g] = false;
    skip[g] = true;
#pragma unroll
    for (int q = 0; q < W; ++q) cs[g][q] = 0;
    if (it >= nslab || first >= te || first + 32 <= tb) continue;  // warp-uniform
    const unsigned long long i = s * 32 + lane;  // operand index within its level
    const bool valid = i < cnt && first + lane >= tb && first + lane < te;
    uint32_t x[W];
#pragma unroll
    for (int q = 0; q < W; ++q) x[q] = 0;
    if (i < cnt) load_cs<W>(p.arena, (star ? base_s : base_q) + i, x);
    if (!star) {
#pragma unroll
      for (int q = 0; q < W; ++q) cs[g][q] = x[q];
      cs[g][0] |= 1u;  // x? = eps + x
    } else {
      uint32_t X[W], S[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        X[q] = p.tarena[(slab_s + s) * NW + q * 32 + lane];
        S[q] = (q == 0 && lane == 0) ? kFull : 0u;  // every star contains eps
      }
      // X[u] does not change across the rounds: fetch the split prefixes once per slab
      // (zero for absent splits), then each round shuffles only S[v]
      uint32_t xu[W][MAXK];
#pragma unroll
      for (int q = 0; q < W; ++q) {
#pragma unroll
        for (int k = 0; k < MAXK; ++k) {
          const uint32_t u = spl[q][k] >> 16;
          uint32_t a = __shfl_sync(kFull, X[0], u & 31);
          if (W == 2) {
            const uint32_t a1 = __shfl_sync(kFull, X[W - 1], u & 31);
            a = (u & 32) ? a1 : a;
          }
          xu[q][k] = spl[q][k] != 0xffffffffu ? a : 0u;
        }
      }
      for (uint32_t L = 1; L <= maxlen; ++L) {
        uint32_t add[W];
#pragma unroll
        for (int q = 0; q < W; ++q) add[q] = 0;
#pragma unroll
        for (int q = 0; q < W; ++q) {
#pragma unroll
          for (int k = 0; k < MAXK; ++k) {
            // only the words of length L update in round L, and they have L - 1 proper
            // splits: later split slots are skipped (warp-uniform)
            if ((uint32_t)k + 1 >= L) break;
            const uint32_t v = spl[q][k] & 0xffffu;
            uint32_t sv = __shfl_sync(kFull, S[0], v & 31);
            if (W == 2) {
              const uint32_t sv1 = __shfl_sync(kFull, S[W - 1], v & 31);
              sv = (v & 32) ? sv1 : sv;
            }
            add[q] |= xu[q][k] & sv;
          }
        }
#pragma unroll
        for (int q = 0; q < W; ++q)
          if (len[q] == L) S[q] = X[q] | add[q];
      }
#pragma unroll
      for (int q = 0; q < W; ++q) cs[g][q] = tr(S[q]);
    }
    vv[g] = valid;
    skip[g] = cs_equal<W>(cs[g], x);
    evaluated += valid ? 1u : 0u;
   }
   process_batch<W, G>(p, cs, vv, skip, [&](int g) { return rk[g]; }, &stage);
  }
  stage_flush<W>(p, stage);
  const uint32_t tot = __reduce_add_sync(kFull, evaluated);
  if (lane == 0 && tot) atomicAdd(&p.ctl->evaluated, (unsigned long long)tot);
}

template <int W, int MAXK>
__global__ void __launch_bounds__(256, 2) k_unary_fast(LevelParams p, unsigned long long n_q, unsigned long long n_s,
                                                    unsigned long long base_q, unsigned long long base_s,
                                                    unsigned long long slab_s) {
  unary_fast_body<W, MAXK>(p, n_q, n_s, base_q, base_s, slab_s, blockIdx.x, gridDim.x);
}
// packed: the ? / * operand counts and bases travel in the spec's LevelParams
// (rank_base = 0, unary_* fields)
template <int W, int MAXK>
__global__ void __launch_bounds__(256, 2) k_unary_fast_packed(Packed pk) {
  uint32_t bid, nbid;
  const LevelParams& p = packed_params(pk, bid, nbid);
  unary_fast_body<W, MAXK>(p, p.un_q, p.un_s, p.un_bq, p.un_bs, p.un_slab, bid, nbid);
}

// Bit-sliced unary kernel for wide CSs (W32 >= 4, |IC| > 64): a warp takes a slab of
// 32 operands.  The slab's transposed words X[w] (bit t = operand t's bit w) and the
// star slices S[w] live in the warp's shared memory; round L computes every word of
// length L (a contiguous shortlex range) spread over the lanes,
//   S[w] = X[w] | OR_{proper (u,v) of w} X[u] & S[v],   S[eps] = all ones,
// where v is shorter than w, so S[v] is final (same fixpoint as star_cs: P:636,
// P:641-642).  Per slab that is S_in shared-memory AND/ORs for 32 operands, against
// S_in bit tests of W-word registers per operand in k_unary.  W transposes turn the
// slices into the 32 stars (one per lane).  ? is x | eps per lane.
template <int W>
__global__ void __launch_bounds__(256) k_unary_wide(LevelParams p, unsigned long long n_q, unsigned long long n_s,
                                                   unsigned long long base_q, unsigned long long base_s,
                                                   unsigned long long slab_s) {
  constexpr int NW = 32 * W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* sX = reinterpret_cast<uint32_t*>(smem_raw) + warp * 2 * NW;
  uint32_t* sS = sX + NW;
  constexpr uint32_t kLen = kMaxSplitRows + 3;  // word lengths 0 .. kMaxSplitRows + 1
  __shared__ uint32_t s_lstart[kLen + 1];          // first word of each length (shortlex)
  if (threadIdx.x == 0) {
    uint32_t L = 0;
    for (uint32_t w = 0; w < p.n; ++w)
      while (L < kLen && L <= p.word_len[w]) s_lstart[L++] = w;
    while (L <= kLen) s_lstart[L++] = p.n;
  }
  __syncthreads();
  uint32_t maxlen = 0;
  while (maxlen + 1 < kLen && s_lstart[maxlen + 1] < p.n) ++maxlen;

  const unsigned long long total = n_q + n_s;
  const unsigned long long tb = p.item_begin;  // this rank's operand share [tb, te)
  const unsigned long long te = total < (unsigned long long)p.total_items ? total : (unsigned long long)p.total_items;
  const unsigned long long slabs_q = (n_q + 31) / 32, slabs_s = (n_s + 31) / 32;
  const unsigned long long gwarp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  uint32_t evaluated = 0;
  const unsigned long long nslab = slabs_q + slabs_s;
  for (unsigned long long it = gwarp; it < nslab; it += nwarps) {
    const bool star = it >= slabs_q;
    const unsigned long long s = star ? it - slabs_q : it;
    const unsigned long long cnt = star ? n_s : n_q;
    const unsigned long long first = (star ? n_q : 0) + s * 32;  // unary rank of lane 0
    if (first >= te || first + 32 <= tb) continue;  // warp-uniform
    const unsigned long long i = s * 32 + lane;  // operand index within its level
    const bool valid = i < cnt && first + lane >= tb && first + lane < te;
    uint32_t x[W], cs[1][W];
#pragma unroll
    for (int q = 0; q < W; ++q) x[q] = 0;
    if (i < cnt) load_cs<W>(p.arena, (star ? base_s : base_q) + i, x);
    if (!star) {
#pragma unroll
      for (int q = 0; q < W; ++q) cs[0][q] = x[q];
      cs[0][0] |= 1u;  // x? = eps + x
    } else {
      const uint32_t* T = p.tarena + (slab_s + s) * NW;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        sX[q * 32 + lane] = T[q * 32 + lane];
        sS[q * 32 + lane] = 0u;
      }
      __syncwarp();
      if (lane == 0) sS[0] = kFull;  // every star contains eps
      for (uint32_t L = 1; L <= maxlen; ++L) {
        __syncwarp();
        const uint32_t w1 = s_lstart[L + 1];
        for (uint32_t w = s_lstart[L] + lane; w < w1; w += 32) {
          uint32_t acc = sX[w];
          for (uint32_t k = 0; k + 1 < L; ++k) {
            const uint32_t sp = __ldg(&p.split[(size_t)k * kMaxNW + w]);
            acc |= sX[sp >> 16] & sS[sp & 0xffffu];
          }
          sS[w] = acc;
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < W; ++q) cs[0][q] = transpose32(sS[q * 32 + lane], lane);
      __syncwarp();
    }
    bool vv[1] = {valid}, skip[1] = {cs_equal<W>(cs[0], x)};
    evaluated += valid ? 1u : 0u;
    const unsigned long long rk = p.rank_base + first + lane;
    process_batch<W, 1>(p, cs, vv, skip, [&](int) { return rk; });
  }
  const uint32_t tot = __reduce_add_sync(kFull, evaluated);
  if (lane == 0 && tot) atomicAdd(&p.ctl->evaluated, (unsigned long long)tot);
}

// Seeds (Alg. 1 line 3): one thread, symbols in Sigma order (deterministic).
template <int W>
__global__ void k_seeds(LevelParams p, const uint32_t* seeds, int nsym) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int a = 0; a < nsym; ++a) {
    uint32_t cs[1][W];
#pragma unroll
    for (int q = 0; q < W; ++q) cs[0][q] = seeds[a * kMaxW32 + q];
    bool valid[1] = {true}, skip[1] = {false};
    unsigned long long rank[1] = {(unsigned long long)a};
    process_batch<W, 1, true>(p, cs, valid, skip, [&](int) { return rank[0]; });
    if (*(volatile unsigned long long*)&p.ctl->found_rank != ~0ull) break;
  }
  p.ctl->evaluated = 0;
}

// Level c -> transposed slabs: warp per slab, T[32q + w] bit t = CS_t[32q + w].
template <int W, bool CG = false>
__device__ __forceinline__ void transpose_body(const uint32_t* __restrict__ arena, unsigned long long base,
                                               unsigned long long count, uint32_t* __restrict__ tarena,
                                               unsigned long long slab_base, uint32_t bid, uint32_t nbid) {
  constexpr int NW = 32 * W;
  const uint32_t lane = lane_id();
  const unsigned long long nslabs = (count + 31) / 32;
  const unsigned long long gw = ((unsigned long long)bid * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = ((unsigned long long)nbid * blockDim.x) >> 5;
  for (unsigned long long s = gw; s < nslabs; s += nw) {
    const unsigned long long e = s * 32 + lane;
    uint32_t x[W];
    if (e < count) {
      if (CG) load_cs_cg<W>(arena, base + e, x);
      else load_cs<W>(arena, base + e, x);
    } else {
#pragma unroll
      for (int q = 0; q < W; ++q) x[q] = 0;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) tarena[(slab_base + s) * NW + q * 32 + lane] = transpose32(x[q], lane);
  }
}

template <int W>
__global__ void k_transpose(const uint32_t* __restrict__ arena, unsigned long long base, unsigned long long count,
                            uint32_t* __restrict__ tarena, unsigned long long slab_base) {
  transpose_body<W>(arena, base, count, tarena, slab_base, blockIdx.x, gridDim.x);
}
// packed: spec i transposes its level [un_bq, un_bq + un_q) into slabs from un_slab
template <int W>
__global__ void k_transpose_packed(Packed pk) {
  uint32_t bid, nbid;
  const LevelParams& p = packed_params(pk, bid, nbid);
  transpose_body<W>(p.arena, p.un_bq, p.un_q, const_cast<uint32_t*>(p.tarena), p.un_slab, bid, nbid);
}

// (Re)insert arena entries [base, base + count) into the dedup set (after growth, or
// after a multi-rank level merge; inserting a present key is a no-op).
template <int W>
__global__ void k_rehash(LevelParams p, unsigned long long base, unsigned long long count) {
  for (unsigned long long t = base + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < base + count;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t x[W];
    load_cs<W>(p.arena, t, x);
    if (p.dedup.mode == DEDUP_BITMAP) {
      const uint32_t pos = bm_pos(x[0], p.n);
      atomicOr(&p.dedup.bitmap[pos >> 5], 1u << (pos & 31));
    } else if (p.dedup.mode == DEDUP_HASH64) {
      const unsigned long long key = key64<W>(x);
      const unsigned long long s = hash_cs<W>(x) & p.dedup.mask;
      insert_hash64(p, key, s, p.dedup.table[s]);
    } else if (p.dedup.mode == DEDUP_HASHIN) {
      if constexpr (W == 4 || W == 8) {
        unsigned long long key[W / 2], v0, v1;
        inline_key<W>(x, key);
        const unsigned long long s = hash_cs<W>(x) & p.dedup.mask;
        ld16v(p.dedup.table + s * (W / 2), v0, v1);
        insert_inline<W>(p, key, s, v0, v1);
      }
    } else {
      insert_indexed<W>(p, x, 0, false, t);
    }
  }
}

// ============================================================================
// Device-resident level loop (DevLoop, rei_common.cuh): the small, launch-bound levels
// of a search in ONE persistent cooperative grid.  Per level: thread (0, 0) finishes
// the previous level (its size from the control line) and plans the next one exactly
// like the host's plan_level (Q | S | C by L ascending | U by L ascending, ranks
// row-major, U with L = R triangular); after a grid barrier every thread takes
// candidates by rank (one per thread: the operands, the CS operation -- `?` sets the
// epsilon bit, `*` the shortlex fixpoint pass, concatenation the guide-table fold
// (Alg. 2), union the OR -- then the same dedup / precision / append tail
// as the level kernels).  The previous level is transposed into slabs meanwhile.
// The loop hands the search back to the host before a level with more than
// cand_limit candidates, one that could overflow the cache, one whose plan has too
// many blocks, after a level the host must sort (bitmap mode, >= sort_min entries),
// at the first precise candidate, or past max_cost.

// arrive-and-wait over the whole (co-resident, cooperative) grid
__device__ __forceinline__ void grid_sync(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// concatenation A.B of two CSs, one thread: bit w = A[eps] B[w] | A[w] B[eps] |
// OR over the proper splits (u, v) of w of A[u] B[v] (Alg. 2 / P:637)
template <int W>
__device__ void concat_cs(const uint32_t (&a)[W], const uint32_t (&b)[W], uint32_t (&r)[W], uint32_t n,
                          const uint32_t* s_split, const uint32_t* s_nsplit, int NW) {
  const bool ae = a[0] & 1u, be = b[0] & 1u;
#pragma unroll
  for (int q = 0; q < W; ++q) r[q] = (ae ? b[q] : 0u) | (be ? a[q] : 0u);
  for (uint32_t w = 1; w < n; ++w) {
    if (get_bit<W>(r, w)) continue;
    const uint32_t m = s_nsplit[w];
    for (uint32_t k = 0; k < m; ++k) {
      const uint32_t sp = s_split[k * NW + w];
      if (get_bit<W>(a, sp >> 16) & get_bit<W>(b, sp & 0xffffu)) {
#pragma unroll
        for (int q = 0; q < W; ++q)
          if ((w >> 5) == (uint32_t)q) r[q] |= 1u << (w & 31);
        break;
      }
    }
  }
}

// thread (0, 0): finish level st.cost, plan the next non-empty level
__device__ void loop_plan(const DevLoop& d, LevelCtl* ctl) {
  LoopState& st = *d.st;
  const uint32_t c_done = st.cost;
  bool transpose_done = false;
  st.tr_count = 0;
  st.sorting = 0;
  if (c_done) {
    const unsigned long long size = *(volatile unsigned long long*)&ctl->count;
    const bool overflow = *(volatile unsigned int*)&ctl->overflow != 0;
    const unsigned long long found = *(volatile unsigned long long*)&ctl->found_rank;
    d.lvl_eval[c_done] = *(volatile unsigned long long*)&ctl->evaluated;
    d.lvl_ns[c_done] = global_ns() - st.t_level;
    if (overflow) {  // partial level: the host clears it and redoes it
      st.stop = LOOP_OVERFLOW;
      st.next_cost = c_done;
      return;
    }
    d.lvl_size[c_done] = size;
    d.lvl_begin[c_done] = st.arena_used;
    d.lvl_slab[c_done] = st.slabs_used;
    st.last_cost = c_done;
    if (found != ~0ull) {
      st.found_rank = found;
      st.arena_used += size;
      st.stop = LOOP_FOUND;
      st.next_cost = c_done;
      return;
    }
    const bool sort = d.sort_min && size >= d.sort_min;
    // a level to sort is ordered in place this round (the free arena after it is the
    // scatter buffer, so it must hold the level once more), else by the host
    const bool sort_here = sort && st.arena_used + 2 * size <= d.entry_limit;
    st.sorting = sort_here ? 1u : 0u;
    if (!sort || sort_here) {  // transposed this round by every CTA (after the sort)
      st.tr_base = st.arena_used;
      st.tr_count = size;
      st.tr_slab = st.slabs_used;
      st.slabs_used += (size + 31) / 32;
    }
    st.arena_used += size;
    if (sort && !sort_here) {  // the host sorts it (its order is fixed before it is an operand)
      st.stop = LOOP_SORT;
      st.next_cost = c_done + 1;
      return;
    }
    transpose_done = true;
  }
  (void)transpose_done;
  // the next level with a non-empty plan
  const int c1 = (int)d.c1;
  auto size_of = [&](int L) -> unsigned long long { return L >= c1 ? d.lvl_size[L] : 0ull; };
  for (uint32_t c = c_done ? c_done + 1 : d.first_cost; c <= d.max_cost; ++c) {
    d.lvl_size[c] = 0;
    const int cost = (int)c;
    unsigned long long off = 0, items = 0;
    uint32_t nb = 0;
    bool too_many = false;
    auto add = [&](uint32_t kind, unsigned long long a_base, unsigned long long b_base, unsigned long long na,
                   unsigned long long nbb, unsigned long long cnt, bool tri) {
      if (nb == kLoopMaxBlocks) { too_many = true; return; }
      Block b{};
      b.kind = kind;
      b.tri = tri ? 1u : 0u;
      b.a_base = a_base;
      b.b_base = b_base;
      b.na = na;
      b.nb = nbb;
      b.cand_off = off;
      b.cand_count = cnt;
      b.item_off = items;
      d.blocks[nb++] = b;
      off += cnt;
      items += (kind == BK_Q || kind == BK_S) ? na : (tri ? na * na : na * nbb);
    };
    const int lq = cost - (int)d.k_opt, ls = cost - (int)d.k_star;
    const unsigned long long nq = size_of(lq), ns = size_of(ls);
    if (nq) add(BK_Q, d.lvl_begin[lq], 0, nq, 0, nq, false);
    if (ns) add(BK_S, d.lvl_begin[ls], 0, ns, 0, ns, false);
    for (int L = c1; L <= cost - (int)d.k_cat - c1; ++L) {
      const int R = cost - (int)d.k_cat - L;
      const unsigned long long na = size_of(L), nbb = size_of(R);
      if (na && nbb) add(BK_C, d.lvl_begin[L], d.lvl_begin[R], na, nbb, na * nbb, false);
    }
    for (int L = c1; L <= cost - (int)d.k_alt - L; ++L) {
      const int R = cost - (int)d.k_alt - L;
      const unsigned long long na = size_of(L), nbb = size_of(R);
      if (!na || !nbb) continue;
      const bool tri = L == R;
      const unsigned long long cnt = tri ? na * (na - 1) / 2 : na * nbb;
      if (cnt) add(BK_U, d.lvl_begin[L], d.lvl_begin[R], na, nbb, cnt, tri);
    }
    if (!nb && !too_many) continue;  // no level at this cost
    st.next_cost = c;
    if (too_many) { st.stop = LOOP_BLOCKS; return; }
    if (off > d.cand_limit) { st.stop = LOOP_BIG; return; }
    if (st.arena_used + off > d.entry_limit || st.slabs_used + (off + 31) / 32 + 1 > d.slab_limit) {
      st.stop = LOOP_CAPACITY;
      return;
    }
    st.cost = c;
    st.nblocks = nb;
    st.items = items;
    st.out_base = st.arena_used;
    ctl->count = 0;
    ctl->evaluated = 0;
    ctl->eval_c = 0;
    ctl->eval_u = 0;
    st.t_level = global_ns();
    return;
  }
  st.stop = LOOP_MAXCOST;
  st.next_cost = d.max_cost + 1;
}

// Order a finished one-word level in place by the top 12 bits of its bitmap position
// (the locality order of the host's sort_level): bucket counts, one
// exclusive scan, scatter to the free arena after the level, copy back.  Any order
// of a level is valid (it is fixed before the level is an operand, and its
// back-pointers travel with its entries); within a bucket the order is arbitrary.
template <int W>
__device__ void loop_sort(const LevelParams& p0, const DevLoop& d, unsigned long long base,
                          unsigned long long count) {
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  const uint32_t n = p0.n;
  auto bucket = [&](uint32_t cs) -> uint32_t {
    const uint32_t key = n ? __brev(cs) >> (32 - n) : 0u;
    return n > 12 ? key >> (n - 12) : key;
  };
  uint32_t* cs = p0.arena_out;
  unsigned long long* bp = p0.bp;
  const unsigned long long tmp = base + count;  // free arena / back-pointer space
  for (unsigned long long i = tid; i < kLoopSortBuckets; i += nth) d.hist[i] = 0;
  grid_sync(d.bar);
  for (unsigned long long i = tid; i < count; i += nth) atomicAdd(&d.hist[bucket(__ldcg(cs + (base + i) * W))], 1u);
  grid_sync(d.bar);
  if (blockIdx.x == 0) {  // exclusive scan of the 4096 counts: 16 per thread
    __shared__ unsigned int s_sum[256];
    unsigned int v[16], t = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = __ldcg(&d.hist[threadIdx.x * 16 + k]);
      t += v[k];
    }
    s_sum[threadIdx.x] = t;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
      const unsigned int a = threadIdx.x >= (unsigned)off ? s_sum[threadIdx.x - off] : 0u;
      __syncthreads();
      s_sum[threadIdx.x] += a;
      __syncthreads();
    }
    unsigned int run = s_sum[threadIdx.x] - t;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      d.hist[threadIdx.x * 16 + k] = run;
      run += v[k];
    }
  }
  grid_sync(d.bar);
  for (unsigned long long i = tid; i < count; i += nth) {
    uint32_t x[W];
    load_cs_cg<W>(cs, base + i, x);
    const unsigned long long b = __ldcg(bp + base + i);
    const unsigned long long j = atomicAdd(&d.hist[bucket(x[0])], 1u);
    store_cs<W>(cs, tmp + j, x);
    bp[tmp + j] = b;
  }
  grid_sync(d.bar);
  for (unsigned long long i = tid; i < count; i += nth) {
    uint32_t x[W];
    load_cs_cg<W>(cs, tmp + i, x);
    store_cs<W>(cs, base + i, x);
    bp[base + i] = __ldcg(bp + tmp + i);
  }
  grid_sync(d.bar);
}

template <int W>
__global__ void __launch_bounds__(256) k_level_loop(LevelParams p0, DevLoop d) {
  constexpr int NW = 32 * W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_split = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* s_nsplit = s_split + p0.maxk * NW;
  __shared__ LevelParams sp;
  __shared__ Block s_blocks[kLoopMaxBlocks];
  __shared__ unsigned long long s_items, s_tr_base, s_tr_count, s_tr_slab;
  __shared__ uint32_t s_nblocks, s_stop, s_sorting;
  for (int i = threadIdx.x; i < (int)(p0.maxk * NW); i += blockDim.x)
    s_split[i] = p0.split[(i / NW) * kMaxNW + (i % NW)];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s_nsplit[i] = p0.nsplit[i];
  if (threadIdx.x == 0) sp = p0;
  const uint32_t lane = lane_id();
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
  for (;;) {
    grid_sync(d.bar);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      loop_plan(d, p0.ctl);
      __threadfence();
    }
    grid_sync(d.bar);
    if (threadIdx.x == 0) {
      const volatile LoopState* vs = d.st;
      s_stop = vs->stop;
      s_nblocks = vs->nblocks;
      s_items = vs->items;
      s_tr_base = vs->tr_base;
      s_tr_count = vs->tr_count;
      s_tr_slab = vs->tr_slab;
      s_sorting = vs->sorting;
      sp.out_base = vs->out_base;
    }
    __syncthreads();
    if (s_sorting) loop_sort<W>(p0, d, s_tr_base, s_tr_count);
    if (s_tr_count)
      transpose_body<W, true>(p0.arena, s_tr_base, s_tr_count, const_cast<uint32_t*>(p0.tarena), s_tr_slab, blockIdx.x,
                        gridDim.x);
    if (s_stop != LOOP_RUN) break;
    for (int i = threadIdx.x; i < (int)(s_nblocks * sizeof(Block) / 4); i += blockDim.x)
      reinterpret_cast<uint32_t*>(s_blocks)[i] = __ldcg(reinterpret_cast<const uint32_t*>(d.blocks) + i);
    __syncthreads();
    const unsigned long long items = s_items;
    const int nb = (int)s_nblocks;
    uint32_t evaluated = 0;
    for (unsigned long long base = tid - lane; base < items; base += nthreads) {
      if (found_and_stop(sp)) break;
      const unsigned long long item = base + lane;
      bool valid = item < items;
      uint32_t cs[1][W];
      bool skip = false;
      unsigned long long rank = 0;
      // a warp whose 32 candidates are one concatenation row (the same left operand x,
      // 32 consecutive right operands) folds them bit-sliced like k_concat: transpose the
      // 32 y's, lane w ORs x[u] ? T[v] over the proper splits (u, v) of word w (plus the
      // epsilon splits), transpose back -- a few instructions per candidate instead of a
      // per-thread pass over every split of every word
      const int bi = valid ? find_block(s_blocks, nb, item) : -1;
      const int bi0 = __shfl_sync(kFull, bi, 0);
      bool row = d.rows && valid && bi == bi0 && s_blocks[bi].kind == BK_C;
      unsigned long long ri = 0, rj = 0;
      if (row) {
        const unsigned long long local = item - s_blocks[bi].item_off;
        ri = local / s_blocks[bi].nb;
        rj = local % s_blocks[bi].nb;
      }
      const unsigned long long ri0 = __shfl_sync(kFull, ri, 0);  // every lane (no short circuit)
      row = __all_sync(kFull, row && ri == ri0);
      if (row) {
        const Block& b = s_blocks[bi];
        uint32_t x[W], y[W], T[W], acc[W];
        load_cs_cg<W>(p0.arena, b.a_base + ri, x);  // warp-uniform
        load_cs_cg<W>(p0.arena, b.b_base + rj, y);
#pragma unroll
        for (int q = 0; q < W; ++q) T[q] = (uint32_t)q * 32 < p0.n ? transpose32(y[q], lane) : 0u;
        const uint32_t Teps = __shfl_sync(kFull, T[0], 0);
        const uint32_t xe = 0u - (x[0] & 1u);
#pragma unroll
        for (int q = 0; q < W; ++q) {
          acc[q] = (xe & T[q]) | ((0u - ((x[q] >> lane) & 1u)) & Teps);
          const uint32_t w = q * 32 + lane;
          const uint32_t m = w < p0.n ? s_nsplit[w] : 0u;
          const uint32_t km = __reduce_max_sync(kFull, m);
          for (uint32_t k = 0; k < km; ++k) {
            const uint32_t sp = k < m ? s_split[k * NW + w] : 0u;
            const uint32_t u = sp >> 16, v = sp & 0xffffu;
            uint32_t t = __shfl_sync(kFull, T[0], v & 31);
            if (W == 2) {
              const uint32_t t1 = __shfl_sync(kFull, T[W - 1], v & 31);
              t = (v >> 5) ? t1 : t;
            }
            if (k < m && get_bit<W>(x, u)) acc[q] |= t;
          }
        }
#pragma unroll
        for (int q = 0; q < W; ++q) cs[0][q] = (uint32_t)q * 32 < p0.n ? transpose32(acc[q], lane) : 0u;
        rank = b.cand_off + ri * b.nb + rj;
        skip = cs_equal<W>(cs[0], x) || cs_equal<W>(cs[0], y);
      } else if (valid) {
        const Block& b = s_blocks[bi];
        const unsigned long long local = item - b.item_off;
        uint32_t x[W], y[W];
        if (b.kind == BK_Q || b.kind == BK_S) {
          load_cs_cg<W>(p0.arena, b.a_base + local, x);
          if (b.kind == BK_Q) {
#pragma unroll
            for (int q = 0; q < W; ++q) cs[0][q] = x[q] | (q == 0 ? 1u : 0u);
          } else {
            star_cs<W>(x, cs[0], p0.n, s_split, s_nsplit, NW);
          }
          rank = b.cand_off + local;
          skip = cs_equal<W>(cs[0], x);
        } else {
          const unsigned long long ncol = b.tri ? b.na : b.nb;
          const unsigned long long i = local / ncol, j = local % ncol;
          if (b.tri && i >= j) {
            valid = false;
          } else {
            load_cs_cg<W>(p0.arena, b.a_base + i, x);
            load_cs_cg<W>(p0.arena, b.b_base + j, y);
            if (b.kind == BK_C) {
              concat_cs<W>(x, y, cs[0], p0.n, s_split, s_nsplit, NW);
            } else {
#pragma unroll
              for (int q = 0; q < W; ++q) cs[0][q] = x[q] | y[q];
            }
            rank = b.cand_off + (b.tri ? i * b.na - i * (i + 1) / 2 + (j - i - 1) : i * b.nb + j);
            skip = cs_equal<W>(cs[0], x) || cs_equal<W>(cs[0], y);
          }
        }
      }
      if (!valid) {
#pragma unroll
        for (int q = 0; q < W; ++q) cs[0][q] = 0;
      }
      evaluated += valid ? 1u : 0u;
      const bool v1[1] = {valid}, k1[1] = {skip};
      process_batch<W, 1>(sp, cs, v1, k1, [&](int) { return rank; });
    }
    const uint32_t tot = __reduce_add_sync(__activemask(), evaluated);
    if (lane == (uint32_t)(__ffs(__activemask()) - 1) && tot) atomicAdd(&p0.ctl->evaluated, (unsigned long long)tot);
  }
}

// Lagged levels: the next level's first arena index = the previous (still unread) level's
// first index + its count; a precise candidate or an overflow in that level makes the
// next level's kernels exit at once (its found_rank is set; the host redoes or discards it)
__global__ void k_next_base(const LevelCtl* __restrict__ prev, const unsigned long long* __restrict__ prev_base,
                            unsigned long long* __restrict__ base, LevelCtl* __restrict__ next,
                            unsigned long long* __restrict__ rank_off, uint32_t unary_reads_prev) {
  *base = *prev_base + prev->count;
  if (rank_off) *rank_off = prev->count * unary_reads_prev;  // ? and / or * operands of that level
  // a stop in the older level (precise candidate, overflow) -- or one passed down to it
  if (prev->found_rank != ~0ull || prev->overflow) next->found_rank = 0ull;
}

// Device CS operations on explicit operand pairs (tests): thread per pair, direct
// fold over the full guide table (epsilon splits + proper splits).
template <int W>
__global__ void k_ops(LevelParams p, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                      unsigned long long count) {
  constexpr int NW = 32 * W;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_split = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* s_nsplit = s_split + p.maxk * NW;
  for (int i = threadIdx.x; i < (int)(p.maxk * NW); i += blockDim.x)
    s_split[i] = p.split[(i / NW) * kMaxNW + (i % NW)];
  for (int i = threadIdx.x; i < NW; i += blockDim.x) s_nsplit[i] = p.nsplit[i];
  __syncthreads();
  for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t x[W], y[W], r[W];
#pragma unroll
    for (int q = 0; q < W; ++q) { x[q] = a[t * W + q]; y[q] = b ? b[t * W + q] : 0u; r[q] = 0; }
    if (op == 0) {
#pragma unroll
      for (int q = 0; q < W; ++q) r[q] = x[q] | y[q];
    } else if (op == 1) {
      for (uint32_t w = 0; w < p.n; ++w) {
        uint32_t bit = (get_bit<W>(x, 0) & get_bit<W>(y, w)) | (get_bit<W>(x, w) & get_bit<W>(y, 0));
        for (uint32_t k = 0; k < s_nsplit[w]; ++k) {
          const uint32_t sp = s_split[k * NW + w];
          bit |= get_bit<W>(x, sp >> 16) & get_bit<W>(y, sp & 0xffffu);
        }
        if (bit) {
#pragma unroll
          for (int q = 0; q < W; ++q)
            if ((w >> 5) == (uint32_t)q) r[q] |= 1u << (w & 31);
        }
      }
    } else if (op == 2) {
      star_cs<W>(x, r, p.n, s_split, s_nsplit, NW);
    } else if (op == 3) {
#pragma unroll
      for (int q = 0; q < W; ++q) r[q] = x[q];
      r[0] |= 1u;
    } else {
      r[0] = satisfies<W>(x, p) ? 1u : 0u;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) out[t * W + q] = r[q];
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <typename K>
int grid_for(K kernel, int threads, size_t smem, unsigned long long work_units_per_cta_hint,
             unsigned long long work, int waves = 1) {
  // the occupancy query costs host microseconds per launch: cache it per (kernel, smem)
  thread_local std::unordered_map<unsigned long long, int> cache;
  const unsigned long long key = (unsigned long long)(uintptr_t)(const void*)kernel ^ ((unsigned long long)smem << 48);
  int occ = 0;
  auto it = cache.find(key);
  if (it != cache.end()) {
    occ = it->second;
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    cache[key] = occ;
  }
  if (occ <= 0) occ = 1;
  unsigned long long want = (work + work_units_per_cta_hint - 1) / work_units_per_cta_hint;
  unsigned long long full = (unsigned long long)sm_count() * occ * (unsigned long long)waves;
  if (want < 1) want = 1;
  return (int)std::min<unsigned long long>(want, full);
}

size_t pair_smem(const LevelParams& p, int W) {
  const int NW = 32 * W;
  size_t s = p.nblocks * sizeof(Block) + (size_t)p.maxk * NW * 4 + NW * 4;
  if (W > 2) s += (size_t)kWarps * (NW + W) * 4;
  return s;
}

// Concat grids span this many waves of resident CTAs (REI_CONCAT_WAVES, default 16; 1 =
// persistent): with more than one, CTAs retire during the level and the union kernel of
// a concurrent level (higher stream priority) gets SMs even when concat reached them first.
int concat_waves();
template <int W, int MAXK, bool SA>
int launch_concat_wide_k(const LevelParams& p, cudaStream_t st) {
  const size_t smem = p.nblocks * sizeof(Block) + (size_t)2 * MAXK * 32 * W * 4 +
                      (size_t)kWarps * (32 * W + (W == 4 ? REI_WIDE_G : REI_WIDE_G8) * (32 * W + 1)) * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_concat_wide<W, MAXK, SA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_for(k_concat_wide<W, MAXK, SA>, kWarps * 32, smem, kWarps, p.total_items - p.item_begin,
                            concat_waves());
  k_concat_wide<W, MAXK, SA><<<grid, kWarps * 32, smem, st>>>(p);
  return 1;
}

int concat_waves() {
  const char* e = getenv("REI_CONCAT_WAVES");
  return e ? std::max(1, atoi(e)) : 16;
}
int union_waves() {
  const char* e = getenv("REI_UNION_WAVES");
  return e ? std::max(1, atoi(e)) : 1;
}

template <int W, int MAXK, bool SA>
int launch_concat_fast_t(const LevelParams& p, cudaStream_t st) {
  // (one-word CSs append directly: no per-warp stage, more of the SM's L1 for probes)
  const size_t smem = p.nblocks * sizeof(Block) + (size_t)MAXK * 32 * W * 4 +
                      (W == 2 ? (size_t)kWarps * kStage * (W * 4 + 8) + local_cache_bytes(W, kWarps) : 0);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_concat_fast<W, MAXK, SA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifdef REI_CARVEOUT
  cudaFuncSetAttribute(k_concat_fast<W, MAXK, SA>, cudaFuncAttributePreferredSharedMemoryCarveout, REI_CARVEOUT);
#endif
  const int grid = grid_for(k_concat_fast<W, MAXK, SA>, kWarps * 32, smem, kWarps, p.total_items - p.item_begin,
                            concat_waves());
  k_concat_fast<W, MAXK, SA><<<grid, kWarps * 32, smem, st>>>(p);
  return 1;
}

template <int W, bool SA>
int launch_concat_fast_k(const LevelParams& p, cudaStream_t st) {
  if (p.maxk <= 1) return launch_concat_fast_t<W, 1, SA>(p, st);
  if (p.maxk <= 3) return launch_concat_fast_t<W, 3, SA>(p, st);
  if (p.maxk <= 7) return launch_concat_fast_t<W, 7, SA>(p, st);
  return launch_concat_fast_t<W, 15, SA>(p, st);
}

// Sharded-cache levels (p.shards > 1) run the SH instantiations of the generic
// kernels: the fast kernels carry no owner routing at all.
template <int W, bool SH>
int launch_concat_generic(const LevelParams& p, cudaStream_t st) {
  const size_t smem = pair_smem(p, W);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_concat<W, SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_for(k_concat<W, SH>, kWarps * 32, smem, kWarps, p.total_items - p.item_begin, concat_waves());
  k_concat<W, SH><<<grid, kWarps * 32, smem, st>>>(p);
  return 1;
}

template <int W>
int launch_concat_t(const LevelParams& p, bool slice_a, cudaStream_t st) {
  if (p.shards > 1) return launch_concat_generic<W, true>(p, st);
  if constexpr (W <= 2) {
    if (p.maxk <= 15 && !getenv("REI_GENERIC_CONCAT"))
      return slice_a ? launch_concat_fast_k<W, true>(p, st) : launch_concat_fast_k<W, false>(p, st);
  }
  if constexpr (W == 4 || W == 8) {
    if (p.maxk <= 15 && !getenv("REI_GENERIC_CONCAT")) {
      if (p.maxk <= 9)
        return slice_a ? launch_concat_wide_k<W, 9, true>(p, st) : launch_concat_wide_k<W, 9, false>(p, st);
      return slice_a ? launch_concat_wide_k<W, 15, true>(p, st) : launch_concat_wide_k<W, 15, false>(p, st);
    }
  }
  return launch_concat_generic<W, false>(p, st);
}

template <int W, bool SH>
int launch_union_sh(const LevelParams& p, cudaStream_t st) {
  const size_t smem = p.nblocks * sizeof(Block) +
                      (W <= 2 ? (size_t)kWarps * kStage * (W * 4 + 8) + local_cache_bytes(W, kWarps) : 0);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_union<W, SH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifdef REI_CARVEOUT
  cudaFuncSetAttribute(k_union<W, SH>, cudaFuncAttributePreferredSharedMemoryCarveout, REI_CARVEOUT);
#endif
  const int grid = grid_for(k_union<W, SH>, kWarps * 32, smem, kWarps, p.total_items - p.item_begin, union_waves());
  k_union<W, SH><<<grid, kWarps * 32, smem, st>>>(p);
  return 1;
}

template <int W>
int launch_union_t(const LevelParams& p, cudaStream_t st) {
  return p.shards > 1 ? launch_union_sh<W, true>(p, st) : launch_union_sh<W, false>(p, st);
}

template <int W, int MAXK>
int launch_unary_fast_t(const LevelParams& p, unsigned long long n_q, unsigned long long n_s,
                        unsigned long long bq, unsigned long long bs, unsigned long long slab_s, cudaStream_t st) {
  const unsigned long long slabs = (n_q + 31) / 32 + (n_s + 31) / 32;
  const size_t smem = (size_t)8 * kStage * (W * 4 + 8) + local_cache_bytes(W, 8);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_unary_fast<W, MAXK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_for(k_unary_fast<W, MAXK>, 256, smem, 8, slabs);
  k_unary_fast<W, MAXK><<<grid, 256, smem, st>>>(p, n_q, n_s, bq, bs, slab_s);
  return 1;
}

template <int W>
int launch_unary_t(const LevelParams& p, unsigned long long n_q, unsigned long long n_s,
                   unsigned long long bq, unsigned long long bs, unsigned long long off_s,
                   unsigned long long slab_s, cudaStream_t st) {
  if (p.shards > 1) {
    const size_t smem = (size_t)p.maxk * 32 * W * 4 + 32 * W * 4;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_unary<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = grid_for(k_unary<W, true>, 256, smem, 256, n_q + n_s);
    k_unary<W, true><<<grid, 256, smem, st>>>(p, n_q, n_s, bq, bs, off_s);
    return 1;
  }
  if constexpr (W <= 2) {
    if (p.maxk <= 15 && !getenv("REI_GENERIC_UNARY")) {
      if (p.maxk <= 1) return launch_unary_fast_t<W, 1>(p, n_q, n_s, bq, bs, slab_s, st);
      if (p.maxk <= 3) return launch_unary_fast_t<W, 3>(p, n_q, n_s, bq, bs, slab_s, st);
      if (p.maxk <= 7) return launch_unary_fast_t<W, 7>(p, n_q, n_s, bq, bs, slab_s, st);
      return launch_unary_fast_t<W, 15>(p, n_q, n_s, bq, bs, slab_s, st);
    }
  }
  if constexpr (W >= 4) {
    if (!getenv("REI_GENERIC_UNARY")) {
      const unsigned long long slabs = (n_q + 31) / 32 + (n_s + 31) / 32;
      const size_t smem = (size_t)8 * 2 * 32 * W * 4;  // per warp: X and S slices
      const int grid = grid_for(k_unary_wide<W>, 256, smem, 8, slabs);
      k_unary_wide<W><<<grid, 256, smem, st>>>(p, n_q, n_s, bq, bs, slab_s);
      return 1;
    }
  }
  const size_t smem = (size_t)p.maxk * 32 * W * 4 + 32 * W * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_unary<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_for(k_unary<W>, 256, smem, 256, n_q + n_s);
  k_unary<W><<<grid, 256, smem, st>>>(p, n_q, n_s, bq, bs, off_s);
  return 1;
}

template <int W>
int launch_ops_t(const LevelParams& p, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
                 unsigned long long count, cudaStream_t st) {
  const size_t smem = (size_t)p.maxk * 32 * W * 4 + 32 * W * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_ops<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = grid_for(k_ops<W>, 256, smem, 256, count);
  k_ops<W><<<grid, 256, smem, st>>>(p, op, a, b, out, count);
  return 1;
}

// ---- packed launches (f4): one grid serves many specifications (CTA groups)
__global__ void k_ctl_reset_packed(const LevelParams* __restrict__ params, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    LevelCtl* c = params[i].ctl;
    c->found_rank = ~0ull;
    c->count = 0;
    c->evaluated = 0;
    c->overflow = 0;
    c->special_seen = 0;
    c->eval_c = 0;
    c->eval_u = 0;
  }
}
__global__ void k_ctl_gather_packed(const LevelParams* __restrict__ params, uint32_t n, LevelCtl* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = *params[i].ctl;
}

template <int W, int MAXK, bool SA>
int launch_concat_packed_t(const Packed& pk, uint32_t ctas, size_t nblocks_max, cudaStream_t st) {
  const size_t smem = nblocks_max * sizeof(Block) + (size_t)MAXK * 32 * W * 4 +
                      (W == 2 ? (size_t)kWarps * kStage * (W * 4 + 8) + local_cache_bytes(W, kWarps) : 0);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_concat_fast_packed<W, MAXK, SA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_concat_fast_packed<W, MAXK, SA><<<ctas, kWarps * 32, smem, st>>>(pk);
  return 1;
}
template <int W, bool SA>
int launch_concat_packed_k(int maxk, const Packed& pk, uint32_t ctas, size_t nb, cudaStream_t st) {
  if (maxk <= 1) return launch_concat_packed_t<W, 1, SA>(pk, ctas, nb, st);
  if (maxk <= 3) return launch_concat_packed_t<W, 3, SA>(pk, ctas, nb, st);
  if (maxk <= 7) return launch_concat_packed_t<W, 7, SA>(pk, ctas, nb, st);
  return launch_concat_packed_t<W, 15, SA>(pk, ctas, nb, st);
}
template <int W>
int launch_union_packed_t(const Packed& pk, uint32_t ctas, size_t nblocks_max, cudaStream_t st) {
  const size_t smem = nblocks_max * sizeof(Block) +
                      (W <= 2 ? (size_t)kWarps * kStage * (W * 4 + 8) + local_cache_bytes(W, kWarps) : 0);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_union_packed<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_union_packed<W><<<ctas, kWarps * 32, smem, st>>>(pk);
  return 1;
}
template <int W, int MAXK>
int launch_unary_packed_t(const Packed& pk, uint32_t ctas, cudaStream_t st) {
  const size_t smem = (size_t)8 * kStage * (W * 4 + 8) + local_cache_bytes(W, 8);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_unary_fast_packed<W, MAXK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_unary_fast_packed<W, MAXK><<<ctas, 256, smem, st>>>(pk);
  return 1;
}

}  // namespace

int packable(int W32, int maxk) { return (W32 == 1 || W32 == 2) && maxk <= 15 ? 1 : 0; }
int maxk_class(int maxk) { return maxk <= 1 ? 1 : maxk <= 3 ? 3 : maxk <= 7 ? 7 : 15; }

int launch_ctl_reset_packed(const LevelParams* params, uint32_t n, cudaStream_t st) {
  k_ctl_reset_packed<<<std::max(1u, std::min(64u, (n + 255) / 256)), 256, 0, st>>>(params, n);
  return 1;
}
int launch_ctl_gather_packed(const LevelParams* params, uint32_t n, LevelCtl* out, cudaStream_t st) {
  k_ctl_gather_packed<<<std::max(1u, std::min(64u, (n + 255) / 256)), 256, 0, st>>>(params, n, out);
  return 1;
}
int launch_concat_packed(int W32, int maxk, bool slice_a, const Packed& pk, uint32_t ctas, size_t nb, cudaStream_t st) {
  if (W32 == 1) return slice_a ? launch_concat_packed_k<1, true>(maxk, pk, ctas, nb, st)
                               : launch_concat_packed_k<1, false>(maxk, pk, ctas, nb, st);
  if (W32 == 2) return slice_a ? launch_concat_packed_k<2, true>(maxk, pk, ctas, nb, st)
                               : launch_concat_packed_k<2, false>(maxk, pk, ctas, nb, st);
  return 0;
}
int launch_union_packed(int W32, const Packed& pk, uint32_t ctas, size_t nb, cudaStream_t st) {
  if (W32 == 1) return launch_union_packed_t<1>(pk, ctas, nb, st);
  if (W32 == 2) return launch_union_packed_t<2>(pk, ctas, nb, st);
  return 0;
}
int launch_unary_packed(int W32, int maxk, const Packed& pk, uint32_t ctas, cudaStream_t st) {
  auto go = [&](auto w) {
    constexpr int W = decltype(w)::value;
    if (maxk <= 1) return launch_unary_packed_t<W, 1>(pk, ctas, st);
    if (maxk <= 3) return launch_unary_packed_t<W, 3>(pk, ctas, st);
    if (maxk <= 7) return launch_unary_packed_t<W, 7>(pk, ctas, st);
    return launch_unary_packed_t<W, 15>(pk, ctas, st);
  };
  if (W32 == 1) return go(std::integral_constant<int, 1>{});
  if (W32 == 2) return go(std::integral_constant<int, 2>{});
  return 0;
}
int launch_transpose_packed(int W32, const Packed& pk, uint32_t ctas, cudaStream_t st) {
  if (W32 == 1) { k_transpose_packed<1><<<ctas, 256, 0, st>>>(pk); return 1; }
  if (W32 == 2) { k_transpose_packed<2><<<ctas, 256, 0, st>>>(pk); return 1; }
  return 0;
}

#define REI_DISPATCH_W(W32, ...)                 \
  switch (W32) {                                 \
    case 1: { constexpr int W = 1; __VA_ARGS__; }   \
    case 2: { constexpr int W = 2; __VA_ARGS__; }   \
    case 4: { constexpr int W = 4; __VA_ARGS__; }   \
    case 8: { constexpr int W = 8; __VA_ARGS__; }   \
    case 16: { constexpr int W = 16; __VA_ARGS__; } \
    default: return 0;                           \
  }

int launch_seeds(int W32, const LevelParams& p, const uint32_t* seeds, int nsym, cudaStream_t st) {
  REI_DISPATCH_W(W32, k_seeds<W><<<1, 32, 0, st>>>(p, seeds, nsym); return 1);
}

int launch_unary(int W32, const LevelParams& p, uint64_t n_q, uint64_t n_s, uint64_t bq, uint64_t bs,
                 uint64_t off_s, uint64_t slab_s, cudaStream_t st) {
  REI_DISPATCH_W(W32, return launch_unary_t<W>(p, n_q, n_s, bq, bs, off_s, slab_s, st));
}

int launch_concat(int W32, const LevelParams& p, bool slice_a, cudaStream_t st) {
  REI_DISPATCH_W(W32, return launch_concat_t<W>(p, slice_a, st));
}

int launch_union(int W32, const LevelParams& p, cudaStream_t st) {
  REI_DISPATCH_W(W32, return launch_union_t<W>(p, st));
}

int launch_transpose(int W32, const uint32_t* arena, uint64_t base, uint64_t count, uint32_t* tarena,
                     uint64_t slab_base, cudaStream_t st) {
  const unsigned long long slabs = (count + 31) / 32;
  const int grid = (int)std::min<unsigned long long>((slabs + 7) / 8, (unsigned long long)sm_count() * 8);
  REI_DISPATCH_W(W32, k_transpose<W><<<std::max(grid, 1), 256, 0, st>>>(arena, base, count, tarena, slab_base);
                 return 1);
}

int launch_rehash(int W32, const LevelParams& p, uint64_t base, uint64_t count, cudaStream_t st) {
  const int grid = (int)std::min<unsigned long long>((count + 255) / 256, (unsigned long long)sm_count() * 8);
  REI_DISPATCH_W(W32, k_rehash<W><<<std::max(grid, 1), 256, 0, st>>>(p, base, count); return 1);
}

int launch_ops(int W32, const LevelParams& p, int op, const uint32_t* a, const uint32_t* b, uint32_t* out,
               uint64_t count, cudaStream_t st) {
  REI_DISPATCH_W(W32, return launch_ops_t<W>(p, op, a, b, out, count, st));
}

int launch_next_base(const LevelCtl* prev, const unsigned long long* prev_base, unsigned long long* base,
                     LevelCtl* next, unsigned long long* rank_off, uint32_t unary_reads_prev, cudaStream_t st) {
  k_next_base<<<1, 1, 0, st>>>(prev, prev_base, base, next, rank_off, unary_reads_prev);
  return 1;
}

// One cooperative launch of the device level loop; returns 1 (launched) or 0 (not
// eligible: width, or the grid cannot be co-resident).
int launch_level_loop(int W32, const LevelParams& p, const DevLoop& d, cudaStream_t st) {
  auto go = [&](auto w) -> int {
    constexpr int W = decltype(w)::value;
    const size_t smem = (size_t)p.maxk * 32 * W * 4 + 32 * W * 4;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_level_loop<W>, 256, smem) != cudaSuccess || occ < 1)
      return 0;
    static const int per_sm = getenv("REI_LOOP_CTAS_PER_SM") ? std::max(1, atoi(getenv("REI_LOOP_CTAS_PER_SM"))) : 4;  // A/B: 1 / 2 / 4 per SM -> loop 0.87 / 0.70 / 0.68 ms (Table 1 row 1)
    int grid = sm_count() * std::min(occ, per_sm);
    LevelParams pp = p;
    DevLoop dd = d;
    void* args[] = {&pp, &dd};
    if (cudaLaunchCooperativeKernel((const void*)k_level_loop<W>, dim3(grid), dim3(256), args, smem, st) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return 1;
  };
  if (W32 == 1) return go(std::integral_constant<int, 1>{});
  if (W32 == 2) return go(std::integral_constant<int, 2>{});
  return 0;
}

}  // namespace rei
