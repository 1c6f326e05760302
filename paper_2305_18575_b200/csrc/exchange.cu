// exchange.cu -- canonical merge of the per-rank new-CS lists of one cost level
// (multi-GPU sharded level).
//
// Every rank enumerates its share of the level's candidates and appends the CSs
// that are new to *its* dedup set.  The lists are all-gathered in rank order, so
// every rank holds the same byte sequence L = list_0 ++ list_1 ++ ...; each rank
// then keeps the first occurrence of every CS in L (a stable radix sort by CS,
// first-of-run flags, and an order-preserving compaction).  The result -- the
// level's unique CSs with their back-pointers, in an order fixed by L -- is
// identical on every rank, so later levels' candidate ranks mean the same
// operands everywhere.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "rei_common.cuh"
#include "rei_host.h"

namespace rei {
namespace {

template <int W>
__global__ void k_pack_keys(const uint32_t* __restrict__ cs, uint64_t m, unsigned long long* __restrict__ keys,
                            uint32_t* __restrict__ pos) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long k = cs[i * W];
    if (W == 2) k |= (unsigned long long)cs[i * W + 1] << 32;
    keys[i] = k;
    pos[i] = (uint32_t)i;
  }
}

__global__ void k_first_flags(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ pos,
                              uint64_t m, uint8_t* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    flags[pos[i]] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

template <int W>
__global__ void k_select(const uint32_t* __restrict__ cs, const unsigned long long* __restrict__ bp,
                         const uint8_t* __restrict__ flags, const uint32_t* __restrict__ scan, uint64_t m,
                         uint32_t* __restrict__ out_cs, unsigned long long* __restrict__ out_bp) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    const uint64_t o = scan[i];  // exclusive prefix count of kept entries: order preserved
#pragma unroll
    for (int q = 0; q < W; ++q) out_cs[o * W + q] = cs[i * W + q];
    out_bp[o] = bp[i];
  }
}

// Sort key of a one-word CS: its bitmap position (levels.cu bm_pos: the n-bit CS
// bit-reversed).
__global__ void k_level_keys(const uint32_t* __restrict__ cs, uint64_t m, uint32_t n, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ pos) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    keys[i] = n ? __brev(cs[i]) >> (32 - n) : 0u;
    pos[i] = (uint32_t)i;
  }
}

__global__ void k_gather_level(const uint32_t* __restrict__ cs, const unsigned long long* __restrict__ bp,
                               const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ out_cs,
                               unsigned long long* __restrict__ out_bp) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = perm[i];
    out_cs[i] = cs[j];
    out_bp[i] = bp[j];
  }
}

// ---- hash-owner exchange (north_star): records of (CS, back-pointer) --
// A record is W 32-bit CS words followed by the 64-bit back-pointer (2 words).
template <int W>
__device__ __forceinline__ void load_rec(const uint32_t* __restrict__ r, uint32_t (&cs)[W]) {
#pragma unroll
  for (int q = 0; q < W; ++q) cs[q] = r[q];
}

// owner[i] = hash owner of staged entry i; counts[o] += entries owned by o.
template <int W>
__global__ void k_owner_count(const uint32_t* __restrict__ cs, uint64_t m, uint32_t world,
                              uint8_t* __restrict__ owner, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int s_cnt[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x[W];
#pragma unroll
    for (int q = 0; q < W; ++q) x[q] = cs[i * W + q];
    const uint32_t o = owner_of_hash(hash_cs<W>(x), world);
    owner[i] = (uint8_t)o;
    atomicAdd(&s_cnt[o], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)world; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
}

// Scatter staged entries into owner-contiguous records (cursor[o] starts at bucket o's
// offset).  The order inside a bucket is free: the owner's unique list is all-gathered,
// so every rank appends the same bytes.
template <int W>
__global__ void k_owner_scatter(const uint32_t* __restrict__ cs, const unsigned long long* __restrict__ bp,
                                const uint8_t* __restrict__ owner, uint64_t m,
                                unsigned long long* __restrict__ cursor, uint32_t* __restrict__ rec) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long at = atomicAdd(&cursor[owner[i]], 1ull);
    uint32_t* r = rec + at * (W + 2);
#pragma unroll
    for (int q = 0; q < W; ++q) r[q] = cs[i * W + q];
    r[W] = (uint32_t)bp[i];
    r[W + 1] = (uint32_t)(bp[i] >> 32);
  }
}

// Owner dedup of the received records: insert-if-absent into a fresh table of
// (fingerprint, record index + 1) slots; the inserting record is appended to `out`.
template <int W>
__global__ void k_owner_dedup(const uint32_t* __restrict__ rec, uint64_t m, unsigned long long* __restrict__ table,
                              unsigned long long mask, uint32_t* __restrict__ out,
                              unsigned long long* __restrict__ out_count) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t x[W];
    load_rec<W>(rec + i * (W + 2), x);
    const unsigned long long h = hash_cs<W>(x);
    const uint32_t fp = (uint32_t)(h >> 32) | 1u;
    const unsigned long long mine = ((unsigned long long)fp << 32) | (uint32_t)(i + 1);
    unsigned long long s = h & mask;
    bool isnew = false;
    for (;;) {
      const unsigned long long old = atomicCAS(&table[s], 0ull, mine);
      if (old == 0) { isnew = true; break; }
      if ((uint32_t)(old >> 32) == fp) {
        uint32_t y[W];
        load_rec<W>(rec + (uint64_t)((uint32_t)old - 1) * (W + 2), y);
        bool eq = true;
#pragma unroll
        for (int q = 0; q < W; ++q) eq &= x[q] == y[q];
        if (eq) break;
      }
      s = (s + 1) & mask;
    }
    if (isnew) {
      const unsigned long long at = atomicAdd(out_count, 1ull);
      uint32_t* o = out + at * (W + 2);
#pragma unroll
      for (int q = 0; q < W + 2; ++q) o[q] = rec[i * (W + 2) + q];
    }
  }
}

// Records -> the level's arena entries and back-pointers.
template <int W>
__global__ void k_unpack(const uint32_t* __restrict__ rec, uint64_t m, uint32_t* __restrict__ cs,
                         unsigned long long* __restrict__ bp) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = rec + i * (W + 2);
#pragma unroll
    for (int q = 0; q < W; ++q) cs[i * W + q] = r[q];
    bp[i] = (unsigned long long)r[W] | ((unsigned long long)r[W + 1] << 32);
  }
}

// Canonical order of a level computed redundantly on every rank: sort keys = the whole
// CS (one word: its bitmap position, i.e. the CS bit-reversed; two words: the 64 bits).
template <int W>
__global__ void k_canon_keys(const uint32_t* __restrict__ cs, uint64_t m, uint32_t n,
                             unsigned long long* __restrict__ keys, uint32_t* __restrict__ pos) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    keys[i] = W == 1 ? (unsigned long long)(n ? __brev(cs[i]) >> (32 - n) : 0u)
                     : ((unsigned long long)cs[i * W + (W > 1 ? 1 : 0)] << 32) | cs[i * W];
    pos[i] = (uint32_t)i;
  }
}

template <int W>
__global__ void k_gather_entries(const uint32_t* __restrict__ cs, const unsigned long long* __restrict__ bp,
                                 const uint32_t* __restrict__ perm, uint64_t m, uint32_t* __restrict__ out_cs,
                                 unsigned long long* __restrict__ out_bp) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = perm[i];
#pragma unroll
    for (int q = 0; q < W; ++q) out_cs[i * W + q] = cs[(uint64_t)j * W + q];
    out_bp[i] = bp[j];
  }
}

// Scratch buffers grow geometrically and come from the caching allocator (devmem.cu).
template <typename T>
bool ensure(void** p, size_t* cap, size_t bytes, cudaStream_t st) {
  if (*cap >= bytes) return true;
  const size_t want = std::max(bytes, 2 * *cap);
  dev_free(*p, st);
  *p = nullptr;
  *cap = 0;
  if (dev_alloc(p, want, st) != cudaSuccess) return false;
  *cap = want;
  return true;
}

}  // namespace

bool merge_level(int W32, const uint32_t* g_cs, const unsigned long long* g_bp, uint64_t m, uint32_t* out_cs,
                 unsigned long long* out_bp, uint64_t* out_count, MergeScratch& s, cudaStream_t st,
                 std::string& err, uint64_t* launches) {
  *out_count = 0;
  if (m == 0) return true;
  if (W32 > 2) { err = "multi-rank merge supports |IC| <= 64"; return false; }
  if (m >= 0xffffffffull) { err = "level too large for the merge"; return false; }
  const int grid = (int)std::min<uint64_t>((m + 255) / 256, 148 * 8);
  bool ok = ensure<unsigned long long>(&s.keys, &s.keys_cap, m * 8, st) &&
            ensure<unsigned long long>(&s.keys2, &s.keys2_cap, m * 8, st) &&
            ensure<uint32_t>(&s.pos, &s.pos_cap, m * 4, st) &&
            ensure<uint32_t>(&s.pos2, &s.pos2_cap, m * 4, st) &&
            ensure<uint8_t>(&s.flags, &s.flags_cap, m, st) &&
            ensure<uint32_t>(&s.scan, &s.scan_cap, (m + 1) * 4, st);
  if (!ok) { err = "merge scratch allocation failed"; return false; }
  auto* keys = static_cast<unsigned long long*>(s.keys);
  auto* keys2 = static_cast<unsigned long long*>(s.keys2);
  auto* pos = static_cast<uint32_t*>(s.pos);
  auto* pos2 = static_cast<uint32_t*>(s.pos2);
  auto* flags = static_cast<uint8_t*>(s.flags);
  auto* scan = static_cast<uint32_t*>(s.scan);
  if (W32 == 1) k_pack_keys<1><<<grid, 256, 0, st>>>(g_cs, m, keys, pos);
  else k_pack_keys<2><<<grid, 256, 0, st>>>(g_cs, m, keys, pos);
  size_t t1 = 0, t2 = 0;
  const int end_bit = 32 * W32;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys2, pos, pos2, (int)m, 0, end_bit, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, flags, scan, (int)m + 1, st);
  if (!ensure<uint8_t>(&s.temp, &s.temp_cap, std::max(t1, t2), st)) { err = "cub temp"; return false; }
  // stable: equal keys keep gathered order, so the first of each run is the first occurrence
  if (cub::DeviceRadixSort::SortPairs(s.temp, t1, keys, keys2, pos, pos2, (int)m, 0, end_bit, st) != cudaSuccess) {
    err = "merge sort failed";
    return false;
  }
  k_first_flags<<<grid, 256, 0, st>>>(keys2, pos2, m, flags);
  if (cub::DeviceScan::ExclusiveSum(s.temp, t2, flags, scan, (int)m, st) != cudaSuccess) {
    err = "merge scan failed";
    return false;
  }
  if (W32 == 1) k_select<1><<<grid, 256, 0, st>>>(g_cs, g_bp, flags, scan, m, out_cs, out_bp);
  else k_select<2><<<grid, 256, 0, st>>>(g_cs, g_bp, flags, scan, m, out_cs, out_bp);
  uint32_t last_scan = 0;
  uint8_t last_flag = 0;
  cudaMemcpyAsync(&last_scan, scan + m - 1, 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&last_flag, flags + m - 1, 1, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) { err = "merge sync failed"; return false; }
  *out_count = (uint64_t)last_scan + last_flag;
  *launches += 6;
  return cudaGetLastError() == cudaSuccess;
}

// Reorder a finished one-word level by bitmap position (a stable radix sort of the
// level's entries with their back-pointers).  Consecutive cached operands then differ
// mostly in their short-word bits, so the 32 candidates of a warp group (one uniform
// operand x 32 consecutive operands) probe few distinct bitmap sectors.  The order of a
// level is free: it is fixed before the level is used as an operand, back-pointers
// refer to operand indices in that order, and every rank sorts identically.
bool sort_level(uint32_t n, uint32_t* cs, unsigned long long* bp, uint64_t m, MergeScratch& s, cudaStream_t st,
                std::string& err, uint64_t* launches, bool may_skip) {
  if (m < 2) return true;
  if (m >= 0xffffffffull) { err = "level too large to sort"; return false; }
  const int grid = (int)std::min<uint64_t>((m + 255) / 256, 148 * 8);
  bool ok = ensure<unsigned long long>(&s.keys, &s.keys_cap, m * 8, st) &&
            ensure<unsigned long long>(&s.keys2, &s.keys2_cap, m * 8, st) &&
            ensure<uint32_t>(&s.pos, &s.pos_cap, m * 4, st) && ensure<uint32_t>(&s.pos2, &s.pos2_cap, m * 4, st);
  if (!ok) {
    // the order is only a locality optimisation: a single rank short of memory keeps
    // the level as appended (ranks of one search must all sort, so they fail instead)
    cudaGetLastError();
    if (may_skip) return true;
    err = "level sort scratch allocation failed";
    return false;
  }
  auto* keys = static_cast<uint32_t*>(s.keys);
  auto* keys2 = static_cast<uint32_t*>(s.keys2);
  auto* pos = static_cast<uint32_t*>(s.pos);
  auto* pos2 = static_cast<uint32_t*>(s.pos2);
  k_level_keys<<<grid, 256, 0, st>>>(cs, m, n, keys, pos);
  size_t t1 = 0;
  const int end_bit = (int)std::max<uint32_t>(1, n);
  // order by the top 12 key bits only (they select the bitmap sector; one radix pass
  // fewer than the full key); REI_LEVEL_SORT_BITS=b overrides
  const char* sb = getenv("REI_LEVEL_SORT_BITS");
  const int begin_bit = std::max(0, end_bit - (sb ? atoi(sb) : 12));
  cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys2, pos, pos2, (int)m, begin_bit, end_bit, st);
  if (!ensure<uint8_t>(&s.temp, &s.temp_cap, t1, st)) {
    cudaGetLastError();
    if (may_skip) return true;
    err = "cub temp";
    return false;
  }
  if (cub::DeviceRadixSort::SortPairs(s.temp, t1, keys, keys2, pos, pos2, (int)m, begin_bit, end_bit, st) !=
      cudaSuccess) {
    err = "level sort failed";
    return false;
  }
  // gather into the (now free) key buffers, then copy back in place
  auto* tmp_bp = static_cast<unsigned long long*>(s.keys);
  auto* tmp_cs = static_cast<uint32_t*>(s.keys2);
  k_gather_level<<<grid, 256, 0, st>>>(cs, bp, pos2, m, tmp_cs, tmp_bp);
  if (cudaMemcpyAsync(cs, tmp_cs, m * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(bp, tmp_bp, m * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    err = "level sort copy failed";
    return false;
  }
  *launches += 3;
  return cudaGetLastError() == cudaSuccess;
}

void free_merge_scratch(MergeScratch& s) {
  for (void* p : {s.keys, s.keys2, s.pos, s.pos2, s.flags, s.scan, s.temp}) dev_free(p, nullptr);
  s = MergeScratch{};
}

// ---- host side of the hash-owner exchange ------------------------------------------
namespace {
int grid_for(uint64_t m) { return (int)std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, 148 * 8)); }
}  // namespace

bool owner_bucket(int W32, const uint32_t* cs, const unsigned long long* bp, uint64_t m, int world,
                  XScratch& x, cudaStream_t st, uint64_t* counts, std::string& err, uint64_t* launches) {
  for (int o = 0; o < world; ++o) counts[o] = 0;
  const size_t rec = 4ull * (W32 + 2);
  bool ok = ensure<uint8_t>(&x.owner, &x.owner_cap, std::max<uint64_t>(m, 1), st) &&
            ensure<uint8_t>(&x.send, &x.send_cap, std::max<uint64_t>(m, 1) * rec, st) &&
            ensure<uint8_t>(&x.ctr, &x.ctr_cap, 2 * 64 * 8, st);
  if (!ok) { err = "exchange scratch allocation failed"; return false; }
  auto* cnt = static_cast<unsigned long long*>(x.ctr);
  auto* cur = cnt + 64;
  if (cudaMemsetAsync(cnt, 0, 64 * 8, st) != cudaSuccess) { err = "memset failed"; return false; }
  if (m) {
    const int g = grid_for(m);
    auto* own = static_cast<uint8_t*>(x.owner);
    switch (W32) {
      case 1: k_owner_count<1><<<g, 256, 0, st>>>(cs, m, world, own, cnt); break;
      case 2: k_owner_count<2><<<g, 256, 0, st>>>(cs, m, world, own, cnt); break;
      case 4: k_owner_count<4><<<g, 256, 0, st>>>(cs, m, world, own, cnt); break;
      case 8: k_owner_count<8><<<g, 256, 0, st>>>(cs, m, world, own, cnt); break;
      default: k_owner_count<16><<<g, 256, 0, st>>>(cs, m, world, own, cnt); break;
    }
    unsigned long long h[64];
    if (cudaMemcpyAsync(h, cnt, world * 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) { err = "owner count failed"; return false; }
    unsigned long long off[64], run = 0;
    for (int o = 0; o < world; ++o) { counts[o] = h[o]; off[o] = run; run += h[o]; }
    if (cudaMemcpyAsync(cur, off, world * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      err = "owner offsets failed";
      return false;
    }
    auto* r = static_cast<uint32_t*>(x.send);
    switch (W32) {
      case 1: k_owner_scatter<1><<<g, 256, 0, st>>>(cs, bp, own, m, cur, r); break;
      case 2: k_owner_scatter<2><<<g, 256, 0, st>>>(cs, bp, own, m, cur, r); break;
      case 4: k_owner_scatter<4><<<g, 256, 0, st>>>(cs, bp, own, m, cur, r); break;
      case 8: k_owner_scatter<8><<<g, 256, 0, st>>>(cs, bp, own, m, cur, r); break;
      default: k_owner_scatter<16><<<g, 256, 0, st>>>(cs, bp, own, m, cur, r); break;
    }
    *launches += 2;
  }
  return cudaGetLastError() == cudaSuccess;
}

bool ensure_recv(int W32, uint64_t m, XScratch& x, cudaStream_t st) {
  return ensure<uint8_t>(&x.recv, &x.recv_cap, std::max<uint64_t>(m, 1) * 4ull * (W32 + 2), st);
}

bool owner_dedup(int W32, uint64_t m, XScratch& x, cudaStream_t st, uint64_t* out_count, std::string& err,
                 uint64_t* launches) {
  *out_count = 0;
  const size_t rec = 4ull * (W32 + 2);
  uint64_t slots = 1024;
  while (slots < 2 * m) slots <<= 1;
  bool ok = ensure<uint8_t>(&x.table, &x.table_cap, slots * 8, st) &&
            ensure<uint8_t>(&x.uniq, &x.uniq_cap, std::max<uint64_t>(m, 1) * rec, st) &&
            ensure<uint8_t>(&x.ctr, &x.ctr_cap, 2 * 64 * 8, st);
  if (!ok) { err = "owner dedup scratch allocation failed"; return false; }
  if (!m) return true;
  auto* cnt = static_cast<unsigned long long*>(x.ctr);
  if (cudaMemsetAsync(x.table, 0, slots * 8, st) != cudaSuccess || cudaMemsetAsync(cnt, 0, 8, st) != cudaSuccess) {
    err = "owner dedup memset failed";
    return false;
  }
  const int g = grid_for(m);
  auto* rin = static_cast<const uint32_t*>(x.recv);
  auto* tab = static_cast<unsigned long long*>(x.table);
  auto* out = static_cast<uint32_t*>(x.uniq);
  switch (W32) {
    case 1: k_owner_dedup<1><<<g, 256, 0, st>>>(rin, m, tab, slots - 1, out, cnt); break;
    case 2: k_owner_dedup<2><<<g, 256, 0, st>>>(rin, m, tab, slots - 1, out, cnt); break;
    case 4: k_owner_dedup<4><<<g, 256, 0, st>>>(rin, m, tab, slots - 1, out, cnt); break;
    case 8: k_owner_dedup<8><<<g, 256, 0, st>>>(rin, m, tab, slots - 1, out, cnt); break;
    default: k_owner_dedup<16><<<g, 256, 0, st>>>(rin, m, tab, slots - 1, out, cnt); break;
  }
  unsigned long long h = 0;
  if (cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) { err = "owner dedup failed"; return false; }
  *out_count = h;
  *launches += 1;
  return true;
}

bool ensure_gather_recs(int W32, uint64_t m, XScratch& x, cudaStream_t st) {
  return ensure<uint8_t>(&x.gath, &x.gath_cap, std::max<uint64_t>(m, 1) * 4ull * (W32 + 2), st);
}

bool unpack_records(int W32, const uint32_t* rec, uint64_t m, uint32_t* cs, unsigned long long* bp, cudaStream_t st,
                    uint64_t* launches) {
  if (!m) return true;
  const int g = grid_for(m);
  switch (W32) {
    case 1: k_unpack<1><<<g, 256, 0, st>>>(rec, m, cs, bp); break;
    case 2: k_unpack<2><<<g, 256, 0, st>>>(rec, m, cs, bp); break;
    case 4: k_unpack<4><<<g, 256, 0, st>>>(rec, m, cs, bp); break;
    case 8: k_unpack<8><<<g, 256, 0, st>>>(rec, m, cs, bp); break;
    default: k_unpack<16><<<g, 256, 0, st>>>(rec, m, cs, bp); break;
  }
  *launches += 1;
  return cudaGetLastError() == cudaSuccess;
}

bool canon_sort_level(int W32, uint32_t n, uint32_t* cs, unsigned long long* bp, uint64_t m, MergeScratch& s,
                      cudaStream_t st, std::string& err, uint64_t* launches) {
  if (m < 2) return true;
  if (W32 > 2) { err = "canonical level sort supports |IC| <= 64"; return false; }
  if (m >= 0xffffffffull) { err = "level too large to sort"; return false; }
  const int grid = grid_for(m);
  bool ok = ensure<unsigned long long>(&s.keys, &s.keys_cap, m * 8, st) &&
            ensure<unsigned long long>(&s.keys2, &s.keys2_cap, m * 8, st) &&
            ensure<uint32_t>(&s.pos, &s.pos_cap, m * 4, st) && ensure<uint32_t>(&s.pos2, &s.pos2_cap, m * 4, st) &&
            ensure<uint32_t>(&s.flags, &s.flags_cap, m * 4ull * W32, st) &&
            ensure<unsigned long long>(&s.scan, &s.scan_cap, m * 8, st);
  if (!ok) { err = "canonical sort scratch allocation failed"; return false; }
  auto* keys = static_cast<unsigned long long*>(s.keys);
  auto* keys2 = static_cast<unsigned long long*>(s.keys2);
  auto* pos = static_cast<uint32_t*>(s.pos);
  auto* pos2 = static_cast<uint32_t*>(s.pos2);
  if (W32 == 1) k_canon_keys<1><<<grid, 256, 0, st>>>(cs, m, n, keys, pos);
  else k_canon_keys<2><<<grid, 256, 0, st>>>(cs, m, n, keys, pos);
  const int end_bit = W32 == 1 ? (int)std::max<uint32_t>(1, n) : 64;
  size_t t1 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, keys, keys2, pos, pos2, (int)m, 0, end_bit, st);
  if (!ensure<uint8_t>(&s.temp, &s.temp_cap, t1, st)) { err = "cub temp"; return false; }
  if (cub::DeviceRadixSort::SortPairs(s.temp, t1, keys, keys2, pos, pos2, (int)m, 0, end_bit, st) != cudaSuccess) {
    err = "canonical level sort failed";
    return false;
  }
  auto* tmp_cs = static_cast<uint32_t*>(s.flags);
  auto* tmp_bp = static_cast<unsigned long long*>(s.scan);
  if (W32 == 1) k_gather_entries<1><<<grid, 256, 0, st>>>(cs, bp, pos2, m, tmp_cs, tmp_bp);
  else k_gather_entries<2><<<grid, 256, 0, st>>>(cs, bp, pos2, m, tmp_cs, tmp_bp);
  if (cudaMemcpyAsync(cs, tmp_cs, m * 4ull * W32, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(bp, tmp_bp, m * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    err = "canonical level sort copy failed";
    return false;
  }
  *launches += 4;
  return cudaGetLastError() == cudaSuccess;
}

void free_xscratch(XScratch& x) {
  for (void* p : {x.owner, x.send, x.recv, x.uniq, x.gath, x.table, x.ctr}) dev_free(p, nullptr);
  x = XScratch{};
}

}  // namespace rei
