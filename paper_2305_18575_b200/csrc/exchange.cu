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
                std::string& err, uint64_t* launches) {
  if (m < 2) return true;
  if (m >= 0xffffffffull) { err = "level too large to sort"; return false; }
  const int grid = (int)std::min<uint64_t>((m + 255) / 256, 148 * 8);
  bool ok = ensure<unsigned long long>(&s.keys, &s.keys_cap, m * 8, st) &&
            ensure<unsigned long long>(&s.keys2, &s.keys2_cap, m * 8, st) &&
            ensure<uint32_t>(&s.pos, &s.pos_cap, m * 4, st) && ensure<uint32_t>(&s.pos2, &s.pos2_cap, m * 4, st);
  if (!ok) { err = "level sort scratch allocation failed"; return false; }
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
  if (!ensure<uint8_t>(&s.temp, &s.temp_cap, t1, st)) { err = "cub temp"; return false; }
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

}  // namespace rei
