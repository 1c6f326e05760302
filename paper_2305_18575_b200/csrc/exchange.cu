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

template <typename T>
bool ensure(void** p, size_t* cap, size_t bytes, cudaStream_t st) {
  if (*cap >= bytes) return true;
  if (*p) cudaFreeAsync(*p, st);
  *p = nullptr;
  if (cudaMallocAsync(p, bytes, st) != cudaSuccess) return false;
  *cap = bytes;
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

void free_merge_scratch(MergeScratch& s) {
  cudaFree(s.keys); cudaFree(s.keys2); cudaFree(s.pos); cudaFree(s.pos2); cudaFree(s.flags);
  cudaFree(s.scan); cudaFree(s.temp);
  s = MergeScratch{};
}

}  // namespace rei
