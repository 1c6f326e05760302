// devmem.cu -- process-wide caching allocators of the runtime (memory manager).
//
// A context's buffers are large (the bitmap-mode arena of Table 1 row 1 is ~0.5 GB;
// a two-word-CS search grows its cache and hash set to tens of GB) and a serving
// process creates many contexts (one per specification, the paper's 5,160-run
// benchmark suite).  Fresh device memory costs ~8 ms per GB to map
// (measured on B200: a 51 GB arena + 34 GB hash set took 0.7 s), and cudaMallocHost
// costs milliseconds per call, so:
//   * device blocks freed by a context (rei_destroy, or a grown arena's old buffers)
//     are kept, per device, in a size-keyed free list and handed to the next request
//     of the same size class (sizes rounded up to 2 MiB; a cached block up to 1/8
//     larger than the request is accepted).  A context's growth sequence is
//     deterministic, so the next context on the same specification reuses every block.
//     The stream is synchronised before a block enters the list (frees are rare).
//     On cudaErrorMemoryAllocation the idle blocks of that device are released and
//     the allocation retried;
//   * pinned host blocks (control lines, block tables) come from a similar free list.
// rei_release_cached_memory() releases both.  Sharded-cache contexts export their
// buffers through CUDA IPC and allocate with plain cudaMalloc (rei_api.cu).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "rei_host.h"

namespace rei {
namespace {

constexpr size_t kGran = size_t(2) << 20;

struct DevBlock {
  int dev;
  size_t bytes;
};

std::mutex g_mu;
std::map<int, std::multimap<size_t, void*>> g_dev_free;  // device -> (size -> idle block)
std::map<void*, DevBlock> g_dev_blocks;                   // every device block we own
std::multimap<size_t, void*> g_host_free;                 // size -> idle pinned block
std::map<void*, size_t> g_host_size;                      // every pinned block we own

size_t round_up(size_t b) { return (b + kGran - 1) / kGran * kGran; }

// Free-memory estimate per device: one cudaMemGetInfo (0.3-70 ms on B200, measured),
// then this allocator's own cudaMalloc / cudaFree traffic since that query.
struct FreeInfo {
  bool known = false;
  uint64_t free_at_query = 0;
  int64_t net_since = 0;  // bytes cudaMalloc'd minus bytes cudaFree'd since the query
};
std::map<int, FreeInfo> g_free_info;

// Take a cached block of at least `bytes` (<= bytes + bytes/8) on `dev`; nullptr if none.
void* take_cached(int dev, size_t bytes) {
  auto& fl = g_dev_free[dev];
  auto it = fl.lower_bound(bytes);
  if (it == fl.end() || it->first > bytes + bytes / 8) return nullptr;
  void* p = it->second;
  fl.erase(it);
  return p;
}

void release_device(int dev) {  // caller holds g_mu
  auto& fl = g_dev_free[dev];
  for (auto& kv : fl) {
    cudaFree(kv.second);
    g_dev_blocks.erase(kv.second);
    g_free_info[dev].net_since -= (int64_t)kv.first;
  }
  fl.clear();
}

}  // namespace

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  (void)st;
  *p = nullptr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const size_t want = round_up(bytes ? bytes : 1);
  std::lock_guard<std::mutex> lk(g_mu);
  if ((*p = take_cached(dev, want)) != nullptr) return cudaSuccess;
  static const bool trace = getenv("REI_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  e = cudaMalloc(p, want);
  if (trace)
    fprintf(stderr, "[rei_devmem] cudaMalloc %zu bytes: %.3f ms (%s)\n", want,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
            cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // not sticky: clear it, return the idle blocks and retry once
    release_device(dev);
    e = cudaMalloc(p, want);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return e;
  }
  g_dev_blocks[*p] = {dev, want};
  g_free_info[dev].net_since += (int64_t)want;
  return cudaSuccess;
}

uint64_t dev_free_estimate(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  FreeInfo& fi = g_free_info[dev];
  if (!fi.known) {
    size_t fr = 0, tot = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev) cudaSetDevice(dev);
    cudaMemGetInfo(&fr, &tot);
    if (cur != dev) cudaSetDevice(cur);
    fi = FreeInfo{true, (uint64_t)fr, 0};
  }
  int64_t est = (int64_t)fi.free_at_query - fi.net_since;
  auto it = g_dev_free.find(dev);
  if (it != g_dev_free.end())
    for (auto& kv : it->second) est += (int64_t)kv.first;  // idle blocks can be released
  return est > 0 ? (uint64_t)est : 0;
}

void dev_free_estimate_reset(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_free_info[dev].known = false;
}

void dev_free(void* p, cudaStream_t st) {
  if (!p) return;
  cudaStreamSynchronize(st);  // no kernel of this stream may still touch the block
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev_blocks.find(p);
  if (it == g_dev_blocks.end()) {
    cudaFree(p);
    return;
  }
  g_dev_free[it->second.dev].emplace(it->second.bytes, p);
}

uint64_t dev_pool_idle_bytes(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  uint64_t s = 0;
  auto it = g_dev_free.find(dev);
  if (it != g_dev_free.end())
    for (auto& kv : it->second) s += kv.first;
  return s;
}

cudaError_t host_alloc(void** p, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_host_free.lower_bound(bytes);
    if (it != g_host_free.end() && it->first <= 2 * bytes) {  // reuse a block of similar size
      *p = it->second;
      g_host_free.erase(it);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMallocHost(p, bytes);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  g_host_size[*p] = bytes;
  return cudaSuccess;
}

void host_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_host_size.find(p);
  if (it == g_host_size.end()) return;
  g_host_free.emplace(it->second, p);
}

void release_cached_memory() {
  std::lock_guard<std::mutex> lk(g_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_dev_free) {
    cudaSetDevice(kv.first);
    release_device(kv.first);
  }
  cudaSetDevice(cur);
  for (auto& kv : g_host_free) {
    cudaFreeHost(kv.second);
    g_host_size.erase(kv.second);
  }
  g_host_free.clear();
}

}  // namespace rei
