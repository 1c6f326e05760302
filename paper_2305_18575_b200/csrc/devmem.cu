// devmem.cu -- process-wide caching allocators of the runtime (memory manager).
//
// A context's buffers are large (the bitmap-mode arena of Table 1 row 1 is ~0.5 GB)
// and a serving process creates many contexts (one per specification, the paper's
// 5,160-run benchmark suite).  cudaMalloc / cudaMallocHost of fresh
// memory costs milliseconds per call, so:
//   * device memory comes from one cudaMemPool per device whose release threshold is
//     unbounded: blocks freed by rei_destroy stay mapped and are handed to the next
//     rei_init (stream-ordered: cudaMallocFromPoolAsync / cudaFreeAsync on the
//     context's stream);
//   * pinned host blocks (control lines, block tables) come from a size-keyed free
//     list.
// rei_release_cached_memory() trims both.  Buffers that are exported through CUDA IPC
// (sharded-cache contexts) do not use the pool (pool memory needs an IPC-capable pool).
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "rei_host.h"

namespace rei {
namespace {

std::mutex g_mu;
std::map<int, cudaMemPool_t> g_pools;                 // device -> pool
std::multimap<size_t, void*> g_host_free;             // size -> pinned block
std::map<void*, size_t> g_host_size;                  // every pinned block we own

cudaError_t pool_of(int dev, cudaMemPool_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_pools.find(dev);
  if (it != g_pools.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.handleTypes = cudaMemHandleTypeNone;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  cudaError_t e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = ~0ull;  // never release freed blocks on synchronisation
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) return e;
  g_pools[dev] = pool;
  *out = pool;
  return cudaSuccess;
}

}  // namespace

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
  *p = nullptr;
  if (bytes == 0) bytes = 1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  if ((e = pool_of(dev, &pool)) != cudaSuccess) return e;
  e = cudaMallocFromPoolAsync(p, bytes, pool, st);
  if (e == cudaErrorMemoryAllocation) {
    // the idle blocks the pool keeps may not fit this request: return them and retry
    cudaGetLastError();
    cudaStreamSynchronize(st);
    cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocFromPoolAsync(p, bytes, pool, st);
  }
  return e;
}

void dev_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

uint64_t dev_pool_idle_bytes(int dev) {
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_pools.find(dev);
    if (it == g_pools.end()) return 0;
    pool = it->second;
  }
  uint64_t reserved = 0, used = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  return reserved > used ? reserved - used : 0;
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
  std::vector<void*> host;
  std::vector<cudaMemPool_t> pools;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_host_free) {
      host.push_back(kv.second);
      g_host_size.erase(kv.second);
    }
    g_host_free.clear();
    for (auto& kv : g_pools) pools.push_back(kv.second);
  }
  for (void* p : host) cudaFreeHost(p);
  for (cudaMemPool_t pool : pools) cudaMemPoolTrimTo(pool, 0);
}

}  // namespace rei
