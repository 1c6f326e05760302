// partprobe.cu -- does partitioning the dedup probes by table slice pay on B200?
//
// A level of the HBM hash-set workloads (configs[1]-[3]) probes ~1e9-5e9 candidate
// CSs against a multi-GB open-addressing table: every probe is one random DRAM access,
// capped at ~36 G/s (profiles/r02_random_read_ncu.md).  This measures the pieces of
// the alternative "emit, partition by slot range, probe per partition" pipeline:
//   direct   : probe records in generation (random) order           -> G probes/s
//   sorted   : probe records grouped by the top 8 bits of their slot -> G probes/s
//   scatter  : write records to 256 partition lists, warp-aggregated atomics
//   cubsort  : cub::DeviceRadixSort::SortPairs, 8-bit keys, 16-byte values
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o partprobe partprobe.cu
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr unsigned long long kEmpty = ~0ull;

__host__ __device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

struct Rec {
  unsigned long long key, rank;
};

__device__ unsigned long long g_hits;

__global__ void k_fill(unsigned long long* t, unsigned long long n) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    t[i] = kEmpty;
}

__global__ void k_insert(unsigned long long* t, unsigned long long mask, unsigned long long nkeys) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < nkeys;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long key = mix(i * 2 + 1);
    unsigned long long s = mix(key ^ 0x1234) & mask;
    for (;;) {
      const unsigned long long old = atomicCAS(&t[s], kEmpty, key);
      if (old == kEmpty || old == key) break;
      s = (s + 1) & mask;
    }
  }
}

// queries: 90 % keys of the set, 10 % absent keys; partition = top 8 bits of the slot
__global__ void k_queries(Rec* q, uint8_t* part, unsigned long long n, unsigned long long nkeys, int log2slots) {
  const unsigned long long mask = (1ull << log2slots) - 1;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long r = mix(i ^ 0xabcdefull);
    const unsigned long long key = (r % 10) ? mix((r >> 8) % nkeys * 2 + 1) : mix(r * 2);
    q[i].key = key;
    q[i].rank = i;
    part[i] = (uint8_t)(((mix(key ^ 0x1234) & mask) >> (log2slots - 8)) & 255);
  }
}

template <int ILP>
__global__ void __launch_bounds__(256) k_probe(const Rec* __restrict__ q, unsigned long long n,
                                               const unsigned long long* __restrict__ t, unsigned long long mask) {
  unsigned long long hits = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i0 = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i0 < n; i0 += stride * ILP) {
    unsigned long long key[ILP], s[ILP], v[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      const unsigned long long i = i0 + j * stride;
      key[j] = i < n ? __ldcs(&q[i].key) : kEmpty;
      s[j] = mix(key[j] ^ 0x1234) & mask;
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) v[j] = key[j] != kEmpty ? t[s[j]] : kEmpty;
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      if (key[j] == kEmpty) continue;
      while (v[j] != key[j] && v[j] != kEmpty) {
        s[j] = (s[j] + 1) & mask;
        v[j] = t[s[j]];
      }
      hits += v[j] == key[j];
    }
  }
  atomicAdd(&g_hits, hits);
}

// scatter records to 256 partition lists (cursor per partition), lanes of one
// partition aggregated with match_any
__global__ void __launch_bounds__(256) k_scatter(const Rec* __restrict__ q, const uint8_t* __restrict__ part,
                                                 unsigned long long n, Rec* __restrict__ out,
                                                 unsigned long long* __restrict__ cursor) {
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i0 = blockIdx.x * (unsigned long long)blockDim.x; i0 < n; i0 += stride) {
    const unsigned long long i = i0 + threadIdx.x;
    const bool ok = i < n;
    Rec r;
    uint32_t p = 256 + (threadIdx.x & 31);
    if (ok) {
      r = q[i];
      p = part[i];
    }
    const unsigned m = __match_any_sync(0xffffffffu, p);
    const int leader = __ffs(m) - 1;
    const int pos = __popc(m & ((1u << (threadIdx.x & 31)) - 1));
    unsigned long long base = 0;
    if (ok && (int)(threadIdx.x & 31) == leader) base = atomicAdd(&cursor[p * 32], (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (ok) out[base + pos] = r;
  }
}

__global__ void k_hist(const uint8_t* __restrict__ part, unsigned long long n, unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    atomicAdd(&h[part[i]], 1u);
  __syncthreads();
  atomicAdd(&cnt[threadIdx.x * 32], (unsigned long long)h[threadIdx.x]);
}

int main(int argc, char** argv) {
  const int log2slots = argc > 1 ? atoi(argv[1]) : 30;
  const unsigned long long slots = 1ull << log2slots, mask = slots - 1;
  const unsigned long long nkeys = slots * 2 / 5;  // load 0.4
  const unsigned long long n = argc > 2 ? strtoull(argv[2], nullptr, 10) : (1ull << 28);
  unsigned long long *t, *cursor, *cnt;
  Rec *q, *q2;
  uint8_t *part, *part2;
  CK(cudaMalloc(&t, slots * 8));
  CK(cudaMalloc(&q, n * sizeof(Rec)));
  CK(cudaMalloc(&q2, n * sizeof(Rec)));
  CK(cudaMalloc(&part, n));
  CK(cudaMalloc(&part2, n));
  CK(cudaMalloc(&cursor, 256 * 32 * 8));
  CK(cudaMalloc(&cnt, 256 * 32 * 8));
  k_fill<<<4096, 256>>>(t, slots);
  k_insert<<<4096, 256>>>(t, mask, nkeys);
  k_queries<<<4096, 256>>>(q, part, n, nkeys, log2slots);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto report = [&](const char* what, double ms, double bytes) {
    printf("{\"what\": \"%s\", \"log2slots\": %d, \"n\": %llu, \"ms\": %.3f, \"G_per_s\": %.2f, \"GB_per_s\": %.1f}\n",
           what, log2slots, n, ms, n / ms / 1e6, bytes / ms / 1e6);
    fflush(stdout);
  };
  float ms;
  const int grid = 148 * 8;
  // direct probes, generation order
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_probe<4><<<grid, 256>>>(q, n, t, mask);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("direct_ilp4", ms, n * 16.0);
  }
  // CUB sort by partition (8-bit keys, 16-byte values)
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, part, part2, q, q2, (int64_t)n, 0, 8);
  void* tmp;
  CK(cudaMalloc(&tmp, tmp_bytes));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, part, part2, q, q2, (int64_t)n, 0, 8);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("cubsort_u8_rec16", ms, n * 34.0);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_probe<4><<<grid, 256>>>(q2, n, t, mask);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("sorted_probe_ilp4", ms, n * 16.0);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_probe<8><<<grid, 256>>>(q2, n, t, mask);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("sorted_probe_ilp8", ms, n * 16.0);
  }
  // scatter into partition lists (offsets from a histogram)
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemset(cnt, 0, 256 * 32 * 8));
    cudaEventRecord(e0);
    k_hist<<<grid, 256>>>(part, n, cnt);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("hist", ms, n * 1.0);
    unsigned long long h[256 * 32], c[256 * 32] = {0};
    CK(cudaMemcpy(h, cnt, sizeof(h), cudaMemcpyDeviceToHost));
    unsigned long long off = 0;
    for (int p = 0; p < 256; ++p) {
      c[p * 32] = off;
      off += h[p * 32];
    }
    CK(cudaMemcpy(cursor, c, sizeof(c), cudaMemcpyHostToDevice));
    cudaEventRecord(e0);
    k_scatter<<<grid * 4, 256>>>(q, part, n, q2, cursor);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("scatter_matchany", ms, n * 33.0);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_probe<8><<<grid, 256>>>(q2, n, t, mask);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) report("scattered_probe_ilp8", ms, n * 16.0);
  }
  unsigned long long hits;
  CK(cudaMemcpyFromSymbol(&hits, g_hits, 8));
  printf("{\"hits_total\": %llu}\n", hits);
  return 0;
}
