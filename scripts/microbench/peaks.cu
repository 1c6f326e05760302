// peaks.cu -- microbenchmarks of the B200 ceilings the REI roofline needs
// (VERDICT r01 "measure the denominators"):
//   * INT32 issue rates of the ALU pipe (LOP3, IADD3) and the FMA pipe (IMAD),
//     alone and mixed, in lane-ops per clock per SM;
//   * the rate of random 32-byte-sector reads from HBM (the dedup probe pattern)
//     over tables of 0.25-64 GiB, with and without a 32-byte L2 fetch granularity;
//   * the rate of random 64-bit atomicCAS (failing and succeeding) on such tables.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
// Prints one JSON object per measurement.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ unsigned long long g_sink;
__device__ unsigned long long g_clk[2];

__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("{ .reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3; }" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// MODE 0: 8 LOP3 chains; 1: 8 IADD3 chains; 2: 8 IMAD chains; 3: 4 LOP3 + 4 IMAD chains
template <int MODE>
__global__ void k_alu(int iters, uint32_t seed) {
  uint32_t x[8];
  const uint32_t t = threadIdx.x + blockIdx.x * blockDim.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = t * (i + 1) + seed;
  const uint32_t b = seed ^ 0x1234567u, c = seed * 3u + 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0) g_clk[0] = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) x[i] = lop3(x[i], b, c);
        else if (MODE == 1) x[i] = iadd3(x[i], b, c);
        else if (MODE == 2) x[i] = imad(x[i], b, c);
        else x[i] = (i & 1) ? imad(x[i], b, c) : lop3(x[i], b, c);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) g_clk[1] = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i];
  if (s == 0x7fffffffu) g_sink = s;
}

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// K independent random sector reads per lane per iteration; BYTES per read (8, 16, 32).
template <int K, int BYTES>
__global__ void k_gather(const unsigned long long* __restrict__ tab, unsigned long long nsect, int iters,
                         unsigned long long seed) {
  const unsigned long long t = threadIdx.x + (unsigned long long)blockIdx.x * blockDim.x;
  unsigned long long acc = 0, st = mix(t + seed);
  for (int it = 0; it < iters; ++it) {
    unsigned long long v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st = mix(st + k + 1);
      const unsigned long long* p = tab + (st & (nsect - 1)) * 4;
      if (BYTES == 4) {  // (label 4 = a plain 8-byte load, L1-allocating, like the hash probes)
        v[k] = *p;
      } else if (BYTES == 8) {
        v[k] = *(const volatile unsigned long long*)p;
      } else if (BYTES == 16) {
        const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(p);
        v[k] = q.x ^ q.y;
      } else {
        const ulonglong2 q0 = reinterpret_cast<const ulonglong2*>(p)[0];
        const ulonglong2 q1 = reinterpret_cast<const ulonglong2*>(p)[1];
        v[k] = q0.x ^ q0.y ^ q1.x ^ q1.y;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
    st += acc & 1;  // a data dependence so the loads cannot be hoisted past iterations
  }
  if (acc == 0x123456789ull) g_sink = acc;
}

// K random atomicCAS per lane per iteration; SUCCEED = the compare value matches
// (table holds 0 and we swap 0 -> 0, a real write), else it never matches.
template <int K, bool SUCCEED>
__global__ void k_cas(unsigned long long* tab, unsigned long long nslot, int iters, unsigned long long seed) {
  const unsigned long long t = threadIdx.x + (unsigned long long)blockIdx.x * blockDim.x;
  unsigned long long acc = 0, st = mix(t + seed);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st = mix(st + k + 1);
      acc += atomicCAS(tab + (st & (nslot - 1)), SUCCEED ? 0ull : ~0ull, 0ull);
    }
  }
  if (acc == 0x123456789ull) g_sink = acc;
}

// MODE 0: ld.global.cv (fetch again; defeats L2 hits); MODE 1: each CTA confined to its
// own window of `win` sectors (per-SM footprint small, whole-table footprint large).
template <int K, int MODE>
__global__ void k_gather2(const unsigned long long* __restrict__ tab, unsigned long long nsect,
                          unsigned long long win, int iters, unsigned long long seed) {
  const unsigned long long t = threadIdx.x + (unsigned long long)blockIdx.x * blockDim.x;
  const unsigned long long wbase = MODE == 1 ? ((mix(blockIdx.x + seed) % (nsect / win)) * win) : 0;
  unsigned long long acc = 0, st = mix(t + seed);
  for (int it = 0; it < iters; ++it) {
    unsigned long long v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st = mix(st + k + 1);
      const unsigned long long* p = tab + (MODE == 1 ? wbase + (st & (win - 1)) : (st & (nsect - 1))) * 4;
      if (MODE == 0) v[k] = __ldcv(p);
      else v[k] = *(const volatile unsigned long long*)p;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
    st += acc & 1;
  }
  if (acc == 0x123456789ull) g_sink = acc;
}

__global__ void k_fill(unsigned long long* p, size_t n) {
  for (size_t i = threadIdx.x + (size_t)blockIdx.x * blockDim.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0;
}

static int g_sms = 148;

template <class F>
static float time_ms(F launch, int reps = 3) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

template <int MODE>
static void run_alu(const char* name, int blocks_per_sm, int threads) {
  const int iters = 4096;
  const int grid = g_sms * blocks_per_sm;
  float ms = time_ms([&] { k_alu<MODE><<<grid, threads>>>(iters, 7); });
  unsigned long long clk[2];
  CK(cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk)));
  const double ops = (double)grid * threads * iters * 16 * 8;
  const double mhz = (double)(clk[1] - clk[0]) / (ms * 1e3);  // block 0's clock over the kernel
  printf("{\"test\": \"int_pipe\", \"op\": \"%s\", \"grid\": %d, \"block\": %d, \"ms\": %.3f, "
         "\"lane_ops_per_s\": %.4e, \"sm_mhz_est\": %.0f, \"lane_ops_per_clk_per_sm\": %.2f}\n",
         name, grid, threads, ms, ops / (ms * 1e-3), mhz, ops / (ms * 1e-3) / (mhz * 1e6) / g_sms);
}

template <int K, int BYTES>
static void run_gather(unsigned long long* tab, size_t bytes, int blocks_per_sm, bool fetch32) {
  CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, fetch32 ? 32 : 128));
  size_t got = 0;
  CK(cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity));
  const unsigned long long nsect = bytes / 32;
  const int grid = g_sms * blocks_per_sm, threads = 256, iters = 64;
  static unsigned long long seed = 1;
  float ms = time_ms([&] { k_gather<K, BYTES><<<grid, threads>>>(tab, nsect, iters, seed++); });
  const double reads = (double)grid * threads * iters * K;
  printf("{\"test\": \"random_sector_read\", \"table_gib\": %.2f, \"bytes_per_read\": %d, \"inflight_per_lane\": %d, "
         "\"ctas_per_sm\": %d, \"l2_fetch_granularity\": %zu, \"ms\": %.3f, \"reads_per_s\": %.4e, "
         "\"sector_gbs\": %.1f}\n",
         bytes / 1073741824.0, BYTES, K, blocks_per_sm, got, ms, reads / (ms * 1e-3),
         reads * 32 / (ms * 1e-3) / 1e9);
}

template <int K, bool SUCCEED>
static void run_cas(unsigned long long* tab, size_t bytes) {
  const unsigned long long nslot = bytes / 8;
  const int grid = g_sms * 8, threads = 256, iters = 16;
  static unsigned long long seed = 99;
  float ms = time_ms([&] { k_cas<K, SUCCEED><<<grid, threads>>>(tab, nslot, iters, seed++); });
  const double ops = (double)grid * threads * iters * K;
  printf("{\"test\": \"random_cas64\", \"table_gib\": %.2f, \"succeed\": %s, \"inflight_per_lane\": %d, "
         "\"ms\": %.3f, \"cas_per_s\": %.4e, \"sector_gbs\": %.1f}\n",
         bytes / 1073741824.0, SUCCEED ? "true" : "false", K, ms, ops / (ms * 1e-3), ops * 32 / (ms * 1e-3) / 1e9);
}

template <int K, int MODE>
static void run_gather2(const char* what, unsigned long long* tab, size_t bytes, size_t win_bytes) {
  const unsigned long long nsect = bytes / 32, win = win_bytes / 32;
  const int grid = g_sms * 8, threads = 256, iters = 64;
  static unsigned long long seed = 5;
  float ms = time_ms([&] { k_gather2<K, MODE><<<grid, threads>>>(tab, nsect, win, iters, seed++); });
  const double reads = (double)grid * threads * iters * K;
  printf("{\"test\": \"%s\", \"table_gib\": %.2f, \"window_mib\": %.1f, \"inflight_per_lane\": %d, "
         "\"ms\": %.3f, \"reads_per_s\": %.4e, \"sector_gbs\": %.1f}\n",
         what, bytes / 1073741824.0, win_bytes / 1048576.0, K, ms, reads / (ms * 1e-3),
         reads * 32 / (ms * 1e-3) / 1e9);
}

int main2() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  size_t freeb, totalb;
  CK(cudaMemGetInfo(&freeb, &totalb));
  size_t maxb = 64ull << 30;
  while (maxb > freeb * 8 / 10) maxb >>= 1;
  unsigned long long* tab;
  CK(cudaMalloc(&tab, maxb));
  k_fill<<<g_sms * 8, 256>>>(tab, maxb / 8);
  CK(cudaDeviceSynchronize());
  for (size_t b : {(size_t)256 << 20, (size_t)1 << 30, maxb}) run_gather2<8, 0>("random_read_cv", tab, b, b);
  for (size_t w : {(size_t)2 << 20, (size_t)16 << 20, (size_t)64 << 20, (size_t)256 << 20, (size_t)1 << 30, (size_t)4 << 30})
    run_gather2<8, 1>("random_read_cta_window", tab, maxb, w);
  CK(cudaFree(tab));
  return 0;
}

// One random 8-byte-read pass over the largest table (for an ncu capture of the DRAM
// bytes one random read really moves).
int main3() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  size_t freeb, totalb;
  CK(cudaMemGetInfo(&freeb, &totalb));
  size_t maxb = 16ull << 30;
  while (maxb > freeb * 8 / 10) maxb >>= 1;
  unsigned long long* tab;
  CK(cudaMalloc(&tab, maxb));
  k_fill<<<g_sms * 8, 256>>>(tab, maxb / 8);
  CK(cudaDeviceSynchronize());
  run_gather2<8, 0>("random_read_cv", tab, maxb, maxb);
  CK(cudaFree(tab));
  return 0;
}

// The random-read kernel variants once each, for an ncu capture of DRAM bytes per read:
// volatile 8-byte, plain 8-byte, 16-byte and 32-byte reads from a 16 GiB table.
int main4() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  size_t freeb, totalb;
  CK(cudaMemGetInfo(&freeb, &totalb));
  size_t maxb = 16ull << 30;
  while (maxb > freeb * 8 / 10) maxb >>= 1;
  unsigned long long* tab;
  CK(cudaMalloc(&tab, maxb));
  k_fill<<<g_sms * 8, 256>>>(tab, maxb / 8);
  CK(cudaDeviceSynchronize());
  run_gather<8, 8>(tab, maxb, 8, true);
  run_gather<8, 4>(tab, maxb, 8, true);
  run_gather<8, 16>(tab, maxb, 8, true);
  run_gather<8, 32>(tab, maxb, 8, true);
  CK(cudaFree(tab));
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == '2') return main2();
  if (argc > 1 && argv[1][0] == '3') return main3();
  if (argc > 1 && argv[1][0] == '4') return main4();
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d}\n", prop.name, g_sms, prop.l2CacheSize);

  run_alu<0>("lop3", 4, 512);
  run_alu<0>("lop3", 8, 256);
  run_alu<1>("iadd3(2x add)", 4, 512);
  run_alu<2>("imad", 4, 512);
  run_alu<3>("lop3+imad", 4, 512);
  run_alu<3>("lop3+imad", 8, 256);

  size_t freeb, totalb;
  CK(cudaMemGetInfo(&freeb, &totalb));
  size_t maxb = 64ull << 30;
  while (maxb > freeb * 8 / 10) maxb >>= 1;
  unsigned long long* tab;
  CK(cudaMalloc(&tab, maxb));
  k_fill<<<g_sms * 8, 256>>>(tab, maxb / 8);
  CK(cudaDeviceSynchronize());
  for (size_t b = 256ull << 20; b <= maxb; b *= 4) {
    run_gather<8, 8>(tab, b, 8, false);
    run_gather<8, 8>(tab, b, 8, true);
  }
  for (bool f32 : {false, true}) {
    run_gather<4, 8>(tab, maxb, 8, f32);
    run_gather<8, 8>(tab, maxb, 4, f32);
    run_gather<16, 8>(tab, maxb, 4, f32);
    run_gather<8, 16>(tab, maxb, 8, f32);
    run_gather<8, 32>(tab, maxb, 8, f32);
    run_gather<16, 32>(tab, maxb, 4, f32);
  }
  CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 128));
  const size_t big = maxb >= (32ull << 30) ? (32ull << 30) : maxb;
  run_cas<4, false>(tab, big);
  run_cas<4, true>(tab, big);
  run_cas<8, false>(tab, big);
  CK(cudaFree(tab));
  return 0;
}
