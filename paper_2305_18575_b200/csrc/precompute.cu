// precompute.cu -- staged precompute on the device.
//
//  k_enum_keys : one thread per (example string, start offset): every infix
//                w = s[i:j] gets the shortlex key (|w| << 58) | value(w), value =
//                base-|Sigma| digits, first symbol most significant.
//  CUB radix sort + unique: IC(P u N) in shortlex order; epsilon (key 0) is word 0.
//  k_tables    : per IC word, its proper splits w = u v (u, v non-empty) found by
//                binary search of the prefix / suffix keys (the guide table,
//                P:839-845, with the two epsilon splits factored out); the P / N
//                masks and the seed CS of each alphabet symbol.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "rei_common.cuh"
#include "rei_host.h"

namespace rei {

namespace {

constexpr int kKeyShift = 58;

__device__ __forceinline__ unsigned long long key_len(unsigned long long key) { return key >> kKeyShift; }
__device__ __forceinline__ unsigned long long key_val(unsigned long long key) {
  return key & ((1ull << kKeyShift) - 1);
}

__device__ unsigned long long ipow(unsigned long long base, int e) {
  unsigned long long r = 1;
  for (int i = 0; i < e; ++i) r *= base;
  return r;
}

// Binary search of `key` in the sorted IC keys; -1 if absent.
__device__ int find_key(const unsigned long long* ic, int n, unsigned long long key) {
  int lo = 0, hi = n - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    unsigned long long v = ic[mid];
    if (v == key) return mid;
    if (v < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

// blockIdx.x = string, threadIdx.x = start offset i in [0, len].
__global__ void k_enum_keys(const uint8_t* __restrict__ syms, const uint32_t* __restrict__ str_off,
                            const uint32_t* __restrict__ str_len, const uint64_t* __restrict__ key_off,
                            int k, unsigned long long* __restrict__ keys,
                            unsigned long long* __restrict__ ex_keys) {
  const int s = blockIdx.x;
  const int m = (int)str_len[s];
  const int i = threadIdx.x;
  if (i > m) return;
  const uint8_t* w = syms + str_off[s];
  unsigned long long* out = keys + key_off[s] + (uint64_t)i * (m + 1) - (uint64_t)i * (i - 1) / 2;
  unsigned long long v = 0;
  out[0] = 0;  // the empty infix s[i:i]
  for (int j = i; j < m; ++j) {
    v = v * (unsigned long long)k + w[j];
    out[j - i + 1] = ((unsigned long long)(j - i + 1) << kKeyShift) | v;
  }
  if (i == 0) ex_keys[s] = out[m];  // the example itself (for the P / N masks)
}

struct TableOut {
  int n;
  int maxk;
  int maxlen;
  int bad;
  uint32_t pos[kMaxW32];
  uint32_t neg[kMaxW32];
};

// One CTA: thread t handles IC word t (and string t for the masks, symbol t for seeds).
__global__ void k_tables(const unsigned long long* __restrict__ ic, const int* __restrict__ n_ptr,
                         int k, uint32_t* __restrict__ split, uint32_t* __restrict__ nsplit,
                         uint32_t* __restrict__ word_len,
                         const unsigned long long* __restrict__ ex_keys, int nP, int nN,
                         uint32_t* __restrict__ seeds, int nsym, TableOut* __restrict__ out) {
  __shared__ int s_maxk, s_maxlen;
  __shared__ uint32_t s_pos[kMaxW32], s_neg[kMaxW32];
  const int n = *n_ptr;
  if (n > kMaxNW) {  // |IC| > 512: the host rejects the spec (REI_EINVAL); index no table
    if (threadIdx.x == 0) { out->n = n; out->maxk = 0; out->maxlen = 0; out->bad = 0; }
    return;
  }
  if (threadIdx.x == 0) { s_maxk = 0; s_maxlen = 0; }
  if (threadIdx.x < kMaxW32) { s_pos[threadIdx.x] = 0; s_neg[threadIdx.x] = 0; }
  __syncthreads();
  for (int w = threadIdx.x; w < kMaxNW; w += blockDim.x) {
    if (w >= n) { nsplit[w] = 0; word_len[w] = 0; continue; }
    const unsigned long long key = ic[w];
    const int m = (int)key_len(key);
    const unsigned long long V = key_val(key);
    int cnt = 0;
    for (int p = 1; p < m; ++p) {  // proper splits: |u| = p, |v| = m - p
      const unsigned long long d = ipow((unsigned long long)k, m - p);
      const unsigned long long ukey = ((unsigned long long)p << kKeyShift) | (V / d);
      const unsigned long long vkey = ((unsigned long long)(m - p) << kKeyShift) | (V % d);
      const int u = find_key(ic, n, ukey);
      const int v = find_key(ic, n, vkey);
      if (cnt < kMaxSplitRows) split[(size_t)cnt * kMaxNW + w] = ((uint32_t)u << 16) | (uint32_t)v;
      ++cnt;
    }
    nsplit[w] = (uint32_t)cnt;
    word_len[w] = (uint32_t)m;
    atomicMax(&s_maxk, cnt);
    atomicMax(&s_maxlen, m);
  }
  // masks: examples are whole IC words
  for (int e = threadIdx.x; e < nP + nN; e += blockDim.x) {
    const int idx = find_key(ic, n, ex_keys[e]);
    if (idx >= 0) {
      if (e < nP) atomicOr(&s_pos[idx >> 5], 1u << (idx & 31));
      else atomicOr(&s_neg[idx >> 5], 1u << (idx & 31));
    }
  }
  // seeds: CS(a) = {a} if a in IC, else the empty CS (reading A2)
  for (int a = threadIdx.x; a < nsym; a += blockDim.x) {
    const int idx = find_key(ic, n, (1ull << kKeyShift) | (unsigned long long)a);
    for (int q = 0; q < kMaxW32; ++q) seeds[a * kMaxW32 + q] = 0;
    if (idx >= 0) seeds[a * kMaxW32 + (idx >> 5)] = 1u << (idx & 31);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out->n = n;
    out->maxk = s_maxk;
    out->maxlen = s_maxlen;
    out->bad = (s_maxk > kMaxSplitRows) ? 1 : 0;
  }
  if (threadIdx.x < kMaxW32) { out->pos[threadIdx.x] = s_pos[threadIdx.x]; out->neg[threadIdx.x] = s_neg[threadIdx.x]; }
}

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e__ = (x);                                                  \
    if (e__ != cudaSuccess) { err = std::string(#x ": ") + cudaGetErrorString(e__); return false; } \
  } while (0)

}  // namespace

// Host launcher: strings are symbol ranks (0..k-1).  Fills dev tables in `t`.
bool run_precompute(const std::vector<std::vector<uint8_t>>& P, const std::vector<std::vector<uint8_t>>& N,
                    int k, cudaStream_t st, DeviceTables& t, std::string& err, uint64_t* launches) {
  std::vector<std::vector<uint8_t>> all(P);
  all.insert(all.end(), N.begin(), N.end());
  const int nstr = (int)all.size();
  std::vector<uint8_t> syms;
  std::vector<uint32_t> off, len;
  std::vector<uint64_t> koff;
  std::vector<unsigned long long> ex_keys;  // whole-example keys (marshalled with the strings)
  uint64_t total = 0;
  int maxlen = 0;
  for (auto& s : all) {
    off.push_back((uint32_t)syms.size());
    len.push_back((uint32_t)s.size());
    koff.push_back(total);
    const uint64_t m = s.size();
    total += (m + 1) * (m + 2) / 2;
    syms.insert(syms.end(), s.begin(), s.end());
    maxlen = std::max(maxlen, (int)m);
  }
  if (nstr == 0) { err = "empty specification"; return false; }
  if (syms.empty()) syms.push_back(0);

  uint8_t* d_syms = nullptr;
  uint32_t *d_off = nullptr, *d_len = nullptr;
  uint64_t* d_koff = nullptr;
  unsigned long long *d_keys = nullptr, *d_sorted = nullptr, *d_ex = nullptr;
  int* d_n = nullptr;
  void* d_tmp = nullptr;
  TableOut* d_out = nullptr;
  size_t tmp_sort = 0, tmp_uniq = 0;
  // CUB temp sizes first (size queries do not touch the buffers), then ONE scratch
  // block from the caching allocator (devmem.cu) carved into the precompute buffers
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, d_keys, d_sorted, (int)total, 0, 64, st);
  cub::DeviceSelect::Unique(nullptr, tmp_uniq, d_sorted, d_keys, d_n, (int)total, st);
  const size_t sizes[10] = {syms.size(), nstr * 4, nstr * 4, nstr * 8, total * 8, total * 8, sizeof(int),
                            sizeof(TableOut), nstr * 8, std::max(tmp_sort, tmp_uniq)};
  size_t offs[10], scratch_bytes = 0;
  for (int i = 0; i < 10; ++i) {
    offs[i] = scratch_bytes;
    scratch_bytes += (sizes[i] + 255) / 256 * 256;
  }
  void* scratch = nullptr;
  CK(dev_alloc(&scratch, scratch_bytes, st));
  auto at = [&](int i) { return static_cast<void*>(static_cast<char*>(scratch) + offs[i]); };
  d_syms = static_cast<uint8_t*>(at(0));
  d_off = static_cast<uint32_t*>(at(1));
  d_len = static_cast<uint32_t*>(at(2));
  d_koff = static_cast<uint64_t*>(at(3));
  d_keys = static_cast<unsigned long long*>(at(4));
  d_sorted = static_cast<unsigned long long*>(at(5));
  d_n = static_cast<int*>(at(6));
  d_out = static_cast<TableOut*>(at(7));
  d_ex = static_cast<unsigned long long*>(at(8));
  d_tmp = at(9);
  CK(cudaMemcpyAsync(d_syms, syms.data(), syms.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_off, off.data(), nstr * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_len, len.data(), nstr * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_koff, koff.data(), nstr * 8, cudaMemcpyHostToDevice, st));

  k_enum_keys<<<nstr, maxlen + 1, 0, st>>>(d_syms, d_off, d_len, d_koff, k, d_keys, d_ex);
  CK(cudaGetLastError());
  ++*launches;
  CK(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_sort, d_keys, d_sorted, (int)total, 0, 64, st));
  CK(cub::DeviceSelect::Unique(d_tmp, tmp_uniq, d_sorted, d_keys, d_n, (int)total, st));
  *launches += 4;  // CUB passes (approximate: histogram/onesweep/select)

  k_tables<<<1, 512, 0, st>>>(d_keys, d_n, k, t.split, t.nsplit, t.word_len, d_ex, (int)P.size(),
                              (int)N.size(), t.seeds, k, d_out);
  CK(cudaGetLastError());
  ++*launches;
  TableOut h{};
  CK(cudaMemcpyAsync(&h, d_out, sizeof(TableOut), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  t.n = h.n;
  t.maxk = h.maxk;
  t.maxlen = h.maxlen;
  for (int q = 0; q < kMaxW32; ++q) { t.pos[q] = h.pos[q]; t.neg[q] = h.neg[q]; }
  if (h.n > kMaxNW) { err = "|IC| > 512"; }
  if (h.bad) { err = "a word of IC has more than 64 proper splits"; }
  // keep the IC keys for introspection
  t.ic_keys.resize(h.n > 0 ? h.n : 0);
  if (h.n > 0)
    CK(cudaMemcpyAsync(t.ic_keys.data(), d_keys, (size_t)h.n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  dev_free(scratch, st);
  return err.empty();
}

}  // namespace rei
