// gen.cu — HARNESS: device generators for the synthetic input graphs.
//
// Not part of the product and holds none of the method's arithmetic (no
// traversal, no relaxation): it builds CSR graphs bit-identical to the numpy
// generators in graphgen/__init__.py (same counter-based splitmix64 hash, same
// integer thresholds) for configs too large to build on the host, and labels
// connected components for source selection (reading A9).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdint>
#include <cstdio>
#include <string>

static thread_local std::string g_err;

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      char b_[256];                                                               \
      snprintf(b_, sizeof b_, "%s:%d %s: %s", __FILE__, __LINE__, #call,          \
               cudaGetErrorString(e_));                                           \
      g_err = b_;                                                                 \
      return -1;                                                                  \
    }                                                                             \
  } while (0)

extern "C" const char *gen_last_error(void) { return g_err.c_str(); }

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash64(uint64_t key, uint64_t ctr) {
  return mix64(key + (ctr + 1ull) * 0x9E3779B97F4A7C15ull);
}

static const uint64_t SENT = ~0ull;

// raw rMAT sample i -> key(s) (u << 32 | v); self-loops become SENT.
__global__ void k_rmat_keys(int levels, long long nedges, uint64_t key, uint64_t t1, uint64_t t2,
                            uint64_t t3, int symmetric, uint64_t *keys) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < nedges; i += gs) {
    uint64_t u = 0, v = 0;
    uint64_t base = (uint64_t)i * (uint64_t)levels;
    for (int l = 0; l < levels; l++) {
      uint64_t r = hash64(key, base + l) >> 32;
      uint64_t ub = r >= t2;
      uint64_t vb = (r >= t1 && r < t2) || r >= t3;
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    bool loop = u == v;
    if (symmetric) {
      keys[2 * i] = loop ? SENT : ((u << 32) | v);
      keys[2 * i + 1] = loop ? SENT : ((v << 32) | u);
    } else {
      keys[i] = loop ? SENT : ((u << 32) | v);
    }
  }
}

__global__ void k_unique_flags(const uint64_t *keys, long long cnt, uint32_t *flags) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < cnt; i += gs) {
    uint64_t k = keys[i];
    flags[i] = (k != SENT) && (i == 0 || keys[i - 1] != k);
  }
}

__global__ void k_scatter_unique(const uint64_t *keys, const uint32_t *flags, const long long *pos,
                                 long long cnt, uint32_t *targets, uint32_t *srcs) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < cnt; i += gs) {
    if (flags[i]) {
      uint64_t k = keys[i];
      targets[pos[i]] = (uint32_t)(k & 0xFFFFFFFFull);
      srcs[pos[i]] = (uint32_t)(k >> 32);
    }
  }
}

// offsets[x] = first index whose source is >= x (srcs sorted ascending).
__global__ void k_offsets_from_srcs(const uint32_t *srcs, long long n, long long m, long long *off) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < m; i += gs) {
    long long s = srcs[i];
    long long ps = (i == 0) ? -1 : (long long)srcs[i - 1];
    for (long long x = ps + 1; x <= s; x++) off[x] = i;
  }
  if (gt == 0) {
    long long last = (m == 0) ? -1 : (long long)srcs[m - 1];
    for (long long x = last + 1; x <= n; x++) off[x] = m;
  }
}

// Build the CSR of an rMAT graph (drop self-loops, optionally symmetrize, dedup,
// sort).  offsets: device int64[2^levels + 1]; targets: device uint32[cap],
// cap >= nedges * (symmetric ? 2 : 1).  *m_out = number of CSR edges.
extern "C" int gen_rmat_csr(int levels, long long nedges, uint64_t seed, uint64_t t1, uint64_t t2,
                            uint64_t t3, int symmetric, long long *offsets, uint32_t *targets,
                            long long cap, long long *m_out) {
  long long cnt = nedges * (symmetric ? 2 : 1);
  if (cap < cnt) {
    g_err = "targets capacity too small";
    return -1;
  }
  long long n = 1ll << levels;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  CK(cudaMalloc(&k0, (size_t)cnt * 8));
  CK(cudaMalloc(&k1, (size_t)cnt * 8));
  k_rmat_keys<<<4736, 256>>>(levels, nedges, mix64(seed), t1, t2, t3, symmetric, k0);
  CK(cudaGetLastError());
  cub::DoubleBuffer<uint64_t> db(k0, k1);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, cnt, 0, 64));
  void *tmp = nullptr;
  CK(cudaMalloc(&tmp, tb));
  CK(cub::DeviceRadixSort::SortKeys(tmp, tb, db, cnt, 0, 64));
  CK(cudaFree(tmp));
  uint64_t *sorted = db.Current();
  uint64_t *other = db.Alternate();
  // flags (uint32) and positions (int64) reuse the alternate key buffer + a new one
  uint32_t *flags = (uint32_t *)other;               // cnt * 4 bytes  <= cnt * 8
  long long *pos = nullptr;
  CK(cudaMalloc(&pos, (size_t)cnt * 8));
  k_unique_flags<<<4736, 256>>>(sorted, cnt, flags);
  CK(cudaGetLastError());
  tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, pos, cnt));
  CK(cudaMalloc(&tmp, tb));
  CK(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, pos, cnt));
  CK(cudaFree(tmp));
  long long lastpos = 0;
  uint32_t lastflag = 0;
  CK(cudaMemcpy(&lastpos, pos + cnt - 1, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&lastflag, flags + cnt - 1, 4, cudaMemcpyDeviceToHost));
  long long m = lastpos + lastflag;
  uint32_t *srcs = (uint32_t *)other + cnt;          // second half of the alternate buffer
  k_scatter_unique<<<4736, 256>>>(sorted, flags, pos, cnt, targets, srcs);
  CK(cudaGetLastError());
  k_offsets_from_srcs<<<4736, 256>>>(srcs, n, m, offsets);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaFree(pos);
  cudaFree(k0);
  cudaFree(k1);
  *m_out = m;
  return 0;
}

// 3D torus L^3, id = x + L*(y + L*z), 6 neighbours sorted ascending.
__global__ void k_torus(long long L, long long *off, uint32_t *tgt) {
  long long n = L * L * L;
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long v = gt; v < n; v += gs) {
    long long x = v % L, y = (v / L) % L, z = v / (L * L);
    long long nb[6];
    nb[0] = ((x + 1) % L) + L * (y + L * z);
    nb[1] = ((x + L - 1) % L) + L * (y + L * z);
    nb[2] = x + L * (((y + 1) % L) + L * z);
    nb[3] = x + L * (((y + L - 1) % L) + L * z);
    nb[4] = x + L * (y + L * ((z + 1) % L));
    nb[5] = x + L * (y + L * ((z + L - 1) % L));
    for (int i = 1; i < 6; i++)
      for (int j = i; j > 0 && nb[j - 1] > nb[j]; j--) {
        long long t = nb[j];
        nb[j] = nb[j - 1];
        nb[j - 1] = t;
      }
    off[v] = 6 * v;
    for (int i = 0; i < 6; i++) tgt[6 * v + i] = (uint32_t)nb[i];
    if (v == n - 1) off[n] = 6 * n;
  }
}

extern "C" int gen_torus_csr(long long L, long long *offsets, uint32_t *targets) {
  k_torus<<<4736, 256>>>(L, offsets, targets);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}

// w(u,v) = 1 + H(key, min<<32 | max) mod W, one warp per source vertex.
__global__ void k_pair_weights(const long long *off, const uint32_t *tgt, long long n, uint64_t key,
                               uint32_t W, uint32_t *w) {
  long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (long long u = warp; u < n; u += nw) {
    for (long long e = off[u] + lane; e < off[u + 1]; e += 32) {
      uint64_t v = tgt[e];
      uint64_t lo = v < (uint64_t)u ? v : (uint64_t)u;
      uint64_t hi = v < (uint64_t)u ? (uint64_t)u : v;
      w[e] = 1u + (uint32_t)(hash64(key, (lo << 32) | hi) % W);
    }
  }
}

extern "C" int gen_pair_weights(const long long *offsets, const uint32_t *targets, long long n,
                                uint64_t seed, uint32_t W, uint32_t *weights) {
  k_pair_weights<<<4736, 256>>>(offsets, targets, n, mix64(seed), W, weights);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}

// Connected components of a symmetric CSR by min-label hooking + pointer jumping.
__global__ void k_cc_init(uint32_t *lab, long long n) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long v = gt; v < n; v += (long long)gridDim.x * blockDim.x) lab[v] = (uint32_t)v;
}

__global__ void k_cc_hook(const long long *off, const uint32_t *tgt, long long n, uint32_t *lab,
                          int *changed) {
  long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (long long u = warp; u < n; u += nw) {
    uint32_t lu = lab[u];
    for (long long e = off[u] + lane; e < off[u + 1]; e += 32) {
      uint32_t lv = lab[tgt[e]];
      if (lu < lv) {
        atomicMin(lab + lv, lu);
        *changed = 1;
      } else if (lv < lu) {
        atomicMin(lab + lu, lv);
        *changed = 1;
      }
    }
  }
}

__global__ void k_cc_jump(uint32_t *lab, long long n) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long v = gt; v < n; v += (long long)gridDim.x * blockDim.x) {
    uint32_t l = lab[v];
    while (lab[l] != l) l = lab[l];
    lab[v] = l;
  }
}

extern "C" int gen_cc_labels(const long long *offsets, const uint32_t *targets, long long n,
                             uint32_t *labels) {
  int *dch = nullptr;
  CK(cudaMalloc(&dch, 4));
  k_cc_init<<<4736, 256>>>(labels, n);
  for (int it = 0; it < 10000; it++) {
    CK(cudaMemset(dch, 0, 4));
    k_cc_hook<<<4736, 256>>>(offsets, targets, n, labels, dch);
    k_cc_jump<<<4736, 256>>>(labels, n);
    int ch = 0;
    CK(cudaMemcpy(&ch, dch, 4, cudaMemcpyDeviceToHost));
    if (!ch) break;
  }
  CK(cudaDeviceSynchronize());
  cudaFree(dch);
  return 0;
}
