// csc.cuh — in-edge CSC of a directed graph (step a0 of SURVEY §8), built on the
// device without a library sort: a counting transpose.
//
//   1. in-degree histogram      cnt[v] = |{(u, v)}|          (one reduction per edge)
//   2. exclusive scan           in_off = scan(cnt), in_off[n] = m   (hand-written,
//                                                            tiles of 8192, recursive)
//   3. scatter                  in_tgt[cursor[v]++] = u      (warp per source u)
//   4. per-segment sort         each in-list ascending by source id (CSC order; the
//                                pull records take a vertex's first in-neighbours
//                                in this order, PAPER.md:1870-1874 scans them in it)
//        deg <= 16    one thread, a sorting network in registers
//        deg <= 1024  one warp, bitonic sort in shared memory
//        deg <= 8192  one CTA, bitonic sort in shared memory
//        larger       8192-element chunks sorted by CTAs, then merge passes (one CTA
//                     per hub, merge-path split of every pair of runs), ping-ponging
//                     through a buffer the size of the hubs' edges
//
// Device memory beyond the CSC itself: the cursor copy of in_off (8n bytes), the
// class lists and the hubs' merge buffer — about 4m + 8n bytes at most, against the
// 16m bytes of (target, source) keys a key sort needs.  Create-time only, never on
// a traversal's path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gbbs_csc {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER = 8;
constexpr long long SCAN_TILE = (long long)SCAN_THREADS * SCAN_PER;
constexpr int SMALL = 16;         // thread-sorted segments
constexpr int WARP_MAX = 1024;    // warp-sorted segments
constexpr int BLOCK_MAX = 8192;   // CTA-sorted segments (and hub chunks)
constexpr int SORT_WARPS = 8;     // warps per CTA of the warp-class kernel
constexpr int MERGE_THREADS = 512;

// 1. in-degree histogram (counts accumulate in the 64-bit words of in_off)
__global__ void k_indeg(const uint32_t *tgt, long long m, unsigned long long *cnt) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gs)
    atomicAdd(cnt + tgt[e], 1ull);
}

// 2. exclusive scan of a[0..len) in place; sums[b] = total of tile b
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile(long long *a, long long len,
                                                            long long *sums) {
  __shared__ long long wsum[SCAN_THREADS / 32];
  const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_PER;
  long long x[SCAN_PER];
  long long t = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER; i++) {
    x[i] = base + i < len ? a[base + i] : 0;
    t += x[i];
  }
  // exclusive scan of the thread totals: warp shuffles, then the warp sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long inc = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    long long s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  long long run = inc - t + (warp > 0 ? wsum[warp - 1] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_PER; i++) {
    if (base + i < len) a[base + i] = run;
    run += x[i];
  }
  if (threadIdx.x == SCAN_THREADS - 1) sums[blockIdx.x] = run;
}

__global__ void k_scan_add(long long *a, long long len, const long long *sums) {
  const long long add = sums[blockIdx.x];
  const long long base = (long long)blockIdx.x * SCAN_TILE;
  for (long long i = threadIdx.x; i < SCAN_TILE; i += blockDim.x)
    if (base + i < len) a[base + i] += add;
}

// 3. scatter: warp per source vertex, lanes over its out-edges
__global__ void k_scatter(const long long *off, const uint32_t *tgt, long long n,
                          unsigned long long *cur, uint32_t *in_tgt) {
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += nw) {
    const long long a = off[u], b = off[u + 1];
    for (long long e = a + lane; e < b; e += 32) {
      const unsigned long long pos = atomicAdd(cur + tgt[e], 1ull);
      in_tgt[pos] = (uint32_t)u;
    }
  }
}

// work lists of step 4 (device counters in ctr[0..3])
struct Item {
  long long start;  // first edge of the chunk / segment in in_tgt
  int len;
  int pad;
};
struct Hub {
  long long start;  // first edge of the segment in in_tgt
  long long len;
  long long tmp;    // its range in the merge buffer
};

// classify every vertex's in-list: warp class -> wl, CTA class and hub chunks ->
// items, hubs -> hubs (with a range of the merge buffer); counters:
// ctr[0] warp list, ctr[1] items, ctr[2] hubs, ctr[3] hub edges, ctr[4] max hub degree
__global__ void k_classify(const long long *in_off, long long n, uint32_t *wl, Item *items,
                           Hub *hubs, unsigned long long *ctr) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gs) {
    const long long a = in_off[v], d = in_off[v + 1] - a;
    if (d <= SMALL) continue;
    if (d <= WARP_MAX) {
      wl[atomicAdd(ctr, 1ull)] = (uint32_t)v;
      continue;
    }
    const long long nc = (d + BLOCK_MAX - 1) / BLOCK_MAX;
    const unsigned long long i0 = atomicAdd(ctr + 1, (unsigned long long)nc);
    for (long long c = 0; c < nc; c++) {
      items[i0 + c].start = a + c * BLOCK_MAX;
      items[i0 + c].len = (int)min((long long)BLOCK_MAX, d - c * BLOCK_MAX);
    }
    if (nc > 1) {
      const unsigned long long h = atomicAdd(ctr + 2, 1ull);
      hubs[h].start = a;
      hubs[h].len = d;
      hubs[h].tmp = (long long)atomicAdd(ctr + 3, (unsigned long long)d);
      atomicMax(ctr + 4, (unsigned long long)d);
    }
  }
}

// 4a. segments of 2..16 in-edges: one thread, bitonic network on 16 registers
__global__ void k_sort_small(const long long *in_off, long long n, uint32_t *in_tgt) {
  const long long gs = (long long)gridDim.x * blockDim.x;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gs) {
    const long long a = in_off[v];
    const int d = (int)(in_off[v + 1] - a);
    if (d < 2 || d > SMALL) continue;
    uint32_t x[SMALL];
#pragma unroll
    for (int i = 0; i < SMALL; i++) x[i] = i < d ? in_tgt[a + i] : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 2; k <= SMALL; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
        for (int i = 0; i < SMALL; i++) {
          const int l = i ^ j;
          if (l > i) {
            const bool up = (i & k) == 0;
            const uint32_t p = x[i], q = x[l];
            if ((p > q) == up) {
              x[i] = q;
              x[l] = p;
            }
          }
        }
#pragma unroll
    for (int i = 0; i < SMALL; i++)
      if (i < d) in_tgt[a + i] = x[i];
  }
}

// bitonic sort of s[0..P) (P a power of two) by `nt` cooperating threads (index t);
// SYNC() separates the steps
#define GBBS_BITONIC(s, P, t, nt, SYNC)                                     \
  for (int k_ = 2; k_ <= (P); k_ <<= 1)                                     \
    for (int j_ = k_ >> 1; j_ > 0; j_ >>= 1) {                              \
      for (int i_ = (t); i_ < (P) / 2; i_ += (nt)) {                        \
        const int lo_ = 2 * i_ - (i_ & (j_ - 1));                           \
        const int hi_ = lo_ + j_;                                           \
        const bool up_ = (lo_ & k_) == 0;                                   \
        const uint32_t p_ = (s)[lo_], q_ = (s)[hi_];                        \
        if ((p_ > q_) == up_) {                                             \
          (s)[lo_] = q_;                                                    \
          (s)[hi_] = p_;                                                    \
        }                                                                   \
      }                                                                     \
      SYNC;                                                                 \
    }

// 4b. segments of 17..1024 in-edges: one warp each
__global__ void __launch_bounds__(32 * SORT_WARPS) k_sort_warp(const long long *in_off,
                                                               const uint32_t *wl,
                                                               const unsigned long long *ctr,
                                                               uint32_t *in_tgt) {
  __shared__ uint32_t sm[SORT_WARPS][WARP_MAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *s = sm[warp];
  const long long cnt = (long long)ctr[0];
  const long long nw = (long long)gridDim.x * SORT_WARPS;
  for (long long i = (long long)blockIdx.x * SORT_WARPS + warp; i < cnt; i += nw) {
    const uint32_t v = wl[i];
    const long long a = in_off[v];
    const int d = (int)(in_off[v + 1] - a);
    int P = 32;
    while (P < d) P <<= 1;
    for (int k = lane; k < P; k += 32) s[k] = k < d ? in_tgt[a + k] : 0xFFFFFFFFu;
    __syncwarp();
    GBBS_BITONIC(s, P, lane, 32, __syncwarp());
    for (int k = lane; k < d; k += 32) in_tgt[a + k] = s[k];
    __syncwarp();
  }
}

// 4c. segments of 1025..8192 in-edges and the 8192-edge chunks of larger ones:
// one CTA per item
__global__ void __launch_bounds__(1024) k_sort_block(const Item *items,
                                                     const unsigned long long *ctr,
                                                     uint32_t *in_tgt) {
  __shared__ uint32_t s[BLOCK_MAX];
  const long long cnt = (long long)ctr[1];
  for (long long i = blockIdx.x; i < cnt; i += gridDim.x) {
    const long long a = items[i].start;
    const int d = items[i].len;
    int P = 1024;
    while (P < d) P <<= 1;
    for (int k = threadIdx.x; k < P; k += blockDim.x) s[k] = k < d ? in_tgt[a + k] : 0xFFFFFFFFu;
    __syncthreads();
    GBBS_BITONIC(s, P, (int)threadIdx.x, (int)blockDim.x, __syncthreads());
    for (int k = threadIdx.x; k < d; k += blockDim.x) in_tgt[a + k] = s[k];
    __syncthreads();
  }
}

// 4d. one merge pass over every hub: runs of width w in `from` are merged pairwise
// into `to` (merge path: thread t writes outputs [t*K, (t+1)*K) of each pair).
// from_tgt selects whether the source of this pass is in_tgt (else the buffer).
__global__ void __launch_bounds__(MERGE_THREADS) k_merge_pass(const Hub *hubs,
                                                              const unsigned long long *ctr,
                                                              uint32_t *in_tgt, uint32_t *buf,
                                                              long long w, int from_tgt) {
  const long long nh = (long long)ctr[2];
  for (long long h = blockIdx.x; h < nh; h += gridDim.x) {
    const long long len = hubs[h].len;
    const uint32_t *src = from_tgt ? in_tgt + hubs[h].start : buf + hubs[h].tmp;
    uint32_t *dst = from_tgt ? buf + hubs[h].tmp : in_tgt + hubs[h].start;
    for (long long s0 = 0; s0 < len; s0 += 2 * w) {
      const uint32_t *A = src + s0;
      const long long la = min(w, len - s0);
      const uint32_t *B = A + la;
      const long long lb = max(0ll, min(w, len - s0 - la));
      const long long tot = la + lb;
      const long long K = (tot + MERGE_THREADS - 1) / MERGE_THREADS;
      const long long k0 = min(tot, (long long)threadIdx.x * K), k1 = min(tot, k0 + K);
      if (k0 >= k1) continue;
      // merge path: smallest i in [max(0, k0 - lb), min(k0, la)] with A[i] > B[k0 - i - 1]
      long long lo = max(0ll, k0 - lb), hi = min(k0, la);
      while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (A[mid] <= B[k0 - mid - 1]) lo = mid + 1;
        else hi = mid;
      }
      long long i = lo, j = k0 - lo;
      for (long long k = k0; k < k1; k++) {
        if (j >= lb || (i < la && A[i] <= B[j])) dst[s0 + k] = A[i++];
        else dst[s0 + k] = B[j++];
      }
    }
  }
}

// copy every hub's segment from the buffer back into in_tgt (odd number of passes)
__global__ void k_hub_copyback(const Hub *hubs, const unsigned long long *ctr, uint32_t *in_tgt,
                               const uint32_t *buf) {
  const long long nh = (long long)ctr[2];
  for (long long h = blockIdx.x; h < nh; h += gridDim.x)
    for (long long k = threadIdx.x; k < hubs[h].len; k += blockDim.x)
      in_tgt[hubs[h].start + k] = buf[hubs[h].tmp + k];
}

// exclusive scan of a[0..len) in place (recursive over tile sums)
static cudaError_t scan_inplace(long long *a, long long len) {
  const long long nb = (len + SCAN_TILE - 1) / SCAN_TILE;
  long long *sums = nullptr;
  cudaError_t e = cudaMalloc(&sums, (size_t)(nb > 0 ? nb : 1) * 8);
  if (e != cudaSuccess) return e;
  k_scan_tile<<<(unsigned)nb, SCAN_THREADS>>>(a, len, sums);
  e = cudaGetLastError();
  if (e == cudaSuccess && nb > 1) {
    e = scan_inplace(sums, nb);
    if (e == cudaSuccess) {
      k_scan_add<<<(unsigned)nb, 256>>>(a, len, sums);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(sums);
  return e;
}

// in_off[0..n] and in_tgt[0..m) from the CSR (off, tgt); m > 0.  Every in-list ends
// up sorted by source id.
static cudaError_t build_csc(const long long *off, const uint32_t *tgt, long long n, long long m,
                             long long *in_off, uint32_t *in_tgt) {
  cudaError_t e = cudaMemset(in_off, 0, (size_t)(n + 1) * 8);
  if (e != cudaSuccess) return e;
  k_indeg<<<4736, 256>>>(tgt, m, reinterpret_cast<unsigned long long *>(in_off));
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = scan_inplace(in_off, n + 1)) != cudaSuccess) return e;

  unsigned long long *cur = nullptr, *ctr = nullptr;
  uint32_t *wl = nullptr, *buf = nullptr;
  Item *items = nullptr;
  Hub *hubs = nullptr;
  unsigned long long hc[5] = {0, 0, 0, 0, 0};
  // items: vertices above WARP_MAX in-edges (< m / WARP_MAX) plus hub chunks
  const long long max_items = m / WARP_MAX + m / (BLOCK_MAX / 2) + 2, max_hubs = m / BLOCK_MAX + 1;
  const long long max_wl = min(n, m / (SMALL + 1) + 1);
  do {
    if ((e = cudaMalloc(&cur, (size_t)n * 8)) != cudaSuccess) break;
    if ((e = cudaMemcpy(cur, in_off, (size_t)n * 8, cudaMemcpyDeviceToDevice)) != cudaSuccess) break;
    k_scatter<<<4736, 256>>>(off, tgt, n, cur, in_tgt);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) break;
    cudaFree(cur);
    cur = nullptr;

    if ((e = cudaMalloc(&ctr, 5 * 8)) != cudaSuccess) break;
    if ((e = cudaMemset(ctr, 0, 5 * 8)) != cudaSuccess) break;
    if ((e = cudaMalloc(&wl, (size_t)max_wl * 4)) != cudaSuccess) break;
    if ((e = cudaMalloc(&items, (size_t)max_items * sizeof(Item))) != cudaSuccess) break;
    if ((e = cudaMalloc(&hubs, (size_t)max_hubs * sizeof(Hub))) != cudaSuccess) break;
    k_classify<<<1184, 256>>>(in_off, n, wl, items, hubs, ctr);
    k_sort_small<<<1184, 256>>>(in_off, n, in_tgt);
    k_sort_warp<<<1184, 32 * SORT_WARPS>>>(in_off, wl, ctr, in_tgt);
    k_sort_block<<<592, 1024>>>(items, ctr, in_tgt);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if ((e = cudaMemcpy(hc, ctr, 5 * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) break;
    if (hc[2] == 0) break;
    if ((e = cudaMalloc(&buf, (size_t)hc[3] * 4)) != cudaSuccess) break;
    int from_tgt = 1;
    for (long long w = BLOCK_MAX; w < (long long)hc[4]; w <<= 1) {
      k_merge_pass<<<(unsigned)min(hc[2], 4096ull), MERGE_THREADS>>>(hubs, ctr, in_tgt, buf, w,
                                                                      from_tgt);
      from_tgt ^= 1;
    }
    if (!from_tgt) k_hub_copyback<<<(unsigned)min(hc[2], 4096ull), 256>>>(hubs, ctr, in_tgt, buf);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
  } while (0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(cur);
  cudaFree(ctr);
  cudaFree(wl);
  cudaFree(items);
  cudaFree(hubs);
  cudaFree(buf);
  return e;
}

}  // namespace gbbs_csc
