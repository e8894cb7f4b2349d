// Dev microbenchmark (not product): sustained random-gather rate on B200, the
// ceiling of the per-edge probe in the Bellman-Ford / wBFS push (one random
// 2-byte shadow load per relaxed edge) and of the dense pull's bitmap probes.
//
// Each thread streams K coalesced uint32 indices (like targets[]) and gathers
// tab[idx] (uint16, like the shadow) for each, K loads in flight per thread;
// variants: table sizes (L2-resident 8 MB / 32 MB, HBM-sized 512 MB), K, CTAs
// per SM, and a relaxed atomicMin on a uint32 table instead of the load.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb tools/gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <vector>

template <int K, bool ATOM>
__global__ void k_gather(const uint32_t *idx, long long m, const uint16_t *tab, uint32_t *tab32,
                         unsigned long long *sink) {
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (long long base = gt; base < m; base += gs * K) {
    uint32_t ix[K];
#pragma unroll
    for (int j = 0; j < K; j++) {
      const long long e = base + (long long)j * gs;
      ix[j] = e < m ? __ldcs(idx + e) : 0u;
    }
    if (ATOM) {
#pragma unroll
      for (int j = 0; j < K; j++) acc += atomicMin(tab32 + ix[j], (uint32_t)j);
    } else {
      uint16_t v[K];
#pragma unroll
      for (int j = 0; j < K; j++) v[j] = __ldcg(tab + ix[j]);
#pragma unroll
      for (int j = 0; j < K; j++) acc += v[j];
    }
  }
  if (acc == 0xFFFFFFFFu) sink[0] = acc;
}

template <int K, bool ATOM>
static void run(const char *name, const uint32_t *idx, long long m, const uint16_t *tab,
                uint32_t *tab32, unsigned long long *sink, int ctas_per_sm) {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<K, ATOM><<<grid, 256>>>(idx, m, tab, tab32, sink);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    k_gather<K, ATOM><<<grid, 256>>>(idx, m, tab, tab32, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("%-28s K=%2d ctas/sm=%d : %7.1f G gathers/s (%.3f ms)\n", name, K, ctas_per_sm,
         m / (best * 1e-3) / 1e9, best);
}

int main() {
  const long long m = 1ll << 27;  // 128 M indices (512 MB stream)
  uint32_t *idx;
  cudaMalloc(&idx, m * 4);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  for (long long entries : {1ll << 22, 1ll << 24, 1ll << 28}) {  // 8 MB, 32 MB, 512 MB of uint16
    std::vector<uint32_t> h(m);
    unsigned long long x = 88172645463325252ull;
    for (long long i = 0; i < m; i++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[i] = (uint32_t)(x % (unsigned long long)entries);
    }
    cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    uint16_t *tab;
    uint32_t *tab32;
    cudaMalloc(&tab, entries * 2);
    cudaMalloc(&tab32, entries * 4);
    cudaMemset(tab, 1, entries * 2);
    cudaMemset(tab32, 0xFF, entries * 4);
    char nm[64];
    snprintf(nm, sizeof nm, "load u16 table %lld MB", entries * 2 >> 20);
    run<1, false>(nm, idx, m, tab, tab32, sink, 4);
    run<4, false>(nm, idx, m, tab, tab32, sink, 4);
    run<8, false>(nm, idx, m, tab, tab32, sink, 4);
    run<16, false>(nm, idx, m, tab, tab32, sink, 4);
    run<4, false>(nm, idx, m, tab, tab32, sink, 8);
    run<8, false>(nm, idx, m, tab, tab32, sink, 8);
    snprintf(nm, sizeof nm, "atomicMin u32 table %lld MB", entries * 4 >> 20);
    run<4, true>(nm, idx, m, tab, tab32, sink, 4);
    run<8, true>(nm, idx, m, tab, tab32, sink, 8);
    cudaFree(tab);
    cudaFree(tab32);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
