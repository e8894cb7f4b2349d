// Dev microbenchmarks (not product): grid-barrier cost and dependent-load latency on B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned long long *out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// sense-reversing barrier: one arrival atomic per CTA, thread 0 spins on a flag
__device__ __forceinline__ void my_sync(unsigned *count, volatile unsigned *gen, unsigned nb, unsigned &local_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g0 = local_gen;
    __threadfence();
    unsigned old = atomicAdd(count, 1);
    if (old == nb - 1) {
      *count = 0;
      __threadfence();
      atomicExch((unsigned *)gen, g0 + 1);
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen));
      } while (v == g0);
    }
    local_gen = g0 + 1;
  }
  __syncthreads();
}

__global__ void k_mysync(int iters, unsigned *count, unsigned *gen, unsigned long long *out) {
  unsigned lg = *((volatile unsigned *)gen);
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i++) my_sync(count, gen, gridDim.x, lg);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void k_chase(const uint32_t *next, int steps, unsigned long long *out, uint32_t *sink) {
  uint32_t i = 0;
  unsigned long long t0 = clock64();
  for (int s = 0; s < steps; s++) i = __ldcg(next + i);
  unsigned long long t1 = clock64();
  out[0] = t1 - t0;
  sink[0] = i;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned long long *d_out;
  cudaMalloc(&d_out, 64);
  unsigned *cnt, *gen;
  cudaMalloc(&cnt, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4);
  cudaMemset(gen, 0, 4);
  int iters = 2000;
  for (int per : {1, 2, 4}) {
    int G = nsm * per;
    void *args[] = {&iters, &d_out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void *)k_sync, G, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)k_sync, G, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cg grid.sync   G=%4d: %.3f us/sync\n", G, ms * 1e3 / iters);
    void *args2[] = {&iters, &cnt, &gen, &d_out};
    cudaLaunchCooperativeKernel((void *)k_mysync, G, 256, args2, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)k_mysync, G, 256, args2, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("custom barrier G=%4d: %.3f us/sync (err=%s)\n", G, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  // dependent-load latency: L2-resident (8 MB) and DRAM (2 GB) random chains
  for (size_t bytes : {(size_t)8 << 20, (size_t)2 << 30}) {
    size_t n = bytes / 4;
    std::vector<uint32_t> h(n);
    // random cycle with stride to defeat prefetch: i -> (i * 2654435761 + 12345) mod n over a permutation
    std::vector<uint32_t> perm(n);
    for (size_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    uint64_t s = 88172645463325252ull;
    for (size_t i = n - 1; i > 0; i--) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      size_t j = s % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    for (size_t i = 0; i < n; i++) h[perm[i]] = perm[(i + 1) % n];
    uint32_t *d, *sink;
    cudaMalloc(&d, bytes);
    cudaMalloc(&sink, 4);
    cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
    int steps = 20000;
    k_chase<<<1, 1>>>(d, steps, d_out, sink);
    k_chase<<<1, 1>>>(d, steps, d_out, sink);
    unsigned long long cyc;
    cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
    printf("chase %zu MB: %.1f cycles/load = %.3f us at %d MHz\n", bytes >> 20, (double)cyc / steps,
           (double)cyc / steps / (clk / 1000.0), clk / 1000);
    cudaFree(d);
  }
  return 0;
}
