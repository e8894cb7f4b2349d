// gbbs.cu — libgbbs: the C ABI declared in include/gbbs.h.
//
// Host side of the library: graph residency (copy/borrow, device validation,
// in-edge CSC by a hand-written counting transpose, csc.cuh), per-handle scratch, and the launch of the
// persistent traversal kernel (traverse.cuh) for gbbs_bfs / gbbs_bellman_ford.
// No torch types, no exceptions across the ABI, no CPU fallback: every step of
// a traversal runs in the kernels of this file and traverse.cuh.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gbbs.h"
#include "traverse.cuh"
#include "csc.cuh"
#include "sbf.cuh"

using namespace gbbs_dev;

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? GBBS_ENOMEM : GBBS_ECUDA;    \
      return fail(code_, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    }                                                                              \
  } while (0)

extern "C" const char *gbbs_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// the handle
// ---------------------------------------------------------------------------
// control words per traversal scratch: packed counter ring [4], status, rounds,
// count, -, heavy-list counters [2], work queues [8], acquisition ring [4]
constexpr int CNT_WORDS = 22;

struct gbbs_graph {
  int device = 0;
  long long n = 0, m = 0;
  uint32_t flags = 0;
  int ebits = 1;
  uint32_t maxw = 1, minw = 1;
  long long *off = nullptr;
  uint32_t *tgt = nullptr;
  uint32_t *wgt = nullptr;
  bool own_off = true, own_tgt = true, own_wgt = true;
  uint4 *phot = nullptr;     // pull records: (in0, in1, in2, out-degree)
  uint4 *pcold = nullptr;    //               (in3, in4, tail)
  uint2 *phot8 = nullptr;    // GBBS_REC8 layout (traverse.cuh Params)
  uint4 *pc32 = nullptr;
  uint32_t *nin = nullptr;   // no-in-edge mask (+ padding)
  long long ncand = 0;       // vertices with at least one in-edge
  uint16_t *shadow = nullptr;  // 16-bit distance shadow (BF / widest path)
  long long *in_off = nullptr;  // alias of off when symmetric
  uint32_t *in_tgt = nullptr;
  // scratch
  uint32_t *bm[2] = {nullptr, nullptr};
  uint32_t *fv[3] = {nullptr, nullptr, nullptr};  // round lists 0/1, heavy list 2
  long long *fo[3] = {nullptr, nullptr, nullptr};
  long long *fb[3] = {nullptr, nullptr, nullptr};
  uint32_t *iso = nullptr;
  unsigned long long *cnt = nullptr;  // [4] + ctrl
  int *status = nullptr;
  long long *rounds = nullptr;
  uint32_t *tmp_dist = nullptr, *tmp_parent = nullptr;  // for host outputs
  uint32_t *bst[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // batch staging [buf][dist/parent]
  cudaStream_t cstream = nullptr;    // batch: device->host copy stream
  cudaEvent_t cev[2] = {nullptr, nullptr};  // batch: copy of buffer b done
  cudaEvent_t kev[2] = {nullptr, nullptr};  // batch: traversal into buffer b done
  long long *bstat = nullptr;        // batch: per-traversal (status, rounds) slots
  long long bstat_cap = 0;
  struct TeamScratch *team[8] = {};  // batch teams 1..7
  unsigned *bar0 = nullptr;          // team 0's barrier words
  int mg_grid[3] = {0, 0, 0};        // co-resident CTAs of traverse_mg_kernel<ALGO>
  int wb_mg_grid = 0;                // co-resident CTAs of wbfs_mg_kernel
  RoundStat *dstats = nullptr;
  long long dstats_cap = 0;
  unsigned long long *dcount = nullptr;
  long long nwords = 0;
  int grid[3][2] = {{0, 0}, {0, 0}, {0, 0}};  // [algo][stats]
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct BcScratch *bc = nullptr;  // betweenness scratch (lazy)
  struct WbfsScratch *wb = nullptr;  // wBFS bucket structure (lazy)
  long long *tmp_sdist = nullptr;    // signed BF: int64 staging for host outputs
  long long smaxabs = -1;            // signed BF: max |w| of the weights read as int32
  int sgrid[2] = {0, 0};
};

// Every entry point that touches a handle runs on the handle's device and restores
// the caller's current device on return (PyTorch and other callers keep theirs).
struct DeviceGuard {
  int prev = -1;
  int rc = GBBS_OK;
  explicit DeviceGuard(int want) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (prev != want) {
      const cudaError_t e = cudaSetDevice(want);
      if (e != cudaSuccess) rc = fail(GBBS_ECUDA, "cudaSetDevice(%d): %s", want, cudaGetErrorString(e));
    }
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;
};

static void free_bc(gbbs_graph *g);
static void free_wbfs(gbbs_graph *g);
static void free_teams(gbbs_graph *g);

static void free_graph(gbbs_graph *g) {
  if (!g) return;
  if (g->own_off) cudaFree(g->off);
  if (g->own_tgt) cudaFree(g->tgt);
  if (g->own_wgt) cudaFree(g->wgt);
  cudaFree(g->phot);
  cudaFree(g->pcold);
  cudaFree(g->phot8);
  cudaFree(g->pc32);
  cudaFree(g->nin);
  cudaFree(g->shadow);
  if (g->in_off && g->in_off != g->off) cudaFree(g->in_off);
  if (g->in_tgt && g->in_tgt != g->tgt) cudaFree(g->in_tgt);
  for (int i = 0; i < 3; i++) {
    if (i < 2) cudaFree(g->bm[i]);
    cudaFree(g->fv[i]);
    cudaFree(g->fo[i]);
    cudaFree(g->fb[i]);
  }
  cudaFree(g->cnt);
  cudaFree(g->iso);
  cudaFree(g->tmp_dist);
  cudaFree(g->tmp_parent);
  for (int i = 0; i < 2; i++) {
    cudaFree(g->bst[i][0]);
    cudaFree(g->bst[i][1]);
    if (g->cev[i]) cudaEventDestroy(g->cev[i]);
    if (g->kev[i]) cudaEventDestroy(g->kev[i]);
  }
  if (g->cstream) cudaStreamDestroy(g->cstream);
  cudaFree(g->bstat);
  cudaFree(g->dstats);
  if (g->ev[0]) cudaEventDestroy(g->ev[0]);
  if (g->ev[1]) cudaEventDestroy(g->ev[1]);
  free_bc(g);
  free_wbfs(g);
  free_teams(g);
  cudaFree(g->tmp_sdist);
  delete g;
}

// ---------------------------------------------------------------------------
// create-time kernels (a0): validation, max weight, CSC construction
// ---------------------------------------------------------------------------
__global__ void k_validate(const long long *off, const uint32_t *tgt, long long n, long long m,
                           unsigned long long *bad) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  for (long long i = gt; i < n; i += gs)
    if (off[i] > off[i + 1]) atomicOr(bad, 1ull);
  for (long long e = gt; e < m; e += gs)
    if (tgt[e] >= (unsigned long long)n) atomicOr(bad, 2ull);
}

// out[0] = max weight, out[1] = min weight (out[1] preset to 0xFFFFFFFF)
__global__ void k_maxw(const uint32_t *w, long long m, unsigned int *out) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  uint32_t mx = 0, mn = 0xFFFFFFFFu;
  for (long long e = gt; e < m; e += gs) {
    mx = max(mx, w[e]);
    mn = min(mn, w[e]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    atomicMin(out + 1, mn);
  }
}

// max |w| over the weights read as int32 (signed Bellman-Ford range check)
__global__ void k_absmax_i32(const uint32_t *w, long long m, unsigned long long *out) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  unsigned long long mx = 0;
  for (long long e = gt; e < m; e += gs) {
    const long long x = (long long)(int32_t)w[e];
    mx = max(mx, (unsigned long long)(x < 0 ? -x : x));
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

// bit v set iff out-degree(v) > WBFS_HEAVY (wBFS: insertions count the hubs of a bucket)
__global__ void k_heavy_bits(const long long *off, long long n, long long nwords, uint32_t *hv) {
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((v >> 5) >= nwords) return;
  const bool h = v < n && off[v + 1] - off[v] > WBFS_HEAVY;
  const unsigned b = __ballot_sync(0xffffffffu, h);
  if ((threadIdx.x & 31) == 0) hv[v >> 5] = b;
}

// Bit v of word v/32 set iff v has no in- and no out-edges (or v >= n, padding):
// such vertices can never be reached nor be anyone's in-neighbour, so BFS starts
// with them marked visited and dense rounds skip them.
__global__ void k_isolated(const long long *off, const long long *in_off, long long n,
                           long long nwords, uint32_t *iso) {
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((v >> 5) >= nwords) return;
  bool z = true;
  if (v < n) z = off[v] == off[v + 1] && in_off[v] == in_off[v + 1];
  unsigned b = __ballot_sync(0xffffffffu, z);
  if ((threadIdx.x & 31) == 0) iso[v >> 5] = b;
}

// Pull records and the no-in-edge mask (a8).  The early-exit pull
// examines v's in-edges in CSC order and stops at the first visited one; on rMAT
// almost every candidate stops within its first few in-edges (sorted by source,
// the hubs come first), so those are stored inline and a candidate is decided
// without first loading its in-offsets and then its in-edges (two dependent HBM
// round trips per candidate):
//   hot[v]  = (in0, in1, in2, out-degree)   16 B, read for every candidate
//   cold[v] = (in3, in4, tail)              16 B, read only when in0..in2 miss
// where in_k is v's k-th in-neighbour in CSC order (INF past the in-degree) and
// tail = (in_off[v] + 5) << 24 | min(indeg - 5, 2^24 - 1) (0 if indeg <= 5; a
// saturated count means: read in_off[v + 1]).  Same edges, same order, same
// early exit as scanning in_tgt from in_off[v].  Bit v of nin is set iff v has no
// in-edges (or v >= n): such a vertex can never be acquired by a pull, so dense
// rounds do not sweep it (it cannot be marked visited instead: visited vertices
// act as the frontier, reading R2).  *ncand counts the others.
__global__ void k_pull_records(const long long *off, const long long *in_off,
                               const uint32_t *in_tgt, long long n, long long nwords, uint4 *hot,
                               uint4 *cold, uint32_t *nin, unsigned long long *ncand,
                               uint2 *hot8, uint4 *c32) {
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((v >> 5) >= nwords) return;
  bool none = true;
  if (v < n) {
    const long long a = in_off[v], b = in_off[v + 1];
    const long long od = off[v + 1] - off[v];
    const long long d = b - a;
    none = d == 0;
    uint32_t x[5];
    for (int k = 0; k < 5; k++) x[k] = k < d ? in_tgt[a + k] : INF;
    const unsigned long long tail =
        d > 5 ? ((unsigned long long)(a + 5) << 24) | (unsigned long long)min(d - 5, 0xFFFFFFll) : 0ull;
    if (hot8) {
      const uint32_t od31 = (uint32_t)min(od, 0x7FFFFFFFll);
      hot8[v] = make_uint2(x[0], od31 | (d > 1 ? 0x80000000u : 0u));
      c32[2 * v] = make_uint4(x[1], x[2], x[3], x[4]);
      c32[2 * v + 1] = make_uint4((uint32_t)(tail & 0xFFFFFFFFull), (uint32_t)(tail >> 32), od31, 0u);
    } else {
      hot[v] = make_uint4(x[0], x[1], x[2], (uint32_t)min(od, 0xFFFFFFFFll));
      cold[v] = make_uint4(x[3], x[4], (uint32_t)(tail & 0xFFFFFFFFull), (uint32_t)(tail >> 32));
    }
  }
  const unsigned bb = __ballot_sync(0xffffffffu, none);
  if ((threadIdx.x & 31) == 0) {
    nin[v >> 5] = bb;
    atomicAdd(ncand, (unsigned long long)(32 - __popc(bb)));
  }
}

static int bits_for(unsigned long long x) {  // bits needed to represent x (>= 1)
  int b = 1;
  while (b < 64 && (x >> b) != 0) b++;
  return b;
}

static bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static int ensure_device_ok(int *dev_out) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    return fail(GBBS_ECUDA, "libgbbs is built for sm_100a (B200); device %d is sm_%d%d", dev,
                prop.major, prop.minor);
  int coop = 0;
  CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return fail(GBBS_ECUDA, "device %d lacks cooperative launch", dev);
  *dev_out = dev;
  return GBBS_OK;
}

template <int ALGO, bool STATS, bool PM = false>
static int occupancy_grid(int *grid) {
  int dev = 0, nsm = 0, per = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, traverse_kernel<ALGO, STATS, PM>, BLOCK, 0));
  if (per < 1) return fail(GBBS_ECUDA, "traverse kernel cannot be resident");
  *grid = per * nsm;
  return GBBS_OK;
}

// pad: extra bytes allocated past the copy (the in-edge group loads of a8)
static int copy_in(void **dst, const void *src, size_t bytes, size_t pad = 0) {
  CU(cudaMalloc(dst, bytes + pad ? bytes + pad : 16));
  if (bytes) CU(cudaMemcpy(*dst, src, bytes, cudaMemcpyDefault));
  return GBBS_OK;
}

static int create_impl(long long n, long long m, const int64_t *offsets, const uint32_t *targets,
                       const uint32_t *weights, uint32_t flags, gbbs_graph *g) {
  int rc;
  if ((rc = ensure_device_ok(&g->device))) return rc;
  g->n = n;
  g->m = m;
  g->flags = flags;
  g->ebits = bits_for((unsigned long long)m);
  if (g->ebits + bits_for((unsigned long long)n) > 64)
    return fail(GBBS_ERANGE, "bits(n)+bits(m) > 64: frontier counter cannot be packed");

  const bool borrow = flags & GBBS_BORROW;
  if (borrow) {
    if (!is_device_ptr(offsets) || (m > 0 && !is_device_ptr(targets)) ||
        (weights && !is_device_ptr(weights)))
      return fail(GBBS_EINVAL, "GBBS_BORROW requires device pointers");
    g->own_off = g->own_tgt = g->own_wgt = false;
    g->off = (long long *)offsets;
    g->tgt = (uint32_t *)targets;
    g->wgt = (uint32_t *)weights;
    // dense rounds read in-edges with 16-byte vector loads of aligned groups of
    // 4 (the last group may extend up to 12 bytes past targets[m - 1]: see
    // GBBS_BORROW in gbbs.h): copy a misaligned array
    if (((uintptr_t)targets & 15) != 0) {
      g->tgt = nullptr;
      g->own_tgt = true;
      if ((rc = copy_in((void **)&g->tgt, targets, (size_t)m * 4, 16))) return rc;
    }
    if (weights && ((uintptr_t)weights & 15) != 0) {  // same for the weights (list-push groups)
      g->wgt = nullptr;
      g->own_wgt = true;
      if ((rc = copy_in((void **)&g->wgt, weights, (size_t)m * 4, 16))) return rc;
    }
  } else {
    if ((rc = copy_in((void **)&g->off, offsets, (size_t)(n + 1) * 8))) return rc;
    if ((rc = copy_in((void **)&g->tgt, targets, (size_t)m * 4, 16))) return rc;
    if (weights && (rc = copy_in((void **)&g->wgt, weights, (size_t)m * 4, 16))) return rc;
  }
  // endpoints
  long long o0 = -1, on = -1;
  CU(cudaMemcpy(&o0, g->off, 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&on, g->off + n, 8, cudaMemcpyDeviceToHost));
  if (o0 != 0) return fail(GBBS_EINVAL, "offsets[0] = %lld, expected 0", o0);
  if (on != m) return fail(GBBS_EINVAL, "offsets[n] = %lld, expected m = %lld", on, m);

  unsigned long long *dscratch = nullptr;
  CU(cudaMalloc(&dscratch, 16));
  CU(cudaMemset(dscratch, 0, 16));
  if (!(flags & GBBS_NO_VALIDATE)) {
    k_validate<<<1184, 256>>>(g->off, g->tgt, n, m, dscratch);
    CU(cudaGetLastError());
    unsigned long long bad = 0;
    CU(cudaMemcpy(&bad, dscratch, 8, cudaMemcpyDeviceToHost));
    if (bad) {
      cudaFree(dscratch);
      return fail(GBBS_EINVAL, "invalid CSR:%s%s", (bad & 1) ? " decreasing offsets" : "",
                  (bad & 2) ? " target >= n" : "");
    }
  }
  g->maxw = g->minw = 1;
  if (g->wgt && m > 0) {
    unsigned int *mx = (unsigned int *)(dscratch + 1);
    CU(cudaMemset(mx + 1, 0xFF, 4));
    k_maxw<<<1184, 256>>>(g->wgt, m, mx);
    CU(cudaGetLastError());
    CU(cudaMemcpy(&g->maxw, mx, 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&g->minw, mx + 1, 4, cudaMemcpyDeviceToHost));
  }
  cudaFree(dscratch);

  // in-edge CSC for pull rounds
  if (flags & GBBS_SYMMETRIC) {
    g->in_off = g->off;
    g->in_tgt = g->tgt;
  } else {
    CU(cudaMalloc(&g->in_off, (size_t)(n + 1) * 8));
    CU(cudaMalloc(&g->in_tgt, (size_t)(m ? m : 1) * 4 + 16));  // + the group loads' pad
    if (m == 0) {
      CU(cudaMemset(g->in_off, 0, (size_t)(n + 1) * 8));
    } else {
      const cudaError_t e2 = gbbs_csc::build_csc(g->off, g->tgt, n, m, g->in_off, g->in_tgt);
      if (e2 != cudaSuccess)
        return fail(e2 == cudaErrorMemoryAllocation ? GBBS_ENOMEM : GBBS_ECUDA, "CSC build: %s",
                    cudaGetErrorString(e2));
    }
  }

  // per-handle scratch
  g->nwords = (n + 31) / 32;
  for (int i = 0; i < 2; i++) {
    CU(cudaMalloc(&g->bm[i], (size_t)g->nwords * 4));
    CU(cudaMemset(g->bm[i], 0, (size_t)g->nwords * 4));
  }
  for (int i = 0; i < 3; i++) {
    CU(cudaMalloc(&g->fv[i], (size_t)n * 4));
    CU(cudaMalloc(&g->fo[i], (size_t)n * 8));
    CU(cudaMalloc(&g->fb[i], (size_t)n * 8));
  }
  CU(cudaMalloc(&g->shadow, (size_t)n * 2));
  CU(cudaMalloc(&g->iso, (size_t)g->nwords * 4));
  k_isolated<<<(unsigned)((g->nwords * 32 + 255) / 256), 256>>>(g->off, g->in_off, n, g->nwords, g->iso);
  CU(cudaGetLastError());
  CU(cudaMalloc(&g->cnt, CNT_WORDS * 8));  // ring[4], status, rounds, count, -, heavy[2], wq[8], acq[4]
  CU(cudaMemset(g->cnt, 0, CNT_WORDS * 8));
  if (GBBS_REC8) {
    CU(cudaMalloc(&g->phot8, (size_t)n * 8));
    CU(cudaMalloc(&g->pc32, (size_t)n * 32));
  } else {
    CU(cudaMalloc(&g->phot, (size_t)n * 16));
    CU(cudaMalloc(&g->pcold, (size_t)n * 16));
  }
  CU(cudaMalloc(&g->nin, (size_t)g->nwords * 4));
  k_pull_records<<<(unsigned)((g->nwords * 32 + 255) / 256), 256>>>(
      g->off, g->in_off, g->in_tgt, n, g->nwords, g->phot, g->pcold, g->nin, g->cnt + 6, g->phot8,
      g->pc32);
  CU(cudaGetLastError());
  CU(cudaMemcpy(&g->ncand, g->cnt + 6, 8, cudaMemcpyDeviceToHost));
  g->status = (int *)(g->cnt + 4);
  g->rounds = (long long *)(g->cnt + 5);
  g->dcount = g->cnt + 6;
  if ((rc = occupancy_grid<ALGO_BFS, false>(&g->grid[0][0]))) return rc;
  if ((rc = occupancy_grid<ALGO_BFS, true>(&g->grid[0][1]))) return rc;
  if ((rc = occupancy_grid<ALGO_BF, false>(&g->grid[1][0]))) return rc;
  if ((rc = occupancy_grid<ALGO_BF, true>(&g->grid[1][1]))) return rc;
  if ((rc = occupancy_grid<ALGO_WP, false>(&g->grid[2][0]))) return rc;
  if ((rc = occupancy_grid<ALGO_WP, true>(&g->grid[2][1]))) return rc;
  CU(cudaDeviceSynchronize());
  return GBBS_OK;
}

extern "C" int gbbs_graph_create(int64_t n, int64_t m, const int64_t *offsets,
                                 const uint32_t *targets, const uint32_t *weights,
                                 uint32_t flags, gbbs_graph **out) {
  g_last_error.clear();
  if (!out) return fail(GBBS_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > (int64_t)0xFFFFFFFEll) return fail(GBBS_EINVAL, "n = %lld out of [1, 2^32-2]", (long long)n);
  if (m < 0) return fail(GBBS_EINVAL, "m < 0");
  if (!offsets || (m > 0 && !targets)) return fail(GBBS_EINVAL, "NULL offsets/targets");
  if (flags & ~(uint32_t)(GBBS_SYMMETRIC | GBBS_BORROW | GBBS_NO_VALIDATE))
    return fail(GBBS_EINVAL, "unknown flags 0x%x", flags);
  gbbs_graph *g = new (std::nothrow) gbbs_graph();
  if (!g) return fail(GBBS_ENOMEM, "host allocation");
  int rc = create_impl(n, m, offsets, targets, weights, flags, g);
  if (rc != GBBS_OK) {
    free_graph(g);
    return rc;
  }
  *out = g;
  return GBBS_OK;
}

extern "C" void gbbs_graph_destroy(gbbs_graph *g) {
  if (!g) return;
  DeviceGuard dguard(g->device);
  free_graph(g);
}

extern "C" int gbbs_graph_info(const gbbs_graph *g, int64_t *n, int64_t *m, uint32_t *flags) {
  if (!g) return fail(GBBS_EINVAL, "g is NULL");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (flags) *flags = g->flags;
  return GBBS_OK;
}

extern "C" void gbbs_default_opts(gbbs_opts *o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->threshold_den = 20;
  o->mode = GBBS_MODE_AUTO;
}

extern "C" int gbbs_graph_in_edges(const gbbs_graph *g, int64_t *in_offsets,
                                   uint32_t *in_sources) {
  if (!g) return fail(GBBS_EINVAL, "g is NULL");
  int prev = 0;
  CU(cudaGetDevice(&prev));
  CU(cudaSetDevice(g->device));
  cudaError_t e = cudaSuccess;
  if (in_offsets)
    e = cudaMemcpy(in_offsets, g->in_off, (size_t)(g->n + 1) * 8, cudaMemcpyDefault);
  if (e == cudaSuccess && in_sources && g->m > 0)
    e = cudaMemcpy(in_sources, g->in_tgt, (size_t)g->m * 4, cudaMemcpyDefault);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(GBBS_ECUDA, "in-edge copy: %s", cudaGetErrorString(e));
  return GBBS_OK;
}

extern "C" int gbbs_launch_info(const gbbs_graph *g, int32_t *ctas, int32_t *threads) {
  if (!g) return fail(GBBS_EINVAL, "g is NULL");
  if (ctas) *ctas = g->grid[0][0];
  if (threads) *threads = BLOCK;
  return GBBS_OK;
}

// ---------------------------------------------------------------------------
// traversal driver
// ---------------------------------------------------------------------------
__global__ void k_count_reached(const uint32_t *dist, long long n, unsigned long long *out) {
  long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long gs = (long long)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (long long i = gt; i < n; i += gs) c += dist[i] != INF;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

template <int ALGO, bool STATS, bool PM = false>
static int launch(gbbs_graph *g, Params &p, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1,
                  unsigned ctas_per_sm) {
  void *args[] = {&p};
  int grid = g->grid[ALGO][STATS];
  if constexpr (PM) {
    int rc;
    if ((rc = occupancy_grid<ALGO, STATS, true>(&grid))) return rc;
  }
  if (ctas_per_sm) {
    int nsm = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    const long long want = (long long)ctas_per_sm * nsm;
    if (want < grid) grid = (int)want;
  }
  if (ev0) CU(cudaEventRecord(ev0, st));
  CU(cudaLaunchCooperativeKernel((const void *)traverse_kernel<ALGO, STATS, PM>, grid, BLOCK, args,
                                 0, st));
  if (ev1) CU(cudaEventRecord(ev1, st));
  return GBBS_OK;
}

// ---------------------------------------------------------------------------
// NEXT-2: wBFS bucket structure (lazy, per handle; sized for the bucket span)
// ---------------------------------------------------------------------------
struct WbfsScratch {
  uint32_t *bq = nullptr;  // nbq lists x qcap ids
  unsigned long long qcap = 0;
  int nbq = 0;
  uint32_t *xq[3] = {nullptr, nullptr, nullptr};
  uint32_t *tag = nullptr, *hv = nullptr;
  unsigned long long *ctr = nullptr;  // btail[64] bheavy[64] xcnt[6] pub[3]
  int grid[2] = {0, 0};
};

static void free_wbfs(gbbs_graph *g) {
  WbfsScratch *w = g->wb;
  if (!w) return;
  cudaFree(w->bq);
  for (int i = 0; i < 3; i++) cudaFree(w->xq[i]);
  cudaFree(w->tag);
  cudaFree(w->hv);
  cudaFree(w->ctr);
  delete w;
  g->wb = nullptr;
}

constexpr size_t WBFS_DYN_SMEM = sizeof(WbfsWarpSmem) * NWARPS;

template <bool STATS>
static int wbfs_grid(int *grid) {
  int dev = 0, nsm = 0, per = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CU(cudaFuncSetAttribute(wbfs_kernel<STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)WBFS_DYN_SMEM));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wbfs_kernel<STATS>, BLOCK, WBFS_DYN_SMEM));
  if (per < 1) return fail(GBBS_ECUDA, "wbfs kernel cannot be resident");
  *grid = per * nsm;
  return GBBS_OK;
}

// Bucket width and list count: delta = opts.delta, or by default 1 (the paper's
// wBFS) while the span fits 64 lists, else ceil(maxw / 32).  span = floor((delta -
// 1 + maxw) / delta) buckets above the current one can receive entries, so nbq =
// the smallest power of two > span.
static int wbfs_setup(gbbs_graph *g, uint32_t delta, Params &p) {
  const unsigned long long W = g->maxw ? g->maxw : 1;
  unsigned long long D = delta ? delta : (W <= 32 ? 1 : (W + 31) / 32);
  const unsigned long long span = (D - 1 + W) / D;
  if (span >= 64)
    return fail(GBBS_EINVAL, "wbfs: delta %llu too small for max weight %llu (needs (delta-1+maxw)/delta < 64)",
                D, W);
  int nbq = 1;
  while ((unsigned long long)nbq <= span) nbq <<= 1;
  const bool need_near = D > 1 || g->minw == 0;
  WbfsScratch *w = g->wb;
  if (w && w->nbq < nbq) {
    free_wbfs(g);
    w = nullptr;
  }
  if (!w) {
    // list capacity: 2^ceil(log2 n) (a bucket can hold every vertex), or less when
    // the ring would take more than half of the free device memory; a list that
    // overflows is detected when its bucket is extracted (GBBS_ENOMEM)
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    unsigned long long qcap = 1;
    while (qcap < (unsigned long long)g->n) qcap <<= 1;
    while (qcap > (1ull << 16) && (unsigned long long)nbq * qcap * 4 > free_b / 2) qcap >>= 1;
    w = new (std::nothrow) WbfsScratch();
    if (!w) return fail(GBBS_ENOMEM, "host allocation");
    g->wb = w;
    w->nbq = nbq;
    w->qcap = qcap;
    CU(cudaMalloc(&w->bq, (size_t)nbq * qcap * 4));
    CU(cudaMalloc(&w->hv, (size_t)g->nwords * 4));
    CU(cudaMalloc(&w->ctr, (64 + 64 + 6 + 3) * 8));
    k_heavy_bits<<<(unsigned)((g->nwords * 32 + 255) / 256), 256>>>(g->off, g->n, g->nwords, w->hv);
    CU(cudaGetLastError());
    int rc;
    if ((rc = wbfs_grid<false>(&w->grid[0]))) return rc;
    if ((rc = wbfs_grid<true>(&w->grid[1]))) return rc;
  }
  if (need_near && !w->tag) {  // near lists + round tags: only for delta > 1 or w = 0
    for (int i = 0; i < 3; i++) CU(cudaMalloc(&w->xq[i], (size_t)g->n * 4));
    CU(cudaMalloc(&w->tag, (size_t)g->n * 4));
  }
  p.bq = w->bq;
  p.qcap = w->qcap;
  p.nbq = w->nbq;
  p.btail = w->ctr;
  p.bheavy = w->ctr + 64;
  p.xcnt = w->ctr + 128;
  p.pub = w->ctr + 134;
  for (int i = 0; i < 3; i++) p.xq[i] = w->xq[i];
  p.tag = need_near ? w->tag : nullptr;
  p.hv = w->hv;
  p.delta = (uint32_t)D;
  const long long n1 = g->n + 1;
  p.max_rounds = need_near ? (n1 < (1ll << 31) ? n1 * n1 : (1ll << 62)) : n1;
  return GBBS_OK;
}

template <bool STATS>
static int launch_wbfs(gbbs_graph *g, Params &p, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1,
                       unsigned ctas_per_sm) {
  void *args[] = {&p};
  int grid = g->wb->grid[STATS];
  if (ctas_per_sm) {
    int nsm = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    const long long want = (long long)ctas_per_sm * nsm;
    if (want < grid) grid = (int)want;
  }
  if (ev0) CU(cudaEventRecord(ev0, st));
  CU(cudaLaunchCooperativeKernel((const void *)wbfs_kernel<STATS>, grid, BLOCK, args, WBFS_DYN_SMEM,
                                 st));
  if (ev1) CU(cudaEventRecord(ev1, st));
  return GBBS_OK;
}

// ---------------------------------------------------------------------------
// options: defaults and validation shared by every entry point
// ---------------------------------------------------------------------------
enum OptsKind { OPTS_TRAVERSE, OPTS_BATCH, OPTS_SIGNED, OPTS_OTHER };

static int parse_opts(const gbbs_opts *opts, OptsKind kind, gbbs_opts &o) {
  gbbs_default_opts(&o);
  if (!opts) return GBBS_OK;
  o = *opts;
  if (o.threshold_den == 0) o.threshold_den = 20;
  if (o.rules & ~(uint32_t)(GBBS_RULE_PAPER_ONLY | GBBS_RULE_LEVEL_BYTES_ON | GBBS_RULE_LEVEL_BYTES_OFF))
    return fail(GBBS_EINVAL, "unknown opts.rules bits 0x%x", o.rules);
  if ((o.rules & GBBS_RULE_LEVEL_BYTES_ON) && (o.rules & GBBS_RULE_LEVEL_BYTES_OFF))
    return fail(GBBS_EINVAL, "opts.rules asks for level bytes both on and off");
  const int max_mode = (kind == OPTS_BATCH) ? 2 : 3;
  if (o.mode < 0 || o.mode > max_mode) return fail(GBBS_EINVAL, "bad mode %d", o.mode);
  if (o.bsize && (o.bsize < 32 || o.bsize > (uint32_t)TE || (o.bsize & (o.bsize - 1))))
    return fail(GBBS_EINVAL, "bsize %u: a power of two in [32, %d], or 0", o.bsize, TE);
  if (kind == OPTS_BATCH && o.ctas_per_sm != 0)
    return fail(GBBS_EINVAL, "batch calls take ctas_per_sm = 0");
  if (o.teams > (uint32_t)GMAX) return fail(GBBS_EINVAL, "teams %u > %d", o.teams, GMAX);
  if (o.neg_scope > 1) return fail(GBBS_EINVAL, "bad neg_scope %u", o.neg_scope);
  return GBBS_OK;
}

// ---------------------------------------------------------------------------
// batch teams: scratch of the traversals that run beside team 0 in one launch
// ---------------------------------------------------------------------------
struct TeamScratch {
  uint32_t *bm[2] = {nullptr, nullptr};
  uint32_t *fv[3] = {nullptr, nullptr, nullptr};
  long long *fo[3] = {nullptr, nullptr, nullptr};
  long long *fb[3] = {nullptr, nullptr, nullptr};
  unsigned long long *cnt = nullptr;  // same layout as the handle's (CNT_WORDS words)
  uint16_t *shadow = nullptr;
  unsigned *bar = nullptr;
  // wBFS bucket structure of this team (hv is shared with team 0's)
  uint32_t *bq = nullptr;
  unsigned long long *wctr = nullptr;
  uint32_t *xq[3] = {nullptr, nullptr, nullptr};
  uint32_t *tag = nullptr;
  int nbq = 0;
  unsigned long long qcap = 0;
};

static void free_teams(gbbs_graph *g) {
  for (int t = 0; t < 8; t++) {
    TeamScratch *x = g->team[t];
    if (!x) continue;
    for (int i = 0; i < 3; i++) {
      if (i < 2) cudaFree(x->bm[i]);
      cudaFree(x->fv[i]);
      cudaFree(x->fo[i]);
      cudaFree(x->fb[i]);
    }
    cudaFree(x->cnt);
    cudaFree(x->shadow);
    cudaFree(x->bar);
    cudaFree(x->bq);
    cudaFree(x->wctr);
    for (int i = 0; i < 3; i++) cudaFree(x->xq[i]);
    cudaFree(x->tag);
    delete x;
    g->team[t] = nullptr;
  }
  cudaFree(g->bar0);
  g->bar0 = nullptr;
}

static int team_scratch(gbbs_graph *g, int t) {
  if (t == 0) {
    if (!g->bar0) {
      CU(cudaMalloc(&g->bar0, 8));
      CU(cudaMemset(g->bar0, 0, 8));
    }
    return GBBS_OK;
  }
  if (g->team[t]) return GBBS_OK;
  TeamScratch *x = new (std::nothrow) TeamScratch();
  if (!x) return fail(GBBS_ENOMEM, "host allocation");
  g->team[t] = x;
  const size_t n = (size_t)g->n;
  for (int i = 0; i < 2; i++) CU(cudaMalloc(&x->bm[i], (size_t)g->nwords * 4));
  for (int i = 0; i < 3; i++) {
    CU(cudaMalloc(&x->fv[i], n * 4));
    CU(cudaMalloc(&x->fo[i], n * 8));
    CU(cudaMalloc(&x->fb[i], n * 8));
  }
  CU(cudaMalloc(&x->cnt, CNT_WORDS * 8));
  CU(cudaMemset(x->cnt, 0, CNT_WORDS * 8));
  CU(cudaMalloc(&x->shadow, n * 2));
  CU(cudaMalloc(&x->bar, 8));
  CU(cudaMemset(x->bar, 0, 8));
  return GBBS_OK;
}

// Kernel parameters of one traversal (no statistics) on device outputs.
static void fill_params(gbbs_graph *g, int algo, uint32_t src, uint32_t *ddist, uint32_t *dpar,
                        const gbbs_opts &o, Params &p) {
  memset(&p, 0, sizeof p);
  p.n = g->n;
  p.m = g->m;
  p.off = g->off;
  p.tgt = g->tgt;
  p.wgt = g->wgt;
  p.in_off = g->in_off;
  p.in_tgt = g->in_tgt;
  p.dist = ddist;
  p.parent = (algo == ALGO_BFS) ? dpar : nullptr;
  p.bm[0] = g->bm[0];
  p.bm[1] = g->bm[1];
  for (int i = 0; i < 3; i++) {
    p.fv[i] = g->fv[i];
    p.fo[i] = g->fo[i];
    p.fb[i] = g->fb[i];
  }
  p.cnt = g->cnt;
  p.hcnt = g->cnt + 8;
  p.wq = g->cnt + 10;
  p.acq = g->cnt + 18;
  p.status = g->status;
  p.rounds_out = g->rounds;
  p.nwords = g->nwords;
  p.dense_threshold = g->m / (long long)o.threshold_den;
  p.max_rounds = g->n + 1;
  p.ebits = g->ebits;
  p.iso = g->iso;
  p.nin = g->nin;
  p.phot = g->phot;
  p.pcold = g->pcold;
  p.phot8 = g->phot8;
  p.pc32 = g->pc32;
  p.ncand = g->ncand;
  p.rules = (int)o.rules;
  p.shadow = g->shadow;
  // BFS levels as bytes in the (otherwise idle) shadow buffer: measured faster above
  // 2^24 vertices (c4 -6 %, c5 -5 %), slower below (c2 +5 %, c3 +2.5 %)
  const bool lvl_on = algo == ALGO_BFS && !(o.rules & GBBS_RULE_LEVEL_BYTES_OFF) &&
                      ((o.rules & GBBS_RULE_LEVEL_BYTES_ON) || g->n > (1ll << 24));
  p.lvl = lvl_on ? reinterpret_cast<uint8_t *>(g->shadow) : nullptr;
  p.symmetric = (g->flags & GBBS_SYMMETRIC) ? 1 : 0;
  p.mode = o.mode;
  p.bsize = (int)o.bsize;
  p.src = src;
}

// The same for team t of a multi-traversal launch (t = 0: the handle's scratch).
static void fill_params_team(gbbs_graph *g, int algo, uint32_t src, uint32_t *ddist,
                             uint32_t *dpar, const gbbs_opts &o, int t, Params &p) {
  fill_params(g, algo, src, ddist, dpar, o, p);
  if (t == 0) {
    p.bar = g->bar0;
    return;
  }
  TeamScratch *x = g->team[t];
  p.bm[0] = x->bm[0];
  p.bm[1] = x->bm[1];
  for (int i = 0; i < 3; i++) {
    p.fv[i] = x->fv[i];
    p.fo[i] = x->fo[i];
    p.fb[i] = x->fb[i];
  }
  p.cnt = x->cnt;
  p.hcnt = x->cnt + 8;
  p.wq = x->cnt + 10;
  p.acq = x->cnt + 18;
  p.status = (int *)(x->cnt + 4);
  p.rounds_out = (long long *)(x->cnt + 5);
  p.shadow = x->shadow;
  if (p.lvl) p.lvl = reinterpret_cast<uint8_t *>(x->shadow);
  p.bar = x->bar;
}

template <int ALGO>
static int launch_mg(gbbs_graph *g, MultiParams &mp, cudaStream_t st) {
  if (!g->mg_grid[ALGO]) {
    int nsm = 0, per = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, traverse_mg_kernel<ALGO>, BLOCK, 0));
    if (per < 1) return fail(GBBS_ECUDA, "multi-traversal kernel cannot be resident");
    g->mg_grid[ALGO] = per * nsm;
  }
  void *args[] = {&mp};
  CU(cudaLaunchCooperativeKernel((const void *)traverse_mg_kernel<ALGO>, g->mg_grid[ALGO], BLOCK,
                                 args, 0, st));
  return GBBS_OK;
}

// Exact range check (status bit 2: a relaxation candidate d(u) + w reached 2^32 - 1).
// The kernels drop such a candidate as "no improvement", so every finite distance
// they return is exact; the true distance of a vertex does not fit the uint32 output
// iff some edge (u, v) has finite d(u), d(u) + w >= 2^32 - 1 and d(v) = INF.  One
// warp per source vertex; run only when the kernel raised the flag.
__global__ void k_range_check(const long long *off, const uint32_t *tgt, const uint32_t *wgt,
                              long long n, const uint32_t *dist, unsigned long long *bad) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long u = warp; u < n; u += nwarps) {
    const uint32_t du = dist[u];
    if (du == INF) continue;
    for (long long e = off[u] + lane; e < off[u + 1]; e += 32) {
      const unsigned long long c = (unsigned long long)du + (wgt ? wgt[e] : 1u);
      if (c >= INF && dist[tgt[e]] == INF) atomicOr(bad, 1ull);
    }
  }
}

// Clears status bit 2 when the check above finds every distance representable.
// dist: n entries, host or device.
static int range_recheck(gbbs_graph *g, const uint32_t *dist, cudaStream_t st, int *status) {
  if (!(*status & 2)) return GBBS_OK;
  const uint32_t *dd = dist;
  if (!is_device_ptr(dist)) {
    if (!g->tmp_dist) CU(cudaMalloc(&g->tmp_dist, (size_t)g->n * 4));
    CU(cudaMemcpyAsync(g->tmp_dist, dist, (size_t)g->n * 4, cudaMemcpyHostToDevice, st));
    dd = g->tmp_dist;
  }
  CU(cudaMemsetAsync(g->dcount, 0, 8, st));
  k_range_check<<<1184, 256, 0, st>>>(g->off, g->tgt, g->wgt, g->n, dd, g->dcount);
  CU(cudaGetLastError());
  unsigned long long bad = 0;
  CU(cudaMemcpyAsync(&bad, g->dcount, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (!bad) *status &= ~2;
  return GBBS_OK;
}

static int status_error(const gbbs_graph *g, int status, long long max_rounds) {
  if (status & 4)
    return fail(GBBS_ENOMEM, "wbfs: a bucket list exceeded its capacity of %llu entries "
                "(device memory was short at first use; a larger delta needs fewer)",
                g->wb ? g->wb->qcap : 0ull);
  if (status & 2)  // a reachable vertex's distance is >= 2^32 - 1 (k_range_check)
    return fail(GBBS_ERANGE, "a reachable vertex's distance is >= 2^32-1 (max weight %u): "
                "distances do not fit the uint32 output", g->maxw);
  if (status != 0)
    return fail(GBBS_EINTERNAL, "round cap (%lld rounds) exceeded", max_rounds);
  return GBBS_OK;
}

static int run(const gbbs_graph *cg_, int algo, uint32_t src, uint32_t *dist, uint32_t *parent,
               void *stream, const gbbs_opts *opts, gbbs_stats *stats) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (!dist) return fail(GBBS_EINVAL, "dist is NULL");
  if ((long long)src >= g->n) return fail(GBBS_EINVAL, "src %u >= n %lld", src, g->n);
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_TRAVERSE, o)) return rc0;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  cudaStream_t st = (cudaStream_t)stream;

  const bool dist_dev = is_device_ptr(dist);
  const bool par_dev = parent ? is_device_ptr(parent) : true;
  const size_t nb = (size_t)g->n * 4;
  if (!dist_dev && !g->tmp_dist) CU(cudaMalloc(&g->tmp_dist, nb));
  if (!par_dev && !g->tmp_parent) CU(cudaMalloc(&g->tmp_parent, nb));
  uint32_t *ddist = dist_dev ? dist : g->tmp_dist;
  uint32_t *dpar = parent ? (par_dev ? parent : g->tmp_parent) : nullptr;

  const bool want_stats = stats != nullptr;
  const bool want_rounds = want_stats && stats->rounds_out && stats->rounds_cap > 0;
  long long cap = 0;
  if (want_rounds) {
    cap = stats->rounds_cap;
    if (g->dstats_cap < cap) {
      cudaFree(g->dstats);
      g->dstats = nullptr;
      g->dstats_cap = 0;
      CU(cudaMalloc(&g->dstats, (size_t)cap * sizeof(RoundStat)));
      g->dstats_cap = cap;
    }
    CU(cudaMemsetAsync(g->dstats, 0, (size_t)cap * sizeof(RoundStat), st));
  }

  Params p;
  fill_params(g, algo, src, ddist, dpar, o, p);
  p.stats = want_rounds ? g->dstats : nullptr;
  p.stats_cap = cap;

  if (algo == ALGO_WBFS) {
    int rc2 = wbfs_setup(g, o.delta, p);
    if (rc2) return rc2;
  }
#if defined(GBBS_DBG_PHASE) || defined(GBBS_DIAG_TILE)
  static unsigned long long *dbg = nullptr;
  constexpr size_t DBGW = 16 * 16384;
  if (!dbg) cudaMalloc(&dbg, DBGW * 8);
  cudaMemsetAsync(dbg, 0, DBGW * 8, st);
  p.dbg = dbg;
#endif
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (want_stats) {
    if (!g->ev[0]) {
      CU(cudaEventCreate(&g->ev[0]));
      CU(cudaEventCreate(&g->ev[1]));
    }
    ev0 = g->ev[0];
    ev1 = g->ev[1];
  }
  int rc;
  if (algo == ALGO_BFS)
    rc = want_rounds ? launch<ALGO_BFS, true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch<ALGO_BFS, false>(g, p, st, ev0, ev1, o.ctas_per_sm);
  else if (algo == ALGO_BF && o.mode == GBBS_MODE_PULL)
    rc = want_rounds ? launch<ALGO_BF, true, true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch<ALGO_BF, false, true>(g, p, st, ev0, ev1, o.ctas_per_sm);
  else if (algo == ALGO_BF)
    rc = want_rounds ? launch<ALGO_BF, true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch<ALGO_BF, false>(g, p, st, ev0, ev1, o.ctas_per_sm);
  else if (algo == ALGO_WP && o.mode == GBBS_MODE_PULL)
    rc = want_rounds ? launch<ALGO_WP, true, true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch<ALGO_WP, false, true>(g, p, st, ev0, ev1, o.ctas_per_sm);
  else if (algo == ALGO_WP)
    rc = want_rounds ? launch<ALGO_WP, true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch<ALGO_WP, false>(g, p, st, ev0, ev1, o.ctas_per_sm);
  else
    rc = want_rounds ? launch_wbfs<true>(g, p, st, ev0, ev1, o.ctas_per_sm) : launch_wbfs<false>(g, p, st, ev0, ev1, o.ctas_per_sm);
  if (rc) return rc;
  if (!dist_dev) CU(cudaMemcpyAsync(dist, ddist, nb, cudaMemcpyDeviceToHost, st));
  if (parent && !par_dev) CU(cudaMemcpyAsync(parent, dpar, nb, cudaMemcpyDeviceToHost, st));
  struct {
    int status;
    int pad;
    long long rounds;
  } ctrl;
  CU(cudaMemcpyAsync(&ctrl, g->status, 16, cudaMemcpyDeviceToHost, st));
  long long reached = -1;
  if (want_stats) {
    CU(cudaMemsetAsync(g->dcount, 0, 8, st));
    k_count_reached<<<592, 256, 0, st>>>(ddist, g->n, g->dcount);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&reached, g->dcount, 8, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaStreamSynchronize(st));
  if (want_stats) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ev0, ev1));
    stats->kernel_ms = ms;
    stats->rounds = ctrl.rounds;
    stats->reached = reached;
    stats->dense_rounds = 0;
    stats->edges_examined = 0;
    if (want_rounds) {
      long long nr = ctrl.rounds + 1 < cap ? ctrl.rounds + 1 : cap;
      static_assert(sizeof(RoundStat) == sizeof(gbbs_round_stat), "stat layout");
      CU(cudaMemcpy(stats->rounds_out, g->dstats, (size_t)nr * sizeof(RoundStat),
                    cudaMemcpyDeviceToHost));
      for (long long i = 0; i < nr; i++) {
        stats->dense_rounds += stats->rounds_out[i].dense == 1;
        stats->edges_examined += stats->rounds_out[i].edges_examined;
      }
    }
  }
#ifdef GBBS_DIAG_TILE
  {
    std::vector<unsigned long long> hv(16 * 16384);
    cudaMemcpy(hv.data(), dbg, hv.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long h[16] = {0};
    for (size_t w = 0; w < 16384; w++)
      for (int k = 0; k < 8; k++) {
        h[k] += hv[16 * w + k];
        h[8 + k] = std::max(h[8 + k], hv[16 * w + 8 + k]);
      }
    const char *nm[6] = {"search", "OBF", "tgt", "pre", "atom", "flush"};
    for (int k = 0; k < 6; k++) {
      const double c = (double)(k == 5 ? h[7] : h[6]);
      fprintf(stderr, "diag %-6s mean %.2fus max %.2fus\n", nm[k], c ? h[k] / c / 1e3 : 0.0,
              h[8 + k] / 1e3);
    }
    fprintf(stderr, "diag tiles %llu flushes %llu\n", h[6], h[7]);
  }
#endif
#ifdef GBBS_DBG_PHASE
  {
    unsigned long long h[256];
    cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 12 && i < ctrl.rounds; i++)
      fprintf(stderr, "dbg r%d flush: pass1 %.1fus atomic %.1fus pass2 %.1fus maxcnt %llu\n", i,
              h[4 * i] / 1e3, h[4 * i + 1] / 1e3, h[4 * i + 2] / 1e3, h[4 * i + 3]);
  }
#endif
  if (int rc3 = range_recheck(g, ddist, st, &ctrl.status)) return rc3;
  return status_error(g, ctrl.status, p.max_rounds);
}

// Batch of traversals (one per source) into row i of dist/parent, enqueued with
// no host synchronisation between them: each launch is followed by a copy of its
// status word into a per-traversal device slot, and the host synchronises once.
// Host outputs: traversal i writes double-buffered device staging and an event;
// the copy stream waits for it and copies the rows while traversal i+1 computes;
// traversal i+2 waits for the copy event that frees its buffer.
static int run_batch(const gbbs_graph *cg_, int algo, const uint32_t *srcs, int64_t k,
                     uint32_t *dist, uint32_t *parent, void *stream, const gbbs_opts *opts) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (k < 0 || (k > 0 && (!srcs || !dist))) return fail(GBBS_EINVAL, "bad batch arguments");
  for (int64_t i = 0; i < k; i++)
    if ((long long)srcs[i] >= g->n) return fail(GBBS_EINVAL, "srcs[%lld] = %u >= n %lld",
                                                 (long long)i, srcs[i], g->n);
  if (k == 0) return GBBS_OK;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  const size_t n = (size_t)g->n;
  const bool dist_dev = is_device_ptr(dist);
  const bool par_dev = parent ? is_device_ptr(parent) : true;
  const bool host_out = !(dist_dev && par_dev);
  cudaStream_t st = (cudaStream_t)stream;
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_BATCH, o)) return rc0;
  if (g->bstat_cap < k) {
    cudaFree(g->bstat);
    g->bstat = nullptr;
    g->bstat_cap = 0;
    CU(cudaMalloc(&g->bstat, (size_t)k * 16));
    g->bstat_cap = k;
  }
  if (host_out) {
    if (!g->cstream) {
      CU(cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; i++) {
        CU(cudaEventCreateWithFlags(&g->cev[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&g->kev[i], cudaEventDisableTiming));
      }
    }
    for (int b = 0; b < 2; b++)
      for (int j = 0; j < (parent ? 2 : 1); j++)
        if (!g->bst[b][j]) CU(cudaMalloc(&g->bst[b][j], n * 4));
  }
  // device outputs: G traversals per launch (teams).  Default (teams = 0): 8 for
  // BFS on graphs with n <= 2^24 and m <= 2^28, else 1 — measured (tools/
  // teams_probe.py): the c2 8-source BFS batch takes 1.34 / 0.94 / 0.88 ms with
  // 1 / 4 / 8 teams; BFS on c4/c5 and every BF batch got slower with teams
  // (throughput-bound rounds, the teams contend for L2)
  int G = 1;
  if (!host_out) {
    if (o.teams) G = (int)o.teams;
    else if (algo == ALGO_BFS && g->n <= (1ll << 24) && g->m <= (1ll << 28)) G = 8;
  }
  if (G > 1) {
    for (int t = 0; t < G; t++) {
      const int rc = team_scratch(g, t);
      if (rc) return rc;
    }
    for (int64_t i0 = 0; i0 < k; i0 += G) {
      MultiParams mp;
      memset(&mp, 0, sizeof mp);
      mp.G = (int)((k - i0) < G ? (k - i0) : G);
      for (int t = 0; t < mp.G; t++)
        fill_params_team(g, algo, srcs[i0 + t], dist + (i0 + t) * n,
                         parent ? parent + (i0 + t) * n : nullptr, o, t, mp.ps[t]);
      const int rc = (algo == ALGO_BFS) ? launch_mg<ALGO_BFS>(g, mp, st) : launch_mg<ALGO_BF>(g, mp, st);
      if (rc) return rc;
      for (int t = 0; t < mp.G; t++)
        CU(cudaMemcpyAsync(g->bstat + 2 * (i0 + t), mp.ps[t].status, 16,
                           cudaMemcpyDeviceToDevice, st));
    }
  }
  for (int64_t i = (G > 1 ? k : 0); i < k; i++) {
    const int b = (int)(i & 1);
    uint32_t *dd = dist + i * n, *dp = parent ? parent + i * n : nullptr;
    if (host_out) {
      if (i >= 2) CU(cudaStreamWaitEvent(st, g->cev[b], 0));  // copy i-2 freed buffer b
      dd = g->bst[b][0];
      dp = parent ? g->bst[b][1] : nullptr;
    }
    Params p;
    fill_params(g, algo, srcs[i], dd, dp, o, p);
    const int rc = (algo == ALGO_BFS) ? launch<ALGO_BFS, false>(g, p, st, nullptr, nullptr, 0)
                                      : launch<ALGO_BF, false>(g, p, st, nullptr, nullptr, 0);
    if (rc) return rc;
    CU(cudaMemcpyAsync(g->bstat + 2 * i, g->status, 16, cudaMemcpyDeviceToDevice, st));
    if (host_out) {
      CU(cudaEventRecord(g->kev[b], st));
      CU(cudaStreamWaitEvent(g->cstream, g->kev[b], 0));
      CU(cudaMemcpyAsync(dist + i * n, g->bst[b][0], n * 4, cudaMemcpyDefault, g->cstream));
      if (parent)
        CU(cudaMemcpyAsync(parent + i * n, g->bst[b][1], n * 4, cudaMemcpyDefault, g->cstream));
      CU(cudaEventRecord(g->cev[b], g->cstream));
    }
  }
  std::vector<long long> hs((size_t)k * 2);
  CU(cudaMemcpyAsync(hs.data(), g->bstat, (size_t)k * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (host_out) CU(cudaStreamSynchronize(g->cstream));
  for (int64_t i = 0; i < k; i++) {
    int sti = (int)(hs[2 * i] & 0xFFFFFFFF);
    if (int rc3 = range_recheck(g, dist + i * n, st, &sti)) return rc3;
    const int rc = status_error(g, sti, g->n + 1);
    if (rc) return rc;
  }
  return GBBS_OK;
}

extern "C" int gbbs_bfs_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k, uint32_t *dist,
                              uint32_t *parent, void *cuda_stream) {
  return run_batch(g, ALGO_BFS, srcs, k, dist, parent, cuda_stream, nullptr);
}

extern "C" int gbbs_bellman_ford_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                                       uint32_t *dist, void *cuda_stream) {
  return run_batch(g, ALGO_BF, srcs, k, dist, nullptr, cuda_stream, nullptr);
}

extern "C" int gbbs_bfs_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                                 uint32_t *dist, uint32_t *parent, void *cuda_stream,
                                 const gbbs_opts *opts) {
  return run_batch(g, ALGO_BFS, srcs, k, dist, parent, cuda_stream, opts);
}

extern "C" int gbbs_bellman_ford_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                                          uint32_t *dist, void *cuda_stream,
                                          const gbbs_opts *opts) {
  return run_batch(g, ALGO_BF, srcs, k, dist, nullptr, cuda_stream, opts);
}

extern "C" int gbbs_bfs(const gbbs_graph *g, uint32_t src, uint32_t *dist, uint32_t *parent,
                        void *cuda_stream) {
  return run(g, ALGO_BFS, src, dist, parent, cuda_stream, nullptr, nullptr);
}

extern "C" int gbbs_bellman_ford(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                                 void *cuda_stream) {
  return run(g, ALGO_BF, src, dist, nullptr, cuda_stream, nullptr, nullptr);
}

extern "C" int gbbs_bfs_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist, uint32_t *parent,
                           void *cuda_stream, const gbbs_opts *opts, gbbs_stats *stats) {
  return run(g, ALGO_BFS, src, dist, parent, cuda_stream, opts, stats);
}

extern "C" int gbbs_bellman_ford_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                                    void *cuda_stream, const gbbs_opts *opts, gbbs_stats *stats) {
  return run(g, ALGO_BF, src, dist, nullptr, cuda_stream, opts, stats);
}

// ---------------------------------------------------------------------------
// NEXT-4: general-weight (signed) Bellman-Ford (sbf.cuh)
// ---------------------------------------------------------------------------
template <bool STATS>
static int sbf_launch(gbbs_graph *g, Params &p, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
  if (!g->sgrid[STATS]) {
    int nsm = 0, per = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sbf_kernel<STATS>, BLOCK, 0));
    if (per < 1) return fail(GBBS_ECUDA, "signed Bellman-Ford kernel cannot be resident");
    g->sgrid[STATS] = per * nsm;
  }
  void *args[] = {&p};
  if (ev0) CU(cudaEventRecord(ev0, st));
  CU(cudaLaunchCooperativeKernel((const void *)sbf_kernel<STATS>, g->sgrid[STATS], BLOCK, args, 0, st));
  if (ev1) CU(cudaEventRecord(ev1, st));
  return GBBS_OK;
}

extern "C" int gbbs_bellman_ford_signed_ex(const gbbs_graph *cg_, uint32_t src, int64_t *dist,
                                           void *cuda_stream, const gbbs_opts *opts,
                                           gbbs_stats *stats) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (!dist) return fail(GBBS_EINVAL, "dist is NULL");
  if ((long long)src >= g->n) return fail(GBBS_EINVAL, "src %u >= n %lld", src, g->n);
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_SIGNED, o)) return rc0;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (g->smaxabs < 0) {
    g->smaxabs = 1;
    if (g->wgt && g->m > 0) {
      unsigned long long *d = nullptr;
      CU(cudaMalloc(&d, 8));
      CU(cudaMemset(d, 0, 8));
      k_absmax_i32<<<1184, 256>>>(g->wgt, g->m, d);
      cudaError_t e = cudaGetLastError();
      unsigned long long h = 0;
      if (e == cudaSuccess) e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      cudaFree(d);
      if (e != cudaSuccess) return fail(GBBS_ECUDA, "max |w|: %s", cudaGetErrorString(e));
      g->smaxabs = (long long)h;
    }
  }
  // every simple path stays above FLOOR = -2^62 and below +2^62
  if (g->smaxabs > 0 && (unsigned long long)(g->n - 1) > ((1ull << 62) - 1) / (unsigned long long)g->smaxabs)
    return fail(GBBS_ERANGE, "(n-1) * max|w| = %lld * %lld does not fit in 2^62", g->n - 1, g->smaxabs);
  const bool dev_out = is_device_ptr(dist);
  if (!dev_out && !g->tmp_sdist) CU(cudaMalloc(&g->tmp_sdist, (size_t)g->n * 8));
  long long *dd = dev_out ? (long long *)dist : g->tmp_sdist;

  const bool want_rounds = stats && stats->rounds_out && stats->rounds_cap > 0;
  long long cap = 0;
  if (want_rounds) {
    cap = stats->rounds_cap;
    if (g->dstats_cap < cap) {
      cudaFree(g->dstats);
      g->dstats = nullptr;
      g->dstats_cap = 0;
      CU(cudaMalloc(&g->dstats, (size_t)cap * sizeof(RoundStat)));
      g->dstats_cap = cap;
    }
    CU(cudaMemsetAsync(g->dstats, 0, (size_t)cap * sizeof(RoundStat), st));
  }
  Params p;
  memset(&p, 0, sizeof p);
  p.n = g->n;
  p.m = g->m;
  p.off = g->off;
  p.tgt = g->tgt;
  p.wgt = g->wgt;
  p.sdist = dd;
  p.bm[0] = g->bm[0];
  p.bm[1] = g->bm[1];
  for (int i = 0; i < 3; i++) {
    p.fv[i] = g->fv[i];
    p.fo[i] = g->fo[i];
    p.fb[i] = g->fb[i];
  }
  p.cnt = g->cnt;
  p.status = g->status;
  p.rounds_out = g->rounds;
  p.stats = want_rounds ? g->dstats : nullptr;
  p.stats_cap = cap;
  p.nwords = g->nwords;
  p.max_rounds = g->n;  // n rounds: a frontier left after them proves a negative cycle
  p.wq = g->cnt + 10;    // scratch of the early negative-cycle check
  p.ebits = g->ebits;
  p.neg_scope = (int)o.neg_scope;
  p.src = src;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (stats) {
    if (!g->ev[0]) {
      CU(cudaEventCreate(&g->ev[0]));
      CU(cudaEventCreate(&g->ev[1]));
    }
    ev0 = g->ev[0];
    ev1 = g->ev[1];
  }
  int rc = want_rounds ? sbf_launch<true>(g, p, st, ev0, ev1) : sbf_launch<false>(g, p, st, ev0, ev1);
  if (rc) return rc;
  if (!dev_out) CU(cudaMemcpyAsync(dist, dd, (size_t)g->n * 8, cudaMemcpyDeviceToHost, st));
  struct {
    int status;
    int pad;
    long long rounds;
  } ctrl;
  CU(cudaMemcpyAsync(&ctrl, g->status, 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (stats) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ev0, ev1));
    stats->kernel_ms = ms;
    stats->rounds = ctrl.rounds;
    stats->dense_rounds = 0;
    stats->edges_examined = 0;
    stats->reached = -1;
    if (want_rounds) {
      long long nr = ctrl.rounds + 1 < cap ? ctrl.rounds + 1 : cap;
      CU(cudaMemcpy(stats->rounds_out, g->dstats, (size_t)nr * sizeof(RoundStat),
                    cudaMemcpyDeviceToHost));
      for (long long i = 0; i < nr && i < ctrl.rounds; i++)
        stats->edges_examined += stats->rounds_out[i].edges_examined;
    }
  }
  return GBBS_OK;
}

extern "C" int gbbs_bellman_ford_signed(const gbbs_graph *g, uint32_t src, int64_t *dist,
                                        void *cuda_stream) {
  return gbbs_bellman_ford_signed_ex(g, src, dist, cuda_stream, nullptr, nullptr);
}

// Batch of wBFS traversals into device rows, G per launch (teams of
// wbfs_mg_kernel, each with its own bucket ring and scratch).
static int run_wbfs_batch(const gbbs_graph *cg_, const uint32_t *srcs, int64_t k, uint32_t *dist,
                          void *stream, const gbbs_opts *opts) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (k < 0 || (k > 0 && (!srcs || !dist))) return fail(GBBS_EINVAL, "bad batch arguments");
  for (int64_t i = 0; i < k; i++)
    if ((long long)srcs[i] >= g->n) return fail(GBBS_EINVAL, "srcs[%lld] = %u >= n %lld",
                                                 (long long)i, srcs[i], g->n);
  if (k == 0) return GBBS_OK;
  if (!is_device_ptr(dist)) return fail(GBBS_EINVAL, "gbbs_wbfs_batch writes device rows");
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_BATCH, o)) return rc0;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = (size_t)g->n;
  // teams: default 8 on graphs with n <= 2^24 and m <= 2^28, else 1 — measured
  // (tools/teams_probe.py): c2 21.3 / 15.1 / 14.6 ms with 1 / 4 / 8 teams for its 8
  // sources, c4 flat (62-64 ms)
  const int G = (int)(o.teams ? o.teams
                              : ((g->n <= (1ll << 24) && g->m <= (1ll << 28)) ? 8 : 1));
  if (g->bstat_cap < k) {
    cudaFree(g->bstat);
    g->bstat = nullptr;
    g->bstat_cap = 0;
    CU(cudaMalloc(&g->bstat, (size_t)k * 16));
    g->bstat_cap = k;
  }
  for (int t = 0; t < G; t++)
    if (int rc = team_scratch(g, t)) return rc;
  if (!g->wb_mg_grid) {
    int nsm = 0, per = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    CU(cudaFuncSetAttribute(wbfs_mg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)WBFS_DYN_SMEM));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wbfs_mg_kernel, BLOCK, WBFS_DYN_SMEM));
    if (per < 1) return fail(GBBS_ECUDA, "multi-traversal wbfs kernel cannot be resident");
    g->wb_mg_grid = per * nsm;
  }
  for (int64_t i0 = 0; i0 < k; i0 += G) {
    MultiParams mp;
    memset(&mp, 0, sizeof mp);
    mp.G = (int)((k - i0) < G ? (k - i0) : G);
    for (int t = 0; t < mp.G; t++) {
      Params &p = mp.ps[t];
      fill_params_team(g, ALGO_WBFS, srcs[i0 + t], dist + (i0 + t) * n, nullptr, o, t, p);
      Params p0;  // team 0's bucket structure decides delta, nbq and the list capacity
      fill_params(g, ALGO_WBFS, srcs[i0 + t], dist, nullptr, o, p0);
      if (int rc = wbfs_setup(g, o.delta, p0)) return rc;
      p.delta = p0.delta;
      p.nbq = p0.nbq;
      p.qcap = p0.qcap;
      p.hv = p0.hv;
      p.max_rounds = p0.max_rounds;
      if (t == 0) {
        p.bq = p0.bq;
        p.btail = p0.btail;
        p.bheavy = p0.bheavy;
        p.xcnt = p0.xcnt;
        p.pub = p0.pub;
        for (int i = 0; i < 3; i++) p.xq[i] = p0.xq[i];
        p.tag = p0.tag;
        continue;
      }
      TeamScratch *x = g->team[t];
      if (x->nbq < p0.nbq || x->qcap != p0.qcap) {
        cudaFree(x->bq);
        x->bq = nullptr;
        CU(cudaMalloc(&x->bq, (size_t)p0.nbq * p0.qcap * 4));
        x->nbq = p0.nbq;
        x->qcap = p0.qcap;
      }
      if (!x->wctr) CU(cudaMalloc(&x->wctr, (64 + 64 + 6 + 3) * 8));
      if (p0.tag && !x->tag) {
        for (int i = 0; i < 3; i++) CU(cudaMalloc(&x->xq[i], n * 4));
        CU(cudaMalloc(&x->tag, n * 4));
      }
      p.bq = x->bq;
      p.btail = x->wctr;
      p.bheavy = x->wctr + 64;
      p.xcnt = x->wctr + 128;
      p.pub = x->wctr + 134;
      for (int i = 0; i < 3; i++) p.xq[i] = x->xq[i];
      p.tag = p0.tag ? x->tag : nullptr;
    }
    if (mp.G == 1) {  // the plain kernel
      void *a1[] = {&mp.ps[0]};
      CU(cudaLaunchCooperativeKernel((const void *)wbfs_kernel<false>, g->wb->grid[0], BLOCK, a1,
                                     WBFS_DYN_SMEM, st));
    } else {
      void *args[] = {&mp};
      CU(cudaLaunchCooperativeKernel((const void *)wbfs_mg_kernel, g->wb_mg_grid, BLOCK, args,
                                     WBFS_DYN_SMEM, st));
    }
    for (int t = 0; t < mp.G; t++)
      CU(cudaMemcpyAsync(g->bstat + 2 * (i0 + t), mp.ps[t].status, 16, cudaMemcpyDeviceToDevice,
                         st));
  }
  std::vector<long long> hs((size_t)k * 2);
  CU(cudaMemcpyAsync(hs.data(), g->bstat, (size_t)k * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < k; i++) {
    int sti = (int)(hs[2 * i] & 0xFFFFFFFF);
    if (int rc3 = range_recheck(g, dist + i * (size_t)g->n, st, &sti)) return rc3;
    const int rc = status_error(g, sti, -1);
    if (rc) return rc;
  }
  return GBBS_OK;
}

extern "C" int gbbs_wbfs_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                               uint32_t *dist, void *cuda_stream) {
  return run_wbfs_batch(g, srcs, k, dist, cuda_stream, nullptr);
}

extern "C" int gbbs_wbfs_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                                  uint32_t *dist, void *cuda_stream, const gbbs_opts *opts) {
  return run_wbfs_batch(g, srcs, k, dist, cuda_stream, opts);
}

extern "C" int gbbs_wbfs(const gbbs_graph *g, uint32_t src, uint32_t *dist, void *cuda_stream) {
  return run(g, ALGO_WBFS, src, dist, nullptr, cuda_stream, nullptr, nullptr);
}

extern "C" int gbbs_wbfs_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist, void *cuda_stream,
                            const gbbs_opts *opts, gbbs_stats *stats) {
  return run(g, ALGO_WBFS, src, dist, nullptr, cuda_stream, opts, stats);
}

extern "C" int gbbs_widest_path(const gbbs_graph *g, uint32_t src, uint32_t *width, void *cuda_stream) {
  return run(g, ALGO_WP, src, width, nullptr, cuda_stream, nullptr, nullptr);
}

extern "C" int gbbs_widest_path_ex(const gbbs_graph *g, uint32_t src, uint32_t *width,
                                   void *cuda_stream, const gbbs_opts *opts, gbbs_stats *stats) {
  return run(g, ALGO_WP, src, width, nullptr, cuda_stream, opts, stats);
}

// ---------------------------------------------------------------------------
// NEXT-3: single-source betweenness contributions (bc.cuh)
// ---------------------------------------------------------------------------
#include "bc.cuh"

struct BcScratch {
  uint32_t *dist = nullptr;
  double *sigma = nullptr, *delta = nullptr;
  long long *lvl = nullptr;
  long long lvl_cap = 0;
  int grid = 0;
};

static BcScratch *bc_scratch(gbbs_graph *g, int *rc) {
  static thread_local std::string dummy;
  if (g->bc) return g->bc;
  BcScratch *b = new (std::nothrow) BcScratch();
  *rc = GBBS_ENOMEM;
  if (!b) return nullptr;
  b->lvl_cap = g->n + 1 < (1ll << 22) ? g->n + 1 : (1ll << 22);
  bool ok = cudaMalloc(&b->dist, (size_t)g->n * 4) == cudaSuccess &&
            cudaMalloc(&b->sigma, (size_t)g->n * 8) == cudaSuccess &&
            cudaMalloc(&b->delta, (size_t)g->n * 8) == cudaSuccess &&
            cudaMalloc(&b->lvl, (size_t)b->lvl_cap * 24) == cudaSuccess;
  int dev = 0, nsm = 0, per = 0;
  ok = ok && cudaGetDevice(&dev) == cudaSuccess &&
       cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
       cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bc_kernel, BLOCK, 0) == cudaSuccess &&
       per > 0;
  if (!ok) {
    cudaFree(b->dist); cudaFree(b->sigma); cudaFree(b->delta); cudaFree(b->lvl);
    delete b;
    cudaGetLastError();
    fail(GBBS_ENOMEM, "betweenness scratch allocation failed");
    return nullptr;
  }
  b->grid = per * nsm;
  g->bc = b;
  *rc = GBBS_OK;
  return b;
}

// Forward-level direction (reading B3): pull only on symmetric graphs; opts.mode
// SPARSE = always push, DENSE = always pull, else the rule in bc_body.
static void bc_dense(const gbbs_graph *g, const gbbs_opts &o, BcParams &p) {
  p.dense_threshold = g->m / (long long)o.threshold_den;
  if (!(g->flags & GBBS_SYMMETRIC) || o.mode == GBBS_MODE_SPARSE) p.dense_mode = 1;
  else if (o.mode == GBBS_MODE_DENSE) p.dense_mode = 2;
  else p.dense_mode = 0;
}

static void free_bc(gbbs_graph *g) {
  if (!g->bc) return;
  cudaFree(g->bc->dist); cudaFree(g->bc->sigma); cudaFree(g->bc->delta); cudaFree(g->bc->lvl);
  delete g->bc;
  g->bc = nullptr;
}

extern "C" int gbbs_betweenness_ex(const gbbs_graph *cg_, uint32_t src, double *delta,
                                   void *cuda_stream, const gbbs_opts *opts, gbbs_stats *stats) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (!delta) return fail(GBBS_EINVAL, "delta is NULL");
  if ((long long)src >= g->n) return fail(GBBS_EINVAL, "src %u >= n %lld", src, g->n);
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_OTHER, o)) return rc0;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  int rc = GBBS_OK;
  BcScratch *b = bc_scratch(g, &rc);
  if (!b) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const bool dev_out = is_device_ptr(delta);
  BcParams p;
  memset(&p, 0, sizeof p);
  p.n = g->n;
  p.m = g->m;
  p.off = g->off;
  p.tgt = g->tgt;
  p.dist = b->dist;
  p.sigma = b->sigma;
  p.delta = dev_out ? delta : b->delta;
  p.qv = g->fv[0];
  p.qo = g->fo[0];
  p.qb = g->fb[0];
  p.lvl = b->lvl;
  p.lvl_cap = b->lvl_cap;
  p.cnt = g->cnt;
  p.wq = g->cnt + 10;
  p.status = g->status;
  p.rounds_out = g->rounds;
  p.ebits = g->ebits;
  p.src = src;
  bc_dense(g, o, p);
  void *args[] = {&p};
  if (stats) {
    if (!g->ev[0]) {
      CU(cudaEventCreate(&g->ev[0]));
      CU(cudaEventCreate(&g->ev[1]));
    }
    CU(cudaEventRecord(g->ev[0], st));
  }
  CU(cudaLaunchCooperativeKernel((const void *)bc_kernel, b->grid, BLOCK, args, 0, st));
  if (stats) CU(cudaEventRecord(g->ev[1], st));
  if (!dev_out) CU(cudaMemcpyAsync(delta, b->delta, (size_t)g->n * 8, cudaMemcpyDeviceToHost, st));
  struct {
    int status;
    int pad;
    long long rounds;
  } ctrl;
  CU(cudaMemcpyAsync(&ctrl, g->status, 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (stats) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]));
    memset(stats, 0, offsetof(gbbs_stats, rounds_out));
    stats->kernel_ms = ms;
    stats->rounds = ctrl.rounds;
  }
  if (ctrl.status != 0) return fail(GBBS_EINTERNAL, "more than %lld BFS levels", b->lvl_cap);
  return GBBS_OK;
}

// Batch of betweenness traversals into device rows: the plain kernel per source,
// launched back to back on the stream (the team form, several traversals per
// launch, measured slower at every team count — DESIGN.md §6 — and was removed;
// gbbs_opts.teams is accepted and ignored here).
extern "C" int gbbs_betweenness_batch_ex(const gbbs_graph *cg_, const uint32_t *srcs, int64_t k,
                                         double *delta, void *cuda_stream,
                                         const gbbs_opts *opts) {
  g_last_error.clear();
  if (!cg_) return fail(GBBS_EINVAL, "g is NULL");
  gbbs_graph *g = const_cast<gbbs_graph *>(cg_);
  if (k < 0 || (k > 0 && (!srcs || !delta))) return fail(GBBS_EINVAL, "bad batch arguments");
  for (int64_t i = 0; i < k; i++)
    if ((long long)srcs[i] >= g->n) return fail(GBBS_EINVAL, "srcs[%lld] = %u >= n %lld",
                                                 (long long)i, srcs[i], g->n);
  if (k == 0) return GBBS_OK;
  if (!is_device_ptr(delta)) return fail(GBBS_EINVAL, "gbbs_betweenness_batch writes device rows");
  gbbs_opts o;
  if (int rc0 = parse_opts(opts, OPTS_BATCH, o)) return rc0;
  DeviceGuard dguard(g->device);
  if (dguard.rc) return dguard.rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t n = (size_t)g->n;
  int rc = GBBS_OK;
  BcScratch *b = bc_scratch(g, &rc);
  if (!b) return rc;
  if (g->bstat_cap < k) {
    cudaFree(g->bstat);
    g->bstat = nullptr;
    g->bstat_cap = 0;
    CU(cudaMalloc(&g->bstat, (size_t)k * 16));
    g->bstat_cap = k;
  }
  for (int64_t i = 0; i < k; i++) {
    BcParams p;
    memset(&p, 0, sizeof p);
    p.n = g->n;
    p.m = g->m;
    p.off = g->off;
    p.tgt = g->tgt;
    p.dist = b->dist;
    p.sigma = b->sigma;
    p.delta = delta + i * n;
    p.qv = g->fv[0];
    p.qo = g->fo[0];
    p.qb = g->fb[0];
    p.lvl = b->lvl;
    p.lvl_cap = b->lvl_cap;
    p.cnt = g->cnt;
    p.wq = p.cnt + 10;
    p.status = (int *)(p.cnt + 4);
    p.rounds_out = (long long *)(p.cnt + 5);
    p.bar = g->bar0;
    p.ebits = g->ebits;
    p.src = srcs[i];
    bc_dense(g, o, p);
    void *a1[] = {&p};
    CU(cudaLaunchCooperativeKernel((const void *)bc_kernel, b->grid, BLOCK, a1, 0, st));
    CU(cudaMemcpyAsync(g->bstat + 2 * i, p.status, 16, cudaMemcpyDeviceToDevice, st));
  }
  std::vector<long long> hs((size_t)k * 2);
  CU(cudaMemcpyAsync(hs.data(), g->bstat, (size_t)k * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < k; i++)
    if (hs[2 * i] & 0xFFFFFFFF) return fail(GBBS_EINTERNAL, "more than %lld BFS levels", b->lvl_cap);
  return GBBS_OK;
}

extern "C" int gbbs_betweenness_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                                      double *delta, void *cuda_stream) {
  return gbbs_betweenness_batch_ex(g, srcs, k, delta, cuda_stream, nullptr);
}

extern "C" int gbbs_betweenness(const gbbs_graph *g, uint32_t src, double *delta,
                                void *cuda_stream) {
  return gbbs_betweenness_ex(g, src, delta, cuda_stream, nullptr, nullptr);
}
