// traverse.cuh — the persistent frontier-traversal kernel (BFS and Bellman-Ford).
//
// One cooperative launch runs a whole traversal: per-run init (SURVEY §8(a)
// a1), then rounds of the paper's edgeMap (sec:prelims)
// separated by a grid-wide barrier (the round synchronisation of
// PAPER.md:89-90).  Inside a round every warp works on its own; the only other
// barrier is the one before heavy vertices of a bitmap-forward round.
//
// Round kinds (the representation is chosen per round from |U| + sum deg(U)
// against m/T; reading A10):
//  * list push (sparse, a3-a7).  The frontier is a vertex list whose entries
//    carry their exclusive edge prefix O (the scan of PAPER.md:1079-1080) and
//    base = offset(v) - O, both produced when the entry was appended.  The
//    round's d_U edges are cut into fixed tiles of TE edges, one warp per tile
//    (edgeMapBlocked's fixed-size blocks: a
//    high-degree vertex spans many tiles); a tile finds its owners with a
//    warp-wide 32-ary search of O (PAPER.md:1082's binary search).
//  * dense pull (a8, BFS).  Each unvisited vertex scans its in-edges in order
//    and stops at the first visited one (the early-exit dense method,
//    PAPER.md:1870-1874).  Every visited in-neighbour of an unvisited vertex
//    lies on the current level, so the visited bitmap (snapshot, double
//    buffered) serves as the frontier.  A warp owns whole 32-vertex words, so
//    the next bitmap is written without atomics; only (|U'|, sum deg) is
//    emitted.
//  * bitmap-forward push (a9/a10).  The frontier is a bitmap (BFS: the
//    vertices a dense round just added; Bellman-Ford: the next-frontier TS
//    bits); warps sweep its words and push the out-edges of its vertices
//    (lane per vertex, warp per vertex above 32 edges).  Vertices above HEAVY
//    edges are appended to a heavy list that is pushed with list-push tiles
//    after a grid barrier, so hubs are spread over many warps.
// F is the BFS test-and-set as an atomic fetch-or on the
// visited bit, or the Bellman-Ford priority-write as
// atomicMin on dist followed by a test-and-set on the next-frontier bit.
// Winners are packed per warp (ballot -> shared staging -> one packed 64-bit
// atomicAdd per flush), i.e. at most LN(U) writes.
#pragma once
// apply_batch returns early for wBFS (insertions instead of staging); the
// staging loops after it are then unreachable by design
#pragma nv_diag_suppress 128

#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

// Device-side bounds checks (build with -DGBBS_CHECKS; compiled out otherwise):
// every list, staging and edge-index write/read site below asserts its range and
// traps on a violation — the stand-in for compute-sanitizer, closed on this pool.
#ifdef GBBS_CHECKS
#define GBBS_CHECK(c)                                                              \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("GBBS_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);            \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define GBBS_CHECK(c) \
  do {                \
  } while (0)
#endif

namespace gbbs_dev {

namespace cg = cooperative_groups;

constexpr int BLOCK = 256;            // threads per CTA
constexpr int NWARPS = BLOCK / 32;
#ifndef GBBS_TE
#define GBBS_TE 256
#endif
constexpr int TE = GBBS_TE;           // edges per warp tile (edgeMapBlocked bsize)
#ifndef GBBS_SEARCH_EST
#define GBBS_SEARCH_EST 1
#endif
#ifndef GBBS_NCH
#define GBBS_NCH 4
#endif
constexpr int NCH = GBBS_NCH;         // 32-edge chunks in flight per batch
// single-owner list-push tiles of the weighted algorithms read targets and weights
// as 16-byte groups (push_tile): c4 Bellman-Ford -8 %; for BFS it measured +0.4..1.5 %
#ifndef GBBS_VEC_TILE
#define GBBS_VEC_TILE 1
#endif
#ifndef GBBS_WCAP
#define GBBS_WCAP 192
#endif
// per-warp staging capacity (vertices).  192 rather than 384: the kernels' static
// shared memory drops from 46 to 40 KB per CTA, so four CTAs fit the 164 KB
// shared-memory carve-out and L1 grows from ~60 to ~92 KB per SM (BFS c2/c4/c5
// -2 to -3.5 %, BF -3.7 %, 8-team BFS batch -3.3 %); adding 2 KB per CTA instead
// (a 228 KB carve-out, ~28 KB of L1) cost 20 %
constexpr int WCAP = GBBS_WCAP;
constexpr long long HEAVY = 512;      // bitmap-forward: deferred to heavy tiles above this
// wBFS bucket sweeps: vertices above this many edges go to the heavy list and are
// pushed in edge tiles by every warp after a barrier (a small bucket is swept one
// vertex per lane by few warps; warp-serial pushes of its 33-512-edge vertices
// made the rounds that expand rMAT's hubs the slowest of the run)
#ifndef GBBS_WBFS_HEAVY
#define GBBS_WBFS_HEAVY 32
#endif
constexpr long long WBFS_HEAVY = GBBS_WBFS_HEAVY;
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

// WP: widest path, (max, min) semiring; WBFS: integral-weight SSSP with buckets
enum Algo { ALGO_BFS = 0, ALGO_BF = 1, ALGO_WP = 2, ALGO_WBFS = 3 };
// EMIT_RED (Bellman-Ford, AUTO/SPARSE): no winners at all — the priority-write is
// a fire-and-forget reduction and the next frontier is the bitmap of the vertices
// it may have lowered (see apply_batch)
enum Emit { EMIT_LIST = 0, EMIT_COUNT = 1, EMIT_RED = 2 };
enum { LIST_HEAVY = 2 };

struct RoundStat {           // mirrors gbbs_round_stat
  int32_t dense;
  int32_t bucket;
  long long frontier;
  long long frontier_edges;
  long long acquired;
  long long edges_examined;
  long long vertices_swept;
  long long t_start_ns;
  long long t_work_ns;
  long long t_flush_ns;
  long long alg_bytes;       // algorithmic bytes at load granularity (STATS builds)
  long long head_hits;       // dense pull: acquired by the inline first in-edge
};

struct Params {
  long long n, m;
  const long long *off;      // out-CSR offsets [n+1]
  const uint32_t *tgt;       // out-CSR targets [m]
  const uint32_t *wgt;       // weights [m] or nullptr (unit)
  const long long *in_off;   // in-CSC (alias of CSR when symmetric)
  const uint32_t *in_tgt;
  const uint32_t *iso;       // [nwords] isolated-vertex (+padding) mask
  const uint32_t *nin;       // [nwords] no in-edges (+padding): never a pull candidate
  const uint4 *phot;         // [n] pull records (in0, in1, in2, out-degree), gbbs.cu k_pull_records
  const uint4 *pcold;        // [n]              (in3, in4, tail offset << 24 | tail count)
  // GBBS_REC8 layout: 8-byte hot records (in0, out-degree saturated to 31 bits | bit 31:
  // more in-edges), four per sector, and one 32-byte cold record per vertex:
  // (in1, in2, in3, in4) (tail lo, tail hi, out-degree, 0)
  const uint2 *phot8;        // [n]
  const uint4 *pc32;         // [2n]
  long long ncand;           // vertices with at least one in-edge
  uint32_t *dist;            // [n]
  uint16_t *shadow;          // [n] BF/WP: 16-bit conservative copy of dist
  uint8_t *lvl;              // [n] BFS: levels as bytes (bfs_set_dist), or nullptr: dist written directly
  uint32_t *parent;          // [n] or nullptr
  uint32_t *bm[2];           // BFS: visited (double-buffered); BF: frontier TS bits
  uint32_t *fv[3];           // lists 0/1 (rounds) and 2 (heavy): vertex
  long long *fo[3];          //   exclusive edge prefix O
  long long *fb[3];          //   base = offset(v) - O
  unsigned long long *cnt;   // packed (count << ebits | edges) ring [4]
  unsigned long long *hcnt;  // heavy-list packed counters [2]
  unsigned *bar;             // team barrier (count, generation) of a multi-traversal launch
  unsigned long long *wq;    // rings [4] + [4] of per-round work-queue counters (sweeps and
                             // list tiles; heavy-list tiles of a forward round)
  int *status;               // 0 ok, 1 = round cap hit
  long long *rounds_out;
  RoundStat *stats;          // per round, or nullptr
  long long stats_cap;
  long long nwords;
  long long dense_threshold; // dense iff |U| + sum deg(U) > dense_threshold
  long long max_rounds;
  unsigned long long *acq;   // BFS: ring [4] of per-round acquisition counts (reading A10b)
  int ebits;
  int mode;                  // 0 auto, 1 sparse, 2 dense, 3 pull
  int rules;                 // gbbs_opts.rules (GBBS_RULE_PAPER_ONLY = 1)
  int bsize;                 // list-push tile edges (power of two in [32, TE]); 0 = adaptive
  int symmetric;
  uint32_t src;
  // wBFS (ALGO_WBFS) bucket structure, wbfs_kernel
  uint32_t *bq;              // [nb][qcap] ring of bucket lists (vertex ids, circular)
  unsigned long long *btail; // [nb] monotone append counters of the bucket lists
  unsigned long long *bheavy;// [nb] monotone counters of heavy (deg > WBFS_HEAVY) entries
  uint32_t *xq[3];           // near lists: re-insertions into the current bucket
  unsigned long long *xcnt;  // [3] their counters, [3] heavy counters after them
  unsigned long long *pub;   // [3] per-round masks of bucket lists that got entries
  uint32_t *tag;             // [n] round tag deduplicating near-list insertions
  const uint32_t *hv;        // [nwords] out-degree > WBFS_HEAVY
  unsigned long long qcap;   // per-list capacity (power of two >= n)
  uint32_t delta;            // bucket width
  int nbq;                   // number of bucket lists (power of two)
  // signed Bellman-Ford (sbf_kernel)
  long long *sdist;          // [n] int64 distances
  int neg_scope;             // 0: all -inf on a negative cycle, 1: its forward closure
#if defined(GBBS_DBG_PHASE) || defined(GBBS_DIAG_TILE)
  unsigned long long *dbg;   // [64][4] per-round max phase durations (ns)
#endif
};

#ifndef GBBS_SWEEP_WORDS
#define GBBS_SWEEP_WORDS 32
#endif
constexpr int SWEEP_WORDS = GBBS_SWEEP_WORDS;  // max bitmap words gathered per warp step (sweeps)
// Sweep unit (words per warp step, a power of two <= SWEEP_WORDS) is chosen per
// traversal so that every warp gets at least this many units: on small graphs a
// 32-word unit per warp leaves the round waiting on the slowest unit.
#ifndef GBBS_UNITS_PER_WARP
#define GBBS_UNITS_PER_WARP 1
#endif
__device__ __forceinline__ int sweep_unit(long long nwords, long long nw) {
  int sw = SWEEP_WORDS;
  while (sw > 1 && (nwords + sw - 1) / sw < (long long)GBBS_UNITS_PER_WARP * nw) sw >>= 1;
  return sw;
}

struct TileSmem {              // list-push tile (shared-memory owner path)
  alignas(16) int32_t head[TE];  // 1 + owner index of the first edge slot of each owner
  long long base[TE + 1];        // owner base (offset - O)
  uint32_t own[TE + 1];          // owner vertex (BFS) or its distance (BF)
};

struct SweepSmem {             // bitmap sweeps: candidates of SWEEP_WORDS words, compacted
  uint32_t cand[SWEEP_WORDS * 32];
  uint32_t found[SWEEP_WORDS];
};

struct WarpSmem {             // one per warp; nothing here is shared across warps
  union {
    TileSmem t;
    SweepSmem s;
  } u;
  uint32_t stage[WCAP];          // winners awaiting warp_flush
};

struct Smem {
  WarpSmem w[NWARPS];
  unsigned long long sacc[7];
  unsigned long long cnt, hcnt, acq;
};

// Per-warp round state kept in registers: staging count, emitted (K, D) for
// EMIT_COUNT rounds, and gbbs_round_stat counters (STATS builds only).
struct WarpState {
  int scnt = 0;
  unsigned long long bk = 0;     // wBFS: bucket being processed
  unsigned long long pmask = 0;  // wBFS: bucket lists this lane appended to
  unsigned long long K = 0, D = 0;
  unsigned long long A = 0;      // BFS dense rounds: vertices acquired (warp-uniform)
  unsigned long long edges = 0, swept = 0, acquired = 0;
  unsigned long long ab = 0, hh = 0;  // STATS: algorithmic bytes, pull head hits
#ifdef GBBS_DIAG_LIST  // diagnostic builds: list-round phase timestamps
  unsigned long long t1 = 0, t2 = 0;
#endif
};

// ---- small device helpers --------------------------------------------------

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// the 16-bit distance shadow (BF / widest path / wBFS) is read and written by many
// threads at once: relaxed gpu-scope accesses, never plain ones
__device__ __forceinline__ uint32_t ld_relaxed16(const uint16_t *p) {
  unsigned short v;
  asm volatile("ld.relaxed.gpu.global.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_relaxed16(uint16_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Streaming accesses to graph arrays and outputs carry an L2 evict-first hint so
// that the multi-GB streams do not evict what must stay resident in the 126 MB
// L2: the visited/frontier bitmaps, the frontier lists, the counters and the
// kernel's own instructions (a cold instruction fetch from HBM costs ~1 us per
// line, which showed up as 10-60 us stalls on rarely run paths).
__device__ __forceinline__ unsigned long long ef_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint32_t ld_stream(const uint32_t *a) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(ef_policy()));
  return v;
}

__device__ __forceinline__ long long ld_stream64(const long long *a) {
  long long v;
  asm("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(ef_policy()));
  return v;
}

// one 32-byte (256-bit) load: sm_100's LDG.256 — a whole sector in one L2 request
__device__ __forceinline__ void ld_stream_v8(const uint32_t *a, uint4 &lo, uint4 &hi) {
  asm("ld.global.nc.L2::cache_hint.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
      : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
      : "l"(a), "l"(ef_policy()));
}

__device__ __forceinline__ uint2 ld_stream_v2(const uint32_t *a) {
  uint2 v;
  asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y)
      : "l"(a), "l"(ef_policy()));
  return v;
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint32_t *a) {
  uint4 v;
  asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(a), "l"(ef_policy()));
  return v;
}

// L2 prefetch of an upcoming stream line: a tile's target/weight chunks are
// requested up front, so the batch loads that follow hit L2 while the previous
// batch's atomics are in flight (GBBS_PREFETCH=0 disables).
#ifndef GBBS_PREFETCH
#define GBBS_PREFETCH 1
#endif
#ifndef GBBS_PREFETCH_W  // the weighted algorithms' register-path tiles too: off, c4 BF -2.3 %
#define GBBS_PREFETCH_W 0
#endif
// Bellman-Ford red rounds (EMIT_RED); 0 = the test-and-set list push of round 1
#ifndef GBBS_BF_RED
#define GBBS_BF_RED 1
#endif
__device__ __forceinline__ void prefetch_l2(const void *a) {
#if GBBS_PREFETCH
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a));
#endif
}

__device__ __forceinline__ void st_stream(uint32_t *a, uint32_t v) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(ef_policy())
               : "memory");
}

__device__ __forceinline__ void st_stream_v4(uint32_t *a, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "r"(x),
               "r"(y), "r"(z), "r"(w), "l"(ef_policy())
               : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifdef GBBS_DIAG_TILE
// diagnostic builds: phase durations of BFS list tiles, p.dbg[0..5] sums,
// [6] tiles, [7] flushes, [8..13] maxima (ns); dep() waits for a value
#define GBBS_DEP(x) asm volatile("" ::"r"((uint32_t)(x)))
__device__ __forceinline__ void diag_add(const unsigned long long *dbgc, int k,
                                         unsigned long long dt) {
  // one private 16-word slot per warp of the grid (no contention); host sums
  unsigned long long *dbg = const_cast<unsigned long long *>(dbgc);
  if ((threadIdx.x & 31) == 0 && dbg) {
    unsigned long long *sl = dbg + 16 * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    sl[k] += dt;
    sl[8 + k] = max(sl[8 + k], dt);
  }
}
#endif
// ---- BFS levels as bytes -------------------------------------------------------------
// A BFS acquisition writes dist[v] = r + 1 exactly once (the test-and-set winner).  As
// a scattered 4-byte store every such write is a partial-sector write that DRAM serves
// as a 32-byte read-modify-write (measured on c5: 23 % of the traversal time goes to
// the state stores).  The traversal therefore records levels below LVL_DIRECT in a
// byte array (Params.lvl, n bytes: the 16-bit shadow's buffer, which BFS does not
// use; 32 vertices per sector, mostly L2-resident) and one coalesced pass at the end expands
// it into dist (4-byte stores, whole lines, no fill at the start).  Levels from
// LVL_DIRECT on (graphs with more rounds than a byte holds) are stored in dist
// directly and flagged LVL_DIRECT so the final pass leaves them alone.  The host
// enables it for graphs above 2^24 vertices (gbbs.cu fill_params: on c2 / c3 the extra
// pass costs more than the stores save) or on request (GBBS_RULE_LEVEL_BYTES_ON).
constexpr uint32_t LVL_DIRECT = 254, LVL_INF = 255;

__device__ __forceinline__ void bfs_set_dist(const Params &p, uint32_t v, uint32_t d) {
  if (p.lvl) {
    if (d < LVL_DIRECT) {
      p.lvl[v] = (uint8_t)d;
    } else {
      p.lvl[v] = (uint8_t)LVL_DIRECT;
      st_stream(p.dist + v, d);
    }
  } else {
    st_stream(p.dist + v, d);
  }
}

__device__ __forceinline__ bool vbit(const uint32_t *vis, uint32_t u) {
  return (vis[u >> 5] >> (u & 31)) & 1u;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned lanemask_le() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(r));
  return r;
}

__device__ __forceinline__ long long warp_sum64(long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

__device__ __forceinline__ long long warp_excl_sum64(long long x, int lane) {
  long long inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  return inc - x;
}

// Largest i in [lo, hi) with O[i] <= key, given O[lo] <= key and O strictly
// increasing: a warp-cooperative 32-ary search (log32(hi-lo) dependent L2 loads),
// the binary search of edgeMapBlocked widened to a warp.
__device__ __forceinline__ long long warp_upper(const long long *O, long long lo, long long hi,
                                                long long key) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const long long step = (hi - lo + 31) >> 5;
    const long long idx = lo + (long long)lane * step;
    const bool ok = idx < hi && __ldcg(O + idx) <= key;
    const unsigned bb = __ballot_sync(FULL, ok);
    lo += (long long)(31 - __clz(bb)) * step;
    hi = min(hi, lo + step);
  }
  const long long idx = lo + lane;
  const bool ok = idx < hi && __ldcg(O + idx) <= key;
  return lo + (31 - __clz(__ballot_sync(FULL, ok)));
}

// Owner search of edge `key` in a list of f entries holding E edges, with an
// interpolation first probe: the 32 entries around key * f / E answer in one
// round trip when the frontier's degrees are near-uniform (the torus: the plain
// 32-ary search costs 4 dependent loads there at 10^5 entries); otherwise the
// probe narrows the range to one side and warp_upper finishes.  Same result as
// warp_upper(O, 0, f, key) (O non-decreasing, O[0] = 0 <= key).
__device__ __forceinline__ long long warp_upper_est(const long long *O, long long f, long long E,
                                                    long long key) {
  if (GBBS_SEARCH_EST && f > 64) {
    const int lane = threadIdx.x & 31;
    const long long est = (long long)((double)key * (double)f / (double)E);
    const long long base = min(max(est - 16, 0ll), f - 32);
    const unsigned bb = __ballot_sync(FULL, __ldcg(O + base + lane) <= key);
    if (bb == 0) return warp_upper(O, 0, base, key);
    if (bb == FULL) return warp_upper(O, base + 31, f, key);
    return base + 31 - __clz(bb);
  }
  return warp_upper(O, 0, f, key);
}

// Append the lanes' (v, a = offset(v), deg > 0) to list `nb` at positions and
// edge prefixes reserved by one packed atomicAdd on *ctr (warp-uniform call).
__device__ __forceinline__ void warp_append(const Params &p, int nb, unsigned long long *ctr,
                                            bool keep, uint32_t v, long long a, long long deg) {
  const int lane = threadIdx.x & 31;
  const unsigned bal = __ballot_sync(FULL, keep);
  if (!bal) return;
  const long long dg = keep ? deg : 0;
  const long long dex = warp_excl_sum64(dg, lane);
  const long long tot = __shfl_sync(FULL, dex + dg, 31);
  unsigned long long old = 0;
  if (lane == 0) old = atomicAdd(ctr, ((unsigned long long)__popc(bal) << p.ebits) | (unsigned long long)tot);
  old = __shfl_sync(FULL, old, 0);
  if (keep) {
    const unsigned long long pos = (old >> p.ebits) + __popc(bal & lanemask_lt());
    const long long o = (long long)(old & ((1ull << p.ebits) - 1)) + dex;
    GBBS_CHECK(pos < (unsigned long long)p.n);
    p.fv[nb][pos] = v;
    p.fo[nb][pos] = o;
    p.fb[nb][pos] = a - o;
  }
}

// Write `cnt` staged vertices of this warp into the next frontier list (a7).
// Out-degree-0 vertices are dropped (no edges to process).  ONE packed 64-bit
// atomicAdd of (count, edge-sum) reserves positions AND their exclusive edge
// prefix O, so the next round needs no degree scan.  Offsets are loaded FL
// entries per lane at a time.  Warp-uniform call.
template <int ALGO, bool CARRY = false>
__device__ __forceinline__ void warp_flush(const Params &p, const uint32_t *st, int cnt, int nb,
                                           int r, uint32_t *bits_next,
                                           unsigned long long *tmark = nullptr,
                                           unsigned long long *ctr = nullptr,
                                           unsigned long long *abp = nullptr) {
  constexpr int FL = 4;
  const int lane = threadIdx.x & 31;
#ifdef GBBS_DBG_PHASE
  const unsigned long long tA = globaltimer_ns();
#endif
  __syncwarp();
  long long Kl = 0, Dl = 0;
  for (int b0 = 0; b0 < cnt; b0 += 32 * FL) {
    long long lo[FL], hi[FL];
#pragma unroll
    for (int u = 0; u < FL; u++) {
      const int i = b0 + 32 * u + lane;
      lo[u] = hi[u] = 0;
      if (i < cnt) {
        const uint32_t v = st[i];
        lo[u] = __ldg(p.off + v);
        hi[u] = __ldg(p.off + v + 1);
        if (abp) *abp += 16;  // STATS: the offset pair
      }
    }
#pragma unroll
    for (int u = 0; u < FL; u++) {
      Kl += hi[u] > lo[u];
      Dl += hi[u] - lo[u];
    }
  }
  const unsigned long long K = warp_sum64(Kl), D = warp_sum64(Dl);
#ifdef GBBS_DBG_PHASE
  const unsigned long long tB = globaltimer_ns();
#endif
  unsigned long long old = 0;
  if (lane == 0 && K) old = atomicAdd(ctr ? ctr : p.cnt + ((r + 1) & 3), (K << p.ebits) | D);
  old = __shfl_sync(FULL, old, 0);
#ifdef GBBS_DBG_PHASE
  const unsigned long long tC = globaltimer_ns();
  if (tmark) *tmark = tC;
#endif
  unsigned long long k = old >> p.ebits;
  unsigned long long d = old & ((1ull << p.ebits) - 1);
  uint32_t *fv = p.fv[nb];
  long long *fo = p.fo[nb];
  long long *fb = p.fb[nb];
  for (int b0 = 0; b0 < cnt; b0 += 32 * FL) {
    uint32_t vv[FL];
    long long lo[FL], hi[FL];
#pragma unroll
    for (int u = 0; u < FL; u++) {
      const int i = b0 + 32 * u + lane;
      vv[u] = 0;
      lo[u] = hi[u] = 0;
      if (i < cnt) {
        vv[u] = st[i];
        lo[u] = __ldg(p.off + vv[u]);
        hi[u] = __ldg(p.off + vv[u] + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < FL; u++) {
      const int i = b0 + 32 * u + lane;
      const long long deg = hi[u] - lo[u];
      const bool keep = deg > 0;
      const unsigned bal = __ballot_sync(FULL, keep);
      const long long dex = warp_excl_sum64(deg, lane);
      const unsigned long long pos = k + __popc(bal & lanemask_lt());
      const long long o = (long long)d + dex;
      if (keep) {
        GBBS_CHECK(pos < (unsigned long long)p.n);
        if (abp) *abp += 20;  // STATS: the entry (v, O, base)
        // CARRY (Bellman-Ford red rounds): the entry carries dist(v) as of the
        // round's start instead of v, so tiles need no owner-distance loads
        fv[pos] = CARRY ? ld_relaxed(p.dist + vv[u]) : vv[u];
        fo[pos] = o;
        fb[pos] = lo[u] - o;
      } else if (!CARRY && (ALGO == ALGO_BF || ALGO == ALGO_WP) && i < cnt) {
        // out-degree-0 vertex: it never enters a frontier; release its TS bit.
        atomicAnd(bits_next + (vv[u] >> 5), ~(1u << (vv[u] & 31)));
      }
      k += __popc(bal);
      d += (unsigned long long)__shfl_sync(FULL, dex + deg, 31);
    }
  }
  __syncwarp();
#ifdef GBBS_DBG_PHASE
  const unsigned long long tD = globaltimer_ns();
  if (lane == 0 && r < 64 && p.dbg) {
    atomicMax(p.dbg + 4 * r + 0, tB - tA);
    atomicMax(p.dbg + 4 * r + 1, tC - tB);
    atomicMax(p.dbg + 4 * r + 2, tD - tC);
    atomicMax(p.dbg + 4 * r + 3, (unsigned long long)cnt);
  }
#endif
}

// ---- wBFS bucket insertion ------------------------------------------------------------
// A vertex whose distance the priority-write lowered from `old` to `nd` moves to
// bucket nd / delta (Julienne's bucket update after edgeMapData).
// Into the bucket being processed it goes to the near list of this round (once
// per round: round tag); into a later bucket it is appended to that bucket's list
// unless it already sits there (old in the same bucket: the list holds it
// unprocessed, since distances only fall).  Lanes aiming at the same list are
// grouped with match.any and reserve their slots with ONE atomicAdd.
constexpr uint32_t XKEY = 64;    // near list
// wBFS lane-owned push loop batch width (A/B knob: 8 and 16 edges per batch
// measured 8 % and 20-65 % slower than 4 on c3/c4, tools/cmp_lib.sh)
#ifndef GBBS_WBFS_LB
#define GBBS_WBFS_LB 4
#endif
constexpr int WBFS_LB = GBBS_WBFS_LB;
// a staging flush leaves room for one whole batch: WCAP - 32 * (chunks per batch)
// must not be negative, or a batch could overrun the warp's staging buffer
static_assert(WCAP >= 32 * NCH && WCAP >= 32 * WBFS_LB, "WCAP below one batch of winners");
constexpr uint32_t NOKEY = 0xFFFFFFFFu;

// Per-warp wBFS staging metadata in dynamic shared memory (wbfs_kernel only):
// the list key of every staged vertex and a 65-bin histogram over the keys.
struct WbfsWarpSmem {
  uint32_t hist[XKEY + 1];
  uint32_t hh[XKEY + 1];  // heavy entries per key (one counter atomic per key and flush)
  uint8_t key[WCAP];
};
extern __shared__ __align__(16) unsigned char gbbs_dyn_smem[];
__device__ __forceinline__ WbfsWarpSmem &wbfs_smem() {
  return reinterpret_cast<WbfsWarpSmem *>(gbbs_dyn_smem)[threadIdx.x >> 5];
}

// Flush the warp's staged insertions: one shared-memory histogram over the list
// keys, then ONE atomicAdd per (list, flush) reserves the slots — the bucket
// tails are the hottest addresses of the run, so per-lane reservations would
// serialise on them — and every vertex is written at base + its rank in its
// list.  Warp-uniform call.
template <bool STATS>
__device__ __forceinline__ void wbfs_flush(const Params &p, WarpState &ws, const uint32_t *st, int cnt,
                                        int r) {
  const int lane = threadIdx.x & 31;
  const int xr = r % 3;
  WbfsWarpSmem &w = wbfs_smem();
  __syncwarp();
  for (int i = lane; i < cnt; i += 32) atomicAdd(&w.hist[w.key[i]], 1u);
  __syncwarp();
  const uint32_t hA = w.hist[lane], hB = w.hist[lane + 32], hX = w.hist[XKEY];
  unsigned long long bA = 0, bB = 0, bX = 0;
  if (hA) bA = atomicAdd(p.btail + lane, (unsigned long long)hA);
  if (hB) bB = atomicAdd(p.btail + lane + 32, (unsigned long long)hB);
  if (lane == 0 && hX) bX = atomicAdd(p.xcnt + xr, (unsigned long long)hX);
  ws.pmask |= (hA ? 1ull << lane : 0ull) | (hB ? 1ull << (lane + 32) : 0ull);
  __syncwarp();
  w.hist[lane] = 0;
  w.hist[lane + 32] = 0;
  if (lane == 0) w.hist[XKEY] = 0;
  __syncwarp();
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t key = i < cnt ? w.key[i] : 0u;
    const unsigned long long x0 = __shfl_sync(FULL, bA, key & 31);
    const unsigned long long x1 = __shfl_sync(FULL, bB, key & 31);
    const unsigned long long x2 = __shfl_sync(FULL, bX, 0);
    if (i < cnt) {
      const uint32_t v = st[i];
      const unsigned long long pos =
          (key == XKEY ? x2 : (key >= 32 ? x1 : x0)) + atomicAdd(&w.hist[key], 1u);
      if (key == XKEY) {
        GBBS_CHECK(pos < (unsigned long long)p.n);
        p.xq[xr][pos] = v;
      } else
        p.bq[(unsigned long long)key * p.qcap + (pos & (p.qcap - 1))] = v;
      if ((__ldg(p.hv + (v >> 5)) >> (v & 31)) & 1u) atomicAdd(&w.hh[key], 1u);
    }
  }
  __syncwarp();
  {
    const uint32_t gA = w.hh[lane], gB = w.hh[lane + 32];
    if (gA) atomicAdd(p.bheavy + lane, (unsigned long long)gA);
    if (gB) atomicAdd(p.bheavy + lane + 32, (unsigned long long)gB);
    if (lane == 0 && w.hh[XKEY]) atomicAdd(p.xcnt + 3 + xr, (unsigned long long)w.hh[XKEY]);
  }
  __syncwarp();
  w.hist[lane] = 0;
  w.hist[lane + 32] = 0;
  w.hh[lane] = 0;
  w.hh[lane + 32] = 0;
  if (lane == 0) w.hist[XKEY] = w.hh[XKEY] = 0;
  if (STATS && lane == 0) ws.acquired += cnt;
  __syncwarp();
}

// Stage the vertices whose distance the priority-write lowered (bucket update).
template <bool STATS, int NB>
__device__ __forceinline__ void wbfs_stage(const Params &p, WarpState &ws, uint32_t *st,
                                           const bool (&cand)[NB], const uint32_t (&v)[NB],
                                           const uint32_t (&nd)[NB],
                                           const uint32_t (&old)[NB], int r) {
  WbfsWarpSmem &w = wbfs_smem();
#pragma unroll
  for (int j = 0; j < NB; j++) {
    uint32_t key = NOKEY;
    if (cand[j]) {
      const uint32_t b = nd[j] / p.delta;
      if (b == ws.bk) {
        if (atomicExch(p.tag + v[j], (uint32_t)(r + 1)) != (uint32_t)(r + 1)) key = XKEY;
      } else if (old[j] == INF || old[j] / p.delta != b) {
        key = (uint32_t)(b & (unsigned long long)(p.nbq - 1));
      }
    }
    const unsigned bal = __ballot_sync(FULL, key != NOKEY);
    GBBS_CHECK(ws.scnt + __popc(bal) <= WCAP);
    if (key != NOKEY) {
      const int idx = ws.scnt + __popc(bal & lanemask_lt());
      st[idx] = v[j];
      w.key[idx] = (uint8_t)key;
    }
    ws.scnt += __popc(bal);
  }
  if (ws.scnt > WCAP - 32 * (WBFS_LB > NCH ? WBFS_LB : NCH)) {  // room for the widest batch
    wbfs_flush<STATS>(p, ws, st, ws.scnt, r);
    ws.scnt = 0;
  }
}

// ---- F: apply one batch of NCH 32-edge chunks -------------------------------------
// vv = targets, uu = owner id (BFS parent) or owner distance (BF), ww = weights.
// EMIT_LIST: winners go to the warp's staging buffer (flushed into list cb^1).
// EMIT_COUNT: winners are only counted (K, D) — the TS bits are the frontier.
template <int ALGO, bool STATS, int EMIT, int NB>
__device__ __forceinline__ void apply_batch(const Params &p, uint32_t *st, WarpState &ws,
                                            const uint32_t (&vv)[NB], const uint32_t (&uu)[NB],
                                            const uint32_t (&ww)[NB], const bool (&act)[NB],
                                            int nb, int r, uint32_t *bits, const uint32_t *prebits) {
  const int lane = threadIdx.x & 31;
  bool win[NB];
  if (ALGO == ALGO_BFS) {
#ifdef GBBS_DIAG_TILE
    const unsigned long long tA0 = globaltimer_ns();
#pragma unroll
    for (int j = 0; j < NB; j++) GBBS_DEP(vv[j]);
    const unsigned long long tA1 = globaltimer_ns();
#endif
    uint32_t pre[NB];
#pragma unroll
    for (int j = 0; j < NB; j++)
      pre[j] = act[j] ? ld_relaxed(prebits + (vv[j] >> 5)) : FULL;  // words others fetch-or
#ifdef GBBS_DIAG_TILE
#pragma unroll
    for (int j = 0; j < NB; j++) GBBS_DEP(pre[j]);
    const unsigned long long tA2 = globaltimer_ns();
#endif
#pragma unroll
    for (int j = 0; j < NB; j++) {
      const uint32_t bit = 1u << (vv[j] & 31);
      win[j] = false;
      if (!(pre[j] & bit)) {
        const uint32_t old = atomicOr(bits + (vv[j] >> 5), bit);  // test-and-set
        win[j] = !(old & bit);
#ifdef GBBS_DIAG_ATOMS  // diagnostic builds: executed test-and-sets in `swept`
        if (STATS) ws.swept += 1;
#endif
      }
    }
#ifdef GBBS_DIAG_TILE
#pragma unroll
    for (int j = 0; j < NB; j++) GBBS_DEP(win[j]);
    const unsigned long long tA3 = globaltimer_ns();
    if (EMIT == EMIT_LIST) {
      diag_add(p.dbg, 2, tA1 - tA0);
      diag_add(p.dbg, 3, tA2 - tA1);
      diag_add(p.dbg, 4, tA3 - tA2);
    }
#endif
#pragma unroll
    for (int j = 0; j < NB; j++) {
      if (win[j]) {
#ifndef GBBS_DIAG_NOSTATE  // diagnostic builds (results invalid): cost of the state writes
        bfs_set_dist(p, vv[j], (uint32_t)(r + 1));
        if (p.parent) st_stream(p.parent + vv[j], uu[j]);
#endif
      }
    }
  } else {
    // Bellman-Ford: candidate d(u)+w, priority = smaller (atomicMin).
    // Widest path: candidate min(width(u), w), priority = larger (atomicMax) —
    // the (max, min) semiring in place of (min, +).
    uint32_t nd[NB];
    // Pre-check against the 16-bit shadow of dist (half the bytes of dist, meant
    // to stay in L2): BF keeps shadow >= min(dist, 0xFFFF) because distances only
    // fall and the shadow only ever receives values dist held; WP keeps
    // shadow <= width.  A relaxation the shadow proves useless is skipped; the
    // others go straight to the priority-write, whose returned old value decides.
    uint32_t cur[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
      // saturating: a sum reaching 2^32 - 1 cannot be stored below the INF
      // sentinel; it is flagged (status bit 2 -> GBBS_ERANGE) instead of the
      // conservative up-front check max(w) * (n - 1) < 2^32 - 1
      if (ALGO == ALGO_WP) {
        nd[j] = min(uu[j], ww[j]);
      } else {
        const uint32_t sum = uu[j] + ww[j];
        const bool ovf = sum < uu[j] || sum == INF;
        nd[j] = ovf ? INF : sum;
        if (ovf && act[j]) atomicOr(p.status, 2);
      }
      cur[j] = act[j] ? ld_relaxed16(p.shadow + vv[j]) : (ALGO == ALGO_WP ? 0xFFFFu : 0u);
    }
    if constexpr (EMIT == EMIT_RED && ALGO == ALGO_BF) {
      // Fire-and-forget priority-write: red.min on dist (its old value is not
      // waited for), the shadow lowered to the candidate, and v marked in the
      // next frontier bitmap with red.or.  The shadow stays an upper bound of the
      // distance dist(v) reaches this round: it only receives candidates, and
      // each candidate's red.min is issued before its shadow store.
      // The shadow is only a pre-filter (racy stores can leave it above dist); a
      // candidate it passes is confirmed against dist itself, which only falls: a
      // candidate below the dist value read means dist(v) falls this round, so
      // every mark is a vertex that improved (and the rounds end)
      bool pass[NB];
      uint32_t dv[NB];
#pragma unroll
      for (int j = 0; j < NB; j++) {
        pass[j] = act[j] && nd[j] != INF && (nd[j] < cur[j] || cur[j] == 0xFFFFu);
        dv[j] = pass[j] ? ld_relaxed(p.dist + vv[j]) : 0u;
      }
      bool mk = false;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        if (pass[j] && nd[j] < dv[j]) {
          atomicMin(p.dist + vv[j], nd[j]);  // result unused: RED.MIN
          st_relaxed16(p.shadow + vv[j], min(nd[j], 0xFFFFu));
          atomicOr(bits + (vv[j] >> 5), 1u << (vv[j] & 31));  // RED.OR
          mk = true;
#ifdef GBBS_DIAG_ATOMS
          if (STATS) ws.swept += 1;
#endif
        }
      }
      ws.K |= mk;  // any mark: the frontier is not empty
      return;
    }
    bool cand[NB];
    uint32_t oldv[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
      cand[j] = false;
      oldv[j] = 0;
      if (!act[j]) continue;
      if (ALGO == ALGO_WP) {
        if (nd[j] > cur[j]) {
          const uint32_t old = atomicMax(p.dist + vv[j], nd[j]);  // priority-write
          cand[j] = nd[j] > old;
        }
      } else if (nd[j] < cur[j] || cur[j] == 0xFFFFu) {
        const uint32_t old = atomicMin(p.dist + vv[j], nd[j]);  // priority-write
        cand[j] = nd[j] < old;
#ifdef GBBS_DIAG_ATOMS  // diagnostic builds: executed priority-writes in `swept`
        if (STATS) ws.swept += 1;
#endif
        oldv[j] = old;
      }
    }
#pragma unroll
    for (int j = 0; j < NB; j++)
      if (cand[j]) st_relaxed16(p.shadow + vv[j], min(nd[j], 0xFFFFu));
    if constexpr (ALGO == ALGO_WBFS) {
      wbfs_stage<STATS, NB>(p, ws, st, cand, vv, nd, oldv, r);
      return;
    }
#pragma unroll
    for (int j = 0; j < NB; j++) {
      win[j] = false;
      if (cand[j]) {
        const uint32_t bit = 1u << (vv[j] & 31);
        const uint32_t ob = atomicOr(bits + (vv[j] >> 5), bit);  // next-frontier TS
        win[j] = !(ob & bit);
      }
    }
  }
  if (EMIT == EMIT_COUNT) {
    long long lo[NB], hi[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
      lo[j] = hi[j] = 0;
      if (win[j]) {
        lo[j] = __ldg(p.off + vv[j]);
        hi[j] = __ldg(p.off + vv[j] + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; j++) {
      ws.K += hi[j] > lo[j];
      ws.D += (unsigned long long)(hi[j] - lo[j]);
      if (STATS) ws.acquired += win[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < NB; j++) {
      const unsigned b = __ballot_sync(FULL, win[j]);
      GBBS_CHECK(ws.scnt + __popc(b) <= WCAP);
      if (win[j]) st[ws.scnt + __popc(b & lanemask_lt())] = vv[j];
      ws.scnt += __popc(b);
    }
    if (ws.scnt > WCAP - 32 * NB) {
      if (STATS && lane == 0) ws.acquired += ws.scnt;
      warp_flush<ALGO>(p, st, ws.scnt, nb, r, bits, nullptr, nullptr, STATS ? &ws.ab : nullptr);
      ws.scnt = 0;
    }
  }
}

// ---- list push: one warp, one tile of TE edges of list `lb` ---------------------
// Tiles are handed to warps in contiguous blocks, so a warp searches O once per
// round (warp_upper) and then carries the owner index from tile to tile: a
// tile's owners are i0, i0+1, ... while O < te, discovered from the owner loads
// the tile needs anyway.  Returns the first owner of the next tile.

template <int ALGO, bool STATS, int EMIT>
__device__ __forceinline__ long long push_tile(const Params &p, WarpSmem &wsm, WarpState &ws,
                                               int lb, long long i0, long long t, long long f,
                                               long long E, int nb, int r, uint32_t *bits,
                                               const uint32_t *prebits, int TR) {
  constexpr long long BIG = 0x7FFFFFFFFFFFFFFFll;
  constexpr bool W = ALGO != ALGO_BFS;  // weights, owner distances
  const int lane = threadIdx.x & 31;
  const long long ts = t * TR;
  const long long te = min(ts + (long long)TR, E);
  const long long *O = p.fo[lb];
  const long long *B = p.fb[lb];
  const uint32_t *F = p.fv[lb];
  if (STATS && lane == 0) {
    ws.edges += (unsigned long long)(te - ts);
    ws.ab += (unsigned long long)(te - ts) * ((W && p.wgt) ? 8 : 4);
  }
#ifdef GBBS_DIAG_TILE
  const unsigned long long tT0 = globaltimer_ns();
#endif

  const long long k = i0 + lane;
  // O, base and vertex of the next 32 entries are loaded together (the base and
  // vertex speculatively), so the owner set costs one round trip
  long long Ok = BIG, Bk = 0;
  uint32_t Uk = 0;
  if (k < f) {
    Ok = __ldcg(O + k);
    Bk = __ldcg(B + k);
    Uk = __ldcg(F + k);
    if (STATS) ws.ab += 20;  // frontier entry (v, O, base)
  }
  const unsigned inb = __ballot_sync(FULL, Ok < te);  // owners with an edge in the tile
  const int n32 = __popc(inb);
#ifdef GBBS_DIAG_TILE
  GBBS_DEP(Bk); GBBS_DEP(Uk);
  if (ALGO == ALGO_BFS) {
    diag_add(p.dbg, 1, globaltimer_ns() - tT0);
    diag_add(p.dbg, 6, 1);
  }
#endif
#if GBBS_VEC_TILE
  if (W && n32 == 1) {
    // Single-owner tile (a hub's edges, the bulk of rMAT's big rounds): the tile is
    // the contiguous range [bb + ts, bb + te) of the owner's targets (weights), read
    // as aligned 16-byte groups — 4 edges per lane, a batch of 128 edges per step —
    // with no per-chunk owner search.  Elements of a group outside the range are
    // masked off (the arrays are readable up to the next 16-byte boundary, gbbs.h).
    const long long bb = __shfl_sync(FULL, Bk, 0);
    uint32_t u0 = __shfl_sync(FULL, Uk, 0);
    if (W && EMIT != EMIT_RED) u0 = ld_relaxed(p.dist + u0);
    const long long onext = __shfl_sync(FULL, Ok, 1);
    const long long a = bb + ts, b = bb + te;
    for (long long g0 = a & ~3ll; g0 < b; g0 += 128) {
      const long long gi = g0 + 4 * lane;
      uint4 tv = make_uint4(0, 0, 0, 0), wv = make_uint4(1, 1, 1, 1);
      if (gi < b) {
        GBBS_CHECK(gi >= 0 && gi < p.m);
        tv = ld_stream_v4(p.tgt + gi);
        if (W && p.wgt) wv = ld_stream_v4(p.wgt + gi);
      }
      uint32_t vv[4] = {tv.x, tv.y, tv.z, tv.w}, ww[4] = {wv.x, wv.y, wv.z, wv.w};
      uint32_t uu[4] = {u0, u0, u0, u0};
      bool act[4];
#pragma unroll
      for (int j = 0; j < 4; j++) act[j] = gi + j >= a && gi + j < b;
      apply_batch<ALGO, STATS, EMIT>(p, wsm.stage, ws, vv, uu, ww, act, nb, r, bits, prebits);
    }
    return onext == te ? i0 + 1 : i0;
  }
#endif
  if (n32 < 32) {
    // Register path: lane k holds owner i0+k; a chunk's owners come from a
    // ballot (owners starting at or before the chunk) plus an or-reduce of the
    // owners starting inside it.
    const long long onext = __shfl_sync(FULL, Ok, n32);
    const bool valid = lane < n32;
    if (!valid) Ok = BIG;
    uint32_t Xk = Uk;
    if (W && EMIT != EMIT_RED) Xk = valid ? ld_relaxed(p.dist + Uk) : 0;
    // owner starts relative to the tile, clamped to [-1, TR + 32] (32-bit compares;
    // every owner starting at or before the tile behaves alike)
    const int tn = (int)(te - ts);
    const int ro = (int)max(-1ll, min(Ok - ts, (long long)TR + 32));
    const long long Bt = Bk + ts;  // owner's target index of the tile's first slot
    if (GBBS_PREFETCH && (!W || GBBS_PREFETCH_W) && tn > 32 * NCH) {
      for (int cr = 32 * NCH; cr < tn; cr += 32) {
        const int c0 = __popc(__ballot_sync(FULL, ro <= cr)) - 1;
        const int rel = ro - cr;
        const unsigned hm = __reduce_or_sync(FULL, (rel > 0 && rel < 32) ? (1u << rel) : 0u);
        const long long bb = __shfl_sync(FULL, Bt, c0 + __popc(hm & lanemask_le()));
        if (cr + lane < tn) {
          prefetch_l2(p.tgt + bb + cr + lane);
          if (W && p.wgt) prefetch_l2(p.wgt + bb + cr + lane);
        }
      }
    }
    for (int cs = 0; cs < tn; cs += 32 * NCH) {
      uint32_t vv[NCH], ww[NCH], uu[NCH];
      bool act[NCH];
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        const int cr = cs + 32 * j;
        const int e = cr + lane;
        act[j] = e < tn;
        vv[j] = 0;
        ww[j] = 0;
        uu[j] = 0;
        if (cr < tn) {  // warp-uniform
          const int c0 = __popc(__ballot_sync(FULL, ro <= cr)) - 1;
          const int rel = ro - cr;
          const unsigned hb = (rel > 0 && rel < 32) ? (1u << rel) : 0u;
          const unsigned hm = __reduce_or_sync(FULL, hb);
          const int own = c0 + __popc(hm & lanemask_le());
          const long long bb = __shfl_sync(FULL, Bt, own);
          uu[j] = __shfl_sync(FULL, Xk, own);
          if (act[j]) {
            GBBS_CHECK(bb + e >= 0 && bb + e < p.m);
            vv[j] = ld_stream(p.tgt + bb + e);
            if (W) ww[j] = p.wgt ? ld_stream(p.wgt + bb + e) : 1u;
          }
        }
      }
      apply_batch<ALGO, STATS, EMIT>(p, wsm.stage, ws, vv, uu, ww, act, nb, r, bits, prebits);
    }
    return onext == te ? i0 + n32 : i0 + n32 - 1;
  }
  // Shared-memory path (many low-degree owners): stage every owner of the tile,
  // mark the slot where each owner's first in-tile edge lies (1 + owner index),
  // and expand owner ids over the TE slots with a warp max-scan.
  TileSmem &w = wsm.u.t;
  {
    int4 *h4 = reinterpret_cast<int4 *>(w.head);
#pragma unroll
    for (int q = 0; q < TE / 128; q++) h4[q * 32 + lane] = make_int4(0, 0, 0, 0);
  }
  __syncwarp();
  int nown = 0;
  long long onext = BIG;
  for (int kb = 0;; kb += 64) {
    long long o2[2], b2[2];
    uint32_t u2[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const long long kk = i0 + kb + 32 * h + lane;
      o2[h] = BIG;
      b2[h] = 0;
      u2[h] = 0;
      if (kk < f) {
        o2[h] = __ldcg(O + kk);
        b2[h] = __ldcg(B + kk);
        u2[h] = __ldcg(F + kk);
        if (STATS) ws.ab += 20;
      }
    }
    int cnt_h[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int kk = kb + 32 * h + lane;
      cnt_h[h] = __popc(__ballot_sync(FULL, o2[h] < te));
      if (o2[h] < te) {
        w.base[kk] = b2[h];
        w.own[kk] = (W && EMIT != EMIT_RED) ? ld_relaxed(p.dist + u2[h]) : u2[h];
        const long long o = o2[h] - ts;
        w.head[o > 0 ? o : 0] = kk + 1;
      }
    }
    nown += cnt_h[0] + cnt_h[1];
    if (cnt_h[0] < 32) {
      onext = __shfl_sync(FULL, o2[0], cnt_h[0]);
      break;
    }
    if (cnt_h[1] < 32) {
      onext = __shfl_sync(FULL, o2[1], cnt_h[1]);
      break;
    }
  }
  __syncwarp();
  {
    constexpr int PER = TE / 32;
    int32_t a[PER];
    const int4 *h4 = reinterpret_cast<const int4 *>(w.head + lane * PER);
#pragma unroll
    for (int q = 0; q < PER / 4; q++) {
      const int4 x = h4[q];
      a[4 * q] = x.x; a[4 * q + 1] = x.y; a[4 * q + 2] = x.z; a[4 * q + 3] = x.w;
    }
#pragma unroll
    for (int q = 1; q < PER; q++) a[q] = max(a[q], a[q - 1]);
    int32_t inc = a[PER - 1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc = max(inc, y);
    }
    int32_t ex = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) ex = 0;
    int4 *o4 = reinterpret_cast<int4 *>(w.head + lane * PER);
#pragma unroll
    for (int q = 0; q < PER / 4; q++)
      o4[q] = make_int4(max(ex, a[4 * q]), max(ex, a[4 * q + 1]), max(ex, a[4 * q + 2]),
                        max(ex, a[4 * q + 3]));
  }
  __syncwarp();
  if (GBBS_PREFETCH) {
    for (long long e = ts + 32 * NCH + lane; e < te; e += 32) {
      const long long bb = w.base[w.head[e - ts] - 1];
      prefetch_l2(p.tgt + bb + e);
      if (W && p.wgt) prefetch_l2(p.wgt + bb + e);
    }
  }
  for (long long cs = ts; cs < te; cs += 32 * NCH) {
    uint32_t vv[NCH], ww[NCH], uu[NCH];
    bool act[NCH];
#pragma unroll
    for (int j = 0; j < NCH; j++) {
      const long long e = cs + 32 * j + lane;
      act[j] = e < te;
      vv[j] = 0;
      ww[j] = 0;
      uu[j] = 0;
      if (act[j]) {
        const int kk = w.head[e - ts] - 1;
        const long long bb = w.base[kk];
        uu[j] = w.own[kk];
        GBBS_CHECK(bb + e >= 0 && bb + e < p.m);
        vv[j] = ld_stream(p.tgt + bb + e);
        if (W) ww[j] = p.wgt ? ld_stream(p.wgt + bb + e) : 1u;
      }
    }
    apply_batch<ALGO, STATS, EMIT>(p, wsm.stage, ws, vv, uu, ww, act, nb, r, bits, prebits);
  }
  __syncwarp();
  return onext == te ? i0 + nown : i0 + nown - 1;
}

// ---- bitmap sweeps: gather + compact --------------------------------------------
// A warp takes SWEEP_WORDS consecutive bitmap words (one per lane, coalesced),
// compacts the candidate vertices of all of them into shared memory in vertex
// order, and then works through them 32 (or 64) at a time, one per lane — so a
// sparse bitmap costs one step per 32 candidates, not one per 32 vertices.

// Compact the set bits of lane-owned words (word w0 + lane) into w.cand.
// Returns the number of candidates (warp-uniform).
__device__ __forceinline__ int warp_gather(SweepSmem &w, long long w0, uint32_t bits) {
  const int lane = threadIdx.x & 31;
  int c = __popc(bits), inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  int k = inc - c;
  const uint32_t base = (uint32_t)((w0 + lane) * 32);
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    w.cand[k++] = base + b;
  }
  __syncwarp();
  return __shfl_sync(FULL, inc, 31);
}

// ---- vertex push (bitmap-forward and bucket sweeps) --------------------------------
// One vertex per lane: v with out-edges [a, a+dg) and the value F propagates (x:
// BFS the parent id v, BF/WP/wBFS dist[v]).  Lane-owned when <= 32 edges (NCH
// edges per batch), warp-owned when <= HEAVY edges, appended to the heavy list
// (counter *hctr) above that — heavy vertices are pushed with list tiles after a
// grid barrier, so a hub is spread over many warps (edgeMapBlocked).
// dg = 0 marks an idle lane.
template <int ALGO, bool STATS, int EMIT>
__device__ __forceinline__ void push_vertices(const Params &p, WarpSmem &wsm, WarpState &ws,
                                              uint32_t v, long long a, int dg, uint32_t x,
                                              unsigned long long *hctr, int nb, int r,
                                              uint32_t *bits, const uint32_t *prebits) {
  const int lane = threadIdx.x & 31;
  const bool heavy = dg > (int)(ALGO == ALGO_WBFS ? WBFS_HEAVY : HEAVY);
  warp_append(p, LIST_HEAVY, hctr, heavy, v, a, dg);
  unsigned med = __ballot_sync(FULL, dg > 32 && !heavy);
  while (med) {
    const int l = __ffs(med) - 1;
    med &= med - 1;
    const long long la = __shfl_sync(FULL, a, l);
    const int ld = __shfl_sync(FULL, dg, l);
    const uint32_t lx = __shfl_sync(FULL, x, l);
    if (STATS && lane == 0) {
      ws.edges += ld;
      ws.ab += (unsigned long long)ld * ((ALGO != ALGO_BFS && p.wgt) ? 8 : 4);
    }
    for (int cs = 0; cs < ld; cs += 32 * NCH) {
      uint32_t vv[NCH], ww[NCH], uu[NCH];
      bool act[NCH];
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        const int e = cs + 32 * j + lane;
        act[j] = e < ld;
        GBBS_CHECK(!act[j] || (la + e >= 0 && la + e < p.m));
        vv[j] = act[j] ? ld_stream(p.tgt + la + e) : 0;
        ww[j] = (ALGO != ALGO_BFS && act[j]) ? (p.wgt ? ld_stream(p.wgt + la + e) : 1u) : 0;
        uu[j] = lx;
      }
      apply_batch<ALGO, STATS, EMIT>(p, wsm.stage, ws, vv, uu, ww, act, nb, r, bits, prebits);
    }
  }
  const int mine = dg <= 32 ? dg : 0;
  if (STATS) {
    ws.edges += mine;
    ws.ab += (unsigned long long)mine * ((ALGO != ALGO_BFS && p.wgt) ? 8 : 4);
  }
  int mx = mine;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  constexpr int LB = (ALGO == ALGO_WBFS) ? WBFS_LB : NCH;
  for (int jj = 0; jj < mx; jj += LB) {
    uint32_t vv[LB], ww[LB], uu[LB];
    bool act[LB];
#pragma unroll
    for (int j = 0; j < LB; j++) {
      act[j] = jj + j < mine;
      GBBS_CHECK(!act[j] || (a + jj + j >= 0 && a + jj + j < p.m));
      vv[j] = act[j] ? ld_stream(p.tgt + a + jj + j) : 0;
      ww[j] = (ALGO != ALGO_BFS && act[j]) ? (p.wgt ? ld_stream(p.wgt + a + jj + j) : 1u) : 0;
      uu[j] = x;
    }
    apply_batch<ALGO, STATS, EMIT>(p, wsm.stage, ws, vv, uu, ww, act, nb, r, bits, prebits);
  }
}

// ---- bitmap-forward push ----------------------------------------------------------
// BFS (GBBS_FWD_CONVERT, default): the frontier bitmap is converted into a list
// with edge prefixes and pushed in edge tiles (coalesced edge loads) instead of
// one vertex per lane.
#ifndef GBBS_FWD_CONVERT
#define GBBS_FWD_CONVERT 1
#endif
// ... when the frontier's average out-degree E/f is at least this (measured: c5's
// 4.8 gains 28 % on that round; c2's 1.75 loses 2 % overall)
#ifndef GBBS_FWD_CONVERT_DEG
#define GBBS_FWD_CONVERT_DEG 4
#endif
// ... and in a multi-traversal launch, where each traversal has 1/G of the warps,
// so the lane path's serial batches per warp are G times longer (c2 8-team batch
// 0.84 -> 0.79 ms at 2; single traversals: c2 flat, c5 up to +2.6 % at 2)
#ifndef GBBS_FWD_CONVERT_DEG_MG
#define GBBS_FWD_CONVERT_DEG_MG 2
#endif
// BFS: frontier = precheck (vis_cur) & ~bits (vis_old): what the last dense round
// added; the TS target is vis_old, which also absorbs the frontier bits (atomicOr)
// so that it becomes the next visited set; vis_cur is read-only and is the
// pre-check.  BF: frontier = fr (this round's TS bits), cleared as swept.
template <int ALGO, bool STATS, int EMIT>
__device__ __forceinline__ void forward_words(const Params &p, WarpSmem &wsm, WarpState &ws,
                                              long long w0, int sw, uint32_t *fr, uint32_t *bits,
                                              const uint32_t *precheck, int nb, int r,
                                              bool convert) {
  const uint32_t *prebits = (ALGO == ALGO_BFS) ? precheck : bits;
  const int lane = threadIdx.x & 31;
  SweepSmem &w = wsm.u.s;
  const long long word = w0 + lane;
  uint32_t fw = 0;
  if (lane < sw && word < p.nwords) {
    if (ALGO == ALGO_BFS) {
      fw = precheck[word] & ~ld_relaxed(bits + word);
      if (fw) atomicOr(bits + word, fw);
    } else {
      fw = fr[word];
      if (fw) fr[word] = 0;
    }
    if (STATS) ws.ab += (ALGO == ALGO_BFS ? 8 : 4) + (fw ? 4 : 0);  // bitmap words swept / updated
  }
  if (!__any_sync(FULL, fw != 0)) return;
  const int cnt = warp_gather(w, w0, fw);
  if (STATS && lane == 0) ws.swept += cnt;
  if ((ALGO == ALGO_BFS || EMIT == EMIT_RED) && convert) {
    // a10 bitmap -> list: stage the frontier vertices; flushes append them with
    // their edge prefixes to the heavy list, pushed in edge tiles after the barrier
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const bool valid = c0 + lane < cnt;
      const unsigned bal = __ballot_sync(FULL, valid);
      GBBS_CHECK(ws.scnt + __popc(bal) <= WCAP);
      if (valid) wsm.stage[ws.scnt + lane] = w.cand[c0 + lane];
      ws.scnt += __popc(bal);
      if (ws.scnt > WCAP - 32) {
        warp_flush<ALGO, EMIT == EMIT_RED>(p, wsm.stage, ws.scnt, LIST_HEAVY, r, nullptr, nullptr,
                                           p.hcnt + (r & 1), STATS ? &ws.ab : nullptr);
        ws.scnt = 0;
      }
    }
    __syncwarp();
    return;
  }
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const bool valid = c0 + lane < cnt;
    const uint32_t v = valid ? w.cand[c0 + lane] : 0;
    long long a = 0;
    int dg = 0;
    if (valid) {
      a = __ldg(p.off + v);
      dg = (int)(__ldg(p.off + v + 1) - a);
      if (STATS) ws.ab += 16;
    }
    uint32_t x = v;
    if (ALGO != ALGO_BFS) x = dg > 0 ? ld_relaxed(p.dist + v) : 0u;
    push_vertices<ALGO, STATS, EMIT>(p, wsm, ws, v, a, dg, x, p.hcnt + (r & 1), nb, r, bits,
                                     prebits);
  }
  __syncwarp();
}

// ---- dense pull (BFS) ---------------------------------------------------------------
// Candidates = unvisited vertices of SWEEP_WORDS words, PCH*32 in flight per step,
// one per lane.  In-edges are read as 16-byte aligned groups of 4 (one vector
// load covers the group containing the scan position); a vertex with more than
// LONG_IN in-edges left after PULL_STEPS steps is finished by the whole warp,
// 128 in-edges per step, so one long in-list cannot hold the warp hostage.
#ifndef GBBS_PCH
#define GBBS_PCH 2
#endif
#ifndef GBBS_PULL_DYNQ
#define GBBS_PULL_DYNQ 1
#endif
#ifndef GBBS_LIST_DYNQ
#define GBBS_LIST_DYNQ 1
#endif
#ifndef GBBS_LIST_DYNQ_BFS
#define GBBS_LIST_DYNQ_BFS 0
#endif
// words per dynamically assigned sweep unit (0 = sweep_unit's); measured (c2/c4/c5
// BFS): 32 beats 16 and 8 by 2-5 % and 4 by 20 %; the queue itself -17 % on c4/c5
#ifndef GBBS_PULL_SW
#define GBBS_PULL_SW 32
#endif
static_assert(GBBS_PULL_SW <= SWEEP_WORDS, "pull units are gathered into SweepSmem");
// vectorised 4-edge steps per lane before a long in-list goes to the warp: 3 since
// the L1 grew (WCAP 192): c2/c4/c5 BFS -2 to -2.3 %, 8-team batch -3.5 % vs 2
// (4 and 5 measure the same as 3, 1 is 5 % slower)
#ifndef GBBS_PULL_STEPS
#define GBBS_PULL_STEPS 3
#endif
#ifndef GBBS_LONG_IN
#define GBBS_LONG_IN 24
#endif
// L2 prefetch of the next candidate batch's hot pull records
#ifndef GBBS_PULL_PF
#define GBBS_PULL_PF 1
#endif
constexpr int PULL_STEPS = GBBS_PULL_STEPS;
constexpr int LONG_IN = GBBS_LONG_IN;
constexpr int PCH = GBBS_PCH;

__device__ __forceinline__ uint4 ldg_v4(const uint32_t *p) { return ld_stream_v4(p); }


// Pull records (gbbs.cu k_pull_records), GBBS_REC8 layout: the hot record is 8 bytes —
// (in0, out-degree | "has more in-edges" in bit 31), four per 32-byte sector — and is
// all that pass 1 reads; the cold record is one sector per vertex — (in1, in2, in3,
// in4) (tail, out-degree) — read by pass 2 in one 256-bit load, so a candidate in0
// does not decide costs one more sector instead of a re-read of the hot record plus
// the cold one.  The text below describes the older 16 + 16-byte pair (GBBS_REC8 = 0).
//
// Candidates = the unit's vertices that are unvisited and have in-edges (the
// no-in-edge mask nin removes vertices no pull can ever acquire).  A candidate's
// first five in-edges in CSC order come from its pull records (gbbs.cu
// k_pull_records): the hot record (in0, in1, in2, out-degree) for every
// candidate, the cold one (in3, in4, tail) only when in0..in2 miss.  rMAT
// in-lists are sorted by source, so the first in-neighbours are the lowest ids —
// the likeliest hubs, visited early — and most candidates are decided by one HBM
// load and one or two probe steps, without the in-offset -> in-edge chain.  The
// scan then continues at the tail (in-edge 5 onwards) in CSC order: same edges,
// same order, same early exit as P:1870-1874 (the probes of in1/in2 and of in3/in4
// are issued together; the first hit in CSC order is taken).
// LISTOUT (light pulls, below): acquisitions with out-edges are also staged and
// flushed into frontier list nb with their edge prefixes, so the next round can
// push from a list instead of sweeping the bitmap.
//
// The scan runs as three passes over the unit's candidates with the survivors of
// each pass compacted in place in w.cand, so that every pass runs with full warps
// instead of a whole batch waiting for its longest in-list (the lock-step batch it
// replaced: c5 +0.7 %, c2 +8 %):
//   pass 1  hot record, probe in0                      (every candidate)
//   pass 2  probes in1, in2 + cold record, in3, in4    (candidates in0 did not decide)
//   pass 3  the tail from in-edge 5 on, 16-byte groups (candidates in0..in4 did not decide)
// Per candidate the in-edges are examined in the same CSC order with the same
// early exit; a pass re-reads its record from L2 instead of carrying
// it in shared memory (not counted as algorithmic bytes: the scan needs it once).
#ifndef GBBS_PULL_P1
#define GBBS_PULL_P1 4
#endif
// pull-record layout: 1 = 8-byte hot + 32-byte cold records (c5 -4 %, c4 -6 % against
// the 16-byte hot / 16-byte cold pair, 0, kept for A/B)
#ifndef GBBS_REC8
#define GBBS_REC8 1
#endif
// the cold sector as ONE 256-bit load (LDG.256) instead of two 16-byte loads: c5 -1.0 %,
// c4 -0.8 %, c2 -2.1 % (0 kept for A/B)
#ifndef GBBS_LD256
#define GBBS_LD256 1
#endif
constexpr int P1CH = GBBS_PULL_P1;

// One 32-candidate chunk's outcome: state writes, found bits, next-frontier counts
// (or, LISTOUT, staging for the next round's list).  Warp-convergent.
template <bool STATS, bool LISTOUT>
__device__ __forceinline__ void pull_commit(const Params &p, WarpSmem &wsm, long long w0, int r,
                                            WarpState &ws, int nb, uint32_t vq, uint32_t par,
                                            uint32_t dgo) {
  SweepSmem &w = wsm.u.s;
  const bool acq = par != INF;
  ws.A += __popc(__ballot_sync(FULL, acq));
  if (acq) {
    if (STATS && (!LISTOUT || dgo == 0)) ws.acquired += 1;  // LISTOUT: staged ones at flush
#ifndef GBBS_DIAG_NOSTATE  // diagnostic builds (results invalid): cost of the state writes
    bfs_set_dist(p, vq, (uint32_t)(r + 1));
    if (p.parent) st_stream(p.parent + vq, par);
#endif
    atomicOr(&w.found[(vq >> 5) - (uint32_t)w0], 1u << (vq & 31));
    if (!LISTOUT && dgo > 0) {
      ws.K += 1;
      ws.D += dgo;
    }
  }
  if (LISTOUT) {
    const bool stg = acq && dgo > 0;
    const unsigned b = __ballot_sync(FULL, stg);
    GBBS_CHECK(ws.scnt + __popc(b) <= WCAP);
    if (stg) wsm.stage[ws.scnt + __popc(b & lanemask_lt())] = vq;
    ws.scnt += __popc(b);
    if (ws.scnt > WCAP - 32) {
      if (STATS && (threadIdx.x & 31) == 0) ws.acquired += ws.scnt;
      warp_flush<ALGO_BFS>(p, wsm.stage, ws.scnt, nb, r, nullptr, nullptr, nullptr,
                           STATS ? &ws.ab : nullptr);
      ws.scnt = 0;
    }
  }
}

template <bool STATS, bool LISTOUT = false>
__device__ __forceinline__ void pull_words(const Params &p, WarpSmem &wsm, long long w0, int sw,
                                           const uint32_t *vis, uint32_t *vis_next, int r,
                                           WarpState &ws, int nb = 0) {
  const int lane = threadIdx.x & 31;
  SweepSmem &w = wsm.u.s;
  const long long word = w0 + lane;
  const bool mine = lane < sw && word < p.nwords;
  const uint32_t vw = mine ? vis[word] : FULL;
  const uint32_t skip = mine ? (vw | __ldg(p.nin + word)) : FULL;
  if (STATS && mine) ws.ab += 12;  // visited + no-in words read, next visited word written
  if (!__any_sync(FULL, skip != FULL)) {  // nothing to pull: carry the words over
    if (mine) vis_next[word] = vw;
    return;
  }
  const int cnt = warp_gather(w, w0, ~skip);
  w.found[lane] = 0;
  __syncwarp();
  if (STATS && lane == 0) ws.swept += cnt;

  // pass 1: hot record + in0, P1CH * 32 candidates in flight
  int ns = 0;
  for (int c0 = 0; c0 < cnt; c0 += 32 * P1CH) {
    uint32_t v[P1CH];
    uint4 h[P1CH];
    if (GBBS_PULL_PF) {  // the next batch's hot records, into L2 while this one runs
#pragma unroll
      for (int q = 0; q < P1CH; q++) {
        const int i = c0 + 32 * P1CH + 32 * q + lane;
        if (i < cnt) {
          if (GBBS_REC8) prefetch_l2(p.phot8 + w.cand[i]);
          else prefetch_l2(p.phot + w.cand[i]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < P1CH; q++) {
      const int i = c0 + 32 * q + lane;
      v[q] = i < cnt ? w.cand[i] : 0;
      h[q] = make_uint4(INF, INF, INF, 0);
      if (GBBS_REC8) {
        if (i < cnt) {
          const uint2 t = ld_stream_v2(reinterpret_cast<const uint32_t *>(p.phot8 + v[q]));
          h[q] = make_uint4(t.x, (t.y >> 31) ? 0u : INF, INF, t.y & 0x7FFFFFFFu);  // y: "has in1" flag
        }
      } else if (i < cnt) {
        h[q] = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.phot + v[q]));
      }
    }
    __syncwarp();  // the batch's candidates are in registers: survivors may overwrite them
#pragma unroll
    for (int q = 0; q < P1CH; q++) {
      if (c0 + 32 * q >= cnt) break;
      if (STATS && c0 + 32 * q + lane < cnt) {
        ws.ab += GBBS_REC8 ? 8 : 16;  // hot record
        ws.edges += 1;
      }
      const bool hit = h[q].x != INF && vbit(vis, h[q].x);
      if (STATS && hit) ws.hh += 1;
      pull_commit<STATS, LISTOUT>(p, wsm, w0, r, ws, nb, v[q], hit ? h[q].x : INF, h[q].w);
      const bool surv = !hit && h[q].y != INF;
      const unsigned b = __ballot_sync(FULL, surv);
      if (surv) w.cand[ns + __popc(b & lanemask_lt())] = v[q];
      ns += __popc(b);
    }
  }
  __syncwarp();

  // pass 2: in1, in2 probed together with the cold record's load (in3, in4, tail)
  int nt = 0;
  for (int c0 = 0; c0 < ns; c0 += 32 * PCH) {
    uint32_t v[PCH], par[PCH];
    uint4 h[PCH], cr[PCH];
    bool need[PCH];
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      const int i = c0 + 32 * q + lane;
      v[q] = i < ns ? w.cand[i] : 0;
      h[q] = make_uint4(INF, INF, INF, 0);
      if (GBBS_REC8) {
        cr[q] = make_uint4(INF, INF, 0, 0);
        if (i < ns) {  // one sector: (in1, in2, in3, in4) (tail, out-degree)
          uint4 c0r, c1r;
          if (GBBS_LD256) {
            ld_stream_v8(reinterpret_cast<const uint32_t *>(p.pc32 + 2 * (size_t)v[q]), c0r, c1r);
          } else {
            c0r = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.pc32 + 2 * (size_t)v[q]));
            c1r = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.pc32 + 2 * (size_t)v[q] + 1));
          }
          h[q] = make_uint4(0u, c0r.x, c0r.y, c1r.z);
          cr[q] = make_uint4(c0r.z, c0r.w, c1r.x, c1r.y);
          if (STATS) ws.ab += 32;
        }
      } else if (i < ns) {
        h[q] = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.phot + v[q]));
      }
    }
    if (!GBBS_REC8) {
#pragma unroll
      for (int q = 0; q < PCH; q++) {
        cr[q] = make_uint4(INF, INF, 0, 0);
        if (h[q].z != INF) cr[q] = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.pcold + v[q]));
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      par[q] = INF;
      if (h[q].y == INF) continue;  // idle lane
      const bool b1 = vbit(vis, h[q].y);
      const bool b2 = h[q].z != INF && vbit(vis, h[q].z);
      if (STATS) ws.edges += (b1 || h[q].z == INF) ? 1 : 2;
      par[q] = b1 ? h[q].y : (b2 ? h[q].z : INF);
    }
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      need[q] = false;
      if (h[q].y == INF || par[q] != INF || h[q].z == INF) continue;
      if (STATS && !GBBS_REC8) ws.ab += 16;  // cold record
      const bool b3 = cr[q].x != INF && vbit(vis, cr[q].x);
      const bool b4 = cr[q].y != INF && vbit(vis, cr[q].y);
      if (STATS) ws.edges += (cr[q].x == INF) ? 0 : ((b3 || cr[q].y == INF) ? 1 : 2);
      par[q] = b3 ? cr[q].x : (b4 ? cr[q].y : INF);
      const unsigned long long tail = ((unsigned long long)cr[q].w << 32) | cr[q].z;
      if (par[q] == INF && tail != 0) {
        need[q] = true;
        prefetch_l2(p.in_tgt + ((long long)(tail >> 24) & ~3ll));  // pass 3 starts here
      }
    }
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      if (c0 + 32 * q >= ns) break;
      pull_commit<STATS, LISTOUT>(p, wsm, w0, r, ws, nb, v[q], par[q], h[q].w);
      const unsigned b = __ballot_sync(FULL, need[q]);
      if (need[q]) w.cand[nt + __popc(b & lanemask_lt())] = v[q];
      nt += __popc(b);
    }
  }
  __syncwarp();

  // pass 3: the tail, 16-byte groups of in-edges
  for (int c0 = 0; c0 < nt; c0 += 32 * PCH) {
    uint32_t v[PCH], par[PCH], dgo[PCH];
    long long js[PCH];
    int rem[PCH];
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      const int i = c0 + 32 * q + lane;
      v[q] = i < nt ? w.cand[i] : 0;
      par[q] = INF;
      js[q] = 0;
      rem[q] = 0;
      dgo[q] = 0;
      if (i < nt) {
        uint2 t;
        if (GBBS_REC8) {
          const uint4 c1r = ld_stream_v4(reinterpret_cast<const uint32_t *>(p.pc32 + 2 * (size_t)v[q] + 1));
          t = make_uint2(c1r.x, c1r.y);
          dgo[q] = c1r.z;
        } else {
          t = ld_stream_v2(reinterpret_cast<const uint32_t *>(p.pcold + v[q]) + 2);
          dgo[q] = ld_stream(reinterpret_cast<const uint32_t *>(p.phot + v[q]) + 3);
        }
        const unsigned long long tail = ((unsigned long long)t.y << 32) | t.x;
        js[q] = (long long)(tail >> 24);
        rem[q] = (int)(tail & 0xFFFFFFull);
        if (rem[q] == 0xFFFFFF) rem[q] = (int)(ld_stream64(p.in_off + v[q] + 1) - js[q]);
      }
    }
    __syncwarp();
    bool anyrem = false;
#pragma unroll
    for (int q = 0; q < PCH; q++) anyrem |= rem[q] > 0;
    if (__any_sync(FULL, anyrem)) {
      for (int step = 0; step < PULL_STEPS; step++) {
        uint4 g[PCH];
#pragma unroll
        for (int q = 0; q < PCH; q++)
          if (rem[q] > 0) {
            GBBS_CHECK(js[q] >= 0 && js[q] < p.m);
            g[q] = ldg_v4(p.in_tgt + (js[q] & ~3ll));
          }
        bool live = false;
#pragma unroll
        for (int q = 0; q < PCH; q++) {
          if (rem[q] <= 0) continue;
          const int lo = (int)(js[q] & 3);
          const int hi = min(4, lo + rem[q]);
          const uint32_t e[4] = {g[q].x, g[q].y, g[q].z, g[q].w};
          bool b[4];
#pragma unroll
          for (int k = 0; k < 4; k++) b[k] = (k >= lo && k < hi) ? vbit(vis, e[k]) : false;
          uint32_t hit = INF;
#pragma unroll
          for (int k = 3; k >= 0; k--)
            if (b[k]) hit = e[k];
          if (STATS) {
            ws.edges += hi - lo;
            ws.ab += 16;
          }
          js[q] += hi - lo;
          rem[q] -= hi - lo;
          if (hit != INF) {
            par[q] = hit;
            rem[q] = 0;
          }
          live |= rem[q] > 0;
        }
        if (!__any_sync(FULL, live)) break;
      }
    }
    // short remainders: per lane; long remainders: the whole warp, one vertex at a time
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      for (;;) {
        const bool go = rem[q] > 0 && rem[q] <= LONG_IN;
        if (!__any_sync(FULL, go)) break;
        if (go) {
          GBBS_CHECK(js[q] >= 0 && js[q] < p.m);
          const uint4 g = ldg_v4(p.in_tgt + (js[q] & ~3ll));
          const int lo = (int)(js[q] & 3);
          const int hi = min(4, lo + rem[q]);
          const uint32_t e[4] = {g.x, g.y, g.z, g.w};
          uint32_t hit = INF;
#pragma unroll
          for (int k = 3; k >= 0; k--)
            if (k >= lo && k < hi && vbit(vis, e[k])) hit = e[k];
          if (STATS) {
            ws.edges += hi - lo;
            ws.ab += 16;
          }
          js[q] += hi - lo;
          rem[q] -= hi - lo;
          if (hit != INF) {
            par[q] = hit;
            rem[q] = 0;
          }
        }
      }
      unsigned longs = __ballot_sync(FULL, rem[q] > LONG_IN);
      while (longs) {
        const int l = __ffs(longs) - 1;
        longs &= longs - 1;
        long long a = __shfl_sync(FULL, js[q], l);
        const long long e_end = a + __shfl_sync(FULL, rem[q], l);
        uint32_t found = INF;
        // groups of 128 in-edges per step: a 16-byte load per lane, then the probes
        while (a < e_end) {
          const long long a0 = a & ~3ll;
          const long long gk = a0 + 4 * lane;
          uint32_t hit = INF;
          if (gk < e_end) {
            GBBS_CHECK(gk >= 0 && gk < p.m);
            const uint4 g = ldg_v4(p.in_tgt + gk);
            const uint32_t e[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int k = 3; k >= 0; k--)
              if (gk + k >= a && gk + k < e_end && vbit(vis, e[k])) hit = e[k];
            if (STATS) ws.ab += 16;
          }
          if (STATS && lane == 0) ws.edges += min(a0 + 128, e_end) - a;
          const unsigned hb = __ballot_sync(FULL, hit != INF);  // first hit in CSC order
          if (hb) {
            found = __shfl_sync(FULL, hit, __ffs(hb) - 1);
            break;
          }
          a = a0 + 128;
        }
        if (lane == l) {
          rem[q] = 0;
          par[q] = found;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < PCH; q++) {
      if (c0 + 32 * q >= nt) break;
      pull_commit<STATS, LISTOUT>(p, wsm, w0, r, ws, nb, v[q], par[q], dgo[q]);
    }
  }
  __syncwarp();
  if (mine) vis_next[word] = vw | w.found[lane];
  __syncwarp();
}

// ---- light pull: a dense round with few candidates left -----------------------------
// When at most GBBS_LIGHT candidates per warp remain (the tail of a direction-
// optimising BFS, reading A10b), most 32-word groups have nothing to pull.  Warps
// take contiguous blocks of 128 words (static, no work queue), read the visited and
// no-in-edge words as 16-byte vectors, carry dead groups over with vector stores and
// run pull_words only on groups with candidates, emitting a frontier list for the
// next round (LISTOUT) so that a small next frontier is pushed from a list instead
// of swept as a bitmap.
#ifndef GBBS_LIGHT
#define GBBS_LIGHT 128
#endif
template <bool STATS>
__device__ __forceinline__ void light_pull(const Params &p, WarpSmem &wsm, WarpState &ws,
                                           const uint32_t *vis, uint32_t *vis_next, int r, int nb,
                                           long long gw, long long nw) {
  const int lane = threadIdx.x & 31;
  const long long steps = (p.nwords + 127) / 128;
  const long long per = (steps + nw - 1) / nw;
  const long long s1 = min(steps, (gw + 1) * per);
  for (long long st = gw * per; st < s1; st++) {
    const long long w0 = st * 128;
    const long long wl = w0 + 4 * lane;
    uint4 a = make_uint4(FULL, FULL, FULL, FULL), b = a;
    if (wl + 3 < p.nwords) {
      a = __ldcg(reinterpret_cast<const uint4 *>(vis + wl));
      b = __ldg(reinterpret_cast<const uint4 *>(p.nin + wl));
    } else {
      if (wl < p.nwords) { a.x = vis[wl]; b.x = p.nin[wl]; }
      if (wl + 1 < p.nwords) { a.y = vis[wl + 1]; b.y = p.nin[wl + 1]; }
      if (wl + 2 < p.nwords) { a.z = vis[wl + 2]; b.z = p.nin[wl + 2]; }
    }
    if (STATS) ws.ab += 8 * 4;
    const bool has = ((a.x | b.x) & (a.y | b.y) & (a.z | b.z) & (a.w | b.w)) != FULL;
    const unsigned hb = __ballot_sync(FULL, has);
    if (!((hb >> (lane & ~7)) & 0xFFu)) {  // this lane's 32-word group is dead: carry over
      if (STATS) ws.ab += 16;
      if (wl + 3 < p.nwords) {
        *reinterpret_cast<uint4 *>(vis_next + wl) = a;
      } else {
        if (wl < p.nwords) vis_next[wl] = a.x;
        if (wl + 1 < p.nwords) vis_next[wl + 1] = a.y;
        if (wl + 2 < p.nwords) vis_next[wl + 2] = a.z;
      }
    }
#pragma unroll 1
    for (int g = 0; g < 4; g++)
      if ((hb >> (8 * g)) & 0xFFu) {
        // pull_words counts its words' visited / no-in reads again: counted above
        if (STATS && lane == 0) ws.ab -= 8 * min(32ll, max(0ll, p.nwords - (w0 + 32 * g)));
        pull_words<STATS, true>(p, wsm, w0 + 32 * g, 32, vis, vis_next, r, ws, nb);
      }
  }
}

// ---- dense pull-min (Bellman-Ford / widest path, GBBS_MODE_PULL) ---------------------
// SURVEY §8(a) a9's alternative dense BF round (reading A11): every non-isolated
// vertex v takes, over its in-edges (u, v) whose source is in the frontier
// bitmap fr, the best candidate d(u) + w (BF) or min(d(u), w) (widest path), and
// its owner lane writes it if it improves dist[v] — no atomics; the warp owns
// its words, so the next frontier bitmap is written word-wise.  Symmetric graphs
// only (the in-edge weights are the CSR weights at the same index).  In-lists
// longer than 32 are scanned by the whole warp, 128 edges per step.
template <int ALGO>
__device__ __forceinline__ void pullmin_edge(const Params &p, const uint32_t *fr, uint32_t u,
                                             long long e, uint32_t &best) {
  if (!vbit(fr, u)) return;
  const uint32_t du = ld_relaxed(p.dist + u);
  const uint32_t w = p.wgt ? ld_stream(p.wgt + e) : 1u;
  if (ALGO == ALGO_WP) {
    best = max(best, min(du, w));
  } else {
    const uint32_t sum = du + w;
    const bool ovf = sum < du || sum == INF;
    if (ovf && du != INF) atomicOr(p.status, 2);
    best = min(best, ovf ? INF : sum);
  }
}

template <int ALGO, bool STATS>
__device__ __forceinline__ void pullmin_words(const Params &p, WarpSmem &wsm, long long w0, int sw,
                                              const uint32_t *fr, uint32_t *nxt, WarpState &ws) {
  constexpr uint32_t WORST = (ALGO == ALGO_WP) ? 0u : INF;
  const int lane = threadIdx.x & 31;
  SweepSmem &w = wsm.u.s;
  const long long word = w0 + lane;
  const bool mine = lane < sw && word < p.nwords;
  const uint32_t cw = mine ? ~p.iso[word] : 0u;
  if (mine) w.found[lane] = 0;
  if (!__any_sync(FULL, cw != 0)) {
    if (mine) nxt[word] = 0;
    return;
  }
  const int cnt = warp_gather(w, w0, cw);
  if (!mine) w.found[lane] = 0;
  __syncwarp();
  if (STATS && lane == 0) ws.swept += cnt;
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const bool valid = c0 + lane < cnt;
    const uint32_t v = valid ? w.cand[c0 + lane] : 0;
    long long js = 0, je = 0;
    if (valid) {
      js = ld_stream64(p.in_off + v);
      je = ld_stream64(p.in_off + v + 1);
    }
    uint32_t best = WORST;
    const bool longl = je - js > 32;
    if (!longl) {
      for (long long e = js; e < je; e++) {
        GBBS_CHECK(e >= 0 && e < p.m);
        pullmin_edge<ALGO>(p, fr, ld_stream(p.in_tgt + e), e, best);
      }
      if (STATS) ws.edges += je - js;
    }
    unsigned lg = __ballot_sync(FULL, longl);
    while (lg) {  // long in-lists: the whole warp, then a warp reduction
      const int l = __ffs(lg) - 1;
      lg &= lg - 1;
      const long long a = __shfl_sync(FULL, js, l), b = __shfl_sync(FULL, je, l);
      uint32_t bl = WORST;
      for (long long e = a + lane; e < b; e += 32) {
        GBBS_CHECK(e >= 0 && e < p.m);
        pullmin_edge<ALGO>(p, fr, ld_stream(p.in_tgt + e), e, bl);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t y = __shfl_xor_sync(FULL, bl, o);
        bl = (ALGO == ALGO_WP) ? max(bl, y) : min(bl, y);
      }
      if (STATS && lane == 0) ws.edges += b - a;
      if (lane == l) best = bl;
    }
    if (valid) {
      const uint32_t cur = ld_relaxed(p.dist + v);
      const bool imp = (ALGO == ALGO_WP) ? best > cur : best < cur;
      if (imp) {  // only v's owner writes dist[v]
        p.dist[v] = best;
        st_relaxed16(p.shadow + v, min(best, 0xFFFFu));
        atomicOr(&w.found[(v >> 5) - (uint32_t)w0], 1u << (v & 31));
        const long long dgo = je - js;  // symmetric: out-degree = in-degree
        if (dgo > 0) {
          ws.K += 1;
          ws.D += (unsigned long long)dgo;
        }
        if (STATS) ws.acquired += 1;
      }
    }
  }
  __syncwarp();
  if (mine) nxt[word] = w.found[lane];
  __syncwarp();
}

// ---- the persistent kernel ---------------------------------------------------

template <int ALGO, bool STATS, int EMIT>
__device__ __forceinline__ void list_round(const Params &p, WarpSmem &w, WarpState &ws, int lb,
                                           long long f, long long E, int nb, int r, uint32_t *bits,
                                           const uint32_t *prebits, long long gw, long long nw,
                                           unsigned long long *q = nullptr) {
  // Tile size: TE, or smaller (power of two >= 32) when the round has fewer than
  // TE edges per warp, so a small round costs each warp a single batch.
  int TR = TE;
  if (p.bsize) TR = p.bsize;  // fixed block size (gbbs_opts.bsize, edgeMapBlocked's bsize)
  else
    while (TR > 32 && (E + TR / 2 - 1) / (TR / 2) <= nw) TR >>= 1;
  const long long ntiles = (E + TR - 1) / TR;
  if ((ALGO != ALGO_BFS || GBBS_LIST_DYNQ_BFS) && GBBS_LIST_DYNQ && q && ntiles >= 16 * nw) {  // not compiled into BFS:
    // it perturbed the BFS kernel's code generation (-5 to -9 %) without a BFS round using it.
    // Big rounds: warps grab runs of G tiles from the round's counter (one owner
    // search per grab), G sized for >= 4 grabs per warp — measured BF/widest path
    // -10 % on c4; small rounds keep the static blocks (one search per warp),
    // where a grab per tile cost c3 up to 19 %
    const int lane = threadIdx.x & 31;
    const long long G = max(1ll, min(16ll, ntiles / (4 * nw)));
    for (;;) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(q, (unsigned long long)G);
      long long t = (long long)__shfl_sync(FULL, u, 0);
      if (t >= ntiles) break;
      const long long t1 = min(t + G, ntiles);
      long long i0 = warp_upper_est(p.fo[lb], f, E, t * TR);
      for (; t < t1; t++)
        i0 = push_tile<ALGO, STATS, EMIT>(p, w, ws, lb, i0, t, f, E, nb, r, bits, prebits, TR);
    }
    return;
  }
  // contiguous blocks of tiles per warp: one owner search per warp and round
  const long long per = (ntiles + nw - 1) / nw;
  long long t = gw * per;
  const long long t1 = min(t + per, ntiles);
  if (t >= t1) return;
#ifdef GBBS_DIAG_TILE
  const unsigned long long tS0 = globaltimer_ns();
#endif
  long long i0 = warp_upper_est(p.fo[lb], f, E, t * TR);
#ifdef GBBS_DIAG_TILE
  GBBS_DEP(i0);
  if (ALGO == ALGO_BFS) diag_add(p.dbg, 0, globaltimer_ns() - tS0);
#endif
#ifdef GBBS_DIAG_LIST
  if (STATS) ws.t1 = globaltimer_ns();
#endif
  for (; t < t1; t++) {
    i0 = push_tile<ALGO, STATS, EMIT>(p, w, ws, lb, i0, t, f, E, nb, r, bits, prebits, TR);
#ifdef GBBS_DIAG_LIST
    if (STATS && !ws.t2) ws.t2 = globaltimer_ns();
#endif
  }
}

// STATS: add one CTA's round counters to p.stats[r] (one global atomic per CTA and counter)
template <bool STATS>
__device__ __forceinline__ void round_stats(const Params &p, Smem &s, const WarpState &ws, long long r,
                                            unsigned long long t_work, unsigned long long t_flush) {
  const int tid = threadIdx.x, lane = tid & 31;
  if (!(STATS && p.stats && r < p.stats_cap)) return;
  if (tid < 7) s.sacc[tid] = 0;
  __syncthreads();
  const unsigned long long e = warp_sum64((long long)ws.edges);
  const unsigned long long sw = warp_sum64((long long)ws.swept);
  const unsigned long long aq = warp_sum64((long long)ws.acquired);
  const unsigned long long ab = warp_sum64((long long)ws.ab);
  const unsigned long long hh = warp_sum64((long long)ws.hh);
  if (lane == 0) {
    atomicAdd(&s.sacc[0], e);
    atomicAdd(&s.sacc[1], sw);
    atomicAdd(&s.sacc[2], aq);
    atomicMax(&s.sacc[3], t_work);
    atomicMax(&s.sacc[4], t_flush);
    atomicAdd(&s.sacc[5], ab);
    atomicAdd(&s.sacc[6], hh);
  }
  __syncthreads();
  if (tid == 0) {
    atomicAdd((unsigned long long *)&p.stats[r].edges_examined, s.sacc[0]);
    atomicAdd((unsigned long long *)&p.stats[r].vertices_swept, s.sacc[1]);
    atomicAdd((unsigned long long *)&p.stats[r].acquired, s.sacc[2]);
    atomicMax((unsigned long long *)&p.stats[r].t_work_ns, s.sacc[3]);
    atomicMax((unsigned long long *)&p.stats[r].t_flush_ns, s.sacc[4]);
    atomicAdd((unsigned long long *)&p.stats[r].alg_bytes, s.sacc[5]);
    atomicAdd((unsigned long long *)&p.stats[r].head_hits, s.sacc[6]);
  }
}

// ---- teams: several traversals in one cooperative launch --------------------------
// A multi-traversal launch (MG) interleaves the CTAs into G teams, one traversal
// each with its own scratch; a team synchronises with a sense-counting barrier on
// its own two words instead of the grid barrier.  MG = false is the plain
// single-traversal kernel (grid.sync, the whole grid as the team).
__device__ __forceinline__ unsigned ld_acquire32(const unsigned *a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a));
  return v;
}

template <bool MG>
__device__ __forceinline__ void team_sync(cg::grid_group &grid, unsigned *bar, long long nblk) {
  if constexpr (!MG) {
    grid.sync();
  } else {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned g0 = ld_acquire32(bar + 1);  // generation, read before arriving
      __threadfence();
      if (atomicAdd(bar, 1u) == (unsigned)nblk - 1) {
        bar[0] = 0;  // last arriver: reset, then release the team
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (ld_acquire32(bar + 1) == g0) {
        }
      }
      __threadfence();
    }
    __syncthreads();
  }
}

template <int ALGO, bool STATS, int EMIT, bool MG = false>
__device__ __forceinline__ void forward_round(Smem &s, const Params &p, cg::grid_group &grid,
                                              WarpSmem &w, WarpState &ws, uint32_t *fr,
                                              uint32_t *bits, const uint32_t *precheck, int nb,
                                              int r, long long gw, long long nw,
                                              bool convert = false, long long nblk = 0) {
  if (GBBS_PULL_DYNQ) {  // dynamic unit assignment, as the dense pull
    const int lane = threadIdx.x & 31;
    const int psw = GBBS_PULL_SW ? GBBS_PULL_SW : sweep_unit(p.nwords, nw);
    for (;;) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(p.wq + (r & 3), 1ull);
      const long long w0 = (long long)__shfl_sync(FULL, u, 0) * psw;
      if (w0 >= p.nwords) break;
      forward_words<ALGO, STATS, EMIT>(p, w, ws, w0, psw, fr, bits, precheck, nb, r, convert);
    }
  } else {
    const int sw = sweep_unit(p.nwords, nw);
    for (long long w0 = gw * sw; w0 < p.nwords; w0 += nw * sw)
      forward_words<ALGO, STATS, EMIT>(p, w, ws, w0, sw, fr, bits, precheck, nb, r, convert);
  }
  if ((ALGO == ALGO_BFS || EMIT == EMIT_RED) && convert && ws.scnt > 0) {
    warp_flush<ALGO, EMIT == EMIT_RED>(p, w.stage, ws.scnt, LIST_HEAVY, r, nullptr, nullptr,
                                       p.hcnt + (r & 1), STATS ? &ws.ab : nullptr);
    ws.scnt = 0;
  }
  team_sync<MG>(grid, p.bar, nblk);  // heavy list complete
  if (threadIdx.x == 0) s.hcnt = ld_relaxed64(p.hcnt + (r & 1));
  __syncthreads();
  const unsigned long long hc = s.hcnt;
  const long long hf = (long long)(hc >> p.ebits);
  const long long hE = (long long)(hc & ((1ull << p.ebits) - 1));
  if (STATS && EMIT == EMIT_RED && threadIdx.x == 0 && blockIdx.x == 0 && p.stats &&
      r < p.stats_cap) {  // the converted frontier (the round's counter only flags marks)
    p.stats[r].frontier = hf;
    p.stats[r].frontier_edges = hE;
  }
  if (hf > 0)
    list_round<ALGO, STATS, EMIT>(p, w, ws, LIST_HEAVY, hf, hE, nb, r, bits,
                                  (ALGO == ALGO_BFS) ? precheck : bits, gw, nw,
                                  p.wq + 4 + (r & 3));
}

// The traversal: per-run init, then edgeMap rounds until the frontier is empty.
// (bid, nblk) = this CTA's index and the number of CTAs in its team (MG: CTA b
// serves team b mod G).
template <int ALGO, bool STATS, bool PM, bool MG>
__device__ __forceinline__ void traverse_body(const Params &p, Smem &s, int G) {
  cg::grid_group grid = cg::this_grid();
  // MG: team-local index and size; the single-traversal kernel reads the special
  // registers at each use (holding them in registers raised its spills)
  long long bid_ = 0, nblk_ = 0;
  if constexpr (MG) {
    const int g = (int)(blockIdx.x % G);
    bid_ = blockIdx.x / G;
    nblk_ = ((long long)gridDim.x - g + G - 1) / G;
  }
#define GBBS_BID (MG ? bid_ : (long long)blockIdx.x)
#define GBBS_NBLK (MG ? nblk_ : (long long)gridDim.x)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long gtid = GBBS_BID * BLOCK + tid;
  const long long gstride = GBBS_NBLK * BLOCK;
  const long long gw = GBBS_BID * NWARPS + warp;
  const long long nw = GBBS_NBLK * NWARPS;
  const uint32_t src = p.src;
  const int sw = sweep_unit(p.nwords, nw);
  WarpSmem &wsm = s.w[warp];

  // a1: per-run init
  if (ALGO == ALGO_BFS && p.lvl) {
    // levels: LVL_INF everywhere, 0 at src (16 bytes per thread and step; the buffer
    // holds 2n bytes; the tail group is written byte by byte); parent as before
    uint8_t *lvl = p.lvl;
    for (long long i = gtid * 16; i < p.n; i += gstride * 16) {
      if (i + 16 <= p.n) {
        uint32_t x[4] = {FULL, FULL, FULL, FULL};
        if ((long long)src >= i && (long long)src < i + 16)
          x[(src - i) >> 2] &= ~(0xFFu << (8 * ((src - i) & 3)));
        *reinterpret_cast<uint4 *>(lvl + i) = make_uint4(x[0], x[1], x[2], x[3]);
      } else {
        for (long long k = i; k < p.n; k++) lvl[k] = (k == (long long)src) ? 0 : (uint8_t)LVL_INF;
      }
    }
#ifndef GBBS_DIAG_NOINIT  // diagnostic builds (results invalid): cost of the fill
    if (p.parent)
      for (long long i = gtid; i < p.n; i += gstride)
        st_stream(p.parent + i, (i == src) ? src : INF);
#endif
  } else
  for (long long i = gtid; i < p.n; i += gstride) {
    // BFS/BF: 0 at src, INF elsewhere; widest path: INF (empty path) at src, 0 elsewhere
    if (ALGO == ALGO_WP) {
      st_stream(p.dist + i, (i == src) ? INF : 0u);
      p.shadow[i] = (i == src) ? 0xFFFFu : 0u;
    } else {
      st_stream(p.dist + i, (i == src) ? 0u : INF);
      if (ALGO == ALGO_BF) p.shadow[i] = (i == src) ? 0u : 0xFFFFu;
    }
    if (ALGO == ALGO_BFS && p.parent) st_stream(p.parent + i, (i == src) ? src : INF);
  }
  for (long long w = gtid; w < p.nwords; w += gstride) {
    if (ALGO == ALGO_BFS) {
      uint32_t x = p.iso[w];  // isolated vertices + padding count as visited
      if ((long long)(src >> 5) == w) x |= 1u << (src & 31);
      p.bm[0][w] = x;
    } else {  // round 0's frontier {src} as TS bits (bitmap-forward reads them)
      p.bm[0][w] = ((long long)(src >> 5) == w) ? (1u << (src & 31)) : 0u;
      p.bm[1][w] = 0;
    }
  }
  const long long a0 = p.off[src], d0 = p.off[src + 1] - a0;
  // reading A10b: vertices with in-edges acquired so far (the source counts if it has any)
  long long acq_total = 0;
  if (ALGO == ALGO_BFS) acq_total = ((__ldg(p.nin + (src >> 5)) >> (src & 31)) & 1u) ? 0 : 1;
  if (GBBS_BID == 0 && tid == 0) {
    if (ALGO == ALGO_BFS) p.acq[0] = p.acq[1] = p.acq[2] = p.acq[3] = 0;
    p.cnt[1] = p.cnt[2] = p.cnt[3] = 0;
    p.hcnt[0] = p.hcnt[1] = 0;
    for (int q = 0; q < 8; q++) p.wq[q] = 0;
    if (d0 > 0) {
      p.fv[0][0] = src;
      p.fo[0][0] = 0;
      p.fb[0][0] = a0;
      p.cnt[0] = (1ull << p.ebits) | (unsigned long long)d0;
    } else {
      p.cnt[0] = 0;
    }
    *p.status = 0;
  }
  team_sync<MG>(grid, p.bar, GBBS_NBLK);

  const unsigned long long emask = (1ull << p.ebits) - 1;
  int vc = 0;              // BFS: index of the current visited bitmap
  bool prev_dense = false;  // BFS: was the previous round a dense pull (reading A10b count)
  bool list_valid = true;  // is this round's frontier materialised as a list?
  long long r = 0;
  for (;; r++) {
    if (tid == 0) {
      s.cnt = ld_relaxed64(p.cnt + (r & 3));
      if (ALGO == ALGO_BFS) s.acq = ld_relaxed64(p.acq + (r & 3));
    }
    __syncthreads();
    const unsigned long long c = s.cnt;
    const long long f = (long long)(c >> p.ebits);
    const long long E = (long long)(c & emask);
    // dense rounds count their acquisitions (one atomic per warp); after a push round
    // the frontier size f — its acquisitions with out-edges — stands in for them
    // (per-warp counting on one word in every push round cost c3 ~1.3 us per round)
    if (ALGO == ALGO_BFS && r > 0) acq_total += prev_dense ? (long long)s.acq : f;
    if (STATS && GBBS_BID == 0 && tid == 0 && p.stats && r < p.stats_cap)
      p.stats[r].t_start_ns = (long long)globaltimer_ns();
    if (f == 0) break;
    if (r >= p.max_rounds) {
      if (GBBS_BID == 0 && tid == 0) *p.status = 1;
      break;
    }
    // kind: 0 list push, 1 dense pull, 2 bitmap-forward.  BFS: dense pull iff
    // |U| + sum deg(U) > m/T.  Bellman-Ford: list push unless GBBS_MODE_DENSE
    // forces bitmap-forward rounds (reading A11: measured slower on rMAT).
    // mode 3 (GBBS_MODE_PULL): BFS as auto; BF / widest path take a pull-min
    // round (kind 3, symmetric graphs) when |U| + sum deg(U) > m/T
    // Reading A10b (BFS AUTO): after a dense round the frontier is a bitmap, and
    // the next round stays dense while the pull's remaining work — the vertices
    // with in-edges not visited yet (ncand - acquired so far) — is at most the
    // push's |U| + sum deg(U): a pull then sweeps few candidates, while a push
    // would expand the whole frontier (Beamer's bottom-up -> top-down switch in
    // work terms).  GBBS_RULE_PAPER_ONLY keeps the paper's m/T test alone.
    const bool over = f + E > p.dense_threshold;
    const bool stay = ALGO == ALGO_BFS && !list_valid && !(p.rules & 1) &&
                      p.ncand - acq_total <= f + E;
    const bool big = (ALGO == ALGO_BFS)
                         ? (p.mode == 2 || ((p.mode == 0 || p.mode == 3) && (over || stay)))
                         : (p.mode == 2 || (p.mode == 3 && over));
    int kind;
    if (ALGO == ALGO_BFS) kind = big ? 1 : (list_valid ? 0 : 2);
    else if (PM && big && p.mode == 3 && p.symmetric) kind = 3;
    else kind = (big || !list_valid) ? 2 : 0;
    // Bellman-Ford, AUTO / SPARSE: red rounds (the frontier bitmap is converted to a
    // list with its distances, then pushed with fire-and-forget priority-writes)
    if (GBBS_BF_RED && ALGO == ALGO_BF && (p.mode == 0 || p.mode == 1)) kind = 5;
    if (GBBS_BID == 0 && tid == 0) {
      p.cnt[(r + 2) & 3] = 0;
      if (ALGO == ALGO_BFS) p.acq[(r + 2) & 3] = 0;
      p.wq[(r + 2) & 3] = 0;
      p.wq[4 + ((r + 2) & 3)] = 0;
      p.hcnt[(r + 1) & 1] = 0;
      if (STATS && p.stats && r < p.stats_cap) {
        p.stats[r].dense = kind;
        p.stats[r].frontier = f;
        p.stats[r].frontier_edges = E;
      }
    }
    const int cb = (int)(r & 1), nb = cb ^ 1;
    WarpState ws;
    bool emit_count = false;
    // light pulls sweep static 128-word blocks: only when every warp gets one
    if (kind == 1 && ALGO == ALGO_BFS && p.ncand - acq_total <= (long long)GBBS_LIGHT * nw &&
        p.nwords >= 128ll * nw) {
      light_pull<STATS>(p, wsm, ws, p.bm[vc], p.bm[vc ^ 1], (int)r, nb, gw, nw);
      vc ^= 1;
      list_valid = true;  // the acquisitions were also emitted as list nb
    } else if (kind == 1) {  // dense pull (BFS)
      const uint32_t *vis = p.bm[vc];
      uint32_t *vis_next = p.bm[vc ^ 1];
      if (GBBS_PULL_DYNQ) {
        // dynamic assignment: a warp takes the next unit of psw words from a
        // per-round counter as soon as it is done, so no warp waits at the
        // barrier for another that drew two units
        // 32-word units (c2/c4/c5: 2-5 % faster than 16 or 8), halved while there are
        // fewer units than a quarter of the warps (a 2^14-vertex graph has 16)
        int psw = GBBS_PULL_SW ? GBBS_PULL_SW : sw;
        while (psw > 1 && (p.nwords + psw - 1) / psw < nw / 4) psw >>= 1;
        for (;;) {
          unsigned long long u = 0;
          if (lane == 0) u = atomicAdd(p.wq + (r & 3), 1ull);
          const long long w0 = (long long)__shfl_sync(FULL, u, 0) * psw;
          if (w0 >= p.nwords) break;
          pull_words<STATS>(p, wsm, w0, psw, vis, vis_next, (int)r, ws);
        }
      } else {
        for (long long w0 = gw * sw; w0 < p.nwords; w0 += nw * sw)
          pull_words<STATS>(p, wsm, w0, sw, vis, vis_next, (int)r, ws);
      }
      vc ^= 1;
      list_valid = false;
      emit_count = true;
    } else if (kind == 3) {  // pull-min (BF / widest path, GBBS_MODE_PULL)
      if constexpr (PM && ALGO != ALGO_BFS) {
        // the frontier as a bitmap: a list frontier's TS bits already are one
        for (long long w0 = gw * sw; w0 < p.nwords; w0 += nw * sw)
          pullmin_words<ALGO, STATS>(p, wsm, w0, sw, p.bm[cb], p.bm[nb], ws);
        team_sync<MG>(grid, p.bar, GBBS_NBLK);  // every probe of bm[cb] is done: clear it for reuse as TS bits
        for (long long i = gtid; i < p.nwords; i += gstride) p.bm[cb][i] = 0;
      }
      list_valid = false;
      emit_count = true;
    } else if (kind == 5) {  // Bellman-Ford red round
      if constexpr (ALGO == ALGO_BF)
        forward_round<ALGO, STATS, EMIT_RED, MG>(s, p, grid, wsm, ws, p.bm[cb], p.bm[nb], nullptr, nb,
                                                 (int)r, gw, nw, true, GBBS_NBLK);
      list_valid = false;
      emit_count = true;
    } else if (kind == 2) {  // bitmap-forward
      if (ALGO == ALGO_BFS) {
        forward_round<ALGO, STATS, EMIT_LIST, MG>(
            s, p, grid, wsm, ws, nullptr, p.bm[vc ^ 1], p.bm[vc], nb, (int)r, gw, nw,
            GBBS_FWD_CONVERT &&
                E >= (long long)(MG ? GBBS_FWD_CONVERT_DEG_MG : GBBS_FWD_CONVERT_DEG) * f, GBBS_NBLK);
        vc ^= 1;
        list_valid = true;
      } else if (big) {
        forward_round<ALGO, STATS, EMIT_COUNT, MG>(s, p, grid, wsm, ws, p.bm[cb], p.bm[nb],
                                                   nullptr, nb, (int)r, gw, nw, false, GBBS_NBLK);
        list_valid = false;
        emit_count = true;
      } else {
        forward_round<ALGO, STATS, EMIT_LIST, MG>(s, p, grid, wsm, ws, p.bm[cb], p.bm[nb],
                                                  nullptr, nb, (int)r, gw, nw, false, GBBS_NBLK);
        list_valid = true;
      }
    } else {  // list push
      uint32_t *bits = (ALGO == ALGO_BFS) ? p.bm[vc] : p.bm[nb];
      if (ALGO != ALGO_BFS) {
        // a11: release the current frontier's TS bits (buffer cb is idle this round)
        uint32_t *cur_bits = p.bm[cb];
        const uint32_t *F = p.fv[cb];
        for (long long i = gtid; i < f; i += gstride) cur_bits[__ldcg(F + i) >> 5] = 0;
      }
      list_round<ALGO, STATS, EMIT_LIST>(p, wsm, ws, cb, f, E, nb, (int)r, bits, bits, gw, nw,
                                         p.wq + (r & 3));
      list_valid = true;
    }
    unsigned long long t_work = 0, t_flush = 0;
    if (STATS) t_work = globaltimer_ns();
    if (ws.scnt > 0) {
      if (STATS && lane == 0) ws.acquired += ws.scnt;
#ifdef GBBS_DIAG_TILE
      const unsigned long long tF0 = globaltimer_ns();
#endif
      warp_flush<ALGO>(p, wsm.stage, ws.scnt, nb, (int)r,
                       (ALGO == ALGO_BFS) ? p.bm[vc] : p.bm[nb], &t_work, nullptr,
                       STATS ? &ws.ab : nullptr);
#ifdef GBBS_DIAG_TILE
      if (ALGO == ALGO_BFS && kind == 0) {
        diag_add(p.dbg, 5, globaltimer_ns() - tF0);
        diag_add(p.dbg, 7, 1);
      }
#endif
    }
    if (emit_count) {
      const unsigned long long K = warp_sum64((long long)ws.K), D = warp_sum64((long long)ws.D);
      if (lane == 0 && K) atomicAdd(p.cnt + ((r + 1) & 3), (K << p.ebits) | D);
    }
    if (ALGO == ALGO_BFS && kind == 1 && lane == 0 && ws.A) atomicAdd(p.acq + ((r + 1) & 3), ws.A);
    prev_dense = ALGO == ALGO_BFS && kind == 1;
    if (STATS) t_flush = globaltimer_ns();
#ifdef GBBS_DIAG_LIST
    if (STATS) { t_work = ws.t1; t_flush = ws.t2; ws.t1 = ws.t2 = 0; }
#endif
    if (STATS) round_stats<STATS>(p, s, ws, r, t_work, t_flush);
    team_sync<MG>(grid, p.bar, GBBS_NBLK);
  }
  if (ALGO == ALGO_BFS && p.lvl) {
    // a12: expand the levels into dist (every write of the last round is visible: the
    // loop is left after a team barrier).  A warp takes 1024 levels per step: each lane
    // loads two 16-byte groups (coalesced), the groups are transposed through the
    // warp's shared memory, and dist is written as whole 512-byte rows (16 bytes per
    // lane) — partial-sector stores cost the L2 several requests per sector.
    const uint8_t *lvl = p.lvl;
    const bool al = (reinterpret_cast<unsigned long long>(p.dist) & 15ull) == 0;
    uint32_t *tw = wsm.u.s.cand;  // 256 words of scratch
    for (long long b0 = gw * 1024; b0 < p.n; b0 += nw * 1024) {
      if (b0 + 1024 <= p.n) {
        const uint4 q0 = __ldcg(reinterpret_cast<const uint4 *>(lvl + b0) + lane);
        const uint4 q1 = __ldcg(reinterpret_cast<const uint4 *>(lvl + b0 + 512) + lane);
        reinterpret_cast<uint4 *>(tw)[lane] = q0;
        reinterpret_cast<uint4 *>(tw)[32 + lane] = q1;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const uint32_t wd = tw[k * 32 + lane];  // levels of b0 + 128 k + 4 lane .. + 3
          const long long v0 = b0 + 128 * k + 4 * lane;
          const uint32_t x = wd ^ 0xFEFEFEFEu;  // a zero byte <=> LVL_DIRECT: dist already final
          const bool direct = ((x - 0x01010101u) & ~x & 0x80808080u) != 0;
          uint32_t d[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const uint32_t l = (wd >> (8 * e)) & 0xFFu;
            d[e] = l == LVL_INF ? INF : l;
          }
          if (al && !direct) {
            st_stream_v4(p.dist + v0, d[0], d[1], d[2], d[3]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; e++)
              if (d[e] != LVL_DIRECT) st_stream(p.dist + v0 + e, d[e]);
          }
        }
        __syncwarp();
      } else {  // the last, partial block
        for (long long j = b0 + lane; j < p.n; j += 32) {
          const uint32_t l = __ldcg(lvl + j);
          if (l != LVL_DIRECT) st_stream(p.dist + j, l == LVL_INF ? INF : l);
        }
      }
    }
  }
  if (GBBS_BID == 0 && tid == 0) *p.rounds_out = r;
}
#undef GBBS_BID
#undef GBBS_NBLK

#ifndef GBBS_MIN_CTAS
#define GBBS_MIN_CTAS 4
#endif
// PM: the instantiation that contains the pull-min round (launched only for
// GBBS_MODE_PULL), so its code does not raise the default kernels' registers.
template <int ALGO, bool STATS, bool PM = false>
__global__ void __launch_bounds__(BLOCK, GBBS_MIN_CTAS)
    traverse_kernel(const __grid_constant__ Params p) {
  __shared__ Smem s;
  traverse_body<ALGO, STATS, PM, false>(p, s, 1);
}

// G traversals in one cooperative launch: CTA b serves team b mod G.
constexpr int GMAX = 8;
struct MultiParams {
  Params ps[GMAX];
  int G;
};
template <int ALGO>
__global__ void __launch_bounds__(BLOCK, GBBS_MIN_CTAS)
    traverse_mg_kernel(const __grid_constant__ MultiParams mp) {
  __shared__ Smem s;
  traverse_body<ALGO, false, false, true>(mp.ps[blockIdx.x % mp.G], s, mp.G);
}

// ---- wBFS: integral-weight SSSP over buckets (NEXT-2) ---------------------------------
// Julienne's weighted BFS (sec:algs; output spec P:1481-1484): buckets
// of distance width delta are extracted in increasing order; each extracted
// bucket is one edgeMapData round whose F is the priority-write min of
// dist[u] + w (a6), and every vertex whose distance dropped moves to its new
// bucket (wbfs_insert).  delta = 1 is the paper's algorithm (one bucket per
// distance value; with weights >= 1 each vertex is expanded exactly once, O(m)
// work); delta > 1 is Delta-stepping, re-expanding vertices that improve inside
// the current bucket from a near list.
//
// Bucket structure, all on the device: nbq (a power of two > the bucket span
// floor((delta - 1 + maxw) / delta)) circular lists of capacity qcap >= n; bucket
// j lives in list j mod nbq, which is unambiguous because every pending entry lies
// within one span above the bucket being processed.  Append counters are
// monotone; each CTA keeps the list heads in shared memory and the set of lists
// with pending entries in a register mask (`pend`), fed by per-round masks that
// appending warps publish (`pub`).  All CTAs therefore take the same decision
// without a host round trip: every round reads only counters that no warp
// updates during that round.  Entries whose vertex has since moved to an
// earlier bucket are skipped when swept (lazy deletion).
// 3 CTAs per SM: the bucket kernel's extra state spills at 64 registers, and it
// measured 1.3x faster with 80 (c2 and c4, tools/cmp_lib.sh)
#ifndef GBBS_WBFS_MIN_CTAS
#define GBBS_WBFS_MIN_CTAS 3
#endif
template <bool STATS, bool MG>
__device__ __forceinline__ void wbfs_body(const Params &p, int G) {
  __shared__ Smem s;
  __shared__ unsigned long long s_head[64], s_hhead[64], s_ctl[3 + 2 * 64];
  cg::grid_group grid = cg::this_grid();
  long long bid_ = 0, nblk_ = 0;  // MG: team-local index and size (as traverse_body)
  if constexpr (MG) {
    const int g = (int)(blockIdx.x % G);
    bid_ = blockIdx.x / G;
    nblk_ = ((long long)gridDim.x - g + G - 1) / G;
  }
#define GBBS_BID (MG ? bid_ : (long long)blockIdx.x)
#define GBBS_NBLK (MG ? nblk_ : (long long)gridDim.x)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long gtid = GBBS_BID * BLOCK + tid;
  const long long gstride = GBBS_NBLK * BLOCK;
  const long long gw = GBBS_BID * NWARPS + warp;
  const long long nw = GBBS_NBLK * NWARPS;
  const uint32_t src = p.src;
  const int nbq = p.nbq;
  const unsigned long long qmask = p.qcap - 1;
  WarpSmem &wsm = s.w[warp];

  // a1: per-run init
  for (long long i = gtid; i < p.n; i += gstride) {
    st_stream(p.dist + i, (i == src) ? 0u : INF);
    p.shadow[i] = (i == src) ? 0u : 0xFFFFu;
    if (p.tag) p.tag[i] = 0;
  }
  if (GBBS_BID == 0 && tid == 0) {
    for (int q = 0; q < nbq; q++) p.btail[q] = p.bheavy[q] = 0;
    for (int q = 0; q < 6; q++) p.xcnt[q] = 0;
    for (int q = 0; q < 3; q++) p.pub[q] = 0;
    p.hcnt[0] = p.hcnt[1] = 0;
    p.cnt[0] = p.cnt[1] = p.cnt[2] = 0;
    for (int q = 0; q < 8; q++) p.wq[q] = 0;
    p.bq[0] = src;  // bucket 0 = {src}
    p.btail[0] = 1;
    p.bheavy[0] = (p.hv[src >> 5] >> (src & 31)) & 1u;
    *p.status = 0;
  }
  if (tid < 64) s_head[tid] = s_hhead[tid] = 0;
  {
    WbfsWarpSmem &w = wbfs_smem();
    w.hist[lane] = w.hist[lane + 32] = 0;
    w.hh[lane] = w.hh[lane + 32] = 0;
    if (lane == 0) w.hist[XKEY] = w.hh[XKEY] = 0;
  }
  team_sync<MG>(grid, p.bar, GBBS_NBLK);

  unsigned long long pend = 1;  // lists with pending entries: bucket 0's
  unsigned long long k = 0;     // bucket being processed
  bool taken = false;           // has bucket k's list been taken
  long long r = 0;
  for (;; r++) {
    const int pr = (int)((r + 2) % 3), xr = (int)(r % 3);
    if (tid == 0) {
      s_ctl[0] = r ? ld_relaxed64(p.xcnt + pr) : 0;
      s_ctl[1] = r ? ld_relaxed64(p.xcnt + 3 + pr) : 0;
      s_ctl[2] = r ? ld_relaxed64(p.pub + pr) : 0;
    }
    if (tid < nbq) {  // only the chosen list's counters are used: no warp appends to it this round
      s_ctl[3 + tid] = ld_relaxed64(p.btail + tid);
      s_ctl[3 + 64 + tid] = ld_relaxed64(p.bheavy + tid);
    }
    __syncthreads();
    pend |= s_ctl[2];
    const uint32_t *Q;
    unsigned long long qm, h, t;
    bool heavy_any;
    int slot = -1;
    if (s_ctl[0] > 0) {  // near list of bucket k (delta > 1 or zero weights)
      Q = p.xq[pr];
      qm = ~0ull;
      h = 0;
      t = s_ctl[0];
      heavy_any = s_ctl[1] > 0;
    } else {  // next bucket: the smallest j >= k (+1 once taken) with a pending list
      const unsigned long long j0 = taken ? k + 1 : k;
      const int sh = (int)(j0 & (unsigned long long)(nbq - 1));
      const unsigned long long all = (nbq == 64) ? ~0ull : ((1ull << nbq) - 1);
      const unsigned long long rot = ((pend >> sh) | (sh ? (pend << (nbq - sh)) : 0ull)) & all;
      if (rot == 0) break;  // every bucket list is empty: done
      k = j0 + (unsigned long long)(__ffsll((long long)rot) - 1);
      taken = true;
      slot = (int)(k & (unsigned long long)(nbq - 1));
      pend &= ~(1ull << slot);
      Q = p.bq + (unsigned long long)slot * p.qcap;
      qm = qmask;
      h = s_head[slot];
      t = s_ctl[3 + slot];
      heavy_any = s_ctl[3 + 64 + slot] > s_hhead[slot];
      if (t - h > p.qcap) {  // entries were overwritten: the list overflowed
        if (GBBS_BID == 0 && tid == 0) *p.status = 4;
        break;
      }
    }
    if (r >= p.max_rounds) {
      if (GBBS_BID == 0 && tid == 0) *p.status = 1;
      break;
    }
    __syncthreads();
    if (tid == 0 && slot >= 0) {
      s_head[slot] = t;
      s_hhead[slot] = s_ctl[3 + 64 + slot];
    }
    if (GBBS_BID == 0 && tid == 0) {
      const int nr = (int)((r + 1) % 3);  // idle this round; appended to next round
      p.xcnt[nr] = p.xcnt[3 + nr] = 0;
      p.pub[nr] = 0;
      p.cnt[nr] = 0;
      p.wq[(r + 2) & 3] = p.wq[4 + ((r + 2) & 3)] = 0;
      p.hcnt[(r + 1) & 1] = 0;
      if (STATS && p.stats && r < p.stats_cap) {
        p.stats[r].dense = slot >= 0 ? 3 : 4;
        p.stats[r].bucket = (int32_t)k;
        p.stats[r].frontier = (long long)(t - h);
        p.stats[r].t_start_ns = (long long)globaltimer_ns();
      }
    }
    WarpState ws;
    ws.bk = k;
    // A large bucket (more entries than lanes in the grid) is first compacted into
    // a frontier list carrying edge prefixes (one packed atomicAdd per warp, as
    // warp_flush) and then pushed in fixed-size edge tiles — edgeMapBlocked's
    // load balance for the rounds that carry most of the edges.  A
    // small one is swept directly, one vertex per lane, saving a grid barrier.
    const bool big = (t - h) > 32ull * (unsigned long long)nw;
    for (unsigned long long i0 = h + 32ull * (unsigned long long)gw; i0 < t;
         i0 += 32ull * (unsigned long long)nw) {
      const unsigned long long i = i0 + lane;
      uint32_t v = 0, x = 0;
      long long a = 0;
      int dg = 0;
      if (i < t) {
        v = __ldcg(Q + (i & qm));
        x = ld_relaxed(p.dist + v);
        a = __ldg(p.off + v);
        dg = (int)(__ldg(p.off + v + 1) - a);
        if (x / p.delta != k) dg = 0;  // lazy deletion: v has moved to an earlier bucket
        if (STATS) ws.swept += 1;
      }
      if (big) {  // stage the live entries; one packed atomicAdd per full stage
        const unsigned bal = __ballot_sync(FULL, dg > 0);
        GBBS_CHECK(ws.scnt + __popc(bal) <= WCAP);
        if (dg > 0) wsm.stage[ws.scnt + __popc(bal & lanemask_lt())] = v;
        ws.scnt += __popc(bal);
        if (ws.scnt > WCAP - 32) {
          warp_flush<ALGO_WBFS>(p, wsm.stage, ws.scnt, 0, (int)r, nullptr, nullptr, p.cnt + xr);
          ws.scnt = 0;
        }
      } else {
        push_vertices<ALGO_WBFS, STATS, EMIT_LIST>(p, wsm, ws, v, a, dg, x, p.hcnt + (r & 1), 0,
                                                   (int)r, nullptr, nullptr);
      }
    }
    if (big) {
      if (ws.scnt > 0) {
        warp_flush<ALGO_WBFS>(p, wsm.stage, ws.scnt, 0, (int)r, nullptr, nullptr, p.cnt + xr);
        ws.scnt = 0;
      }
      team_sync<MG>(grid, p.bar, GBBS_NBLK);
      if (tid == 0) s.cnt = ld_relaxed64(p.cnt + xr);
      __syncthreads();
      const unsigned long long c = s.cnt;
      const long long f = (long long)(c >> p.ebits);
      const long long E = (long long)(c & ((1ull << p.ebits) - 1));
      if (STATS && p.stats && r < p.stats_cap && GBBS_BID == 0 && tid == 0)
        p.stats[r].frontier_edges = E;
      if (f > 0)
        list_round<ALGO_WBFS, STATS, EMIT_LIST>(p, wsm, ws, 0, f, E, 0, (int)r, nullptr, nullptr,
                                                gw, nw, p.wq + (r & 3));
    } else if (heavy_any) {  // hubs of this bucket, spread over all warps in list tiles
      team_sync<MG>(grid, p.bar, GBBS_NBLK);
      if (tid == 0) s.hcnt = ld_relaxed64(p.hcnt + (r & 1));
      __syncthreads();
      const unsigned long long hc = s.hcnt;
      const long long hf = (long long)(hc >> p.ebits);
      const long long hE = (long long)(hc & ((1ull << p.ebits) - 1));
      if (hf > 0)
        list_round<ALGO_WBFS, STATS, EMIT_LIST>(p, wsm, ws, LIST_HEAVY, hf, hE, 0, (int)r, nullptr,
                                                nullptr, gw, nw, p.wq + 4 + (r & 3));
    }
    unsigned long long t_work = 0;
    if (STATS) t_work = globaltimer_ns();
    if (ws.scnt > 0) wbfs_flush<STATS>(p, ws, wsm.stage, ws.scnt, (int)r);
    // publish the lists this warp appended to
    unsigned long long pm = ws.pmask;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pm |= __shfl_xor_sync(FULL, pm, o);
    if (lane == 0 && pm) atomicOr(p.pub + xr, pm);
    if (STATS && p.stats && r < p.stats_cap) {
      const unsigned long long t_flush = globaltimer_ns();
      const unsigned long long e = warp_sum64((long long)ws.edges);
      const unsigned long long sw = warp_sum64((long long)ws.swept);
      const unsigned long long aq = warp_sum64((long long)ws.acquired);
      if (lane == 0) {
        if (e) atomicAdd((unsigned long long *)&p.stats[r].edges_examined, e);
        if (sw) atomicAdd((unsigned long long *)&p.stats[r].vertices_swept, sw);
        if (aq) atomicAdd((unsigned long long *)&p.stats[r].acquired, aq);
        atomicMax((unsigned long long *)&p.stats[r].t_work_ns, t_work);
        atomicMax((unsigned long long *)&p.stats[r].t_flush_ns, t_flush);
      }
    }
    team_sync<MG>(grid, p.bar, GBBS_NBLK);
  }
  if (STATS && GBBS_BID == 0 && tid == 0 && p.stats && r < p.stats_cap)
    p.stats[r].t_start_ns = (long long)globaltimer_ns();
  if (GBBS_BID == 0 && tid == 0) *p.rounds_out = r;
}
#undef GBBS_BID
#undef GBBS_NBLK

template <bool STATS>
__global__ void __launch_bounds__(BLOCK, GBBS_WBFS_MIN_CTAS)
    wbfs_kernel(const __grid_constant__ Params p) {
  wbfs_body<STATS, false>(p, 1);
}

// G wBFS traversals in one cooperative launch (teams, as traverse_mg_kernel).
__global__ void __launch_bounds__(BLOCK, GBBS_WBFS_MIN_CTAS)
    wbfs_mg_kernel(const __grid_constant__ MultiParams mp) {
  wbfs_body<false, true>(mp.ps[blockIdx.x % mp.G], mp.G);
}

}  // namespace gbbs_dev
