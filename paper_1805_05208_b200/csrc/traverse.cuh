// traverse.cuh — the persistent frontier-traversal kernel (BFS and Bellman-Ford).
//
// One cooperative launch runs the whole traversal: init, then
// rounds of the paper's edgeMap (sec:prelims) separated by
// a grid-wide barrier (the round synchronisation of PAPER.md:89-90).  Each
// round is either
//   * sparse push (a3-a7): the frontier is a vertex list whose entries carry
//     their exclusive edge prefix O (the scan of PAPER.md:1079-1080, computed
//     when the entry was appended, see flush()) and base = offset - O.  The
//     round's d_U edges are cut into fixed tiles of TE edges (edgeMapBlocked's
//     blocks); a tile finds its first/last
//     owner by a warp-wide 32-ary search of O, expands owner ids over its
//     edges with a shared-memory max-scan, loads targets coalesced, and
//     applies F: BFS test-and-set as an atomic fetch-or
//     on the visited bit, Bellman-Ford priority-write as
//     atomicMin on dist followed by a test-and-set on the next-frontier bit.
//     Winners are packed (warp ballot -> shared staging -> one global atomic per
//     flush), i.e. at most LN(U) writes;
//   * dense pull (a8, BFS only): every unvisited vertex scans its in-edges in
//     order and stops at the first one from the frontier (the early-exit dense
//     method of PAPER.md:1870-1874).  A warp owns one 32-vertex bitmap word,
//     so the next visited word is written without atomics.
// The direction is chosen per round from |U| + sum deg(U) against m/T
// (reading A10), read from the packed counter that the
// previous round's flushes produced.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

namespace gbbs_dev {

namespace cg = cooperative_groups;

constexpr int BLOCK = 256;            // threads per CTA
constexpr int NWARPS = BLOCK / 32;
constexpr int EPT = 4;                // edges per thread per tile
constexpr int TE = BLOCK * EPT;       // edges per tile (edgeMapBlocked bsize)
constexpr int CAP = 2 * TE;           // shared staging capacity (vertices)
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr int KBITS = 11;             // head = (tag << KBITS) | owner slot
constexpr int32_t KMASK = (1 << KBITS) - 1;
constexpr int32_t TAG_MAX = (1 << (31 - KBITS)) - 1;

enum Algo { ALGO_BFS = 0, ALGO_BF = 1 };

struct RoundStat {           // mirrors gbbs_round_stat
  int32_t dense;
  int32_t reserved;
  long long frontier;
  long long frontier_edges;
  long long acquired;
  long long edges_examined;
  long long vertices_swept;
  long long t_start_ns;
};

struct Params {
  long long n, m;
  const long long *off;      // out-CSR offsets [n+1]
  const uint32_t *tgt;       // out-CSR targets [m]
  const uint32_t *wgt;       // weights [m] or nullptr (unit)
  const long long *in_off;   // in-CSC (alias of CSR when symmetric)
  const uint32_t *in_tgt;
  uint32_t *dist;            // [n]
  uint32_t *parent;          // [n] or nullptr
  uint32_t *bm[2];           // BFS: visited (double-buffered); BF: next-frontier bits
  uint32_t *fv[2];           // frontier lists: vertex
  long long *fo[2];          //                 exclusive edge prefix O
  long long *fb[2];          //                 base = offset(v) - O
  unsigned long long *cnt;   // packed (count << ebits | edges) ring [4]
  int *status;               // 0 ok, 1 = round cap hit
  long long *rounds_out;
  RoundStat *stats;          // per round, or nullptr
  long long stats_cap;
  long long nwords;
  long long dense_threshold; // dense iff |U| + sum deg(U) > dense_threshold
  long long max_rounds;
  int ebits;
  int mode;                  // 0 auto, 1 sparse, 2 dense
  uint32_t src;
};

struct Smem {
  int64_t own_base[TE];
  uint32_t own_u[TE];
  uint32_t own_du[TE];
  int32_t head[TE];
  uint32_t stage[CAP];
  unsigned long long wk[NWARPS];
  unsigned long long wd[NWARPS];
  int32_t wmax[NWARPS];
  long long i0, i1;
  unsigned long long base_k, base_d;
  unsigned long long cnt;
  int stage_n;
  int tag;
};

// ---- small device helpers --------------------------------------------------

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ long long warp_sum64(long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ long long warp_excl_sum64(long long x, int lane) {
  long long inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  return inc - x;
}

// Largest i in [0, f) with O[i] <= key (O strictly increasing, O[0] = 0 <= key).
// Warp-cooperative 32-ary search: ~log32(f) dependent L2 round trips.
__device__ __forceinline__ long long warp_owner_search(const long long *O, long long f,
                                                       long long key, int lane) {
  long long lo = 0, hi = f;
  while (hi - lo > 32) {
    long long step = (hi - lo + 31) >> 5;
    long long idx = lo + (long long)lane * step;
    bool ok = idx < hi && __ldcg(O + idx) <= key;
    unsigned b = __ballot_sync(0xffffffffu, ok);
    int last = 31 - __clz(b);
    lo = lo + (long long)last * step;
    long long nh = lo + step;
    hi = nh < hi ? nh : hi;
  }
  long long idx = lo + lane;
  bool ok = idx < hi && __ldcg(O + idx) <= key;
  unsigned b = __ballot_sync(0xffffffffu, ok);
  return lo + (31 - __clz(b));
}

// Append the calling lanes with `win` set to the shared staging buffer.
__device__ __forceinline__ void stage_push(Smem &s, bool win, uint32_t v, int lane) {
  unsigned b = __ballot_sync(0xffffffffu, win);
  if (b == 0) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(&s.stage_n, __popc(b));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (win) s.stage[base + __popc(b & lanemask_lt())] = v;
}

// Flush the staging buffer into the next frontier list (a7).  Entries with
// out-degree 0 are dropped (they have no edges to process); the others are
// written at positions reserved with ONE 64-bit atomicAdd of the packed
// (count, edge-sum) pair, which also yields their exclusive edge prefix O —
// so the next round needs no separate degree scan.  Block-uniform call.
template <int ALGO, bool STATS>
__device__ void flush(Smem &s, const Params &p, int nb, int r, uint32_t *bits_next) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cnt = s.stage_n;  // read after the caller's __syncthreads
  if (cnt == 0) return;
  int per = (cnt + NWARPS - 1) / NWARPS;
  per = (per + 31) & ~31;
  const int lo = warp * per;
  const int hi = min(lo + per, cnt);
  const unsigned long long emask = (1ull << p.ebits) - 1;

  unsigned long long K = 0, D = 0;
  for (int b0 = lo; b0 < hi; b0 += 32) {
    int i = b0 + lane;
    long long deg = 0;
    if (i < hi) {
      uint32_t v = s.stage[i];
      deg = __ldg(p.off + v + 1) - __ldg(p.off + v);
    }
    K += __popc(__ballot_sync(0xffffffffu, deg > 0));
    D += (unsigned long long)warp_sum64(deg);
  }
  if (lane == 0) { s.wk[warp] = K; s.wd[warp] = D; }
  __syncthreads();
  if (tid == 0) {
    unsigned long long ak = 0, ad = 0;
    for (int w = 0; w < NWARPS; w++) {
      unsigned long long k = s.wk[w], d = s.wd[w];
      s.wk[w] = ak; s.wd[w] = ad;
      ak += k; ad += d;
    }
    unsigned long long old = 0;
    if (ak > 0) old = atomicAdd(p.cnt + ((r + 1) & 3), (ak << p.ebits) | ad);
    s.base_k = old >> p.ebits;
    s.base_d = old & emask;
    if (STATS && p.stats && r < p.stats_cap)
      atomicAdd((unsigned long long *)&p.stats[r].acquired, (unsigned long long)cnt);
  }
  __syncthreads();
  unsigned long long k = s.base_k + s.wk[warp];
  unsigned long long d = s.base_d + s.wd[warp];
  uint32_t *fv = p.fv[nb];
  long long *fo = p.fo[nb];
  long long *fb = p.fb[nb];
  for (int b0 = lo; b0 < hi; b0 += 32) {
    int i = b0 + lane;
    long long deg = 0, a = 0;
    uint32_t v = 0;
    if (i < hi) {
      v = s.stage[i];
      a = __ldg(p.off + v);
      deg = __ldg(p.off + v + 1) - a;
    }
    bool keep = deg > 0;
    unsigned bal = __ballot_sync(0xffffffffu, keep);
    long long dex = warp_excl_sum64(deg, lane);
    if (keep) {
      unsigned long long pos = k + __popc(bal & lanemask_lt());
      long long o = (long long)d + dex;
      fv[pos] = v;
      fo[pos] = o;
      fb[pos] = a - o;
    } else if (ALGO == ALGO_BF && i < hi) {
      // out-degree-0 vertex: it never enters a frontier; release its TS bit.
      atomicAnd(bits_next + (v >> 5), ~(1u << (v & 31)));
    }
    k += __popc(bal);
    d += (unsigned long long)__shfl_sync(0xffffffffu, dex + deg, 31);
  }
  __syncthreads();
  if (tid == 0) s.stage_n = 0;
  __syncthreads();
}

// ---- sparse push: one tile of TE edges --------------------------------------

template <int ALGO, bool STATS>
__device__ void push_tile(Smem &s, const Params &p, long long tile, long long f, long long E,
                          int cb, int r, uint32_t *bits) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long ts = tile * TE;
  const long long te = min(ts + (long long)TE, E);
  const long long *O = p.fo[cb];
  const long long *B = p.fb[cb];
  const uint32_t *F = p.fv[cb];

  if (warp == 0) {
    long long i0 = warp_owner_search(O, f, ts, lane);
    if (lane == 0) s.i0 = i0;
  } else if (warp == 1) {
    long long i1 = warp_owner_search(O, f, te - 1, lane);
    if (lane == 0) s.i1 = i1;
  }
  if (tid == 0) {
    if (++s.tag >= TAG_MAX) {  // tag wrap: clear heads (rare)
      for (int i = 0; i < TE; i++) s.head[i] = 0;
      s.tag = 1;
    }
  }
  __syncthreads();
  const long long i0 = s.i0;
  const int nown = (int)(s.i1 - i0 + 1);
  const int32_t tagv = s.tag << KBITS;
  // Stage the owners of this tile: u, base, (BF) current dist[u]; mark heads.
  for (int kk = tid; kk < nown; kk += BLOCK) {
    long long i = i0 + kk;
    uint32_t u = __ldcg(F + i);
    s.own_u[kk] = u;
    s.own_base[kk] = __ldcg(B + i);
    if (ALGO == ALGO_BF) s.own_du[kk] = ld_relaxed(p.dist + u);
    if (nown > 1) {
      long long o = __ldcg(O + i) - ts;
      s.head[o > 0 ? o : 0] = tagv | kk;
    }
  }
  __syncthreads();
  if (nown > 1) {
    // inclusive max-scan of head[] (owner id of every edge slot in the tile)
    int4 h = reinterpret_cast<int4 *>(s.head)[tid];
    int32_t a0 = h.x, a1 = max(a0, h.y), a2 = max(a1, h.z), a3 = max(a2, h.w);
    int32_t inc = a3;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc = max(inc, y);
    }
    if (lane == 31) s.wmax[warp] = inc;
    int32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0;
    __syncthreads();
    for (int w = 0; w < warp; w++) ex = max(ex, s.wmax[w]);
    reinterpret_cast<int4 *>(s.head)[tid] = make_int4(max(ex, a0), max(ex, a1), max(ex, a2), max(ex, a3));
    __syncthreads();
  }

  uint32_t vv[EPT];
  uint32_t ww[EPT];
  int kk[EPT];
  bool act[EPT];
#pragma unroll
  for (int j = 0; j < EPT; j++) {
    int pos = j * BLOCK + tid;
    long long e = ts + pos;
    act[j] = e < te;
    kk[j] = 0;
    if (act[j]) {
      int k = nown > 1 ? (s.head[pos] & KMASK) : 0;
      kk[j] = k;
      long long idx = s.own_base[k] + e;
      vv[j] = __ldcs(p.tgt + idx);
      if (ALGO == ALGO_BF) ww[j] = p.wgt ? __ldcs(p.wgt + idx) : 1u;
    }
  }
  const uint32_t next_d = (uint32_t)(r + 1);
#pragma unroll
  for (int j = 0; j < EPT; j++) {
    bool win = false;
    uint32_t v = vv[j];
    if (ALGO == ALGO_BFS) {
      if (act[j]) {
        uint32_t bit = 1u << (v & 31);
        if (!(ld_relaxed(bits + (v >> 5)) & bit)) {
          uint32_t old = atomicOr(bits + (v >> 5), bit);   // test-and-set
          if (!(old & bit)) {
            win = true;
            p.dist[v] = next_d;
            if (p.parent) p.parent[v] = s.own_u[kk[j]];
          }
        }
      }
    } else {
      if (act[j]) {
        unsigned long long nd = (unsigned long long)s.own_du[kk[j]] + ww[j];
        if (nd < (unsigned long long)ld_relaxed(p.dist + v)) {
          uint32_t old = atomicMin(p.dist + v, (uint32_t)nd);  // priority-write
          if (nd < old) {
            uint32_t bit = 1u << (v & 31);
            uint32_t ob = atomicOr(bits + (v >> 5), bit);      // next-frontier TS
            win = !(ob & bit);
          }
        }
      }
    }
    stage_push(s, win, v, lane);
  }
  if (STATS && p.stats && r < p.stats_cap) {
    long long ne = te - ts;
    if (tid == 0) atomicAdd((unsigned long long *)&p.stats[r].edges_examined, (unsigned long long)ne);
  }
  __syncthreads();
}

// ---- dense pull (BFS): 8 bitmap words (256 vertices) per CTA iteration -------

template <bool STATS>
__device__ void pull_chunk(Smem &s, const Params &p, long long chunk, const uint32_t *vis,
                           uint32_t *vis_next, int r) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long word = chunk * NWARPS + warp;
  if (word >= p.nwords) return;
  const uint32_t vw = vis[word];
  uint32_t nw = vw;
  if (vw != 0xFFFFFFFFu) {
    const uint32_t v = (uint32_t)(word * 32 + lane);
    const bool need = !((vw >> lane) & 1u);
    uint32_t par = INF;
    long long loaded = 0;
    if (need) {
      long long j = __ldg(p.in_off + v);
      const long long e = __ldg(p.in_off + v + 1);
      for (; j < e && par == INF; j += 4) {
        uint32_t u0 = __ldg(p.in_tgt + j);
        uint32_t u1 = j + 1 < e ? __ldg(p.in_tgt + j + 1) : u0;
        uint32_t u2 = j + 2 < e ? __ldg(p.in_tgt + j + 2) : u0;
        uint32_t u3 = j + 3 < e ? __ldg(p.in_tgt + j + 3) : u0;
        bool b0 = (vis[u0 >> 5] >> (u0 & 31)) & 1u;
        bool b1 = (vis[u1 >> 5] >> (u1 & 31)) & 1u;
        bool b2 = (vis[u2 >> 5] >> (u2 & 31)) & 1u;
        bool b3 = (vis[u3 >> 5] >> (u3 & 31)) & 1u;
        if (STATS) loaded += min(4ll, e - j);
        par = b0 ? u0 : b1 ? u1 : b2 ? u2 : b3 ? u3 : INF;
      }
    }
    const bool found = par != INF;
    const unsigned nb = __ballot_sync(0xffffffffu, found);
    nw |= nb;
    if (found) {
      p.dist[v] = (uint32_t)(r + 1);
      if (p.parent) p.parent[v] = par;
    }
    stage_push(s, found, v, lane);
    if (STATS && p.stats && r < p.stats_cap) {
      long long sl = warp_sum64(loaded);
      int sw = __popc(__ballot_sync(0xffffffffu, need));
      if (lane == 0) {
        atomicAdd((unsigned long long *)&p.stats[r].edges_examined, (unsigned long long)sl);
        atomicAdd((unsigned long long *)&p.stats[r].vertices_swept, (unsigned long long)sw);
      }
    }
  }
  if (lane == 0) vis_next[word] = nw;
}

// ---- the persistent kernel ---------------------------------------------------

template <int ALGO, bool STATS>
__global__ void __launch_bounds__(BLOCK) traverse_kernel(Params p) {
  __shared__ Smem s;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  const long long gtid = (long long)blockIdx.x * BLOCK + tid;
  const long long gstride = (long long)gridDim.x * BLOCK;
  const uint32_t src = p.src;

  // a1: per-run init
  for (long long i = gtid; i < p.n; i += gstride) {
    p.dist[i] = (i == src) ? 0u : INF;
    if (ALGO == ALGO_BFS && p.parent) p.parent[i] = (i == src) ? src : INF;
  }
  for (long long w = gtid; w < p.nwords; w += gstride) {
    if (ALGO == ALGO_BFS) {
      uint32_t x = 0;
      long long lo = w * 32;
      if (lo + 32 > p.n) x = 0xFFFFFFFFu << (uint32_t)(p.n - lo);  // padding = visited
      if ((long long)(src >> 5) == w) x |= 1u << (src & 31);
      p.bm[0][w] = x;
    } else {
      p.bm[0][w] = 0;
      p.bm[1][w] = 0;
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    long long a = p.off[src], d0 = p.off[src + 1] - a;
    p.cnt[1] = p.cnt[2] = p.cnt[3] = 0;
    if (d0 > 0) {
      p.fv[0][0] = src;
      p.fo[0][0] = 0;
      p.fb[0][0] = a;
      p.cnt[0] = (1ull << p.ebits) | (unsigned long long)d0;
    } else {
      p.cnt[0] = 0;
    }
    *p.status = 0;
  }
  if (tid == 0) { s.stage_n = 0; s.tag = 0; }
  for (int i = tid; i < TE; i += BLOCK) s.head[i] = 0;
  grid.sync();

  const unsigned long long emask = (1ull << p.ebits) - 1;
  int vc = 0;  // BFS: index of the current visited bitmap
  long long r = 0;
  for (;; r++) {
    if (tid == 0) s.cnt = ld_relaxed64(p.cnt + (r & 3));
    __syncthreads();
    const unsigned long long c = s.cnt;
    const long long f = (long long)(c >> p.ebits);
    const long long E = (long long)(c & emask);
    if (STATS && blockIdx.x == 0 && tid == 0 && p.stats && r < p.stats_cap)
      p.stats[r].t_start_ns = (long long)globaltimer_ns();
    if (f == 0) break;
    if (r >= p.max_rounds) {
      if (blockIdx.x == 0 && tid == 0) *p.status = 1;
      break;
    }
    bool dense = false;
    if (ALGO == ALGO_BFS)
      dense = p.mode == 2 || (p.mode == 0 && f + E > p.dense_threshold);
    if (blockIdx.x == 0 && tid == 0) {
      p.cnt[(r + 2) & 3] = 0;
      if (STATS && p.stats && r < p.stats_cap) {
        p.stats[r].dense = dense;
        p.stats[r].frontier = f;
        p.stats[r].frontier_edges = E;
      }
    }
    const int cb = (int)(r & 1), nbuf = cb ^ 1;
    if (dense) {
      const uint32_t *vis = p.bm[vc];
      uint32_t *vis_next = p.bm[vc ^ 1];
      const long long nchunks = (p.nwords + NWARPS - 1) / NWARPS;
      for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        pull_chunk<STATS>(s, p, ch, vis, vis_next, (int)r);
        __syncthreads();
        if (s.stage_n > CAP - BLOCK) flush<ALGO, STATS>(s, p, nbuf, (int)r, nullptr);
      }
      vc ^= 1;
    } else {
      uint32_t *bits = (ALGO == ALGO_BFS) ? p.bm[vc] : p.bm[nbuf];
      if (ALGO == ALGO_BF) {
        // a11: release the current frontier's TS bits (buffer cb is idle this round)
        uint32_t *cur_bits = p.bm[cb];
        const uint32_t *F = p.fv[cb];
        for (long long i = gtid; i < f; i += gstride) cur_bits[__ldcg(F + i) >> 5] = 0;
      }
      const long long ntiles = (E + TE - 1) / TE;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        push_tile<ALGO, STATS>(s, p, t, f, E, cb, (int)r, bits);
        if (s.stage_n > CAP - TE) flush<ALGO, STATS>(s, p, nbuf, (int)r, bits);
      }
    }
    __syncthreads();
    flush<ALGO, STATS>(s, p, nbuf, (int)r, (ALGO == ALGO_BF) ? p.bm[nbuf] : nullptr);
    grid.sync();
  }
  if (blockIdx.x == 0 && tid == 0) *p.rounds_out = r;
}

}  // namespace gbbs_dev
