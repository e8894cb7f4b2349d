// sbf.cuh — NEXT-4: general-weight (signed) frontier Bellman-Ford.
//
// Output spec PAPER.md:1487-1490 (sec:benchmark, "General-Weight SSSP
// (Bellman-Ford)"): D[v] = the shortest-path distance from src, infinity if v is
// unreachable, and "All distances must be -infinity if G contains a
// negative-weight cycle reachable from src".  Algorithm
// (sec:algs): rounds of edgeMap whose F is the priority-write min of
// d(u) + w(u,v); a vertex enters the next frontier when its
// distance dropped.
//
// Distances are int64 (weights are the graph's 32-bit weights read as int32).
// Without a reachable negative cycle every shortest path is simple, so the
// frontier empties within n rounds; a frontier still non-empty after round n-1
// proves a reachable negative cycle (reading N2).  Then:
//  * scope 0 (default, the paper's sentence read literally, reading N1): every
//    distance is -infinity;
//  * scope 1 (SPEC's reading): exactly the vertices reachable from a reachable
//    negative cycle get -infinity.  Seeds are the targets of edges still
//    relaxable after the n rounds plus vertices whose distance reached FLOOR;
//    every such vertex lies downstream of a negative cycle, and every reachable
//    negative cycle contains one (the sum of d(v) - d(u) - w over its edges
//    would otherwise be >= 0).  The -infinity region is their forward closure.
// Candidates saturate at FLOOR = -2^62: no simple path reaches it because
// (n-1) * max|w| < 2^62 is required (GBBS_ERANGE otherwise), so a distance at
// FLOOR certifies a negative cycle and int64 arithmetic never overflows.
//
// Early detection (reading N4): a relaxation that lowers d(v) records its edge
// (parent, weight) for v.  From round SBF_DETECT on, at every power-of-two
// round, pointer doubling over the parent pointers finds the vertices whose
// parent chain does not end at the source; one of them leads into a cycle of the
// parent graph, which is walked and its recorded weights summed.  Every recorded
// pair is a real edge, so a negative sum proves a reachable negative cycle (a
// non-negative one — possible, as the records race — proves nothing and the
// rounds go on).  Scope 0 then fills -infinity at once; scope 1 freezes the
// cycle's forward closure at -infinity (frozen vertices relax nothing) and goes
// on with the rest, so the run ends when the remaining frontier empties.  The
// n-round rule above stays as the backstop (a cycle longer than SBF_WALK, or
// records that keep racing).
// Work distribution as the list push of traverse.cuh: the frontier list carries
// edge prefixes, warps take fixed tiles of SBF_TE edges (edgeMapBlocked's
// blocks), owners expanded over the tile in shared memory.
#pragma once

#include "traverse.cuh"

namespace gbbs_dev {

constexpr long long SBF_INF = 0x7FFFFFFFFFFFFFFFll;
constexpr long long SBF_NEGINF = (long long)0x8000000000000000ull;
constexpr long long SBF_FLOOR = -(1ll << 62);
constexpr int SBF_TE = 128;
constexpr long long SBF_DETECT = 64;    // first round of the early negative-cycle check
constexpr long long SBF_WALK = 1 << 16; // longest parent cycle walked

struct SbfWarpSmem {
  alignas(16) int32_t head[SBF_TE];
  long long base[SBF_TE + 1];
  long long dval[SBF_TE + 1];
  uint32_t own[SBF_TE + 1];
  uint32_t stage[WCAP];
};

__device__ __forceinline__ long long sbf_weight(const Params &p, long long e) {
  return p.wgt ? (long long)(int32_t)ld_stream(p.wgt + e) : 1ll;
}

// One tile [t*SBF_TE, ...) of the round's edge space (frontier list lb).
template <bool STATS>
__device__ __forceinline__ void sbf_tile(const Params &p, SbfWarpSmem &w, WarpState &ws, int lb,
                                         long long t, long long f, long long E, int nb, int r,
                                         uint32_t *bits) {
  constexpr long long BIG = 0x7FFFFFFFFFFFFFFFll;
  const int lane = threadIdx.x & 31;
  const long long ts = t * SBF_TE;
  const long long te = min(ts + (long long)SBF_TE, E);
  const long long *O = p.fo[lb];
  const long long *B = p.fb[lb];
  const uint32_t *F = p.fv[lb];
  if (STATS && lane == 0) ws.edges += (unsigned long long)(te - ts);
  const long long i0 = warp_upper_est(O, f, E, ts);
  {
    int4 *h4 = reinterpret_cast<int4 *>(w.head);
    h4[lane] = make_int4(0, 0, 0, 0);  // SBF_TE = 128 = 32 lanes x 4
  }
  __syncwarp();
  for (int kb = 0;; kb += 32) {
    const long long kk = i0 + kb + lane;
    long long o = BIG;
    if (kk < f) o = __ldcg(O + kk);
    const bool in = o < te;
    if (in) {
      w.base[kb + lane] = __ldcg(B + kk);
      const uint32_t u = __ldcg(F + kk);
      w.own[kb + lane] = u;
      w.dval[kb + lane] = __ldcg(p.sdist + u);  // coherent: updated last round
      w.head[o > ts ? o - ts : 0] = kb + lane + 1;
    }
    if (__popc(__ballot_sync(FULL, in)) < 32) break;
  }
  __syncwarp();
  {
    int4 *h4 = reinterpret_cast<int4 *>(w.head);
    int4 x = h4[lane];
    int32_t a0 = x.x, a1 = max(a0, x.y), a2 = max(a1, x.z), a3 = max(a2, x.w);
    int32_t inc = a3;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc = max(inc, y);
    }
    int32_t ex = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) ex = 0;
    h4[lane] = make_int4(max(ex, a0), max(ex, a1), max(ex, a2), max(ex, a3));
  }
  __syncwarp();
  for (long long cs = ts; cs < te; cs += 32) {
    const long long e = cs + lane;
    bool win = false;
    uint32_t v = 0;
    if (e < te) {
      const int kk = w.head[e - ts] - 1;
      const long long bb = w.base[kk];
      const long long du = w.dval[kk];
      GBBS_CHECK(bb + e >= 0 && bb + e < p.m);
      v = ld_stream(p.tgt + bb + e);
      const long long we = sbf_weight(p, bb + e);
      long long nd = du + we;
      if (nd < SBF_FLOOR) nd = SBF_FLOOR;
      const long long cur = (long long)ld_relaxed64((const unsigned long long *)(p.sdist + v));
      if (du != SBF_NEGINF && nd < cur) {  // a frozen (-infinity) owner relaxes nothing
        const long long old = atomicMin(p.sdist + v, nd);  // priority-write (min)
        if (nd < old) {
          // the relaxing edge, for the parent-cycle check (racy, each store one real edge)
          p.fo[2][v] = (long long)(((unsigned long long)w.own[kk] << 32) | (uint32_t)(int32_t)we);
          const uint32_t bit = 1u << (v & 31);
          win = !(atomicOr(bits + (v >> 5), bit) & bit);  // next-frontier TS
        }
      }
    }
    const unsigned b = __ballot_sync(FULL, win);
    GBBS_CHECK(ws.scnt + __popc(b) <= WCAP);
    if (win) w.stage[ws.scnt + __popc(b & lanemask_lt())] = v;
    ws.scnt += __popc(b);
    if (ws.scnt > WCAP - 32) {
      if (STATS && lane == 0) ws.acquired += ws.scnt;
      warp_flush<ALGO_BF>(p, w.stage, ws.scnt, nb, r, bits);
      ws.scnt = 0;
    }
  }
  __syncwarp();
}

// Forward closure of the set R (bitmap, X = expanded set, both zeroed by the
// caller except R's seeds): every vertex reachable from R joins R; then every
// vertex of R gets -infinity.  ctr[0..2]: zeroed change counters.
__device__ __forceinline__ void sbf_closure(const Params &p, cg::grid_group &grid, uint32_t *R,
                                            uint32_t *X, unsigned long long *ctr,
                                            unsigned long long &s_cnt) {
  const int tid = threadIdx.x;
  const long long gtid = (long long)blockIdx.x * BLOCK + tid;
  const long long gstride = (long long)gridDim.x * BLOCK;
  for (long long sweep = 0;; sweep++) {  // expand reached, not yet expanded vertices
    grid.sync();
    if (tid == 0) s_cnt = ld_relaxed64(ctr + (sweep % 3));
    if (blockIdx.x == 0 && tid == 0) ctr[(sweep + 2) % 3] = 0;
    __syncthreads();
    if (sweep > 0 && s_cnt == 0) break;
    bool changed = false;
    for (long long w = gtid; w < p.nwords; w += gstride) {
      unsigned todo = ld_relaxed(R + w) & ~X[w];
      if (!todo) continue;
      X[w] |= todo;
      changed = true;
      while (todo) {
        const uint32_t u = (uint32_t)(w * 32 + __ffs(todo) - 1);
        todo &= todo - 1;
        for (long long e = p.off[u]; e < p.off[u + 1]; e++) {
          const uint32_t v = p.tgt[e];
          atomicOr(R + (v >> 5), 1u << (v & 31));
        }
      }
    }
    if (changed) atomicAdd(ctr + ((sweep + 1) % 3), 1ull);
  }
  for (long long i = gtid; i < p.n; i += gstride)
    if ((ld_relaxed(R + (i >> 5)) >> (i & 31)) & 1u) p.sdist[i] = SBF_NEGINF;
  grid.sync();
}

// Early negative-cycle check (reading N4), between rounds (all threads, uniform
// result).  J = p.fv[2]: ancestor by pointer doubling; M (first half of p.fb[2]):
// the smallest vertex among the ancestors J covered; seen (second half): one
// bit per cycle representative; parent records p.fo[2]; scratch p.wq[0..1].
// After more doublings than n, J[v] of a vertex whose parent chain misses the
// roots lies on a cycle of the parent graph and M[J[v]] is that cycle's smallest
// vertex.  Racing records can close cycles that are not negative, so every
// cycle is walked (by one thread, from its smallest vertex) and its recorded
// weights summed.  Returns the smallest vertex of a negative cycle, or -1.
__device__ __forceinline__ long long sbf_detect(const Params &p, cg::grid_group &grid,
                                                unsigned long long &s_cnt) {
  const int tid = threadIdx.x;
  const long long gtid = (long long)blockIdx.x * BLOCK + tid;
  const long long gstride = (long long)gridDim.x * BLOCK;
  uint32_t *J = p.fv[2];
  uint32_t *M = reinterpret_cast<uint32_t *>(p.fb[2]);
  uint32_t *seen = M + p.n;
  const long long *pw = p.fo[2];
  // resolved vertices point to themselves: the source, the unreached, the frozen
  for (long long v = gtid; v < p.n; v += gstride) {
    const long long d = __ldcg(p.sdist + v);
    J[v] = (v == p.src || d == SBF_INF || d == SBF_NEGINF)
               ? (uint32_t)v
               : (uint32_t)((unsigned long long)__ldcg(pw + v) >> 32);
    M[v] = (uint32_t)v;
  }
  for (long long w = gtid; w < p.nwords; w += gstride) seen[w] = 0;
  if (blockIdx.x == 0 && tid == 0) p.wq[1] = ~0ull;
  int steps = 1;
  while ((1ll << steps) < p.n) steps++;
  for (int k = 0; k <= steps; k++) {  // in place: J[v] only moves up v's chain
    grid.sync();
    for (long long v = gtid; v < p.n; v += gstride) {
      const uint32_t j = __ldcg(J + v);
      M[v] = min(__ldcg(M + v), __ldcg(M + j));
      J[v] = __ldcg(J + j);
    }
  }
  grid.sync();
  for (long long v = gtid; v < p.n; v += gstride) {
    const uint32_t x = __ldcg(J + v);  // resolved v: x = v; else src or a cycle vertex
    if (x == p.src) continue;
    const long long dx = __ldcg(p.sdist + x);
    if (dx == SBF_NEGINF || dx == SBF_INF) continue;
    const uint32_t c = __ldcg(M + x);  // the cycle's smallest vertex
    const uint32_t bit = 1u << (c & 31);
    if (atomicOr(seen + (c >> 5), bit) & bit) continue;  // walked by another thread
    long long sum = 0, len = 0;
    uint32_t y = c;
    do {
      const unsigned long long rec = (unsigned long long)__ldcg(pw + y);
      sum += (long long)(int32_t)(uint32_t)(rec & 0xFFFFFFFFull);
      y = (uint32_t)(rec >> 32);
      len++;
    } while (y != c && len < SBF_WALK);
    if (y == c && sum < 0) atomicMin(p.wq + 1, (unsigned long long)c);
  }
  grid.sync();
  if (tid == 0) s_cnt = ld_relaxed64(p.wq + 1);
  __syncthreads();
  return s_cnt == ~0ull ? -1 : (long long)s_cnt;
}

template <bool STATS>
__global__ void __launch_bounds__(BLOCK, GBBS_MIN_CTAS) sbf_kernel(Params p) {
  __shared__ SbfWarpSmem sw[NWARPS];
  __shared__ unsigned long long s_cnt;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long gtid = (long long)blockIdx.x * BLOCK + tid;
  const long long gstride = (long long)gridDim.x * BLOCK;
  const long long gw = (long long)blockIdx.x * NWARPS + warp;
  const long long nw = (long long)gridDim.x * NWARPS;
  const uint32_t src = p.src;
  SbfWarpSmem &wsm = sw[warp];
  const unsigned long long emask = (1ull << p.ebits) - 1;

  // a1: init
  for (long long i = gtid; i < p.n; i += gstride) p.sdist[i] = (i == src) ? 0 : SBF_INF;
  for (long long w = gtid; w < p.nwords; w += gstride) p.bm[0][w] = p.bm[1][w] = 0;
  const long long a0 = p.off[src], d0 = p.off[src + 1] - a0;
  if (blockIdx.x == 0 && tid == 0) {
    p.cnt[1] = p.cnt[2] = p.cnt[3] = 0;
    if (d0 > 0) {
      p.fv[0][0] = src;
      p.fo[0][0] = 0;
      p.fb[0][0] = a0;
      p.cnt[0] = (1ull << p.ebits) | (unsigned long long)d0;
      p.bm[0][src >> 5] = 1u << (src & 31);
    } else {
      p.cnt[0] = 0;
    }
    *p.status = 0;
  }
  grid.sync();

  long long r = 0;
  bool negcycle = false;
  for (;; r++) {
    if (r >= SBF_DETECT && (r & (r - 1)) == 0 && r < p.max_rounds) {  // uniform
      const long long c = sbf_detect(p, grid, s_cnt);
      if (c >= 0) {
        if (blockIdx.x == 0 && tid == 0) *p.status = 2;
        if (p.neg_scope == 0) {  // reading N1: every distance is -infinity
          if (blockIdx.x == 0 && tid == 0) *p.rounds_out = r;
          for (long long i = gtid; i < p.n; i += gstride) p.sdist[i] = SBF_NEGINF;
          return;
        }
        // scope 1: freeze the cycle's forward closure at -infinity and go on
        uint32_t *R = reinterpret_cast<uint32_t *>(p.fb[2]), *X = R + p.nwords;
        for (long long w = gtid; w < p.nwords; w += gstride) R[w] = X[w] = 0;
        if (blockIdx.x == 0 && tid == 0) p.wq[2] = p.wq[3] = p.wq[4] = 0;
        grid.sync();
        if (blockIdx.x == 0 && tid == 0) {
          uint32_t x = (uint32_t)c;
          do {
            R[x >> 5] |= 1u << (x & 31);
            x = (uint32_t)((unsigned long long)p.fo[2][x] >> 32);
          } while (x != (uint32_t)c);
        }
        sbf_closure(p, grid, R, X, p.wq + 2, s_cnt);
      }
    }
    if (tid == 0) s_cnt = ld_relaxed64(p.cnt + (r & 3));
    __syncthreads();
    const unsigned long long c = s_cnt;
    const long long f = (long long)(c >> p.ebits);
    const long long E = (long long)(c & emask);
    if (STATS && blockIdx.x == 0 && tid == 0 && p.stats && r < p.stats_cap)
      p.stats[r].t_start_ns = (long long)globaltimer_ns();
    if (f == 0) break;
    if (r >= p.max_rounds) {  // still relaxing after n rounds: a reachable negative cycle
      negcycle = true;
      break;
    }
    const int cb = (int)(r & 1), nb = cb ^ 1;
    if (blockIdx.x == 0 && tid == 0) {
      p.cnt[(r + 2) & 3] = 0;
      if (STATS && p.stats && r < p.stats_cap) {
        p.stats[r].frontier = f;
        p.stats[r].frontier_edges = E;
      }
    }
    // a11: release the current frontier's TS bits (buffer cb is idle this round)
    for (long long i = gtid; i < f; i += gstride) p.bm[cb][__ldcg(p.fv[cb] + i) >> 5] = 0;
    WarpState ws;
    const long long ntiles = (E + SBF_TE - 1) / SBF_TE;
    for (long long t = gw; t < ntiles; t += nw)
      sbf_tile<STATS>(p, wsm, ws, cb, t, f, E, nb, (int)r, p.bm[nb]);
    if (ws.scnt > 0) {
      if (STATS && lane == 0) ws.acquired += ws.scnt;
      warp_flush<ALGO_BF>(p, wsm.stage, ws.scnt, nb, (int)r, p.bm[nb]);
    }
    if (STATS && p.stats && r < p.stats_cap) {
      const unsigned long long e = warp_sum64((long long)ws.edges);
      const unsigned long long aq = warp_sum64((long long)ws.acquired);
      if (lane == 0) {
        if (e) atomicAdd((unsigned long long *)&p.stats[r].edges_examined, e);
        if (aq) atomicAdd((unsigned long long *)&p.stats[r].acquired, aq);
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && tid == 0) *p.rounds_out = r;
  if (!negcycle) return;  // uniform
  if (blockIdx.x == 0 && tid == 0) *p.status = 2;
  if (p.neg_scope == 0) {  // reading N1: every distance is -infinity
    for (long long i = gtid; i < p.n; i += gstride) p.sdist[i] = SBF_NEGINF;
    return;
  }
  // reading N2 (scope 1): forward closure of the seeds.  bm[0] = reached set V,
  // bm[1] = expanded set X; sweep s counts its expansions in cnt[(s+1) % 3].
  grid.sync();
  for (long long w = gtid; w < p.nwords; w += gstride) p.bm[0][w] = p.bm[1][w] = 0;
  if (blockIdx.x == 0 && tid == 0) p.cnt[0] = p.cnt[1] = p.cnt[2] = 0;
  grid.sync();
  for (long long u = gw; u < p.n; u += nw) {  // seeds: one warp per vertex
    const long long du = __ldcg(p.sdist + u);
    if (du == SBF_INF) continue;
    if (du == SBF_FLOOR || du == SBF_NEGINF) {  // NEGINF: frozen by an early check
      if (lane == 0) atomicOr(p.bm[0] + (u >> 5), 1u << (u & 31));
      continue;
    }
    const long long a = p.off[u], b = p.off[u + 1];
    for (long long e = a + lane; e < b; e += 32) {
      const uint32_t v = p.tgt[e];
      long long nd = du + sbf_weight(p, e);
      if (nd < SBF_FLOOR) nd = SBF_FLOOR;
      if (nd < __ldcg(p.sdist + v)) atomicOr(p.bm[0] + (v >> 5), 1u << (v & 31));
    }
  }
  sbf_closure(p, grid, p.bm[0], p.bm[1], p.cnt, s_cnt);
}

}  // namespace gbbs_dev
