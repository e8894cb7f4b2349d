// bc.cuh — single-source betweenness contributions (NEXT-3), one persistent
// cooperative kernel per call.
//
// PAPER.md:98-101 (sec:algs): "It uses fetch-and-add to compute the total number
// of shortest-paths through vertices"; output spec PAPER.md:1493-1496: for every
// v, the contribution to v's centrality from all (src, t) shortest paths through
// v — Brandes' dependency delta_src(v).
//
//  forward  level r -> r+1 over the level-r vertex list (edge tiles as in the
//           list push of traverse.cuh): for edge (u, v) the test-and-set is an
//           atomicCAS(dist[v], INF, r+1) whose returned value also says whether
//           v lies on level r+1 (won or lost to a same-level writer), and the
//           fetch-and-add is atomicAdd(sigma[v], sigma[u]) in fp64.  Winners are
//           appended to a cumulative level queue (all levels kept, in order).
//  dense    forward level on a symmetric graph (Ligra's dense edgeMap, P:1851-1874,
//           reading B3): every unvisited vertex v sums sigma over its neighbours
//           on level r (owner-computes, no atomics) and joins level r+1 iff the
//           sum is positive; used when |U| + sum deg(U) > m/T and the unvisited
//           vertices carry fewer edges than the frontier (no early exit here).
//  backward levels L-1 .. 1: for every edge (u, v) of a level-l vertex u with
//           dist[v] = l+1, delta[u] += sigma[u] / sigma[v] * (1 + delta[v])
//           (Brandes' recurrence), a grid barrier between levels.
// delta[src] = 0 and unreached vertices keep 0 (reading B1).
#pragma once

#include "traverse.cuh"

// Backward-pass A/B knobs (tools/bc_probe.py): SEG = one atomicAdd per (owner,
// chunk) after a segmented warp sum (c2 -10 %, c4 -4 % time); SPEC = load the
// target's sigma and delta speculatively beside its level (measured 35-55 %
// slower: two extra random fp64 sectors per non-DAG edge).
#ifndef GBBS_BC_SPEC
#define GBBS_BC_SPEC 0
#endif
#ifndef GBBS_BC_SEG
#define GBBS_BC_SEG 1
#endif
// Dense forward levels (reading B3) need the unvisited vertices' edges below
// 1/RATIO of the frontier's: a pulled edge (lane-serial, no early exit) costs more
// than a pushed one
#ifndef GBBS_BC_PULL_RATIO
#define GBBS_BC_PULL_RATIO 4
#endif
#ifndef GBBS_BC_DYNQ_FWD
#define GBBS_BC_DYNQ_FWD 1
#endif
#ifndef GBBS_BC_DYNQ_BACK
#define GBBS_BC_DYNQ_BACK 1
#endif

namespace gbbs_dev {

struct BcParams {
  long long n, m;
  const long long *off;
  const uint32_t *tgt;
  uint32_t *dist;            // [n] level of each vertex (INF = unreached)
  double *sigma;             // [n] shortest-path counts
  double *delta;             // [n] output
  uint32_t *qv;              // cumulative level queue: vertex
  long long *qo;             //   exclusive edge prefix O within its level
  long long *qb;             //   base = offset(v) - O
  long long *lvl;            // [3 * lvl_cap]: start, count, edges per level
  long long lvl_cap;
  unsigned long long *cnt;   // packed (count << ebits | edges) ring [4]
  unsigned long long *wq;    // [8] tile work-queue counters: forward ring [4], backward ring [4]
  unsigned *bar;             // team barrier words (multi-traversal launches)
  int *status;
  long long *rounds_out;
  int ebits;
  uint32_t src;
  long long dense_threshold;  // m / T
  int dense_mode;             // 0: the rule above, 1: never (push), 2: always (pull)
};

struct BcWarpSmem {
  alignas(16) int32_t head[TE];
  long long base[TE + 1];
  uint32_t own[TE + 1];
  uint32_t stage[WCAP];
};

struct BcSmem {
  BcWarpSmem w[NWARPS];
  unsigned long long cnt;
};

// Append staged vertices (all with out-degree > 0 are kept) to the next level.
__device__ __forceinline__ void bc_flush(const BcParams &p, const uint32_t *st, int cnt,
                                         long long qbase, unsigned long long *ctr) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  long long Kl = 0, Dl = 0;
  for (int i = lane; i < cnt; i += 32) {
    const uint32_t v = st[i];
    const long long dg = __ldg(p.off + v + 1) - __ldg(p.off + v);
    Kl += dg > 0;
    Dl += dg;
  }
  const unsigned long long K = warp_sum64(Kl), D = warp_sum64(Dl);
  unsigned long long old = 0;
  if (lane == 0 && K) old = atomicAdd(ctr, (K << p.ebits) | D);
  old = __shfl_sync(FULL, old, 0);
  unsigned long long k = old >> p.ebits, d = old & ((1ull << p.ebits) - 1);
  for (int b0 = 0; b0 < cnt; b0 += 32) {
    const int i = b0 + lane;
    uint32_t v = 0;
    long long a = 0, deg = 0;
    if (i < cnt) {
      v = st[i];
      a = __ldg(p.off + v);
      deg = __ldg(p.off + v + 1) - a;
    }
    const bool keep = deg > 0;
    const unsigned bal = __ballot_sync(FULL, keep);
    const long long dex = warp_excl_sum64(deg, lane);
    if (keep) {
      const unsigned long long pos = qbase + k + __popc(bal & lanemask_lt());
      const long long o = (long long)d + dex;
      GBBS_CHECK(pos < (unsigned long long)p.n);
      p.qv[pos] = v;
      p.qo[pos] = o;
      p.qb[pos] = a - o;
    }
    k += __popc(bal);
    d += (unsigned long long)__shfl_sync(FULL, dex + deg, 31);
  }
  __syncwarp();
}

// One warp tile of level-l edges: owners staged in shared memory (1 + index at
// the slot of each owner's first in-tile edge, expanded by a warp max-scan).
// BACK = false: forward (CAS + sigma fetch-and-add, stage winners);
// BACK = true : backward (accumulate delta of the owners).
template <bool BACK>
__device__ __forceinline__ long long bc_tile(const BcParams &p, BcWarpSmem &w, int &scnt,
                                             const uint32_t *F, const long long *O,
                                             const long long *B, long long f, long long E,
                                             long long i0, long long t, int l, long long qnext,
                                             unsigned long long *ctr) {
  constexpr long long BIG = 0x7FFFFFFFFFFFFFFFll;
  const int lane = threadIdx.x & 31;
  const long long ts = t * TE;
  const long long te = min(ts + (long long)TE, E);
  {
    int4 *h4 = reinterpret_cast<int4 *>(w.head);
#pragma unroll
    for (int q = 0; q < TE / 128; q++) h4[q * 32 + lane] = make_int4(0, 0, 0, 0);
  }
  __syncwarp();
  int nown = 0;
  long long onext = BIG;
  for (int kb = 0;; kb += 32) {
    const long long kk = i0 + kb + lane;
    long long o = BIG, b = 0;
    uint32_t u = 0;
    if (kk < f) {
      o = __ldcg(O + kk);
      b = __ldcg(B + kk);
      u = __ldcg(F + kk);
    }
    const int c = __popc(__ballot_sync(FULL, o < te));
    if (o < te) {
      w.base[kb + lane] = b;
      w.own[kb + lane] = u;
      const long long r = o - ts;
      w.head[r > 0 ? r : 0] = kb + lane + 1;
    }
    nown += c;
    if (c < 32) {
      onext = __shfl_sync(FULL, o, c);
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
  const uint32_t nl = (uint32_t)(l + 1);
  for (long long cs = ts; cs < te; cs += 32 * NCH) {
    uint32_t vv[NCH], uu[NCH];
    bool act[NCH];
#pragma unroll
    for (int j = 0; j < NCH; j++) {
      const long long e = cs + 32 * j + lane;
      act[j] = e < te;
      vv[j] = 0;
      uu[j] = 0;
      if (act[j]) {
        const int kk = w.head[e - ts] - 1;
        uu[j] = w.own[kk];
        GBBS_CHECK(w.base[kk] + e >= 0 && w.base[kk] + e < p.m);
        vv[j] = ld_stream(p.tgt + w.base[kk] + e);
      }
    }
    if (!BACK) {
      bool win[NCH];
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        win[j] = false;
        if (!act[j]) continue;
        uint32_t cur = p.dist[vv[j]];
        bool same = cur == nl;
        if (cur == INF) {
          const uint32_t old = atomicCAS(p.dist + vv[j], INF, nl);  // test-and-set
          win[j] = old == INF;
          same = win[j] || old == nl;
        }
        if (same) atomicAdd(p.sigma + vv[j], p.sigma[uu[j]]);  // fetch-and-add
      }
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        const unsigned b = __ballot_sync(FULL, win[j]);
        if (win[j]) w.stage[scnt + __popc(b & lanemask_lt())] = vv[j];
        scnt += __popc(b);
      }
      if (scnt > WCAP - 32 * NCH) {
        bc_flush(p, w.stage, scnt, qnext, ctr);
        scnt = 0;
      }
    } else {
#if GBBS_BC_SPEC  // level, sigma and delta of the target loaded together
      uint32_t dv[NCH];
      double sv[NCH], tv[NCH], su[NCH];
#pragma unroll
      for (int j = 0; j < NCH; j++) {
        dv[j] = act[j] ? p.dist[vv[j]] : INF;
        sv[j] = act[j] ? p.sigma[vv[j]] : 1.0;
        tv[j] = act[j] ? p.delta[vv[j]] : 0.0;
        su[j] = act[j] ? p.sigma[uu[j]] : 0.0;
      }
#endif
#pragma unroll
      for (int j = 0; j < NCH; j++) {
#if GBBS_BC_SPEC
        double c = (dv[j] == nl) ? su[j] / sv[j] * (1.0 + tv[j]) : 0.0;
#else
        double c = 0.0;
        if (act[j] && p.dist[vv[j]] == nl)
          c = p.sigma[uu[j]] / p.sigma[vv[j]] * (1.0 + p.delta[vv[j]]);
#endif
#if !GBBS_BC_SEG
        const unsigned same = __match_any_sync(FULL, act[j] ? uu[j] : INF);
        if (same == FULL) {  // one owner for the whole chunk (a hub): reduce first
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
          if (lane == 0 && c != 0.0) atomicAdd(p.delta + uu[j], c);
        } else if (c != 0.0) {
          atomicAdd(p.delta + uu[j], c);
        }
        continue;
#endif
        // segmented sum over runs of the same owner (edges of an owner are
        // contiguous in the chunk): ONE atomicAdd per (owner, chunk)
        const uint32_t ow = act[j] ? uu[j] : INF;
        const uint32_t prev = __shfl_up_sync(FULL, ow, 1);
        const unsigned heads = __ballot_sync(FULL, lane == 0 || prev != ow);
        const int seg0 = 31 - __clz(heads & lanemask_le());  // first lane of my run
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(FULL, c, o);
          if (lane - o >= seg0) c += y;
        }
        const uint32_t next = __shfl_down_sync(FULL, ow, 1);
        const bool last = lane == 31 || next != ow;
        if (last && ow != INF && c != 0.0) atomicAdd(p.delta + ow, c);
      }
    }
  }
  __syncwarp();
  return onext == te ? i0 + nown : i0 + nown - 1;
}

// Dense forward level l (reading B3): units of BC_PULLV vertices from the level's
// counter; a lane takes an unvisited vertex and sums sigma over its level-l
// neighbours (4 edge loads in flight), vertices above 32 edges are summed by the
// whole warp; winners get level l+1 and sigma with plain stores (each is written
// by its owner only) and are appended to the level queue as in the push.
constexpr int BC_PULLV = 1024;
__device__ __forceinline__ void bc_pull_level(const BcParams &p, BcWarpSmem &w, int &scnt, int l,
                                              long long qnext, unsigned long long *ctr,
                                              unsigned long long *q) {
  const int lane = threadIdx.x & 31;
  const uint32_t lv = (uint32_t)l, nl = (uint32_t)(l + 1);
  for (;;) {
    unsigned long long u0 = 0;
    if (lane == 0) u0 = atomicAdd(q, 1ull);
    const long long v0 = (long long)__shfl_sync(FULL, u0, 0) * BC_PULLV;
    if (v0 >= p.n) break;
    const long long v1 = min(v0 + (long long)BC_PULLV, p.n);
    for (long long vb = v0; vb < v1; vb += 32) {
      const long long v = vb + lane;
      long long a = 0;
      int dg = 0;
      if (v < v1 && ld_relaxed(p.dist + v) == INF) {
        a = __ldg(p.off + v);
        dg = (int)(__ldg(p.off + v + 1) - a);
      }
      double sum = 0.0;
      unsigned big = __ballot_sync(FULL, dg > 32);
      while (big) {
        const int b = __ffs(big) - 1;
        big &= big - 1;
        const long long ba = __shfl_sync(FULL, a, b);
        const int bd = __shfl_sync(FULL, dg, b);
        double t = 0.0;
        for (int e0 = 0; e0 < bd; e0 += 128) {
          uint32_t u[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int e = e0 + 32 * j + lane;
            GBBS_CHECK(e >= bd || (ba + e >= 0 && ba + e < p.m));
            u[j] = e < bd ? ld_stream(p.tgt + ba + e) : 0u;
          }
          uint32_t d[4];
#pragma unroll
          for (int j = 0; j < 4; j++) d[j] = (e0 + 32 * j + lane < bd) ? p.dist[u[j]] : INF;
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (d[j] == lv) t += p.sigma[u[j]];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
        if (lane == b) sum = t;
      }
      const int mine = dg <= 32 ? dg : 0;
      int mx = mine;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
      for (int jj = 0; jj < mx; jj += 4) {
        uint32_t u[4], d[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          GBBS_CHECK(jj + j >= mine || (a + jj + j >= 0 && a + jj + j < p.m));
          u[j] = jj + j < mine ? ld_stream(p.tgt + a + jj + j) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) d[j] = jj + j < mine ? p.dist[u[j]] : INF;
#pragma unroll
        for (int j = 0; j < 4; j++)
          if (d[j] == lv) sum += p.sigma[u[j]];
      }
      const bool win = sum > 0.0;
      if (win) {
        p.dist[v] = nl;
        p.sigma[v] = sum;
      }
      const unsigned bw = __ballot_sync(FULL, win);
      if (win) w.stage[scnt + __popc(bw & lanemask_lt())] = (uint32_t)v;
      scnt += __popc(bw);
      if (scnt > WCAP - 32) {
        bc_flush(p, w.stage, scnt, qnext, ctr);
        scnt = 0;
      }
    }
  }
}

template <bool BACK>
__device__ __forceinline__ void bc_level(const BcParams &p, BcWarpSmem &w, int &scnt,
                                         long long start, long long f, long long E, int l,
                                         long long qnext, unsigned long long *ctr, long long gw,
                                         long long nw, unsigned long long *q) {
  const uint32_t *F = p.qv + start;
  const long long *O = p.qo + start;
  const long long *B = p.qb + start;
  const long long ntiles = (E + TE - 1) / TE;
  if (((BACK && GBBS_BC_DYNQ_BACK) || (!BACK && GBBS_BC_DYNQ_FWD)) && ntiles >= 16 * nw) {
    // big level: runs of G tiles from the level's counter
    const int lane = threadIdx.x & 31;
    const long long G = max(1ll, min(16ll, ntiles / (4 * nw)));
    for (;;) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(q, (unsigned long long)G);
      long long t = (long long)__shfl_sync(FULL, u, 0);
      if (t >= ntiles) break;
      const long long t1 = min(t + G, ntiles);
      long long i0 = warp_upper_est(O, f, E, t * TE);
      for (; t < t1; t++) i0 = bc_tile<BACK>(p, w, scnt, F, O, B, f, E, i0, t, l, qnext, ctr);
    }
    return;
  }
  const long long per = (ntiles + nw - 1) / nw;
  long long t = gw * per;
  const long long t1 = min(t + per, ntiles);
  if (t >= t1) return;
  long long i0 = warp_upper_est(O, f, E, t * TE);
  for (; t < t1; t++) i0 = bc_tile<BACK>(p, w, scnt, F, O, B, f, E, i0, t, l, qnext, ctr);
}

template <bool MG>
__device__ __forceinline__ void bc_body(const BcParams &p, int G) {
  __shared__ BcSmem s;
  cg::grid_group grid = cg::this_grid();
  long long bid_ = 0, nblk_ = 0;  // MG: team-local index and size (as traverse_body)
  if constexpr (MG) {
    const int g = (int)(blockIdx.x % G);
    bid_ = blockIdx.x / G;
    nblk_ = ((long long)gridDim.x - g + G - 1) / G;
  }
#define GBBS_BID (MG ? bid_ : (long long)blockIdx.x)
#define GBBS_NBLK (MG ? nblk_ : (long long)gridDim.x)
  const int tid = threadIdx.x, warp = tid >> 5;
  const long long gtid = GBBS_BID * BLOCK + tid;
  const long long gstride = GBBS_NBLK * BLOCK;
  const long long gw = GBBS_BID * NWARPS + warp;
  const long long nw = GBBS_NBLK * NWARPS;
  const uint32_t src = p.src;
  BcWarpSmem &w = s.w[warp];

  for (long long i = gtid; i < p.n; i += gstride) {
    p.dist[i] = (i == src) ? 0u : INF;
    p.sigma[i] = (i == src) ? 1.0 : 0.0;
    p.delta[i] = 0.0;
  }
  if (GBBS_BID == 0 && tid == 0) {
    const long long a = p.off[src], d0 = p.off[src + 1] - a;
    p.cnt[1] = p.cnt[2] = p.cnt[3] = 0;
    if (d0 > 0) {
      p.qv[0] = src;
      p.qo[0] = 0;
      p.qb[0] = a;
      p.cnt[0] = (1ull << p.ebits) | (unsigned long long)d0;
    } else {
      p.cnt[0] = 0;
    }
    *p.status = 0;
    for (int q = 0; q < 8; q++) p.wq[q] = 0;
  }
  team_sync<MG>(grid, p.bar, GBBS_NBLK);

  const unsigned long long emask = (1ull << p.ebits) - 1;
  long long start = 0;  // queue position of the current level
  long long seenE = 0;  // edges of the listed levels' vertices (so far and this one)
  int l = 0;
  for (;; l++) {
    if (tid == 0) s.cnt = ld_relaxed64(p.cnt + (l & 3));
    __syncthreads();
    const long long f = (long long)(s.cnt >> p.ebits), E = (long long)(s.cnt & emask);
    if (f == 0) break;
    if (l >= p.lvl_cap) {
      if (GBBS_BID == 0 && tid == 0) *p.status = 1;
      break;
    }
    if (GBBS_BID == 0 && tid == 0) {
      p.cnt[(l + 2) & 3] = 0;
      p.wq[(l + 2) & 3] = 0;
      p.lvl[3 * l] = start;
      p.lvl[3 * l + 1] = f;
      p.lvl[3 * l + 2] = E;
    }
    int scnt = 0;
    seenE += E;
    // dense iff the paper's rule holds and the pull (every edge of every unvisited
    // vertex: m - seenE on a symmetric graph) reads fewer edges than the push (E)
    const bool dense = p.dense_mode == 2 ||
                       (p.dense_mode == 0 && f + E > p.dense_threshold &&
                        GBBS_BC_PULL_RATIO * (p.m - seenE) < E);
    if (dense)
      bc_pull_level(p, w, scnt, l, start + f, p.cnt + ((l + 1) & 3), p.wq + (l & 3));
    else
      bc_level<false>(p, w, scnt, start, f, E, l, start + f, p.cnt + ((l + 1) & 3), gw, nw,
                      p.wq + (l & 3));
    if (scnt > 0) bc_flush(p, w.stage, scnt, start + f, p.cnt + ((l + 1) & 3));
    start += f;
    team_sync<MG>(grid, p.bar, GBBS_NBLK);
  }
  const int L = l;  // levels with a non-empty list: 0 .. L-1
#ifdef GBBS_DIAG_BC_FORWARD_ONLY  // measurement-only build
  if (L > 0) {
    if (GBBS_BID == 0 && tid == 0) *p.rounds_out = L;
    return;
  }
#endif
  for (int b = L - 1; b >= 1; b--) {
    const long long st0 = p.lvl[3 * b], f = p.lvl[3 * b + 1], E = p.lvl[3 * b + 2];
    int scnt = 0;
    if (GBBS_BID == 0 && tid == 0) p.wq[4 + ((b - 2) & 3)] = 0;  // used two levels down
    bc_level<true>(p, w, scnt, st0, f, E, b, 0, nullptr, gw, nw, p.wq + 4 + (b & 3));
    team_sync<MG>(grid, p.bar, GBBS_NBLK);
  }
  if (GBBS_BID == 0 && tid == 0) *p.rounds_out = L;
}
#undef GBBS_BID
#undef GBBS_NBLK

__global__ void __launch_bounds__(BLOCK) bc_kernel(const __grid_constant__ BcParams p) {
  bc_body<false>(p, 1);
}

}  // namespace gbbs_dev
