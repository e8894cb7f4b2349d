/*
 * oracle.c — CPU ORACLE FOR THE FRONTIER BFS / BELLMAN-FORD HOT PATH.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke()
 * entry point in __graft_entry__.py and bench.py's cpu_baseline / reference
 * leg may load or execute it.  It shares no source, header, helper, table or
 * constant with paper_1805_05208_b200/csrc (the CUDA path); neither side
 * includes or links the other.
 *
 * Everything here is plain, sequential, single-threaded C written to be
 * checked against the paper by eye.  It implements the *definitions* of the
 * outputs, not the paper's parallel algorithm, because both frontier methods
 * reach exactly (bit for bit) the unique shortest-path distances:
 *
 *   BFS  (sec:benchmark "Breadth-First Search"):
 *        D[v] = shortest-path (hop) distance from src to v, infinity if
 *        unreachable.
 *   Bellman-Ford (sec:benchmark "General-Weight SSSP"):
 *        D[v] = shortest-path distance from src to v, infinity if
 *        unreachable.  (The -infinity clause for reachable negative cycles
 *        cannot arise: weights are unsigned; reading A13.)
 *
 * Graph representation (sec:prelims): CSR with
 * offsets[n+1] (int64) and targets[m] (uint32), optional weights[m]
 * (uint32; NULL = unit weights, reading A17).  Edges are followed
 * u -> targets[e] for e in [offsets[u], offsets[u+1]) (reading A4).
 *
 * Sentinels (reading A2): unreachable = 0xFFFFFFFF in uint32 outputs,
 * UINT64_MAX in the uint64 outputs of the weighted routines.
 * Parent of src = src (reading A3).
 *
 * Functions:
 *   oracle_bfs              — textbook FIFO-queue BFS.
 *   oracle_dijkstra         — textbook Dijkstra with an indexed binary heap
 *                             (decrease-key), uint64 accumulation.
 *   oracle_bellman_ford     — textbook Bellman-Ford: repeated passes that
 *                             relax every edge until a pass changes nothing
 *                             (at most n-1 useful passes).
 *   oracle_frontier_bellman_ford — the paper's frontier formulation
 *                             (sec:algs "BFS, wBFS,
 *                             Bellman-Ford"): each round relaxes only the
 *                             out-edges of vertices whose distance dropped in
 *                             the previous round; run sequentially.
 *   oracle_check_bfs        — O(n+m) certificate for a BFS output.
 *   oracle_check_sssp       — O(n+m) certificate for an SSSP output (w >= 1).
 *   oracle_reached_edges    — sum of out-degrees of reached vertices (the
 *                             TEPS numerator, reading A20).
 *
 * Error convention: 0 = OK, negative = error (see ORACLE_E* below).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL -1
#define ORACLE_ENOMEM -2
#define ORACLE_ERANGE -3   /* a finite distance does not fit in uint32 */
#define ORACLE_EFAIL -4    /* certificate violated; *bad holds a witness */
#define ORACLE_ENA -5      /* certificate not applicable (a zero weight) */

#define INF32 0xFFFFFFFFu
#define INF64 UINT64_MAX

static int check_args(int64_t n, const int64_t *off, const uint32_t *tgt,
                      uint32_t src) {
  if (n < 1 || off == NULL || (off[n] > 0 && tgt == NULL)) return ORACLE_EINVAL;
  if ((int64_t)src >= n) return ORACLE_EINVAL;
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* BFS: FIFO queue.  dist/parent are caller-owned arrays of length n;       */
/* parent may be NULL.                                                       */
/* ------------------------------------------------------------------------ */
int oracle_bfs(int64_t n, const int64_t *off, const uint32_t *tgt,
               uint32_t src, uint32_t *dist, uint32_t *parent) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  uint32_t *queue = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  if (!queue) return ORACLE_ENOMEM;
  for (int64_t v = 0; v < n; v++) {
    dist[v] = INF32;
    if (parent) parent[v] = INF32;
  }
  int64_t head = 0, tail = 0;
  dist[src] = 0;
  if (parent) parent[src] = src;
  queue[tail++] = src;
  while (head < tail) {
    uint32_t u = queue[head++];
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      if (dist[v] == INF32) {
        dist[v] = dist[u] + 1;
        if (parent) parent[v] = u;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Dijkstra with an indexed binary min-heap keyed by dist (uint64).         */
/* weights NULL = unit weights.  dist is uint64[n] (INF64 = unreachable),    */
/* parent uint32[n] or NULL.                                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t *heap;    /* heap[i] = vertex */
  int64_t *pos;      /* pos[v] = index in heap, -1 if absent */
  const uint64_t *key;
  int64_t size;
} heap_t;

static void heap_swap(heap_t *h, int64_t i, int64_t j) {
  uint32_t a = h->heap[i], b = h->heap[j];
  h->heap[i] = b;
  h->heap[j] = a;
  h->pos[b] = i;
  h->pos[a] = j;
}

static void heap_up(heap_t *h, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h->key[h->heap[p]] <= h->key[h->heap[i]]) break;
    heap_swap(h, i, p);
    i = p;
  }
}

static void heap_down(heap_t *h, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->size && h->key[h->heap[l]] < h->key[h->heap[s]]) s = l;
    if (r < h->size && h->key[h->heap[r]] < h->key[h->heap[s]]) s = r;
    if (s == i) break;
    heap_swap(h, i, s);
    i = s;
  }
}

int oracle_dijkstra(int64_t n, const int64_t *off, const uint32_t *tgt,
                    const uint32_t *w, uint32_t src, uint64_t *dist,
                    uint32_t *parent) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  heap_t h;
  h.heap = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  h.pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  char *done = (char *)calloc((size_t)n, 1);
  if (!h.heap || !h.pos || !done) {
    free(h.heap); free(h.pos); free(done);
    return ORACLE_ENOMEM;
  }
  h.key = dist;
  h.size = 0;
  for (int64_t v = 0; v < n; v++) {
    dist[v] = INF64;
    h.pos[v] = -1;
    if (parent) parent[v] = INF32;
  }
  dist[src] = 0;
  if (parent) parent[src] = src;
  h.heap[0] = src;
  h.pos[src] = 0;
  h.size = 1;
  while (h.size > 0) {
    uint32_t u = h.heap[0];
    heap_swap(&h, 0, h.size - 1);
    h.size--;
    h.pos[u] = -1;
    if (h.size > 0) heap_down(&h, 0);
    done[u] = 1;
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      if (done[v]) continue;
      uint64_t nd = dist[u] + (w ? (uint64_t)w[e] : 1u);
      if (nd < dist[v]) {
        dist[v] = nd;
        if (parent) parent[v] = u;
        if (h.pos[v] < 0) {
          h.heap[h.size] = v;
          h.pos[v] = h.size;
          h.size++;
        }
        heap_up(&h, h.pos[v]);
      }
    }
  }
  free(h.heap); free(h.pos); free(done);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Textbook Bellman-Ford: relax all edges, pass after pass, until no change.*/
/* With non-negative weights at most n-1 passes change anything; a change in*/
/* pass n would mean a negative cycle, impossible here (returns EINVAL).    */
/* ------------------------------------------------------------------------ */
int oracle_bellman_ford(int64_t n, const int64_t *off, const uint32_t *tgt,
                        const uint32_t *w, uint32_t src, uint64_t *dist,
                        int64_t *passes) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  for (int64_t v = 0; v < n; v++) dist[v] = INF64;
  dist[src] = 0;
  int64_t pass = 0;
  for (;;) {
    int changed = 0;
    for (int64_t u = 0; u < n; u++) {
      if (dist[u] == INF64) continue;
      for (int64_t e = off[u]; e < off[u + 1]; e++) {
        uint64_t nd = dist[u] + (w ? (uint64_t)w[e] : 1u);
        if (nd < dist[tgt[e]]) {
          dist[tgt[e]] = nd;
          changed = 1;
        }
      }
    }
    pass++;
    if (!changed) break;
    if (pass > n) return ORACLE_EINVAL;
  }
  if (passes) *passes = pass;
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* The paper's frontier Bellman-Ford, run sequentially:    */
/* frontier F = {src}; each round, for u in F and each edge (u,v,w), write  */
/* D[v] = min(D[v], D[u]+w) (the priority-write); v joins the next frontier */
/* iff the write lowered D[v].  Stop when the frontier is empty.  The next  */
/* frontier is a set (a vertex is added once per round).                    */
/* ------------------------------------------------------------------------ */
int oracle_frontier_bellman_ford(int64_t n, const int64_t *off,
                                 const uint32_t *tgt, const uint32_t *w,
                                 uint32_t src, uint64_t *dist,
                                 int64_t *rounds) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  uint32_t *cur = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  uint32_t *nxt = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  char *in_next = (char *)calloc((size_t)n, 1);
  if (!cur || !nxt || !in_next) {
    free(cur); free(nxt); free(in_next);
    return ORACLE_ENOMEM;
  }
  for (int64_t v = 0; v < n; v++) dist[v] = INF64;
  dist[src] = 0;
  int64_t fc = 1, r = 0;
  cur[0] = src;
  while (fc > 0) {
    if (r >= n) { /* more than n rounds: impossible for w >= 0 */
      free(cur); free(nxt); free(in_next);
      return ORACLE_EINVAL;
    }
    int64_t nc = 0;
    for (int64_t i = 0; i < fc; i++) {
      uint32_t u = cur[i];
      for (int64_t e = off[u]; e < off[u + 1]; e++) {
        uint32_t v = tgt[e];
        uint64_t nd = dist[u] + (w ? (uint64_t)w[e] : 1u);
        if (nd < dist[v]) {
          dist[v] = nd;
          if (!in_next[v]) {
            in_next[v] = 1;
            nxt[nc++] = v;
          }
        }
      }
    }
    for (int64_t i = 0; i < nc; i++) in_next[nxt[i]] = 0;
    uint32_t *t = cur; cur = nxt; nxt = t;
    fc = nc;
    r++;
  }
  if (rounds) *rounds = r;
  free(cur); free(nxt); free(in_next);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Certificates (independent of every routine above).                       */
/*                                                                          */
/* BFS: (1) dist[src]=0; (2) for every edge u->v with dist[u] finite,       */
/* dist[v] <= dist[u]+1; (3) every reached v != src has a tight in-edge     */
/* u->v with dist[u]+1 == dist[v] — and, if parent is given, that edge is    */
/* parent[v]->v; (4) parent[src]=src and parent[v]=INF iff dist[v]=INF.     */
/* (1)+(2) give dist <= true distance; (3) gives a path of length dist[v],  */
/* so dist >= true distance.  Hence dist is exact and parents are valid.    */
/* On failure *bad = a witness vertex.                                      */
/* ------------------------------------------------------------------------ */
int oracle_check_bfs(int64_t n, const int64_t *off, const uint32_t *tgt,
                     uint32_t src, const uint32_t *dist,
                     const uint32_t *parent, int64_t *bad) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  int64_t dummy;
  if (!bad) bad = &dummy;
  *bad = -1;
  if (dist[src] != 0) { *bad = src; return ORACLE_EFAIL; }
  if (parent && parent[src] != src) { *bad = src; return ORACLE_EFAIL; }
  char *ok = (char *)calloc((size_t)n, 1);
  if (!ok) return ORACLE_ENOMEM;
  for (int64_t u = 0; u < n; u++) {
    if (dist[u] == INF32) continue;
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      if ((uint64_t)dist[v] > (uint64_t)dist[u] + 1) {
        *bad = v; free(ok); return ORACLE_EFAIL;
      }
      if ((uint64_t)dist[u] + 1 == (uint64_t)dist[v] &&
          (parent == NULL || parent[v] == (uint32_t)u))
        ok[v] = 1;
    }
  }
  for (int64_t v = 0; v < n; v++) {
    if (v == (int64_t)src) continue;
    if (dist[v] == INF32) {
      if (parent && parent[v] != INF32) { *bad = v; free(ok); return ORACLE_EFAIL; }
    } else if (!ok[v]) {
      *bad = v; free(ok); return ORACLE_EFAIL;
    }
  }
  free(ok);
  return ORACLE_OK;
}

/* SSSP with all weights >= 1 (weights NULL = unit): (1) dist[src]=0;       */
/* (2) every edge with dist[u] finite has dist[v] <= dist[u]+w; (3) every   */
/* reached v != src has a tight in-edge dist[u]+w == dist[v].  With w >= 1  */
/* tight edges strictly decrease dist, so following them backwards ends at  */
/* src: dist[v] is a real path length.  Returns ORACLE_ENA if some weight   */
/* is 0 (the certificate then proves nothing).                              */
int oracle_check_sssp(int64_t n, const int64_t *off, const uint32_t *tgt,
                      const uint32_t *w, uint32_t src, const uint32_t *dist,
                      int64_t *bad) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL) return ORACLE_EINVAL;
  int64_t dummy;
  if (!bad) bad = &dummy;
  *bad = -1;
  int64_t m = off[n];
  if (w)
    for (int64_t e = 0; e < m; e++)
      if (w[e] == 0) return ORACLE_ENA;
  if (dist[src] != 0) { *bad = src; return ORACLE_EFAIL; }
  char *ok = (char *)calloc((size_t)n, 1);
  if (!ok) return ORACLE_ENOMEM;
  for (int64_t u = 0; u < n; u++) {
    if (dist[u] == INF32) continue;
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      uint64_t nd = (uint64_t)dist[u] + (w ? (uint64_t)w[e] : 1u);
      if ((uint64_t)dist[v] > nd) { *bad = v; free(ok); return ORACLE_EFAIL; }
      if ((uint64_t)dist[v] == nd) ok[v] = 1;
    }
  }
  for (int64_t v = 0; v < n; v++) {
    if (v == (int64_t)src || dist[v] == INF32) continue;
    if (!ok[v]) { *bad = v; free(ok); return ORACLE_EFAIL; }
  }
  free(ok);
  return ORACLE_OK;
}

/* TEPS numerator: sum of out-degrees over vertices with finite dist.       */
int64_t oracle_reached_edges(int64_t n, const int64_t *off,
                             const uint32_t *dist) {
  int64_t s = 0;
  for (int64_t v = 0; v < n; v++)
    if (dist[v] != INF32) s += off[v + 1] - off[v];
  return s;
}

/* ------------------------------------------------------------------------ */
/* Widest (bottleneck) path, PAPER.md:114-136 (sec:algs "Widest Path"),     */
/* output spec PAPER.md:1499-1504: width[v] = max over src->v paths of the  */
/* minimum edge weight.  The definition computed by the textbook modified   */
/* Dijkstra ("Sequentially, the algorithm can be solved as quickly as SSSP  */
/* using a modified version of Dijkstra's algorithm"):    */
/* extract the vertex of largest width, relax width[v] = max(width[v],      */
/* min(width[u], w)).  Readings W1/W2: width[src] = INF32 (empty */
/* path), unreachable = 0.  weights NULL = unit.                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t *heap;
  int64_t *pos;
  const uint32_t *key;
  int64_t size;
} mheap_t; /* max-heap on key */

static void mheap_swap(mheap_t *h, int64_t i, int64_t j) {
  uint32_t a = h->heap[i], b = h->heap[j];
  h->heap[i] = b;
  h->heap[j] = a;
  h->pos[b] = i;
  h->pos[a] = j;
}

static void mheap_up(mheap_t *h, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h->key[h->heap[p]] >= h->key[h->heap[i]]) break;
    mheap_swap(h, i, p);
    i = p;
  }
}

static void mheap_down(mheap_t *h, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->size && h->key[h->heap[l]] > h->key[h->heap[s]]) s = l;
    if (r < h->size && h->key[h->heap[r]] > h->key[h->heap[s]]) s = r;
    if (s == i) break;
    mheap_swap(h, i, s);
    i = s;
  }
}

int oracle_widest_path(int64_t n, const int64_t *off, const uint32_t *tgt,
                       const uint32_t *w, uint32_t src, uint32_t *width) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (width == NULL) return ORACLE_EINVAL;
  mheap_t h;
  h.heap = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  h.pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  char *done = (char *)calloc((size_t)n, 1);
  if (!h.heap || !h.pos || !done) {
    free(h.heap); free(h.pos); free(done);
    return ORACLE_ENOMEM;
  }
  h.key = width;
  for (int64_t v = 0; v < n; v++) {
    width[v] = 0;
    h.pos[v] = -1;
  }
  width[src] = INF32;
  h.heap[0] = src;
  h.pos[src] = 0;
  h.size = 1;
  while (h.size > 0) {
    uint32_t u = h.heap[0];
    mheap_swap(&h, 0, h.size - 1);
    h.size--;
    h.pos[u] = -1;
    if (h.size > 0) mheap_down(&h, 0);
    done[u] = 1;
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      if (done[v]) continue;
      uint32_t we = w ? w[e] : 1u;
      uint32_t cand = width[u] < we ? width[u] : we;
      if (cand > width[v]) {
        width[v] = cand;
        if (h.pos[v] < 0) {
          h.heap[h.size] = v;
          h.pos[v] = h.size;
          h.size++;
        }
        mheap_up(&h, h.pos[v]);
      }
    }
  }
  free(h.heap); free(h.pos); free(done);
  return ORACLE_OK;
}

/* Widest-path certificate, O(n+m): (1) width[src] = INF32; (2) no edge can  */
/* improve: width[v] >= min(width[u], w) for every edge; (3) a BFS from src  */
/* over tight edges (min(width[u], w) == width[v] > 0) reaches exactly the   */
/* vertices with width > 0.  (2) gives width >= true width along an optimal */
/* path; every vertex reached by (3) has width <= true width by induction;  */
/* so (2)+(3) imply exact widths.                                           */
int oracle_check_widest(int64_t n, const int64_t *off, const uint32_t *tgt,
                        const uint32_t *w, uint32_t src, const uint32_t *width,
                        int64_t *bad) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (width == NULL) return ORACLE_EINVAL;
  int64_t dummy;
  if (!bad) bad = &dummy;
  *bad = -1;
  if (width[src] != INF32) { *bad = src; return ORACLE_EFAIL; }
  for (int64_t u = 0; u < n; u++) {
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t we = w ? w[e] : 1u;
      uint32_t cand = width[u] < we ? width[u] : we;
      if (width[tgt[e]] < cand) { *bad = tgt[e]; return ORACLE_EFAIL; }
    }
  }
  char *seen = (char *)calloc((size_t)n, 1);
  uint32_t *queue = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  if (!seen || !queue) { free(seen); free(queue); return ORACLE_ENOMEM; }
  int64_t head = 0, tail = 0;
  seen[src] = 1;
  queue[tail++] = src;
  while (head < tail) {
    uint32_t u = queue[head++];
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      uint32_t we = w ? w[e] : 1u;
      uint32_t cand = width[u] < we ? width[u] : we;
      if (!seen[v] && width[v] > 0 && cand == width[v]) {
        seen[v] = 1;
        queue[tail++] = v;
      }
    }
  }
  for (int64_t v = 0; v < n; v++) {
    if ((width[v] > 0) != (seen[v] != 0)) { *bad = v; free(seen); free(queue); return ORACLE_EFAIL; }
  }
  free(seen); free(queue);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Single-source betweenness contributions, PAPER.md:98-101 (sec:algs) and   */
/* the output spec PAPER.md:1493-1496: S[v] = contribution to v's centrality */
/* from all (src, t) shortest paths through v = Brandes' dependency          */
/* delta_src(v) = sum_{t != src, v} sigma_st(v) / sigma_st.  Textbook        */
/* Brandes: BFS from src counting shortest paths sigma (double), then        */
/* vertices in reverse BFS order accumulate                                  */
/* delta[v] = sum_{v->w, d[w] = d[v]+1} sigma[v]/sigma[w] * (1 + delta[w]).   */
/* Reading B1: endpoints are excluded, so delta[src] = 0 and     */
/* unreached vertices get 0.  sigma may be NULL.                             */
/* ------------------------------------------------------------------------ */
int oracle_bc(int64_t n, const int64_t *off, const uint32_t *tgt, uint32_t src,
              double *delta, double *sigma_out) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (delta == NULL) return ORACLE_EINVAL;
  uint32_t *order = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  uint32_t *d = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
  double *sigma = (double *)calloc((size_t)n, sizeof(double));
  if (!order || !d || !sigma) {
    free(order); free(d); free(sigma);
    return ORACLE_ENOMEM;
  }
  for (int64_t v = 0; v < n; v++) {
    d[v] = INF32;
    delta[v] = 0.0;
  }
  int64_t head = 0, tail = 0;
  d[src] = 0;
  sigma[src] = 1.0;
  order[tail++] = src;
  while (head < tail) {
    uint32_t u = order[head++];
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      uint32_t v = tgt[e];
      if (d[v] == INF32) {
        d[v] = d[u] + 1;
        order[tail++] = v;
      }
      if (d[v] == d[u] + 1) sigma[v] += sigma[u];
    }
  }
  for (int64_t i = tail - 1; i >= 0; i--) {
    uint32_t v = order[i];
    double acc = 0.0;
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      uint32_t w = tgt[e];
      if (d[w] == d[v] + 1) acc += sigma[v] / sigma[w] * (1.0 + delta[w]);
    }
    delta[v] = acc;
  }
  delta[src] = 0.0;
  if (sigma_out)
    for (int64_t v = 0; v < n; v++) sigma_out[v] = sigma[v];
  free(order); free(d); free(sigma);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: general-weight SSSP (sec:benchmark "General- */
/* Weight SSSP (Bellman-Ford)"): D[v] = shortest-path distance from src,    */
/* infinity if unreachable; "All distances must be -infinity if G contains  */
/* a negative-weight cycle reachable from src".  Weights are int32 (w[e]    */
/* read as two's complement; NULL = unit weights), distances int64 with     */
/* INT64_MAX = infinity and INT64_MIN = -infinity.                          */
/*                                                                          */
/* Textbook Bellman-Ford: n-1 passes relaxing every edge (u,v) with D[u]    */
/* finite.  Afterwards an edge that still relaxes proves a negative cycle   */
/* reachable from src (a walk beating every simple path), and every         */
/* reachable negative cycle has such an edge.  scope 0 (reading N1, the     */
/* sentence read literally): then every D[v] = -infinity.  scope 1 (reading */
/* N2): D[v] = -infinity exactly for v reachable from the target of a still */
/* relaxing edge (depth-first search over out-edges).  *negcycle = 1 if a   */
/* reachable negative cycle exists.  Distances of simple paths fit int64    */
/* when (n-1) * max|w| < 2^62; larger inputs return ORACLE_ERANGE.          */
/* ------------------------------------------------------------------------ */
int oracle_bellman_ford_signed(int64_t n, const int64_t *off, const uint32_t *tgt,
                               const uint32_t *w, uint32_t src, int scope,
                               int64_t *dist, int *negcycle) {
  int rc = check_args(n, off, tgt, src);
  if (rc) return rc;
  if (dist == NULL || (scope != 0 && scope != 1)) return ORACLE_EINVAL;
  const int64_t m = off[n];
  int64_t maxabs = 1;
  for (int64_t e = 0; w && e < m; e++) {
    int64_t x = (int32_t)w[e];
    if (x < 0) x = -x;
    if (x > maxabs) maxabs = x;
  }
  if ((n - 1) > ((INT64_C(1) << 62) - 1) / maxabs) return ORACLE_ERANGE;
  for (int64_t v = 0; v < n; v++) dist[v] = INT64_MAX;
  dist[src] = 0;
  for (int64_t pass = 0; pass < n - 1; pass++) {
    int changed = 0;
    for (int64_t u = 0; u < n; u++) {
      if (dist[u] == INT64_MAX) continue;
      for (int64_t e = off[u]; e < off[u + 1]; e++) {
        int64_t nd = dist[u] + (w ? (int64_t)(int32_t)w[e] : 1);
        if (nd < dist[tgt[e]]) {
          dist[tgt[e]] = nd;
          changed = 1;
        }
      }
    }
    if (!changed) break;
  }
  /* pass n: edges that still relax */
  unsigned char *mark = (unsigned char *)calloc((size_t)n, 1);
  int64_t *stack = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  if (!mark || !stack) {
    free(mark);
    free(stack);
    return ORACLE_ENOMEM;
  }
  int64_t sp = 0;
  int found = 0;
  for (int64_t u = 0; u < n; u++) {
    if (dist[u] == INT64_MAX) continue;
    for (int64_t e = off[u]; e < off[u + 1]; e++) {
      int64_t nd = dist[u] + (w ? (int64_t)(int32_t)w[e] : 1);
      if (nd < dist[tgt[e]]) {
        found = 1;
        if (!mark[tgt[e]]) {
          mark[tgt[e]] = 1;
          stack[sp++] = tgt[e];
        }
      }
    }
  }
  if (negcycle) *negcycle = found;
  if (found && scope == 0) {
    for (int64_t v = 0; v < n; v++) dist[v] = INT64_MIN;
  } else if (found) {
    while (sp > 0) { /* forward closure of the seeds */
      int64_t u = stack[--sp];
      for (int64_t e = off[u]; e < off[u + 1]; e++) {
        if (!mark[tgt[e]]) {
          mark[tgt[e]] = 1;
          stack[sp++] = tgt[e];
        }
      }
    }
    for (int64_t v = 0; v < n; v++)
      if (mark[v]) dist[v] = INT64_MIN;
  }
  free(mark);
  free(stack);
  return ORACLE_OK;
}
