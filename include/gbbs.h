/*
 * gbbs.h — C ABI of libgbbs: frontier BFS and frontier Bellman-Ford on one
 * NVIDIA B200 (sm_100a), after arxiv 1805.05208 (GBBS, "Theoretically
 * Efficient Parallel Graph Algorithms Can Be Fast and Scalable").
 *
 * Citations are to /root/reference/PAPER.md lines ("P:<line>") with the
 * section they fall in; SURVEY.md §8(b) is the design contract.
 *
 * The library implements the paper's edgeMap primitive (P:1851-1874,
 * sec:prelims "Ligra, Ligra+, and Julienne") instantiated two ways:
 *   - BFS: F = test-and-set acquire of unvisited neighbours (P:84-93,
 *     sec:algs; TS semantics P:1821-1825);
 *   - Bellman-Ford: F = priority-write of the minimum distance (P:93-97,
 *     sec:algs; PW semantics P:1826-1831).
 * Each round chooses a sparse (push over a vertex list, with the edge work cut
 * into fixed-size blocks as in edgeMapBlocked) or dense (pull
 * over in-edges with early exit) method from the number of edges
 * incident to the frontier.
 *
 * Conventions common to every call:
 *   - Status: 0 = GBBS_OK, negative = error.  No C++ exception crosses the
 *     ABI.  gbbs_last_error() returns a thread-local message for the last
 *     failing call on the calling thread.
 *   - Vertex ids are uint32 in [0, n); edge indices and offsets are int64.
 *   - Unreached vertices get GBBS_INF (0xFFFFFFFF) in dist and parent
 *     (reading A2); parent[src] = src (reading A3).
 *   - Pointers may be host or device memory (classified with
 *     cudaPointerGetAttributes); device pointers must be on the current
 *     device.  The CUDA device is the one current when the graph is created.
 *   - A gbbs_graph owns per-handle scratch, so calls on ONE handle must not
 *     run concurrently (different handles may).
 */
#ifndef GBBS_H
#define GBBS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define GBBS_OK 0
#define GBBS_EINVAL (-1)    /* bad argument or malformed CSR               */
#define GBBS_ERANGE (-2)    /* sizes/weights outside what uint32 state holds */
#define GBBS_ENOMEM (-3)    /* device or host allocation failed            */
#define GBBS_ECUDA (-4)     /* CUDA error, including "no sm_100 device"     */
#define GBBS_EINTERNAL (-5) /* round cap hit (cannot happen for w >= 0)    */

#define GBBS_INF 0xFFFFFFFFu

/* ---- gbbs_graph_create flags ------------------------------------------- */
/* The caller asserts the CSR is symmetric (u->v iff v->u).  The in-edge CSC
 * used by dense (pull) rounds then aliases the CSR instead of being built.
 * An incorrect assertion makes dense-round results undefined. */
#define GBBS_SYMMETRIC 0x1u
/* Use device arrays in place (zero copy).  The caller keeps offsets, targets
 * and weights alive and unmodified until gbbs_graph_destroy.  Host pointers
 * with this flag are an error (GBBS_EINVAL).  Dense rounds of symmetric graphs
 * and list pushes of a hub's edges read targets (and weights) in aligned
 * 16-byte groups, so borrowed targets and weights arrays must be readable up
 * to the next 16-byte boundary past element m - 1 (true of any cudaMalloc or
 * PyTorch allocation, whose sizes are rounded up to 512 bytes); a targets or
 * weights pointer that is not 16-byte aligned is copied instead. */
#define GBBS_BORROW 0x2u
/* Skip the O(n+m) device validation of the CSR (offsets/targets). */
#define GBBS_NO_VALIDATE 0x4u

typedef struct gbbs_graph gbbs_graph;

/*
 * gbbs_graph_create — make a graph resident in HBM.
 *
 * n        number of vertices, 1 <= n <= 2^32 - 2.
 * m        number of directed edges (CSR entries), m >= 0.
 * offsets  int64[n+1], offsets[0] = 0, non-decreasing, offsets[n] = m
 *          (CSR, P:1813-1817 sec:prelims).  Host or device.
 * targets  uint32[m], targets[e] < n: out-neighbours of u are
 *          targets[offsets[u] .. offsets[u+1]).  Host or device.  Self-loops
 *          and duplicates are accepted (reading A18) and only cost work.
 * weights  uint32[m] edge weights for Bellman-Ford, or NULL for unit weights
 *          (reading A17).  Host or device.
 * flags    GBBS_SYMMETRIC | GBBS_BORROW | GBBS_NO_VALIDATE.
 * out      receives the handle; set to NULL on any error (nothing leaks).
 *
 * Ownership: without GBBS_BORROW the library copies every array into its own
 * device memory, so the caller may free its arrays as soon as this returns.
 * For non-symmetric graphs an in-edge CSC (in-lists sorted by source) is built
 * here on the device.  Per-handle traversal scratch (frontier lists, bitmaps,
 * counters) is allocated once here.
 *
 * Errors: GBBS_EINVAL  n out of range, m < 0, NULL required pointer,
 *                      offsets[0] != 0, offsets[n] != m, decreasing offsets,
 *                      a target >= n (unless GBBS_NO_VALIDATE);
 *         GBBS_ERANGE  n and m too large to pack the frontier counter
 *                      (bits(n) + bits(m) > 64);
 *         GBBS_ENOMEM, GBBS_ECUDA.
 */
int gbbs_graph_create(int64_t n, int64_t m, const int64_t *offsets,
                      const uint32_t *targets, const uint32_t *weights,
                      uint32_t flags, gbbs_graph **out);

/* Free library-owned device memory; borrowed arrays are not freed.  NULL-safe. */
void gbbs_graph_destroy(gbbs_graph *g);

/* Query sizes/flags of a handle (any pointer may be NULL). */
int gbbs_graph_info(const gbbs_graph *g, int64_t *n, int64_t *m,
                    uint32_t *flags);

/*
 * gbbs_bfs — breadth-first search from src along out-edges
 * (output spec P:1475-1478, sec:benchmark; algorithm, sec:algs).
 *
 * dist    uint32[n], caller-owned, host or device: dist[v] = hop distance
 *         from src, GBBS_INF if unreachable.  Required.
 * parent  uint32[n] or NULL: parent[v] = an in-neighbour u of v with
 *         dist[u] = dist[v] - 1 (which one is unspecified: the test-and-set
 *         winner in push rounds, the first frontier in-neighbour in CSC order
 *         in pull rounds, reading A15); parent[src] = src; GBBS_INF if
 *         unreached.
 * cuda_stream  a cudaStream_t (NULL = legacy default stream).  All work is
 *         enqueued on it and the call synchronizes it before returning, so the
 *         status covers kernel errors; CUDA events recorded on the stream
 *         around the call time it.
 *
 * Errors: GBBS_EINVAL (g NULL, dist NULL, src >= n; outputs untouched),
 *         GBBS_ECUDA, GBBS_EINTERNAL.
 */
int gbbs_bfs(const gbbs_graph *g, uint32_t src, uint32_t *dist,
             uint32_t *parent, void *cuda_stream);

/*
 * gbbs_bfs_batch / gbbs_bellman_ford_batch — k traversals, one per source
 * srcs[0..k) (host array), with results in row i of dist (and parent):
 * dist[i*n .. (i+1)*n).  Same results as k single calls.  With host outputs
 * (pinned memory recommended) the device->host copy of traversal i overlaps
 * traversal i+1 (double-buffered device staging of 8n bytes, allocated on first
 * use, and a copy stream owned by the handle); device outputs are written in
 * place.  The call returns when every row is written.
 * Errors: GBBS_EINVAL (g NULL, k < 0, srcs or dist NULL with k > 0, a source
 * >= n; nothing is run), else as gbbs_bfs / gbbs_bellman_ford for the first
 * failing source (rows of the sources before it are complete).
 */
int gbbs_bfs_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                   uint32_t *dist, uint32_t *parent, void *cuda_stream);
int gbbs_bellman_ford_batch(const gbbs_graph *g, const uint32_t *srcs,
                            int64_t k, uint32_t *dist, void *cuda_stream);
/* The k launches are enqueued without host synchronisation between them
 * (each traversal's status word is kept in a device slot and checked after
 * the single synchronisation at the end); _ex variants with options below. */

/*
 * gbbs_bellman_ford — frontier Bellman-Ford from src (output spec
 * P:1487-1490, sec:benchmark; algorithm, sec:algs).  Weights are the
 * uint32 weights given at create (non-negative, so no negative cycles;
 * reading A13), or 1 if none were given.
 *
 * dist    uint32[n], caller-owned, host or device: shortest weighted
 *         distance from src, GBBS_INF if unreachable.
 * Same stream/synchronization/error conventions as gbbs_bfs, plus
 * GBBS_ERANGE iff some reachable vertex's shortest distance is >= 2^32 - 1
 * (it does not fit below the uint32 sentinel): candidates d(u) + w reaching
 * 2^32 - 1 are dropped as "no improvement" during the run, so every finite
 * distance returned is exact; when the run dropped one, an O(m) check after
 * it returns GBBS_ERANGE only if an edge (u, v) has finite d(u),
 * d(u) + w >= 2^32 - 1 and d(v) = GBBS_INF (dist then holds the exact finite
 * distances and GBBS_INF for the vertices that do not fit).  GBBS_EINTERNAL
 * if more than n+1 rounds run (impossible with w >= 0).
 */
int gbbs_bellman_ford(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                      void *cuda_stream);

/*
 * gbbs_widest_path — widest (bottleneck) path from src by Bellman-Ford over
 * the (max, min) semiring (sec:algs "Widest Path"; output spec
 * P:1499-1504): width[v] = max over src->v paths of the minimum edge weight
 * on the path.  Readings W1/W2: width[src] = GBBS_INF (the empty
 * path has no bottleneck); unreachable vertices get 0 (the max-semiring
 * identity; the paper's "infinity if unreachable" repeats the SSSP phrasing).
 * Weights as for gbbs_bellman_ford (NULL = unit).  Same stream, options and
 * error conventions as gbbs_bellman_ford (no GBBS_ERANGE: widths never exceed
 * the largest weight).
 */
int gbbs_widest_path(const gbbs_graph *g, uint32_t src, uint32_t *width,
                     void *cuda_stream);

/*
 * gbbs_betweenness — single-source betweenness contributions (P:98-101,
 * sec:algs; output spec P:1493-1496): delta[v] = sum over t != src, v of
 * sigma_st(v) / sigma_st, Brandes' dependency of src on v, following
 * out-edges (the paper's input is undirected; pass a symmetric CSR).  The
 * forward pass counts shortest paths with an atomicCAS test-and-set on the
 * level and an fp64 fetch-and-add on sigma, or, on a symmetric graph for a
 * level where |U| + sum deg(U) > m/T and the unvisited vertices carry under a
 * quarter of the frontier's edges, by pulling (each unvisited vertex sums
 * sigma over its neighbours on the level; reading B3; _ex: opts.mode
 * GBBS_MODE_SPARSE forces push, GBBS_MODE_DENSE pull); the backward pass
 * accumulates delta level by level.  delta[src] = 0 and unreached vertices get 0
 * (reading B1).
 *
 * delta   double[n], caller-owned, host or device.  fp64 accumulation in a
 *         nondeterministic order: results agree with a sequential Brandes to
 *         rounding (DESIGN.md tolerance), not bit for bit.
 * Errors: GBBS_EINVAL (g or delta NULL, src >= n), GBBS_ENOMEM (scratch:
 *         12n + 24*levels bytes on first use), GBBS_ECUDA, GBBS_EINTERNAL
 *         (more than 2^22 BFS levels).
 */
int gbbs_betweenness(const gbbs_graph *g, uint32_t src, double *delta,
                     void *cuda_stream);

/*
 * gbbs_wbfs — integral-weight SSSP ("weighted BFS", output spec P:1481-1484,
 * sec:benchmark; algorithm, sec:algs, after Julienne): dist[v] = the
 * shortest weighted distance from src, GBBS_INF if unreachable — the same
 * result as gbbs_bellman_ford, reached by extracting distance buckets in
 * increasing order, each bucket one edgeMap round with the priority-write min
 * (PAPER.md:1826-1831), vertices whose distance dropped moved to their new
 * bucket.  With the default bucket width 1 and weights >= 1 every reached
 * vertex is expanded exactly once (O(m) work) and every distinct finite
 * distance is an extracted bucket (a bucket whose entries all moved to earlier
 * buckets still costs a round).  gbbs_opts.delta > 1 selects Delta-stepping
 * buckets with a near list.
 *
 * Weights, dist, stream and error conventions as gbbs_bellman_ford (including
 * GBBS_ERANGE), plus GBBS_EINVAL if floor((delta - 1 + maxw) / delta) >= 64
 * (the bucket ring holds 64 lists), and GBBS_ENOMEM if a bucket list
 * overflows its capacity.  The bucket structure is allocated on the first call
 * and kept with the handle: nbq lists (the power of two above that span, <= 64)
 * of 2^ceil(log2 n) vertex ids each — fewer when that would take over half of
 * the free device memory — plus 16n bytes (near lists and round tags only when
 * delta > 1 or a weight is 0).
 */
int gbbs_wbfs(const gbbs_graph *g, uint32_t src, uint32_t *dist,
              void *cuda_stream);

/*
 * gbbs_bellman_ford_signed — general-weight SSSP by frontier Bellman-Ford
 * (output spec P:1487-1490, sec:benchmark; algorithm, sec:algs) with the
 * graph's weights read as int32 (two's complement of the uint32 weights given
 * at create; NULL weights = 1).
 *
 * dist    int64[n], caller-owned, host or device: the shortest-path distance
 *         from src; GBBS_DIST_INF if unreachable.  If a negative-weight cycle
 *         is reachable from src, "all distances must be -infinity":
 *         with gbbs_opts.neg_scope = 0 (default) every entry is
 *         GBBS_DIST_NEGINF; with neg_scope = 1 exactly the vertices reachable
 *         from such a cycle are GBBS_DIST_NEGINF and the others keep their
 *         finite distance or GBBS_DIST_INF.
 * Cost: O(diam) rounds without a reachable negative cycle.  With one: from
 * round 64 on, at every power-of-two round, the parent records of the
 * relaxations (each a real edge) are checked for a cycle by pointer doubling
 * (O(n log n) work); a parent cycle whose recorded weights sum below 0 proves
 * a reachable negative cycle (reading N4) — neg_scope 0 then ends
 * at once, neg_scope 1 fixes that cycle's forward closure at -infinity and
 * continues with the other vertices.  Backstop: a frontier still non-empty
 * after round n - 1 also proves one (then, for neg_scope = 1, one edge pass and
 * a reachability sweep find every affected vertex).
 * Same stream/synchronization conventions as gbbs_bfs.
 * Errors: GBBS_EINVAL (g or dist NULL, src >= n, bad options), GBBS_ERANGE
 *         if (n - 1) * max|w| >= 2^62, GBBS_ENOMEM (8n bytes of staging for
 *         a host dist), GBBS_ECUDA.
 */
#define GBBS_DIST_INF INT64_MAX
#define GBBS_DIST_NEGINF INT64_MIN
int gbbs_bellman_ford_signed(const gbbs_graph *g, uint32_t src, int64_t *dist,
                             void *cuda_stream);

/*
 * gbbs_wbfs_batch — k wBFS traversals (sources srcs[0..k), host array) into
 * device rows dist[i*n .. (i+1)*n); same results as k gbbs_wbfs calls.  The
 * traversals run concurrently, `teams` per cooperative launch (gbbs_opts.teams
 * in gbbs_wbfs_batch_ex; default 8 on graphs with n <= 2^24 and m <= 2^28,
 * else 1), each team with its own bucket ring and
 * scratch allocated on first use.  Errors as gbbs_wbfs, plus GBBS_EINVAL for
 * host rows.
 */
int gbbs_wbfs_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                    uint32_t *dist, void *cuda_stream);

/*
 * gbbs_betweenness_batch — k single-source betweenness computations (sources
 * srcs[0..k), host array) into device rows delta[i*n .. (i+1)*n) (double),
 * the same values as k gbbs_betweenness calls up to fp64 summation order.  The
 * traversals are launched back to back on the stream with one synchronisation
 * at the end (gbbs_opts.teams is accepted and ignored: several betweenness
 * traversals per launch measured slower at every team count, their levels are
 * throughput-bound).
 * Errors as gbbs_betweenness, plus GBBS_EINVAL for host rows.
 */
int gbbs_betweenness_batch(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                           double *delta, void *cuda_stream);

/* ---- extended calls (bench / tests) ------------------------------------ */

/* Representation choice per round (threshold rule reading A10).
 * BFS AUTO: a round is dense (pull over in-edges, early exit) iff
 *   |U| + sum_{u in U} outdeg(u) > m / T (reading A10), or —
 *   reading A10b, unless gbbs_opts.rules has GBBS_RULE_PAPER_ONLY — the
 *   previous round was dense (the frontier is a bitmap) and the pull's
 *   remaining work, the vertices with in-edges not yet visited, is at most
 *   |U| + sum deg(U); else sparse (push).
 * Bellman-Ford AUTO / SPARSE: every round converts the frontier bitmap into a
 *   list carrying each vertex's distance and pushes it in edge tiles with
 *   fire-and-forget priority-writes (round kind 5); DENSE forces the
 *   bitmap-forward push (the frontier as a bitmap, reading A11), kept as the
 *   measured alternative. */
#define GBBS_MODE_AUTO 0
#define GBBS_MODE_SPARSE 1 /* always push                                 */
#define GBBS_MODE_DENSE 2  /* BFS: always pull; BF: bitmap-forward push   */
#define GBBS_MODE_PULL 3   /* BFS: as AUTO; BF / widest path on symmetric
                              graphs: a pull-min round (every vertex takes
                              the best candidate over its in-edges from the
                              frontier, no atomics) whenever
                              |U| + sum deg(U) > m/T, else list push
                              (SURVEY 8(a) a9's alternative, reading A11) */

typedef struct {
  uint32_t threshold_den; /* T; 0 selects the default 20                  */
  int32_t mode;           /* GBBS_MODE_*                                   */
  uint32_t ctas_per_sm;   /* persistent-kernel CTAs per SM; 0 = as many as
                             are co-resident (default).  Fewer CTAs make
                             the per-round grid barrier cheaper (many small
                             rounds) at the cost of latency hiding.        */
  uint32_t delta;         /* gbbs_wbfs bucket width; 0 = default: 1 (the
                             paper's one bucket per distance) while
                             maxw <= 32, else ceil(maxw / 32).  Other
                             calls ignore it.                              */
  uint32_t neg_scope;     /* gbbs_bellman_ford_signed, when a negative cycle
                             is reachable from src: 0 (default) = every
                             distance is GBBS_DIST_NEGINF (PAPER.md:1489
                             read literally, reading N1); 1 = exactly the
                             vertices reachable from such a cycle
                             (reading N2).  Other calls ignore it.         */
  uint32_t bsize;         /* edges per warp tile of a list-push round
                             (edgeMapBlocked's block size):
                             a power of two in [32, 256]; 0 (default) =
                             256, halved while the round has fewer than
                             two tiles per warp                            */
  uint32_t teams;         /* batch calls with device outputs: traversals
                             run concurrently in one cooperative launch,
                             the CTAs interleaved into this many teams of
                             independent traversals (1-8).  0 = auto: 8 for
                             BFS on graphs with n <= 2^24 and m <= 2^28
                             (latency-bound traversals overlap), else 1.
                             Teams 1-7 allocate their own scratch (~60n
                             bytes of lists each) on first use.  Other
                             calls ignore it.                              */
  uint32_t rules;         /* direction-rule flags: GBBS_RULE_PAPER_ONLY
                             (BFS AUTO takes the paper's m/T test alone,
                             without reading A10b's stay-dense test);
                             GBBS_RULE_LEVEL_BYTES_ON / _OFF (BFS keeps
                             the levels of a traversal as one byte per
                             vertex and expands them into dist in a last
                             coalesced pass, instead of one scattered
                             4-byte store per acquisition — same dist,
                             P:1475-1478; default: on above 2^24
                             vertices).  Other bits must be zero.         */
} gbbs_opts;

#define GBBS_RULE_PAPER_ONLY 0x1
#define GBBS_RULE_LEVEL_BYTES_ON 0x2
#define GBBS_RULE_LEVEL_BYTES_OFF 0x4

/* One record per round, filled only when gbbs_stats.rounds_out != NULL. */
typedef struct {
  int32_t dense;          /* round kind: 0 = list push, 1 = dense pull,
                             2 = bitmap-forward push, 3 = pull-min (BF /
                             widest path, GBBS_MODE_PULL) or, for wBFS, a
                             bucket list, 4 = wBFS near list (same bucket),
                             5 = Bellman-Ford red round (bitmap -> list with
                             distances, then a push whose priority-writes
                             are reductions; frontier = the marked bitmap) */
  int32_t bucket;         /* wBFS: the bucket the round processed; else 0 */
  int64_t frontier;       /* |U|: frontier vertices with out-degree > 0   */
  int64_t frontier_edges; /* sum of out-degrees of U                       */
  int64_t acquired;       /* vertices won this round (incl. out-degree 0) */
  int64_t edges_examined; /* push: edges of U; pull: in-edges loaded      */
  int64_t vertices_swept; /* pull: unvisited vertices examined; bitmap-
                             forward: frontier vertices swept            */
  int64_t t_start_ns;     /* device %globaltimer when the round started;
                             the record after the last round holds the
                             end time when rounds_cap allows             */
  int64_t t_work_ns;      /* latest end of edge work over all CTAs      */
  int64_t t_flush_ns;     /* latest end of the final flush over all CTAs */
  int64_t alg_bytes;      /* algorithmic bytes the round loaded or stored
                             at the granularity of its loads:
                             offsets and per-vertex pull records, targets,
                             weights, frontier lists and bitmap words
                             swept; probes of the L2-resident bitmaps and
                             dist / parent state are not counted          */
  int64_t head_hits;      /* dense pull: vertices acquired by their first
                             in-edge (the inline record, no in-list load) */
} gbbs_round_stat;

typedef struct {
  int64_t rounds;          /* rounds executed (edgeMap calls)             */
  int64_t dense_rounds;    /* rounds of kind 1 (dense pull)               */
  int64_t edges_examined;  /* total over rounds                           */
  int64_t reached;         /* vertices with finite dist                  */
  double kernel_ms;        /* device time of the traversal kernel, from
                              CUDA events recorded on cuda_stream around
                              its launch                                 */
  gbbs_round_stat *rounds_out; /* host array or NULL                       */
  int64_t rounds_cap;      /* capacity of rounds_out                      */
} gbbs_stats;

/* Defaults: T = 20, GBBS_MODE_AUTO. */
void gbbs_default_opts(gbbs_opts *o);

/* As gbbs_bfs / gbbs_bellman_ford with options (NULL = defaults) and optional
 * statistics (NULL = none).  Collecting per-round records adds counters to
 * the kernels; do not time runs that collect them.  GBBS_EINVAL also for a
 * bad mode or unknown rules bits. */
int gbbs_bfs_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                uint32_t *parent, void *cuda_stream, const gbbs_opts *opts,
                gbbs_stats *stats);
int gbbs_bellman_ford_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                         void *cuda_stream, const gbbs_opts *opts,
                         gbbs_stats *stats);
int gbbs_betweenness_ex(const gbbs_graph *g, uint32_t src, double *delta,
                        void *cuda_stream, const gbbs_opts *opts,
                        gbbs_stats *stats);
int gbbs_bellman_ford_signed_ex(const gbbs_graph *g, uint32_t src, int64_t *dist,
                                void *cuda_stream, const gbbs_opts *opts,
                                gbbs_stats *stats);
/* Batch calls with options (threshold T, modes 0-2, bsize, teams, wBFS delta;
 * NULL = defaults; ctas_per_sm must be 0). */
int gbbs_wbfs_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                       uint32_t *dist, void *cuda_stream, const gbbs_opts *opts);
int gbbs_betweenness_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                              double *delta, void *cuda_stream,
                              const gbbs_opts *opts);
int gbbs_bfs_batch_ex(const gbbs_graph *g, const uint32_t *srcs, int64_t k,
                      uint32_t *dist, uint32_t *parent, void *cuda_stream,
                      const gbbs_opts *opts);
int gbbs_bellman_ford_batch_ex(const gbbs_graph *g, const uint32_t *srcs,
                               int64_t k, uint32_t *dist, void *cuda_stream,
                               const gbbs_opts *opts);
int gbbs_wbfs_ex(const gbbs_graph *g, uint32_t src, uint32_t *dist,
                 void *cuda_stream, const gbbs_opts *opts, gbbs_stats *stats);
int gbbs_widest_path_ex(const gbbs_graph *g, uint32_t src, uint32_t *width,
                        void *cuda_stream, const gbbs_opts *opts,
                        gbbs_stats *stats);

/* Launch geometry of the persistent traversal kernel on this device:
 * *ctas = co-resident CTAs used, *threads = threads per CTA. */
int gbbs_launch_info(const gbbs_graph *g, int32_t *ctas, int32_t *threads);

/* gbbs_graph_in_edges — copy the handle's in-edge CSC (the transpose the dense
 * pull reads, P:1870-1874 sec:prelims) into caller-owned buffers, host or
 * device: in_offsets int64[n+1], in_sources uint32[m] (each in-list ascending
 * by source id).  For a GBBS_SYMMETRIC graph this is the CSR itself.  Either
 * pointer may be NULL (not copied).  Synchronous.
 * Errors: GBBS_EINVAL (g NULL), GBBS_ECUDA. */
int gbbs_graph_in_edges(const gbbs_graph *g, int64_t *in_offsets, uint32_t *in_sources);

/* Thread-local message describing the last error on this thread ("" if none). */
const char *gbbs_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* GBBS_H */
