#!/usr/bin/env python
"""bench.py — GTEPS of libgbbs's frontier BFS / Bellman-Ford on one B200 per rank.

Contract (task README + DESIGN.md §Measurement):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c5] [--bf-workload c4] [--algo bfs|bf]
One step = one pass of the hot path over the workload's batch: BFS (direction-
optimising, T=20) from each of the config's seeded sources on the resident graph
(default c5, the largest single-GPU config: 8 sources with out-degree >= 1 on the
directed 2^26-vertex rMAT graph), issued as one gbbs_bfs_batch call into device
rows.  The Bellman-Ford leg of the metric is measured in the same run on c4 (BJ's
atomicMin config: 4 seeded LCC sources, weights in [1, 25], reading A6) and
reported under "bellman_ford", beside the NEXT rows on the same graph and a c2 BFS
leg.
Multi-GPU: every rank holds its own copy of the graph and
traverses its own shard of the source sample (rank r: sources 8r .. 8r+7 of the
config's sequential seeded sample, so rank 0's are the N=1 sources; configs with
a single fixed source run it on every rank); value = traversed edges summed over
ranks / max-over-ranks step time (weak scaling, no collective on the data path).
--impl reference times the CPU oracle (sequential C queue-BFS / Dijkstra) — the
only place besides cpu_baseline where bench.py executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GTEPS per B200 for BFS and Bellman-Ford; achieved HBM GB/s vs roofline"
INF = 0xFFFFFFFF


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5",
                    help="headline config (default c5: the largest single-GPU config, BJ's "
                         "large rMAT direction-optimising BFS)")
    ap.add_argument("--algo", default="bfs", choices=["bfs", "bf"])
    ap.add_argument("--bf-workload", default="c4",
                    help="config of the Bellman-Ford leg (default c4: BJ's atomicMin config)")
    ap.add_argument("--threshold", type=int, default=20)
    ap.add_argument("--rules", type=int, default=0, help="gbbs_opts.rules (1 = paper's m/T only)")
    ap.add_argument("--no-legs", action="store_true", help="headline only (no BF / NEXT / c2 legs)")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no legs, no cpu baseline)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """Sample SM clocks and clock-event (throttle) reasons with NVML every `period`
    seconds in a background thread while the timed region runs (the recipe's
    clocks line, B200_PROFILING.md).  Falls back to nvidia-smi if NVML fails."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index, period=0.002):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = None
        self._thr = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for nm, attr in self.NAMES:
                        if bits & getattr(pynvml, attr, 0):
                            self.reasons.add(nm)
                except Exception:  # noqa: BLE001
                    pass
                self._stop.wait(self.period)

        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def stop(self):
        if self._thr is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [getattr(self, "err", "no samples")]}
        self._stop.set()
        self._thr.join()
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs"), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def copy_bandwidth(torch):
    """Stream copy, same method as MEASURED_PEAKS: 1 Gi bf16 copy_, best of 10."""
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * (1 << 30) * 2 / (best * 1e-3) / 1e9


def algorithmic_bytes(recs, n, m, algo):
    """SURVEY §8(d) algorithmic bytes of one traversal: offsets (and per-vertex pull
    records), targets, weights and frontier (lists and bitmap words), at the
    granularity the kernels load them — a 16-byte in-edge vector load counts 16 B
    even after an early exit.  BFS / Bellman-Ford / widest path: the kernels' own
    counters (gbbs_round_stat.alg_bytes, summed by the STATS instantiation at every
    load site).  wBFS has no counters: 24 B per bucket entry swept (id, dist, two
    offsets), 8 B per edge (target + weight), 4 B per insertion.  Probes of the
    L2-resident bitmaps and the dist / parent state are not counted; the state
    bytes (per-run init) are returned separately."""
    if algo in ("bfs", "bf", "wp"):
        alg = sum(r["alg_bytes"] for r in recs)
    else:
        alg = sum(24 * r["vertices_swept"] + 8 * r["edges_examined"] + 4 * r["acquired"]
                  for r in recs)
    state = 8 * n if algo == "bfs" else 4 * n
    return alg, state


def reached_edges(torch, off, d):
    deg = off[1:] - off[:-1]
    return int(deg[d != -1].sum())


def ncu_traffic(workload, algo, what="bytes"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from
    the committed ncu --set full capture (profiles/ncu_traffic.json), or None;
    what="us": that launch's ncu duration."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if what == "us":
            return d.get("_duration_us", {}).get(workload, {}).get(algo)
        return d.get(workload, {}).get(algo)
    except (OSError, ValueError):
        return None


def replica_max(x, world, dist_mod=None, device="cpu"):
    """Max over ranks of a per-rank time (replicas: no data-path collective; this
    is the only reduction).  world == 1: identity."""
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist_mod.all_reduce(t, op=dist_mod.ReduceOp.MAX)
    return float(t.item())


def replica_sum(x, world, dist_mod=None, device="cpu"):
    """Sum over ranks of a per-rank count (the job's traversed edges)."""
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist_mod.all_reduce(t, op=dist_mod.ReduceOp.SUM)
    return float(t.item())


def replica_value(edges_all_ranks_step, step_ms_max):
    """Whole-job GTEPS: edges traversed by all ranks per step / the slowest rank's
    step time (weak scaling: each rank's batch is fixed)."""
    return edges_all_ranks_step / (step_ms_max * 1e-3) / 1e9


def shard_sources(sources, rank, world, per_rank):
    """Rank r's sources: entries [per_rank*r, per_rank*(r+1)) of the sequential
    sample, or the whole (single-source) list on every rank."""
    if len(sources) < per_rank * world:
        return list(sources)
    return list(sources[per_rank * rank: per_rank * (rank + 1)])


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist_mod
    from graphgen import CONFIGS
    from graphgen import device as gdev
    from paper_1805_05208_b200 import gbbs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist_mod.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    peak, peak_src = measured_peaks()

    def load(name, weights):
        t0 = time.time()
        per_rank = CONFIGS[name].nsources
        G = gdev.build_config(name, weights=weights, nsources=per_rank * world)
        G["g"] = gbbs.Graph(G["offsets"], G["targets"], G["weights"], symmetric=G["symmetric"])
        G["mine"] = shard_sources(G["sources"], rank, world, per_rank)
        G["setup_s"] = round(time.time() - t0, 2)
        return G

    def drop(G):
        G["g"].close()
        G.clear()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def one(G, algo, src, dist, par, opts=None, stats=None):
        g = G["g"]
        if algo == "bfs":
            g.bfs(src, dist, par, stream=stream, opts=opts, stats=stats)
        elif algo == "bf":
            g.bellman_ford(src, dist, stream=stream, opts=opts, stats=stats)
        elif algo == "wbfs":
            g.wbfs(src, dist, stream=stream, opts=opts, stats=stats)
        else:
            g.widest_path(src, dist, stream=stream, opts=opts, stats=stats)

    def profile(G, algo, opts):
        """Per source: TEPS numerator (reading A20), rounds, algorithmic bytes (the
        kernels' counters, STATS instantiation, untimed) and relaxations."""
        n, off = G["n"], G["offsets"]
        dist = torch.empty(n, dtype=torch.int32, device=dev)
        par = torch.empty_like(dist)
        out = {}
        for s in G["mine"]:
            st = gbbs.make_stats(1 << 16)
            one(G, algo, s, dist, par, opts, st)
            recs = gbbs.round_records(st)
            alg, state = algorithmic_bytes(recs, n, G["m"], algo)
            reach = reached_edges(torch, off, dist) if algo != "wp" else \
                int((off[1:] - off[:-1])[dist != 0].sum())
            out[s] = dict(m_reach=reach, rounds=st.rounds, dense_rounds=st.dense_rounds,
                          alg_bytes=alg, state_bytes=state,
                          relax=sum(r["edges_examined"] for r in recs),
                          kinds="".join("SDFPBR"[min(r["dense"], 5)] for r in recs))
        return out

    def timed(G, algo, opts, steps, warmup, rows, prows):
        """One step = the batch call over this rank's sources into device rows (the
        launches are enqueued back to back, one synchronisation per step); the step
        time is the slowest rank's.  Also the kernel-only time summed over sources
        (CUDA events libgbbs records around each persistent launch)."""
        srcs = G["mine"]

        def step():
            if algo == "bfs":
                G["g"].bfs_batch(srcs, rows, prows, stream=stream, opts=opts)
            elif algo == "bf":
                G["g"].bellman_ford_batch(srcs, rows, stream=stream, opts=opts)
            elif algo == "wbfs":
                G["g"].wbfs_batch(srcs, rows, stream=stream, opts=opts)
            else:
                for i, s in enumerate(srcs):
                    one(G, algo, s, rows[i], None, opts)
        for _ in range(warmup):
            step()
        if world > 1:
            dist_mod.barrier()
        torch.cuda.synchronize()
        clocks = Clocks(local)
        clocks.start()
        evs = []
        for _ in range(steps):
            flush_buf.fill_(1)  # L2 flush between timed steps (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ck = clocks.stop()
        if world > 1:
            dist_mod.barrier()
        ms = float(np.mean([x.elapsed_time(y) for x, y in evs]))
        tmax = replica_max(ms, world, dist_mod, dev)
        kms = []
        for i, s in enumerate(srcs):
            flush_buf.fill_(1)
            st = gbbs.make_stats(0)
            one(G, algo, s, rows[i], prows[i] if prows is not None else None, opts, st)
            kms.append(st.kernel_ms)
        return tmax, ck, float(np.sum(kms))

    def leg(G, algo, opts, steps, warmup, with_parent=False):
        per = profile(G, algo, opts)
        rows = torch.empty((len(G["mine"]), G["n"]), dtype=torch.int32, device=dev)
        prows = torch.empty_like(rows) if with_parent else None
        t, ck, kms = timed(G, algo, opts, steps, warmup, rows, prows)
        edges = replica_sum(sum(v["m_reach"] for v in per.values()), world, dist_mod, dev)
        alg = sum(v["alg_bytes"] for v in per.values())
        del rows, prows
        return dict(per=per, ms=t, clocks=ck, kernel_ms=kms, edges=edges, alg=alg,
                    value=replica_value(edges, t))

    # ---- headline: c5 direction-optimising BFS (default) --------------------------
    H = load(args.workload, weights=args.algo == "bf")
    cfg, n, m = H["cfg"], H["n"], H["m"]
    sources = H["mine"]
    opts = gbbs.make_opts(args.threshold, gbbs.GBBS_MODE_AUTO, rules=args.rules)
    hl = leg(H, args.algo, opts, args.steps, args.warmup, with_parent=args.algo == "bfs")
    step_ms, clocks, kernel_ms = hl["ms"], hl["clocks"], hl["kernel_ms"]
    per_src, edges_job, alg_bytes = hl["per"], hl["edges"], hl["alg"]
    edges_step = sum(v["m_reach"] for v in per_src.values())
    value = hl["value"]

    # e2e: the public batch API with pinned host output rows: one gbbs_bfs_batch call
    # per step, whose device->host copies of dist/parent (8n bytes per source)
    # overlap the next traversal (sources are a host array)
    hd = torch.empty((len(sources), n), dtype=torch.int32, pin_memory=True)
    hp = torch.empty((len(sources), n), dtype=torch.int32, pin_memory=True)
    hdn, hpn = hd.numpy(), hp.numpy()
    torch.cuda.synchronize()
    e2e = []
    for _ in range(max(2, min(args.steps, 5))):
        if world > 1:
            dist_mod.barrier()
        t = time.perf_counter()
        if args.algo == "bfs":
            gbbs.gbbs_bfs_batch(H["g"].handle, sources, hdn, hpn, stream=stream, opts=opts)
        else:
            gbbs.gbbs_bellman_ford_batch(H["g"].handle, sources, hdn, stream=stream)
        e2e.append(replica_max(time.perf_counter() - t, world, dist_mod, dev))
    e2e_s = float(np.median(e2e))
    del hd, hp, hdn, hpn

    teams = min(8, len(sources)) if (args.algo == "bfs" and n <= (1 << 24) and m <= (1 << 28)) else 1
    launches = -(-len(sources) // teams)
    out = None
    if rank == 0:
        copy_gbs = copy_bandwidth(torch)
        kname = ("gbbs_dev::traverse_mg_kernel<BFS> (persistent; %d traversals per launch, "
                 "%d launches per step)" % (teams, launches)) if teams > 1 else \
            "gbbs_dev::traverse_kernel<%s> (persistent; one launch per traversal)" % args.algo.upper()
        # achieved = algorithmic bytes of the step (kernel counters) / the step's device
        # time (CUDA events around exactly those launches on their stream)
        achieved = alg_bytes / (step_ms * 1e-3) / 1e9
        traffic = ncu_traffic(cfg.name, args.algo)
        d2h = len(sources) * n * (8 if args.algo == "bfs" else 4)
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded counter-based rMAT/torus generators, DESIGN.md §Input recipe)",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "algo": args.algo,
                       "n": n, "m": m, "sources": sources, "threshold_T": args.threshold,
                       "rules": args.rules, "traversals_per_step": len(sources),
                       "edges_per_step": edges_step,
                       "l2": "flushed (256 MB write) before every timed step; graph > L2",
                       "parallelism": f"source-sharded replicas x{world}",
                       "edges_per_step_all_ranks": edges_job},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "traffic_unit": "bytes per launch of the kernel below",
                         "traffic_vs_alg_bytes": (round(traffic / (alg_bytes / len(sources)), 3)
                                                  if traffic else None),
                         "peak_source": peak_src, "copy_gbs_same_run": round(copy_gbs, 1),
                         "frac_of_copy_same_run": round(achieved / copy_gbs, 4),
                         "frac_of_nominal_8tbs": round(achieved / 8000.0, 4),
                         "kernel": kname, "teams": teams,
                         "alg_bytes_per_step": alg_bytes, "kernel_ms_per_step": round(step_ms, 4),
                         "single_traversal_kernel_ms_per_step": round(kernel_ms, 4),
                         "single_traversal_gteps": round(edges_step / (kernel_ms * 1e-3) / 1e9, 3),
                         # context only, not the gate: 4 B per reached edge at peak (a
                         # dense-equivalent count; an early-exit pull never reads most
                         # of those bytes, so this can exceed 1)
                         "dense_equivalent_context": {
                             "bytes_per_reached_edge": 4,
                             "frac": round(4 * edges_step / (step_ms * 1e-3) / 1e9 / peak, 4)}},
            "e2e": {"value": round(edges_job / e2e_s / 1e9, 3), "unit": "GTEPS",
                    "h2d_bytes_per_step": 4 * len(sources) * world, "d2h_bytes_per_step": d2h * world,
                    "note": "gbbs_bfs_batch (one call per step) into pinned host dist/parent "
                            "rows; the library's D2H copy of traversal i overlaps traversal i+1; "
                            "h2d = the source ids (host array, passed as kernel arguments)"},
            "graph500_undirected_gteps": (round(edges_job / 2 / (step_ms * 1e-3) / 1e9, 3)
                                          if cfg.symmetric else None),
            "gpu_launches": args.steps * launches,
            "clocks": clocks,
            "per_source": [{"src": s, **per_src[s]} for s in sources],
            "setup_s": H["setup_s"],
        }
        if not args.profile:
            out["cpu_baseline"] = cpu_baseline(args, H["offsets"], H["targets"], sources, cfg)
    drop(H)
    if args.no_legs or args.profile:
        if world > 1:
            dist_mod.destroy_process_group()
        return out

    # ---- legs: Bellman-Ford (the metric's second half) + NEXT rows on c4 ------------
    B = load(args.bf_workload, weights=True)
    bcfg = B["cfg"]
    legs = {}
    for algo, key in (("bf", "bellman_ford"), ("wbfs", "wbfs"), ("wp", "widest_path")):
        r = leg(B, algo, None, max(2, args.steps // 2), 1)
        legs[key] = r
    # NEXT-3: single-source betweenness on the same graph, this rank's sources per step
    srcs = B["mine"]
    delta = torch.empty((len(srcs), B["n"]), dtype=torch.float64, device=dev)
    B["g"].betweenness_batch(srcs[:1], delta[:1], stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush_buf.fill_(1)
    e0.record(stream)
    B["g"].betweenness_batch(srcs, delta, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    bc_ms = replica_max(e0.elapsed_time(e1), world, dist_mod, dev)
    bc_edges = legs["bellman_ford"]["edges"]
    del delta
    bsrc = B["mine"]
    drop(B)
    # ---- leg: c2 BFS (the medium config; teams of traversals per launch) -------------
    C = load("c2", weights=False)
    c2 = leg(C, "bfs", opts, args.steps, args.warmup, with_parent=True)
    c2src = C["mine"]
    drop(C)

    if rank == 0:
        bf = legs["bellman_ford"]
        bf_relax = sum(v["relax"] for v in bf["per"].values())
        out["bellman_ford"] = {
            "workload": f"{bcfg.name}: {bcfg.note}", "sources": bsrc,
            "value": round(bf["value"], 3), "unit": "GTEPS (effective, reading A20)",
            "relaxations_per_s_G": round(bf_relax / (bf["ms"] * 1e-3) / 1e9, 3),
            "ms_per_step": round(bf["ms"], 4), "kernel_ms_per_step": round(bf["kernel_ms"], 4),
            "weights": f"[1,{bcfg.W}] pair-hash (readings A5, A6)",
            "alg_bytes_per_step": bf["alg"],
            "roofline_frac": round(bf["alg"] / (bf["kernel_ms"] * 1e-3) / 1e9 / peak, 4),
            # every relaxation probes the 16-bit distance shadow at a random address;
            # tools/gather_bench.cu measured 270 G random 2-byte L2 gathers/s on this B200
            "relax_vs_l2_gather_ceiling": round(bf_relax / (bf["kernel_ms"] * 1e-3) / 1e9 / 270.0, 4),
            # ncu dram read+write per launch (mean over the config's sources, committed capture)
            "traffic": ncu_traffic(bcfg.name, "bf"),
            "traffic_vs_alg_bytes": (round(ncu_traffic(bcfg.name, "bf") / (bf["alg"] / len(bsrc)), 3)
                                     if ncu_traffic(bcfg.name, "bf") else None),
            "clocks": bf["clocks"], "rounds": [v["rounds"] for v in bf["per"].values()]}
        for key, note in (("wbfs", "NEXT-2: integral-weight SSSP over distance buckets (bucket width "
                                   "1), same graph and weights as the Bellman-Ford leg"),
                          ("widest_path", "NEXT-1: Bellman-Ford over the (max, min) semiring, same "
                                          "graph and weights")):
            r = legs[key]
            out[key] = {"value": round(r["value"], 3), "unit": "GTEPS (effective)",
                        "ms_per_step": round(r["ms"], 4), "kernel_ms_per_step": round(r["kernel_ms"], 4),
                        "roofline_frac": round(r["alg"] / (r["kernel_ms"] * 1e-3) / 1e9 / peak, 4),
                        "note": note, "rounds": [v["rounds"] for v in r["per"].values()]}
        out["betweenness"] = {
            "value": round(bc_edges / (bc_ms * 1e-3) / 1e9, 3),
            "unit": "GTEPS (m_reach of the BFS per source / time)", "ms_per_step": round(bc_ms, 4),
            "note": "NEXT-3: Brandes dependencies on the Bellman-Ford leg's graph and sources, one "
                    "gbbs_betweenness_batch call into device rows"}
        out["c2_bfs"] = {
            "workload": "c2: " + CONFIGS["c2"].note, "sources": c2src,
            "value": round(c2["value"], 3), "unit": "GTEPS",
            "graph500_undirected_gteps": round(c2["edges"] / 2 / (c2["ms"] * 1e-3) / 1e9, 3),
            "ms_per_step": round(c2["ms"], 4),
            "roofline_frac": round(c2["alg"] / (c2["ms"] * 1e-3) / 1e9 / peak, 4),
            "note": "the medium config: one gbbs_bfs_batch call per step (8 traversals as teams "
                    "of one cooperative launch)",
            "rounds": [v["rounds"] for v in c2["per"].values()]}
    if world > 1:
        dist_mod.destroy_process_group()
    return out


def cpu_baseline(args, off_dev, tgt_dev, sources, cfg):
    """The oracle as it stands (sequential C queue-BFS), 1 core, bounded sample."""
    import oracle
    off = off_dev.cpu().numpy()
    tgt = tgt_dev.cpu().numpy().view(np.uint32)
    done, edges, t_all = [], 0, 0.0
    for s in sources:
        t = time.perf_counter()
        d, _ = oracle.bfs(off, tgt, s)
        dt = time.perf_counter() - t
        edges += oracle.reached_edges(off, d)
        t_all += dt
        done.append(s)
        if t_all > args.cpu_budget_s:
            break
    return {"value": round(edges / t_all / 1e9, 4), "unit": "GTEPS", "cores": 1, "kind": "oracle",
            "sample": f"oracle_bfs (sequential C FIFO BFS) from {len(done)} of {len(sources)} "
                      f"sources of {cfg.name}, {t_all:.1f} s", "cpu": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the same workload (rank 0 only)."""
    if rank != 0:
        return None
    import oracle
    import graphgen
    cfg = graphgen.CONFIGS[args.workload]
    try:
        from graphgen import device as gdev
        import torch
        G = gdev.build_config(cfg.name, weights=args.algo == "bf")
        off = G["offsets"].cpu().numpy()
        tgt = G["targets"].cpu().numpy().view(np.uint32)
        w = G["weights"].cpu().numpy().view(np.uint32) if G["weights"] is not None else None
        sources = G["sources"]
        del G
    except Exception:  # no GPU: build on the host (small configs only)
        off, tgt = graphgen.rmat_graph(cfg.levels, 1 << cfg.log_edges, cfg.graph_seed, *cfg.abc,
                                       symmetric=cfg.symmetric)
        w = graphgen.pair_weights(off, tgt, cfg.weight_seed, cfg.W) if args.algo == "bf" else None
        sources = graphgen.choose_sources(graphgen.largest_component(off, tgt), cfg.nsources,
                                          cfg.source_seed) if cfg.sources == "lcc" else [0]
    times, edges = [], 0
    budget = 120.0 / max(1, args.steps + args.warmup)
    for step in range(args.warmup + args.steps):
        t = time.perf_counter()
        e, used = 0, 0
        for s in sources:
            if args.algo == "bfs":
                d, _ = oracle.bfs(off, tgt, s)
            else:
                d, _ = oracle.dijkstra(off, tgt, w, s)
            e += oracle.reached_edges(off, d)
            used += 1
            if time.perf_counter() - t > budget:
                break
        dt = time.perf_counter() - t
        if step >= args.warmup:
            times.append(dt); edges += e
    v = edges / sum(times) / 1e9
    return {"metric": METRIC, "value": round(v, 4), "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * float(np.mean(times)), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "algo": args.algo},
            "cpu_baseline": {"value": round(v, 4), "unit": "GTEPS", "cores": 1, "kind": "oracle",
                             "sample": f"{used} of {len(sources)} sources per step (budget {budget:.0f} s)"},
            "e2e": {"value": round(v, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local)
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
