#!/usr/bin/env python
"""Benchmark of the xBeam decode-step selection path (BASELINE.json metric) on B200.

One bench "step" = one pass of the whole hot path over one batch: the ND beam-search steps of
C3 (batch 256, BW 256, V 8192, ND 3, 100M-item trie) through the C ABI, plus
finalize (device outputs). Inputs (seeded synthetic logits, 4.0 GiB per pass) are resident in HBM
and larger than L2, so L2 needs no flush between iterations.

  python bench.py [--gpus N --steps K --warmup W]        our CUDA path (one JSON line, rank 0)
  python bench.py --impl reference [...]                 the CPU oracle (reference arm, rank 0)

Multi-GPU (torchrun, one process per GPU): the request batch partitions the work, every rank runs
its own C3 batch (different seeds, the same catalogue), no data-path collective ("scaling":
"weak"); time = max over ranks of CUDA-event time, value = all ranks' candidates / that time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "beam-step candidates/sec (C3: batch 256, BW 256, V 8192, ND 3; raw (b, v) pool per step)"
UNIT = "candidates/s"


# ---- host-side multi-rank logic (covered by tests/test_bench_dist.py with gloo) -------------------
def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_plan(cfg: dict, rank: int, world: int) -> dict:
    """Weak scaling: every rank runs one full batch of the config with its own logit seeds."""
    return {"batch": cfg["batch"], "seed_base": 7919 * (rank + 1), "requests": (rank * cfg["batch"], (rank + 1) * cfg["batch"])}


def step_seeds(plan: dict, nd: int):
    return [plan["seed_base"] * 16 + t for t in range(nd)]


def candidates_per_pass(cfg: dict, batch: int) -> int:
    """Raw (b, v) candidate pool of one ND-step pass: 1 root row at step 1, BW rows after."""
    return batch * (1 + cfg["beam_width"] * (cfg["nd"] - 1)) * cfg["vocab"]


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int, device=None):
    if world > 1:
        import torch.distributed as dist
        if device is not None:
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


# ---- clocks during the timed region (B200_PROFILING.md clocks line) --------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def committed_traffic(dtype="f32"):
    """dram bytes per launch of k_stream from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_k_stream_traffic.json" if dtype == "f32"
                     else f"ncu_k_stream_{dtype}_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except OSError:
        return None


# ---- CPU oracle timing (cpu_baseline and the reference arm) -----------------------------------------
def oracle_sample(voc, cfg, logits_fn, n_req: int, threads: int):
    """Free-running oracle ND-step beam search of n_req requests on a thread pool.
    logits_fn(r, t) -> numpy [rows][V] fp32. Returns (candidates, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import xbeam_oracle as O
    lg = [[logits_fn(r, t) for t in range(cfg["nd"])] for r in range(n_req)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda r: O.run_request(voc, lg[r], cfg["beam_width"]), range(n_req)))
    dt = time.perf_counter() - t0
    return candidates_per_pass(cfg, n_req), dt


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---- our CUDA path -----------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2512_11529_b200 as xgr
    from synth import make_items, make_logits_torch

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    plan = rank_plan(cfg, rank, world)
    B, BW, V, ND = plan["batch"], cfg["beam_width"], cfg["vocab"], cfg["nd"]
    t0 = time.perf_counter()
    items = make_items(cfg["n_items"], V, ND, cfg["trie_key"])
    gen_s = time.perf_counter() - t0
    bs = xgr.BeamSearch(V, ND, BW, B, device=local_rank, flags=xgr.XGR_CFG_TIMING,
                        theta_rows=int(os.environ.get("XGR_THETA_ROWS", "0")))
    t0 = time.perf_counter()
    bs.mask_build(items)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    info = bs.info()
    seeds = step_seeds(plan, ND)
    logits = [make_logits_torch((B, 1 if t == 0 else BW, V), seeds[t], args.sigma, device=dev)
              for t in range(ND)]
    if args.logits == "bf16":   # NEXT f1: the same N(0, sigma^2) draws rounded to bf16
        logits = [x.to(torch.bfloat16) for x in logits]
    in_bytes = sum(x.numel() * x.element_size() for x in logits)
    stream = torch.cuda.current_stream()
    out = {"tokens": torch.empty((B, BW, ND), dtype=torch.int32, device=dev),
           "item_rank": torch.empty((B, BW), dtype=torch.int64, device=dev),
           "score": torch.empty((B, BW), dtype=torch.float32, device=dev),
           "n_live": torch.empty((B,), dtype=torch.int32, device=dev)}

    def one_pass(evs=None):
        if evs:
            evs[0].record(stream)
        for t in range(ND):
            bs.step(logits[t])
            if evs:
                evs[t + 1].record(stream)
        # finalize (a6) is fused into the last step's commit: the item tuples, ranks and scores
        # are in device memory now (bs.outputs_view()); this call only ends the batch
        bs.finalize_in_place()
        if evs:
            evs[ND + 1].record(stream)

    for _ in range(args.warmup):
        one_pass()
    torch.cuda.synchronize()
    bs.kernel_times()                      # drain warm-up records
    launches0 = bs.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(ND + 2)] for _ in range(args.steps)]
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    barrier(world, dev)
    torch.cuda.synchronize()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for k in range(args.steps):
        one_pass(evs[k])
    e_end.record(stream)
    torch.cuda.synchronize()
    barrier(world, dev)
    # the dense-step kernel's library-side CUDA-event times of the eager passes (read before the
    # graph capture, which records the same events as graph nodes)
    kms, kstep = bs.kernel_times()
    launches = bs.launch_count() - launches0   # kernels per timed run (a graph replay runs the same ones)
    # the same pass captured once as a CUDA graph and replayed K times (xSchedule's
    # graph dispatch submits a step's device work at once). This removes the host's per-launch
    # work from the critical path; when capture works it is the headline, eager is kept beside it.
    graph = None
    if not args.profile and not args.no_graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                one_pass()
            for _ in range(max(1, args.warmup)):
                g.replay()
            torch.cuda.synchronize()
            barrier(world, dev)
            gev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
            gev[0].record(stream)
            for k in range(args.steps):
                g.replay()
                gev[k + 1].record(stream)
            torch.cuda.synchronize()
            barrier(world, dev)
            g_total = max_over_ranks(gev[0].elapsed_time(gev[-1]), world, dev)
            g_iter = [gev[k].elapsed_time(gev[k + 1]) for k in range(args.steps)]
            graph = {"total_ms": g_total, "per_iter": g_iter}
            del g
        except Exception as e:   # the eager measurement above stands
            graph = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    clk = clocks.stop()
    total_ms = e_start.elapsed_time(e_end)
    total_ms_max = max_over_ranks(total_ms, world, dev)
    per_iter = [evs[k][0].elapsed_time(evs[k][ND + 1]) for k in range(args.steps)]
    per_step = [[evs[k][t].elapsed_time(evs[k][t + 1]) for k in range(args.steps)] for t in range(ND + 1)]
    main_ms = [float(m) for m, s in zip(kms, kstep)]
    dense_steps = sorted(set(int(s) for s in kstep))

    cand = candidates_per_pass(cfg, B)
    value = cand * world * args.steps / (total_ms_max / 1e3)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
        "p50_ms": statistics.median(per_iter), "p99_ms": sorted(per_iter)[min(len(per_iter) - 1, int(0.99 * len(per_iter)))],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded: Feistel-permuted uniform item tuples, N(0, sigma^2) {args.logits} logits)",
        "config": {"workload": cfg["name"], "batch_per_gpu": B, "beam_width": BW, "vocab": V, "nd": ND,
                   "logits": args.logits,
                   "n_items": cfg["n_items"], "n_items_dedup": int(info["n_items"]), "sigma": args.sigma,
                   "parallelism": f"request-split x{world}",
                   "l2": f"inputs larger than L2 ({in_bytes / 2**30:.2f} GiB per pass), no flush"},
        "step_p50_ms": {f"t{t + 1}" if t < ND else "finalize": statistics.median(per_step[t]) for t in range(ND + 1)},
        "gpu_launches": launches,
        "clocks": clk,
        "setup": {"items_gen_s": round(gen_s, 2), "mask_build_s": round(build_s, 3),
                  "trie_bytes": int(info["bytes"]), "dense_route_steps": dense_steps},
    }

    res["eager"] = {"value": value, "ms_per_step": res["ms_per_step"], "p50_ms": res["p50_ms"],
                    "p99_ms": res["p99_ms"], "how": "per-step host calls (ctypes) on one stream"}
    if graph and "total_ms" in graph:
        gi = graph["per_iter"]
        res["value"] = cand * world * args.steps / (graph["total_ms"] / 1e3)
        res["ms_per_step"] = graph["total_ms"] / args.steps
        res["p50_ms"] = statistics.median(gi)
        res["p99_ms"] = sorted(gi)[min(len(gi) - 1, int(0.99 * len(gi)))]
        res["mode"] = "cuda_graph"
        res["graph"] = {"how": "one pass (ND steps + finalize) captured once in a CUDA graph, replayed K times; "
                               "step_p50_ms / gpu_launches / roofline come from the eager passes"}
    else:
        res["mode"] = "eager"
        if graph:
            res["graph"] = graph

    if rank == 0 and not args.profile:
        # ---- accounting + counters on an identical, untimed pass (separate ctx) ----
        acc = xgr.BeamSearch(V, ND, BW, B, device=local_rank, flags=xgr.XGR_CFG_COUNTERS,
                             theta_rows=int(os.environ.get("XGR_THETA_ROWS", "0")))
        acc.mask_build(items)
        acc.counters()
        algb = None
        counters = {}
        for t in range(ND):
            acc.step(logits[t])
            c = acc.counters()
            if t + 1 in dense_steps:
                a = acc.account()
                algb = a if algb is None else algb
                counters = c
        acc.finalize(on_device=True)
        acc.close()
        peaks, src = measured_peaks()
        peak = float(peaks.get("hbm_gbs", 6650.0))
        if main_ms and algb:
            mean_ms = sum(main_ms) / len(main_ms)
            achieved = algb["alg_bytes"] / (mean_ms / 1e3) / 1e9
            step_dense = statistics.median(per_step[dense_steps[0] - 1]) if dense_steps else None
            tr = committed_traffic(args.logits)
            res["roofline"] = {
                "bound": "hbm", "kernel": "k_stream (dense step: TMA row stream, masked log-softmax, score add, pruned emit)",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs)" if src == "measured" else "fallback 6.65 TB/s",
                "traffic": (tr or {}).get("dram_bytes_per_launch"),
                "traffic_source": (tr or {}).get("source"),
                "alg_bytes_per_launch": algb["alg_bytes"], "full_bytes_per_launch": algb["full_bytes"],
                "kernel_ms_mean": mean_ms, "launches_timed": len(main_ms),
                "dense_step_ms_p50": step_dense,
                "dense_step_frac": (algb["alg_bytes"] / (step_dense / 1e3) / 1e9 / peak) if step_dense else None,
            }
            res["pruning"] = {
                "legal_candidates_dense_step": algb["legal"],
                "survivors": counters.get("survivors"),
                "pruned_fraction": 1.0 - counters.get("survivors", 0) / max(1, counters.get("legal", 1)),
                "rows_read": counters.get("rows_read"), "rows_skip_pre": counters.get("rows_skip_pre"),
                "rows_skip_post": counters.get("rows_skip_post"), "overflow": counters.get("overflow"),
            }

    if not args.no_e2e:
        # ---- end to end through the public API: pinned host logits in, host results out ----
        hl = [x.cpu().pin_memory() for x in logits]
        h2d = sum(x.numel() * x.element_size() for x in hl)
        d2h = B * BW * ND * 4 + B * BW * 8 + B * BW * 4 + B * 4
        ke = max(1, min(args.steps, 5))

        def e2e_pass():
            for t in range(ND):
                bs.step(hl[t])
            bs.finalize(on_device=False)

        e2e_pass()
        torch.cuda.synchronize()
        barrier(world, dev)
        t0 = time.perf_counter()
        for _ in range(ke):
            e2e_pass()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, dev)
        res["e2e"] = {"value": cand * world * ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3 / ke, "steps": ke,
                      "path": "BeamSearch.step(pinned host tensor) -> H2D on the step stream -> xgr_beam_step; xgr_beam_finalize(host outputs)"}
        del hl

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        res["cpu_baseline"] = cpu_baseline(args, cfg, items, logits)
    bs.close()
    return res


def cpu_baseline(args, cfg, items, logits):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload."""
    from oracle import xbeam_oracle as O
    t0 = time.perf_counter()
    voc = O.Vocabulary(items, cfg["vocab"], cfg["nd"])
    vb = time.perf_counter() - t0
    nthr = cores()
    host = {}

    def lf(r, t):
        if (r, t) not in host:
            host[(r, t)] = logits[t][r].float().cpu().numpy()   # bf16 widened exactly
        return host[(r, t)]

    # estimate with one request, then size the sample to ~args.cpu_budget seconds
    c1, s1 = oracle_sample(voc, cfg, lf, 1, 1)
    n_req = max(1, min(cfg["batch"], int(args.cpu_budget / max(s1, 1e-3) * min(nthr, 8) * 0.8)))
    n_req = max(n_req, min(nthr, cfg["batch"]))
    c, s = oracle_sample(voc, cfg, lf, n_req, nthr)
    return {"value": c / s, "unit": UNIT, "cores": nthr, "kind": "oracle",
            "sample": f"{n_req} of {cfg['batch']} requests of {cfg['name']}, full ND={cfg['nd']} steps each, "
                      f"fp64 numpy oracle, thread pool over requests; {s:.1f} s (oracle trie build {vb:.1f} s excluded)",
            "seconds": s}


def run_reference(args, cfg):
    """Reference arm: the CPU oracle timed on the host cores, each step a bounded sample."""
    from oracle import xbeam_oracle as O
    from synth import make_items, make_logits
    V, ND, BW = cfg["vocab"], cfg["nd"], cfg["beam_width"]
    items = make_items(cfg["n_items"], V, ND, cfg["trie_key"])
    voc = O.Vocabulary(items, V, ND)
    del items
    nthr = cores()
    n_req = max(1, min(nthr, cfg["batch"]))
    times = []
    for k in range(args.warmup + args.steps):
        def lf(r, t, k=k):
            return make_logits((1 if t == 0 else BW, V), 104729 * (k + 1) + 31 * r + t, args.sigma)
        c, s = oracle_sample(voc, cfg, lf, n_req, nthr)
        if k >= args.warmup:
            times.append(s)
    tot = sum(times)
    value = candidates_per_pass(cfg, n_req) * args.steps / tot
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded)",
        "config": {"workload": cfg["name"], "batch_per_gpu": cfg["batch"], "beam_width": BW,
                   "vocab": V, "nd": ND, "n_items": cfg["n_items"], "sigma": args.sigma},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthr, "kind": "oracle",
                         "sample": f"each step: {n_req} of {cfg['batch']} requests, full ND steps, "
                                   "fp64 numpy oracle on a thread pool"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--sigma", type=float, default=2.0)
    ap.add_argument("--logits", choices=["f32", "bf16"], default="f32",
                    help="logits element type (bf16: SURVEY 8(f) NEXT f1); the path computes in f32")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager passes only (no CUDA-graph replay)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="timed loop only (for ncu launch lists)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and not args.profile:
        args.warmup = 3
    from synth import config
    cfg = config(args.config)
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, cfg)), flush=True)
        return 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, cfg, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
