#!/usr/bin/env python
"""Benchmark of the xBeam decode-step selection path (BASELINE.json metric) on B200.

One bench "step" = one pass of the whole hot path over one batch: the ND beam-search steps of the
config through the C ABI, plus finalize (device outputs). Inputs (seeded synthetic logits, several
GiB per pass) are resident in HBM and larger than L2, so L2 needs no flush between iterations.

  python bench.py [--gpus N --steps K --warmup W]        our CUDA path, C3 (one JSON line, rank 0)
  python bench.py --config C4 [...]                       request split (strong scaling)
  python bench.py --config C5 [...]                       codebook shard over 8 virtual ranks
  python bench.py --impl reference [...]                  the CPU oracle (reference arm, rank 0)

How the work partitions over N processes (one per GPU):
  weak   (C1-C3, default): every rank runs its own full batch of the config (distinct logit seeds,
         the same catalogue), no data-path collective; value = all ranks' candidates / max time.
  strong (C4): the config's request batch is split, rank r takes requests [r B/N, (r+1) B/N);
         logits are generated per request, so every request's bytes and result are the same for
         any N; no data-path collective.
  shard  (C5): the codebook is split into G = 8 column shards of V/8 (8192) columns ("virtual
         ranks", one xgr ctx each); process p hosts shards [p G/N, (p+1) G/N). Per step two
         collectives: an all-gather of the per-row (m, Z) stats and one of the local top-BW records
         (torch.distributed NCCL all_gather_into_tensor over NVLink; a local stack at N = 1).
         Results are identical for every N (always G = 8 shards).
Time = max over ranks of the CUDA-event time of the K timed passes.
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

UNIT = "candidates/s"
SHARDS = 8          # codebook shards of the shard mode (C5: 65536 / 8 = 8192 columns each)


def metric_name(cfg: dict) -> str:
    return (f"beam-step candidates/sec ({cfg['name']}: batch {cfg['batch']}, BW {cfg['beam_width']}, "
            f"V {cfg['vocab']}, ND {cfg['nd']}; raw (b, v) pool per step)")


# ---- host-side multi-rank logic (covered by tests/test_bench_dist.py with gloo) -------------------
def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def split_mode(cfg: dict, override: str = "auto") -> str:
    if override != "auto":
        return override
    return {"C4": "strong", "C5": "shard"}.get(cfg["name"], "weak")


def rank_plan(cfg: dict, rank: int, world: int, mode: str = "weak") -> dict:
    """The requests (and, in shard mode, the codebook shards) this rank processes."""
    B = cfg["batch"]
    if mode == "weak":
        return {"mode": mode, "batch": B, "seed_base": 7919 * (rank + 1),
                "requests": (rank * B, (rank + 1) * B), "shards": None}
    if mode == "strong":
        if B % world:
            raise ValueError(f"request split: batch {B} not divisible by {world} ranks")
        b = B // world
        return {"mode": mode, "batch": b, "seed_base": None, "requests": (rank * b, (rank + 1) * b),
                "shards": None}
    if mode == "shard":
        if SHARDS % world:
            raise ValueError(f"codebook shard: {SHARDS} shards not divisible by {world} ranks")
        L = SHARDS // world
        return {"mode": mode, "batch": B, "seed_base": None, "requests": (0, B),
                "shards": (rank * L, (rank + 1) * L)}
    raise ValueError(mode)


def step_seeds(plan: dict, nd: int):
    return [plan["seed_base"] * 16 + t for t in range(nd)]


def candidates_per_pass(cfg: dict, batch: int) -> int:
    """Raw (b, v) candidate pool of one ND-step pass: 1 root row at step 1, BW rows after."""
    return batch * (1 + cfg["beam_width"] * (cfg["nd"] - 1)) * cfg["vocab"]


def pass_candidates(cfg: dict, plan: dict, world: int) -> int:
    """Candidates of one pass of the WHOLE job (all ranks)."""
    if plan["mode"] == "weak":
        return candidates_per_pass(cfg, plan["batch"]) * world
    return candidates_per_pass(cfg, cfg["batch"])   # strong / shard: the config's batch, split


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


def shard_all_gather(local, world: int):
    """[L][...] per process -> [world * L][...] in global shard order (rank-major), the layout
    xgr_shard_select / xgr_shard_merge take. A stack at world 1."""
    import torch
    if world == 1:
        return local.contiguous()
    import torch.distributed as dist
    local = local.contiguous()
    out = torch.empty((world * local.shape[0], *local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local)
    return out


def xgr_env() -> dict:
    """Every XGR_* knob in effect (recorded in the JSON config)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("XGR_")}


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


def traffic_key(cfg_name: str, dtype: str, sigma: float, split: str = "") -> str:
    """split: "" for the config's default partition, else its name (e.g. C5 with --split weak)."""
    s = "" if sigma == 2.0 else f"_s{sigma:g}"
    sp = f"_{split}" if split else ""
    return f"ncu_k_stream_{cfg_name}{sp}_{dtype}{s}_traffic.json"


def committed_traffic(cfg_name: str, dtype: str = "f32", sigma: float = 2.0, split: str = ""):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary of
    THIS config / partition / dtype / sigma
    (profiles/ncu_k_stream_<cfg>[_<split>]_<dtype>[_s<sigma>]_traffic.json), or None when no
    capture of it is committed."""
    p = os.path.join(ROOT, "profiles", traffic_key(cfg_name, dtype, sigma, split))
    try:
        with open(p) as f:
            d = json.load(f)
        d.setdefault("file", os.path.relpath(p, ROOT))
        return d
    except OSError:
        return None


# ---- CPU baselines (cpu_baseline and the reference arm) ---------------------------------------------
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


def paper_heap_sample(voc, cfg, logits_fn, n_req: int, threads: int):
    """The paper's own selection (PAPER.md L385 min-heap with early termination, fp32, C, one
    pthread per request slice) on the same logits: oracle/paper_heap_c. Returns (cands, s, stats)
    or None if the C library is not built."""
    try:
        from oracle import paper_heap_c
    except (ImportError, OSError):
        return None
    lg = [[logits_fn(r, t) for t in range(cfg["nd"])] for r in range(n_req)]
    runner = paper_heap_c.PaperHeap(voc.keys, cfg["vocab"], cfg["nd"])
    t0 = time.perf_counter()
    stats = runner.run(lg, cfg["beam_width"], threads)
    dt = time.perf_counter() - t0
    return candidates_per_pass(cfg, n_req), dt, stats


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---- our CUDA path -----------------------------------------------------------------------------
def make_inputs(args, cfg, plan, dev, rank):
    """Per-step device logits of this rank: a list over steps of [batch][rows][cols] tensors."""
    import torch

    from synth import make_logits_rows_torch, make_logits_torch
    B, BW, V, ND = plan["batch"], cfg["beam_width"], cfg["vocab"], cfg["nd"]
    rows = [1 if t == 0 else BW for t in range(ND)]
    if plan["mode"] == "weak":
        seeds = step_seeds(plan, ND)
        logits = [make_logits_torch((B, rows[t], V), seeds[t], args.sigma, device=dev) for t in range(ND)]
    else:
        reqs = list(range(*plan["requests"]))
        if plan["mode"] == "shard":
            vl = V // SHARDS
            c0, c1 = plan["shards"][0] * vl, plan["shards"][1] * vl
        else:
            c0, c1 = 0, V
        logits = [make_logits_rows_torch(reqs, rows[t], V, t, cfg["trie_key"], args.sigma, col0=c0,
                                         ncols=c1 - c0, device=dev) for t in range(ND)]
    if args.logits == "bf16":   # NEXT f1: the same N(0, sigma^2) draws rounded to bf16
        logits = [x.to(torch.bfloat16) for x in logits]
    return logits


class Runner:
    """One rank's contexts and its pass (ND steps + finalize) in the plan's mode."""

    def __init__(self, args, cfg, plan, dev, world, items, flags):
        import paper_2512_11529_b200 as xgr
        self.cfg, self.plan, self.world, self.dev = cfg, plan, world, dev
        B, BW, V, ND = plan["batch"], cfg["beam_width"], cfg["vocab"], cfg["nd"]
        tr = int(os.environ.get("XGR_THETA_ROWS", "0"))
        if plan["mode"] == "shard":
            self.ctxs = [xgr.BeamSearch(V, ND, BW, B, device=dev.index, flags=flags, theta_rows=tr,
                                        nranks=SHARDS, rank=g) for g in range(*plan["shards"])]
        else:
            self.ctxs = [xgr.BeamSearch(V, ND, BW, B, device=dev.index, flags=flags, theta_rows=tr)]
        for bs in self.ctxs:
            bs.mask_build(items)
        self.bs = self.ctxs[0]
        self.stats_ev = None

    def views(self, logits_t):
        """Per local ctx, its [batch][rows][cols] view of this rank's logits of one step."""
        if self.plan["mode"] != "shard":
            return [logits_t]
        vl = self.cfg["vocab"] // SHARDS
        return [logits_t[:, :, j * vl:(j + 1) * vl] for j in range(len(self.ctxs))]

    def one_pass(self, logits, evs=None, stats_evs=None):
        import torch
        stream = torch.cuda.current_stream()
        nd = self.cfg["nd"]
        if evs:
            evs[0].record(stream)
        for t in range(nd):
            if self.plan["mode"] != "shard":
                self.bs.step(logits[t])
            else:
                vs = self.views(logits[t])
                if stats_evs:
                    stats_evs[t][0].record(stream)
                st = [bs.shard_stats(x) for bs, x in zip(self.ctxs, vs)]
                if stats_evs:
                    stats_evs[t][1].record(stream)
                gstats = shard_all_gather(torch.stack(st), self.world)
                recs = [bs.shard_select(gstats)[0] for bs in self.ctxs]
                grecs = shard_all_gather(torch.stack(recs), self.world)
                for bs in self.ctxs:
                    bs.shard_merge(grecs, None)
            if evs:
                evs[t + 1].record(stream)
        # finalize (a6) is fused into the last step's commit: the item tuples, ranks and scores
        # are in device memory now (bs.outputs_view()); this call only ends the batch
        for bs in self.ctxs:
            bs.finalize_in_place()
        if evs:
            evs[nd + 1].record(stream)

    def launch_count(self):
        return sum(bs.launch_count() for bs in self.ctxs)

    def close(self):
        for bs in self.ctxs:
            bs.close()


def run_ours(args, cfg, rank, world, local_rank):
    import torch

    import paper_2512_11529_b200 as xgr
    from synth import make_config_items

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    mode = split_mode(cfg, args.split)
    plan = rank_plan(cfg, rank, world, mode)
    B, BW, V, ND = plan["batch"], cfg["beam_width"], cfg["vocab"], cfg["nd"]
    t0 = time.perf_counter()
    items = make_config_items(cfg)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    run = Runner(args, cfg, plan, dev, world, items, xgr.XGR_CFG_TIMING | (0x10 if args.paper_heap else 0))
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    info = run.bs.info()
    logits = make_inputs(args, cfg, plan, dev, rank)
    in_bytes = sum(x.numel() * x.element_size() for x in logits)
    stream = torch.cuda.current_stream()
    shard = mode == "shard"

    for _ in range(args.warmup):
        run.one_pass(logits)
    torch.cuda.synchronize()
    run.bs.kernel_times()                      # drain warm-up records
    launches0 = run.launch_count()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(ND + 2)] for _ in range(args.steps)]
    sevs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(ND)]
            for _ in range(args.steps)] if shard else [None] * args.steps
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    barrier(world, dev)
    torch.cuda.synchronize()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for k in range(args.steps):
        run.one_pass(logits, evs[k], sevs[k])
    e_end.record(stream)
    torch.cuda.synchronize()
    barrier(world, dev)
    # the dense-step kernel's library-side CUDA-event times of the eager passes (read before the
    # graph capture, which records the same events as graph nodes)
    kms, kstep = run.bs.kernel_times()
    launches = run.launch_count() - launches0   # kernels per timed run (a graph replay runs the same ones)
    # the same pass captured once as a CUDA graph and replayed K times (xSchedule's
    # graph dispatch submits a step's device work at once). This removes the host's per-launch
    # work from the critical path; when capture works it is the headline, eager is kept beside it.
    # The shard mode's collectives stay eager.
    graph = None
    if not args.profile and not args.no_graph and not shard:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run.one_pass(logits)
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
    if shard:   # the shard stats kernels of the dense step (every local shard, one event pair)
        dense_t = 1
        main_ms = [sevs[k][dense_t][0].elapsed_time(sevs[k][dense_t][1]) for k in range(args.steps)]
        dense_steps = [dense_t + 1]
    else:
        # the dense step the roofline is about: the one whose streaming kernel takes longest (a
        # root step wider than 8192 columns also takes the dense route, with one row per request)
        by_step = {}
        for m, st in zip(kms, kstep):
            by_step.setdefault(int(st), []).append(float(m))
        main_step = max(by_step, key=lambda st: sum(by_step[st]) / len(by_step[st])) if by_step else None
        main_ms = by_step.get(main_step, [])
        dense_steps = [main_step] if main_step else []

    cand = pass_candidates(cfg, plan, world)
    value = cand * args.steps / (total_ms_max / 1e3)
    dtype = args.logits
    res = {
        "metric": metric_name(cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
        "p50_ms": statistics.median(per_iter), "p99_ms": sorted(per_iter)[min(len(per_iter) - 1, int(0.99 * len(per_iter)))],
        "higher_is_better": True, "scaling": "weak" if mode == "weak" else "strong", "vs_baseline": None,
        "dtype": "f32",
        "data": f"synthetic (seeded: Feistel-permuted uniform item tuples, N(0, sigma^2) {dtype} logits)",
        "config": {"workload": cfg["name"], "split": mode, "batch": cfg["batch"], "batch_per_gpu": B,
                   "beam_width": BW, "vocab": V, "nd": ND, "logits": dtype,
                   "n_items": cfg["n_items"], "n_items_dedup": int(info["n_items"]), "sigma": args.sigma,
                   "parallelism": {"weak": f"request-split x{world} (a full batch per GPU)",
                                   "strong": f"request-split x{world} ({B} of {cfg['batch']} requests per GPU)",
                                   "shard": f"codebook shard: {SHARDS} shards of {V // SHARDS} columns over {world} GPU(s), "
                                            f"2 all-gathers per step"}[mode],
                   "l2": f"inputs larger than L2 ({in_bytes / 2**30:.2f} GiB per pass per GPU), no flush",
                   "items": "clustered (Zipf per level)" if cfg.get("clustered") else "uniform",
                   "env": xgr_env(),
                   "selection": ("paper heap (per-beam sorted Top-K lists + sequential min-heap, PAPER.md L385; "
                                 "XGR_CFG_PAPER_HEAP baseline)" if args.paper_heap else "theta-pruned streaming")},
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
        res["value"] = cand * args.steps / (graph["total_ms"] / 1e3)
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

    if not args.no_e2e:
        res["e2e"] = e2e(args, cfg, plan, run, logits, world, dev, cand)
    run.close()   # frees the timed contexts (the shard mode's accounting builds its own)

    if not args.profile and (rank == 0 or shard):   # shard accounting exchanges stats: every rank
        res.update(account(args, cfg, plan, dev, items, logits, main_ms, dense_steps, per_step, world))

    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        res["cpu_baseline"] = cpu_baseline(args, cfg, items, logits, plan)
    return res


def account(args, cfg, plan, dev, items, logits, main_ms, dense_steps, per_step, world):
    """Algorithmic bytes, counters and the roofline of the dominant kernel, from an identical
    untimed pass on separate contexts with device counters on (this rank's share of the work)."""
    import torch

    import paper_2512_11529_b200 as xgr
    ND = cfg["nd"]
    shard = plan["mode"] == "shard"
    acc = Runner(args, cfg, plan, dev, world, items, xgr.XGR_CFG_COUNTERS | (0x10 if args.paper_heap else 0))
    out = {}
    algb = None
    counters = {}
    for bs in acc.ctxs:
        bs.counters()
    for t in range(ND):
        if shard:
            st = [bs.shard_stats(x) for bs, x in zip(acc.ctxs, acc.views(logits[t]))]
            gstats = shard_all_gather(torch.stack(st), world)
            recs = [bs.shard_select(gstats)[0] for bs in acc.ctxs]
            grecs = shard_all_gather(torch.stack(recs), world)
            for bs in acc.ctxs:
                bs.shard_merge(grecs, None)
        else:
            acc.bs.step(logits[t])
        cs = [bs.counters() for bs in acc.ctxs]
        if t + 1 in dense_steps and algb is None:
            # every local shard ctx counted together (their stats kernels are timed together)
            accs = [bs.account() for bs in acc.ctxs]
            algb = {k: sum(a[k] for a in accs) for k in accs[0]}
            counters = {k: sum(c[k] for c in cs) for k in cs[0]}
    for bs in acc.ctxs:
        bs.finalize(on_device=True)
    acc.close()
    peaks, src = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    if main_ms and algb:
        mean_ms = sum(main_ms) / len(main_ms)
        achieved = algb["alg_bytes"] / (mean_ms / 1e3) / 1e9
        step_dense = statistics.median(per_step[dense_steps[0] - 1]) if dense_steps else None
        tr = committed_traffic(cfg["name"], args.logits, args.sigma,
                               "" if args.split in ("auto", split_mode(cfg)) else args.split)
        if args.paper_heap:
            tr = None   # no ncu capture of the baseline's kernels is committed
            kname = "k_ph_rows (the paper's per-beam Top-K lists; baseline, XGR_CFG_PAPER_HEAP)"
        elif shard:
            kname = "k_stream stats mode (codebook shard: per-row (m, Z) over each shard's columns; every local shard)"
        elif cfg["vocab"] >= 32768 and args.logits == "f32":
            kname = "k_stream2 (dense step, one CTA per row in two passes: online softmax, then emission from L2)"
        elif cfg["vocab"] > 8192:
            kname = "k_stream, 2-CTA column-split clusters (dense step)"
        else:
            kname = "k_stream (dense step: TMA row stream, masked log-softmax, score add, pruned emit)"
        out["roofline"] = {
            "bound": "hbm", "kernel": kname,
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs)" if src == "measured" else "fallback 6.65 TB/s",
            # the shard line's stats pass is SHARDS launches (one per local shard ctx); the capture is one of them
            "traffic": ((tr or {}).get("dram_bytes_per_launch") or 0) * (SHARDS if shard else 1) or None,
            "traffic_source": (tr or {}).get("source"),
            "traffic_file": (tr or {}).get("file"),
            "alg_bytes_per_launch": algb["alg_bytes"], "full_bytes_per_launch": algb["full_bytes"],
            "kernel_ms_mean": mean_ms, "launches_timed": len(main_ms),
            "dense_step_ms_p50": step_dense,
            "dense_step_frac": (algb["alg_bytes"] / (step_dense / 1e3) / 1e9 / peak) if step_dense else None,
        }
        rr = counters.get("rows_read")
        if rr:
            # bytes of the rows the kernel actually read (rows not skipped before reading: the
            # seed's theta is weaker than theta*, so this exceeds the algorithmic bytes at sigma 4)
            esz = 2 if args.logits == "bf16" else 4
            vl = cfg["vocab"] // (SHARDS if shard else 1)
            rbytes = rr * (vl * esz + vl // 8 + 16)
            out["roofline"]["rows_read_bytes_per_launch"] = rbytes
            out["roofline"]["frac_rows_read"] = rbytes / (mean_ms / 1e3) / 1e9 / peak
        if shard:
            out["roofline"]["note"] = ("the shard select phase re-reads the rows after the stats all-gather "
                                       "(the global lse is needed before any emission), so the dense step "
                                       "moves ~2x the algorithmic bytes")
        out["pruning"] = {
            "legal_candidates_dense_step": algb["legal"],
            "survivors": counters.get("survivors"),
            "pruned_fraction": 1.0 - counters.get("survivors", 0) / max(1, counters.get("legal", 1)),
            "rows_read": counters.get("rows_read"), "rows_skip_pre": counters.get("rows_skip_pre"),
            "rows_skip_post": counters.get("rows_skip_post"), "overflow": counters.get("overflow"),
        }
    return out


def e2e(args, cfg, plan, run, logits, world, dev, cand):
    """End to end through the public API: pinned host logits in (H2D on the step stream inside
    BeamSearch.step), host results out (xgr_beam_finalize with host outputs)."""
    import torch
    in_bytes = sum(x.numel() * x.element_size() for x in logits)
    if plan["mode"] == "shard" or in_bytes * world > 48 * 2**30:
        why = ("shard mode: the host would stage every shard's columns (not a serving layout)"
               if plan["mode"] == "shard" else
               f"{in_bytes * world / 2**30:.0f} GiB of pinned host logits per pass across ranks")
        return {"unavailable": why}
    B, BW, ND = plan["batch"], cfg["beam_width"], cfg["nd"]
    bs = run.bs
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
    del hl
    return {"value": cand * ke / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3 / ke, "steps": ke,
            "path": "BeamSearch.step(pinned host tensor) -> xgr_beam_step_host (H2D on the step stream inside the C ABI); "
                    "xgr_beam_finalize(host outputs)"}


def cpu_baseline(args, cfg, items, logits, plan):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload; and
    the paper's own heap selection (fp32, C, threaded) on the same sample."""
    from oracle import xbeam_oracle as O
    t0 = time.perf_counter()
    voc = O.Vocabulary(items, cfg["vocab"], cfg["nd"])
    vb = time.perf_counter() - t0
    nthr = cores()
    host = {}
    shard_cols = plan["mode"] == "shard" and plan["shards"] != (0, SHARDS)
    if shard_cols:
        return {"unavailable": "this rank holds only some codebook shards"}

    def lf(r, t):
        if (r, t) not in host:
            host[(r, t)] = logits[t][r].float().cpu().numpy()   # bf16 widened exactly
        return host[(r, t)]

    # estimate with one request, then size the sample to ~args.cpu_budget seconds
    c1, s1 = oracle_sample(voc, cfg, lf, 1, 1)
    n_req = max(1, min(plan["batch"], int(args.cpu_budget / max(s1, 1e-3) * min(nthr, 8) * 0.8)))
    n_req = max(n_req, min(nthr, plan["batch"]))
    c, s = oracle_sample(voc, cfg, lf, n_req, nthr)
    out = {"value": c / s, "unit": UNIT, "cores": nthr, "kind": "oracle",
           "sample": f"{n_req} of {cfg['batch']} requests of {cfg['name']}, full ND={cfg['nd']} steps each, "
                     f"fp64 numpy oracle, thread pool over requests; {s:.1f} s (oracle trie build {vb:.1f} s excluded)",
           "seconds": s}
    ph = paper_heap_sample(voc, cfg, lf, n_req, nthr)
    if ph is not None:
        pc, ps, pst = ph
        out["paper_heap"] = {"value": pc / ps, "unit": UNIT, "cores": nthr, "kind": "paper_heap",
                             "sample": f"the same {n_req} requests: PAPER.md L385 heap selection with early termination, "
                                       "fp32, C (oracle/paper_heap.c), one pthread per request slice",
                             "seconds": ps, "heap_visits_fraction": pst.get("visit_frac")}
    return out


def run_reference(args, cfg):
    """Reference arm: the CPU oracle timed on the host cores, each step a bounded sample."""
    from oracle import xbeam_oracle as O
    from synth import make_config_items, make_logits
    V, ND, BW = cfg["vocab"], cfg["nd"], cfg["beam_width"]
    items = make_config_items(cfg)
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
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": UNIT, "n_gpus": 1,
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
    ap.add_argument("--split", choices=["auto", "weak", "strong", "shard"], default="auto",
                    help="how N GPUs partition the work (auto: C4 strong, C5 shard, else weak)")
    ap.add_argument("--sigma", type=float, default=2.0)
    ap.add_argument("--logits", choices=["f32", "bf16"], default="f32",
                    help="logits element type (bf16: SURVEY 8(f) NEXT f1); the path computes in f32")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager passes only (no CUDA-graph replay)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="timed loop only (for ncu launch lists)")
    ap.add_argument("--paper-heap", action="store_true",
                    help="baseline: dense steps select with the paper's heap procedure (XGR_CFG_PAPER_HEAP)")
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
        # NCCL's communicator lines (rank count, transport) on stderr, so a multi-GPU run's log
        # shows the communicator the timings came from; stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist.barrier(device_ids=[local_rank])   # creates the communicator now (its INIT lines)
        print(f"[bench] rank {rank} of {world}: NCCL communicator on cuda:{local_rank}", file=sys.stderr, flush=True)
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
