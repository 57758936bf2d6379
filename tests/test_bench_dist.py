"""Multi-rank host logic of bench.py with the gloo backend on CPU (world size 2): per-rank work
plans are disjoint (weak scaling over requests), the max-over-ranks reduction, barriers, and the
reference arm's rank-0-only rule. No GPU needed."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import bench
    from synth import config
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = config("C3")
    plan = bench.rank_plan(cfg, rank, world)
    seeds = bench.step_seeds(plan, cfg["nd"])
    t = bench.max_over_ranks(float(10 + rank), world, device=torch.device("cpu"))
    bench.barrier(world)
    # C4 request split and C5 codebook shard plans, and the shard exchange's rank-major layout
    c4, c5 = config("C4"), config("C5")
    p4 = bench.rank_plan(c4, rank, world, bench.split_mode(c4))
    p5 = bench.rank_plan(c5, rank, world, bench.split_mode(c5))
    L = p5["shards"][1] - p5["shards"][0]
    local = torch.stack([torch.full((3, 2), float(g)) for g in range(*p5["shards"])])   # [L][...]
    gathered = bench.shard_all_gather(local, world)
    q.put((rank, plan, seeds, t, bench.candidates_per_pass(cfg, plan["batch"]), p4, p5, L,
           gathered[:, 0, 0].tolist(), bench.pass_candidates(c4, p4, world), bench.pass_candidates(c5, p5, world)))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, p0, s0, t0, c0, a4, a5, L0, g0, n4, n5), (r1, p1, s1, t1, c1, b4, b5, L1, g1, m4, m5) = res
    assert t0 == t1 == 11.0                     # max over ranks
    assert set(s0).isdisjoint(s1)               # distinct logit seeds per rank
    assert p0["requests"][1] == p1["requests"][0]   # contiguous, disjoint request ranges
    assert p0["batch"] == p1["batch"] == 256 and c0 == c1 == 256 * (1 + 256 * 2) * 8192
    # C4 strong split: 256 + 256 of the 512 requests, whole-job candidates counted once
    assert a4["mode"] == "strong" and a4["requests"] == (0, 256) and b4["requests"] == (256, 512)
    assert n4 == m4 == 512 * (1 + 512 * 3) * 16384
    # C5 codebook shard: 4 + 4 of the 8 shards; every rank holds the whole batch; the all-gather
    # returns the 8 shards in global order on both ranks
    assert a5["shards"] == (0, 4) and b5["shards"] == (4, 8) and L0 == L1 == 4
    assert g0 == g1 == [float(g) for g in range(8)]
    assert n5 == m5 == 128 * (1 + 512 * 2) * 65536


def test_reference_arm_nonzero_rank_exits(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--impl", "reference"]) == 0


def test_traffic_files_keyed_by_config_partition_dtype_sigma():
    """Each bench line reads the ncu capture of its own config, partition, dtype and sigma, and
    reports null when none is committed (never another config's file)."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.traffic_key("C3", "f32", 2.0) == "ncu_k_stream_C3_f32_traffic.json"
    assert bench.traffic_key("C3", "bf16", 4.0) == "ncu_k_stream_C3_bf16_s4_traffic.json"
    assert bench.traffic_key("C5", "f32", 2.0, "weak") == "ncu_k_stream_C5_weak_f32_traffic.json"
    assert bench.committed_traffic("C9", "f32", 2.0) is None
    for cfg, dt, sg, sp in (("C3", "f32", 2.0, ""), ("C5", "f32", 2.0, "weak")):
        tr = bench.committed_traffic(cfg, dt, sg, sp)
        assert tr is not None and tr["dram_bytes_per_launch"] > 0, (cfg, sp)
        assert bench.traffic_key(cfg, dt, sg, sp) in tr["file"]
