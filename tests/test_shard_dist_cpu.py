"""Host logic of the codebook-shard exchange (ShardedBeamSearch) over a real gloo process group on
CPU, world size 2: the all-gathers are rank-major and the phases run in order. The CUDA phases are
replaced by a recording stand-in (no GPU here); the GPU path itself is covered by the emulated
shard parity tests."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class FakeShardCtx:
    nranks = 2

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def shard_stats(self, logits, stream=None):
        self.calls.append("stats")
        return torch.full((2, 3, 2), float(self.rank))

    def shard_select(self, gstats, stream=None):
        self.calls.append(("select", gstats[:, 0, 0, 0].tolist()))
        return torch.full((2, 3), 10 + self.rank, dtype=torch.int64), torch.full((2,), self.rank, dtype=torch.int32)

    def shard_merge(self, grecs, gn, stream=None):
        self.calls.append(("merge", grecs[:, 0, 0].tolist(), gn[:, 0].tolist()))


def _worker(rank, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    import importlib.util
    spec = importlib.util.spec_from_file_location("xbind", os.path.join(ROOT, "paper_2512_11529_b200", "binding.py"))
    # the binding loads the CUDA library at import; only ShardedBeamSearch is needed here
    src = open(os.path.join(ROOT, "paper_2512_11529_b200", "binding.py")).read()
    cls_src = src[src.index("class ShardedBeamSearch"):]
    ns = {}
    exec(cls_src, ns)
    fake = FakeShardCtx(rank)
    sb = ns["ShardedBeamSearch"](fake)
    sb.step(torch.zeros(2, 3, 4))
    q.put((rank, fake.calls))
    dist.destroy_process_group()


def test_shard_exchange_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        calls = res[r]
        assert calls[0] == "stats"
        assert calls[1] == ("select", [0.0, 1.0])          # rank-major gathered stats
        assert calls[2] == ("merge", [10, 11], [0, 1])     # rank-major records and counts
