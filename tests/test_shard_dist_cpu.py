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
        self.calls.append(("merge", grecs[:, 0, 0].tolist(), gn))


def _worker(rank, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    # the real class from the package (the library loads without a GPU; no CUDA call is made)
    from paper_2512_11529_b200 import ShardedBeamSearch
    fake = FakeShardCtx(rank)
    sb = ShardedBeamSearch(fake)
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
        assert calls[2] == ("merge", [10, 11], None)       # rank-major records; no count exchange
        assert len(calls) == 3
