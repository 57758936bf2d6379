"""Codebook shard emulated on one GPU: G rank contexts, the two all-gathers done as
plain concatenations in rank order (the layout an NCCL all-gather produces). Test helper."""
import torch


class ShardEmulator:
    """G ranks' contexts on one device; the two all-gathers are plain concatenations (the same
    rank-major layout an NCCL all-gather produces)."""

    def __init__(self, xgr, vocab, nd, bw, batch, G, items, flags=0):
        self.G, self.vocab = G, vocab
        self.ranks = [xgr.BeamSearch(vocab, nd, bw, batch, flags=flags, nranks=G, rank=r) for r in range(G)]
        for bs in self.ranks:
            bs.mask_build(items)
        self.bw = bw

    def step(self, logits_full):
        vl = self.vocab // self.G
        sl = [logits_full[:, :, r * vl:(r + 1) * vl] for r in range(self.G)]
        stats = [bs.shard_stats(x) for bs, x in zip(self.ranks, sl)]
        gstats = torch.stack([s.clone() for s in stats]).contiguous()
        outs = [bs.shard_select(gstats) for bs in self.ranks]
        grecs = torch.stack([r.clone() for r, _ in outs]).contiguous()
        # two exchanges per step (stats, records): the merge counts each rank's nonzero records
        for bs in self.ranks:
            bs.shard_merge(grecs, None)
        for bs in self.ranks:
            bs.batch = logits_full.shape[0]
        torch.cuda.synchronize()
