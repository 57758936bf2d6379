"""The seeded generators (synth/) are deterministic and produce what DESIGN.md's recipe says."""
import numpy as np

from synth import config, feistel_permute, make_items, make_logits, prefix_keyed_row


def test_feistel_is_a_permutation():
    for bits in (2, 3, 7, 12, 13):
        y = feistel_permute(np.arange(1 << bits, dtype=np.uint64), bits, 1234)
        assert y.max() < (1 << bits)
        assert np.unique(y).shape[0] == 1 << bits


def test_items_distinct_deterministic_and_in_range():
    c = config("C1")
    a = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    b = make_items(c["n_items"], c["vocab"], c["nd"], c["trie_key"])
    assert a.dtype == np.int32 and a.shape == (200, 3)
    assert np.array_equal(a, b)
    assert len(set(map(tuple, a.tolist()))) == 200
    assert a.min() >= 0 and a.max() < 16
    d = make_items(1000, 256, 3, 77, dup_frac=0.01)
    assert d.shape[0] == 1010 and len(set(map(tuple, d.tolist()))) == 1000


def test_logits_seeded():
    a = make_logits((3, 5), 11, 2.0)
    assert a.dtype == np.float32 and np.array_equal(a, make_logits((3, 5), 11, 2.0))
    assert not np.array_equal(a, make_logits((3, 5), 12, 2.0))


def test_prefix_keyed_rows_exact_grid():
    r = prefix_keyed_row(5, 0, (1, 2), 64)
    assert r.dtype == np.float32
    assert np.all(r * 2 ** 15 == np.round(r * 2 ** 15))
    assert np.array_equal(r, prefix_keyed_row(5, 0, (1, 2), 64))
    assert not np.array_equal(r, prefix_keyed_row(5, 0, (1, 3), 64))


def test_clustered_items_distinct_deterministic_skewed():
    from synth import make_items_clustered
    a = make_items_clustered(200_000, 1024, 3, 5)
    b = make_items_clustered(200_000, 1024, 3, 5)
    assert a.shape == (200_000, 3) and a.dtype == np.int32
    assert np.array_equal(a, b)
    assert a.min() >= 0 and a.max() < 1024
    k = (a[:, 0].astype(np.int64) << 20) | (a[:, 1].astype(np.int64) << 10) | a[:, 2]
    assert np.unique(k).shape[0] == 200_000
    # skew: the most popular first token holds far more than a uniform 1/1024 share
    _, cnt = np.unique(a[:, 0], return_counts=True)
    assert cnt.max() > 20 * 200_000 / 1024
