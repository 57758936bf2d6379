"""Pins of the KV-reorder oracle (oracle/kv_reorder.py) against SPEC.md's worked
examples and the gather-oracle equivalence property: no GPU needed."""
import itertools

import numpy as np
import pytest

from oracle import kv_reorder as K


def _rows(labels):
    return np.array([[ord(c)] for c in labels], dtype=np.int64)


def test_spec_plan_examples():
    s, perm, d = K.plan_reorder([0, 1, 2, 3])           # S:L75 identity
    assert list(d) == [0, 0, 0, 0] and list(perm) == [0, 1, 2, 3]
    s, perm, d = K.plan_reorder([1, 2, 2, 3])
    assert list(d) == [1, 1, 0, 0]
    s, perm, d = K.plan_reorder([2, 0, 1, 0])           # S:L77 stable sort + permutation
    assert list(s) == [0, 0, 1, 2] and list(perm) == [1, 3, 2, 0]
    with pytest.raises(K.ReorderError):
        K.plan_reorder([0, 4, 1, 2])                    # S:L73 out of range


def test_spec_apply_examples():
    r = _rows("ABCD")
    K.apply_reorder_in_place(r, [1, 2, 2, 3])
    assert [chr(x) for x in r[:, 0]] == list("BCCD")
    r = _rows("ABCD")
    K.apply_reorder_in_place(r, [0, 0, 1, 2])
    assert [chr(x) for x in r[:, 0]] == list("AABC")
    r = _rows("ABCD")
    assert K.apply_reorder_in_place(r, [0, 1, 2, 3]) == 0   # S:L86 zero writes
    assert [chr(x) for x in r[:, 0]] == list("ABCD")
    with pytest.raises(K.ReorderError):
        K.apply_reorder_in_place(_rows("ABCD"), [2, 0, 1, 0])   # S:L83 non-monotone rejected


def test_gather_examples_by_hand():
    r = _rows("ABCD")
    assert [chr(x) for x in K.gather(r, [3, 3, 0, 1])[:, 0]] == list("DDAB")
    assert [chr(x) for x in K.gather(r, [2, 0, 1, 0])[:, 0]] == list("CABA")


@pytest.mark.parametrize("bw", [1, 2, 3, 4, 5, 6])
def test_in_place_equals_gather_all_monotone_maps(bw):
    """every non-decreasing map for BW <= 6 (exhaustive)."""
    rows = np.arange(bw * 3).reshape(bw, 3)
    for src in itertools.combinations_with_replacement(range(bw), bw):
        r = rows.copy()
        K.apply_reorder_in_place(r, src)
        assert np.array_equal(r, K.gather(rows, src)), src


@pytest.mark.parametrize("bw", [128, 512])
def test_in_place_equals_gather_random_monotone(bw):
    rng = np.random.default_rng(bw)
    rows = rng.integers(0, 1 << 30, size=(bw, 4))
    for _ in range(200):
        src = np.sort(rng.integers(0, bw, size=bw))
        r = rows.copy()
        K.apply_reorder_in_place(r, src)
        assert np.array_equal(r, K.gather(rows, src))


def test_canonicalised_plan_reproduces_caller_order():
    """Applying the plan to the permuted caller order is the gather of the caller's map, up to the
    returned permutation (callers permute scores/tokens the same way)."""
    rng = np.random.default_rng(7)
    rows = rng.integers(0, 1000, size=(16, 2))
    for _ in range(100):
        src = rng.integers(0, 16, size=16)
        s, perm, _ = K.plan_reorder(src)
        r = rows.copy()
        K.apply_reorder_in_place(r, s)
        assert np.array_equal(r, K.gather(rows, src)[perm])
