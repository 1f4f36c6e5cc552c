"""Pins for the oracle's dispatch structures. CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import dispatch_brute, dispatch_argsort
from moe_inputs import make_ids

GOLD = os.path.join(os.path.dirname(__file__), "golden", "fig2_dispatch.json")


def test_fig2_worked_example():
    """Paper's worked example, Fig. 2, corrected per reading #6."""
    g = json.load(open(GOLD))
    ids = np.array(g["ids"], dtype=np.int32)
    for fn in (dispatch_brute, dispatch_argsort):
        d = fn(ids, g["E"])
        ex = g["expected"]
        assert d["eti"].tolist() == ex["expert_token_indices"]
        assert d["offs"].tolist() == ex["expert_token_offsets"]
        assert d["counts"].tolist() == ex["expert_counts"]
        assert d["tim"].tolist() == ex["token_index_map"]
        assert d["tei"].reshape(-1).tolist() == ex["token_expert_indices"]
        # values printed in the paper, verbatim
        pr = g["printed"]
        assert d["eti"].tolist() == pr["expert_token_indices_P152"]
        assert d["offs"].tolist() == pr["expert_token_offsets_P153"]
        assert d["tim"][0].tolist() == pr["token_index_map_0_P156"]


def _invariants(ids, E, d):
    T, k = ids.shape
    R = T * k
    counts, offs, eti, tim = d["counts"], d["offs"], d["eti"], d["tim"]
    assert offs[0] == 0 and offs[E] == R                         # dropless, no padding
    assert np.all(np.diff(offs) >= 0)
    assert np.array_equal(np.diff(offs), counts)
    assert len(eti) == R
    assert np.array_equal(np.bincount(eti, minlength=T), np.full(T, k))   # every token exactly k times
    assert np.array_equal(np.sort(tim.reshape(-1)), np.arange(R))         # tim is a permutation
    for t in range(T):
        for j in range(k):
            r = tim[t, j]
            e = ids[t, j]
            assert eti[r] == t
            assert offs[e] <= r < offs[e + 1]
            assert d["row_slot"][r] == t * k + j
    for e in range(E):
        seg = eti[offs[e]:offs[e + 1]]
        assert np.all(np.diff(seg) > 0)                           # ascending token ids


@pytest.mark.parametrize("T,E,k,kind", [
    (1, 1, 1, "random"), (1, 8, 8, "random"), (37, 4, 2, "random"), (200, 16, 2, "skewed"),
    (300, 64, 6, "random"), (128, 8, 8, "random"), (99, 5, 1, "random"), (64, 16, 3, "degenerate"),
])
def test_brute_equals_argsort_and_invariants(T, E, k, kind):
    ids = make_ids(T, E, k, seed=T * 7 + E, kind=kind).numpy()
    a = dispatch_brute(ids, E)
    b = dispatch_argsort(ids, E)
    for key in ("counts", "offs", "eti", "tim", "row_slot"):
        assert np.array_equal(a[key], b[key]), key
    _invariants(ids, E, a)


def test_empty_experts_and_all_to_one():
    ids = np.zeros((10, 1), dtype=np.int32)
    d = dispatch_brute(ids, 4)
    assert d["offs"].tolist() == [0, 10, 10, 10, 10]
    assert d["eti"].tolist() == list(range(10))
    ids = np.full((5, 1), 3, dtype=np.int32)
    d = dispatch_argsort(ids, 4)
    assert d["offs"].tolist() == [0, 0, 0, 0, 5]


def test_zero_tokens():
    ids = np.zeros((0, 2), dtype=np.int32)
    for fn in (dispatch_brute, dispatch_argsort):
        d = fn(ids, 4)
        assert d["offs"].tolist() == [0, 0, 0, 0, 0]
        assert len(d["eti"]) == 0
