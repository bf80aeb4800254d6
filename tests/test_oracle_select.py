"""Pins for O7 (top-k) and O8 (elastic diff + slots).

Top-k: the paper's/SPEC's worked examples, and a brute-force
check against Python's own sort of (-value, id) on random rows with forced
duplicates; composite thresholds; the rescale invariance of S:144.
Elastic diff: the S:235 example, exhaustive enumeration of all
subset pairs of a 10-element universe against Python set algebra, and a
10,000-step random walk in which slot contents always equal the backing rows.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


@pytest.mark.parametrize("case", GOLD["topk"])
def test_topk_paper_examples(oracle, case):
    val = np.array(case["val"], np.float32)
    fp = len(val) - 1 if case.get("force_last") else -1
    pos, _, _ = oracle.topk_row(val, case["k"], fp)
    assert pos.tolist() == case["expect"]


def brute_topk(val, k, ids):
    order = sorted(range(len(val)), key=lambda p: (-float(val[p]), ids[p]))
    return sorted(order[:k]), order[:k]


def test_topk_brute_force_with_ties(oracle):
    rng = np.random.default_rng(0)
    for trial in range(1000):
        S = 256
        k = 32
        val = rng.random(S).astype(np.float32)
        dup = rng.integers(0, S, size=(rng.integers(0, 64), 2))
        val[dup[:, 0]] = val[dup[:, 1]]  # exact ties
        if trial % 7 == 0:
            val = np.round(val * 4).astype(np.float32) / 4  # massive ties
        stride, off = (1, 0) if trial % 2 else (3, 2)
        ids = [p * stride + off for p in range(S)]
        want, order = brute_topk(val, k, ids)
        pos, v, th = oracle.topk_row(val, k, -1, stride, off)
        assert pos.tolist() == want
        assert np.array_equal(v, val[pos])
        last = order[-1]
        assert th == oracle.composite(float(val[last]), ids[last])


def test_topk_clamp_force_and_empty(oracle):
    val = np.array([0.3, 0.2, 0.1], np.float32)
    pos, v, th = oracle.topk_row(val, 8, 2)
    assert pos.tolist() == [0, 1, 2] and v[2] == np.inf
    pos, v, th = oracle.topk_row(val[:0], 4)
    assert len(pos) == 0 and th == 0
    pos, _, th = oracle.topk_row(val, 1, 2)  # forced element beats everything
    assert pos.tolist() == [2] and th == oracle.composite(float("inf"), 2)


def test_topk_scale_invariance(oracle):
    """positive rescaling of a weight row leaves the selection unchanged
    (exact power-of-two scale; and x3.7 whenever it creates no new ties)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        val = rng.random(300).astype(np.float32)
        a, _, _ = oracle.topk_row(val, 40)
        b, _, _ = oracle.topk_row(val * np.float32(4.0), 40)
        assert np.array_equal(a, b)
        v37 = val * np.float32(3.7)
        if len(np.unique(v37)) == len(np.unique(val)):
            c, _, _ = oracle.topk_row(v37, 40)
            assert np.array_equal(a, c)


def test_sharded_topk_union_equals_global(oracle):
    """O13: strided shards' local top-k lists contain the global top-k; the merged threshold
    filter reproduces it exactly (P shards, ids = pos * P + r)."""
    rng = np.random.default_rng(2)
    for P in (1, 2, 3, 4, 8):
        for _ in range(30):
            S, k = int(rng.integers(50, 400)), int(rng.integers(1, 60))
            val = (rng.random(S) * 8).round().astype(np.float32)  # many ties
            want, _, _ = oracle.topk_row(val, k)
            cands = []
            for r in range(P):
                loc = val[r::P]
                pos, v, _ = oracle.topk_row(loc, k, -1, P, r)
                cands += [(float(x), int(p) * P + r) for p, x in zip(pos, v)]
            cv = np.array([c[0] for c in cands], np.float32)
            cid = np.array([c[1] for c in cands], np.int32)
            _, _, th = oracle.topk_row(cv, k, -1, cand_id=cid)
            kept = sorted(i for x, i in cands if oracle.composite(x, i) >= th)
            assert kept == want.tolist(), (P, S, k)


@pytest.mark.parametrize("case", GOLD["elastic_diff"])
def test_diff_paper_examples(oracle, case):
    r = oracle.elastic_diff_row(case["prev"], case["cur"], 3)
    assert r["load_tok"][: r["n_load"]].tolist() == case["expect_load"]
    assert r["evict_tok"][: r["n_evict"]].tolist() == case["expect_evict"]


def check_slots(prev, cur, k, slot_in, r):
    """Invariants of reading R13: kept slots never move; new tokens fill freed slots in
    ascending order; afterwards the non-empty slots hold exactly cur."""
    st = r["slot_tok"]
    newt = [t for t in cur if t not in set(prev)]
    assert r["load_tok"][: r["n_load"]].tolist() == newt
    for s in range(k):
        if slot_in[s] >= 0 and slot_in[s] in set(cur):
            assert st[s] == slot_in[s]  # kept slot untouched
    freed = [s for s in range(k) if slot_in[s] < 0 or slot_in[s] not in set(cur)]
    assert r["load_slot"][: r["n_load"]].tolist() == freed[: len(newt)]
    assert sorted(t for t in st if t >= 0) == sorted(cur)


def test_diff_exhaustive_small_universe(oracle):
    """All (prev, cur) pairs of subsets of {0..9} with sizes <= 4 (149,769 pairs)."""
    U = range(10)
    subsets = [list(c) for n in range(5) for c in itertools.combinations(U, n)]
    rng = random.Random(3)
    k = 5
    for prev in subsets:
        slot_in = np.full(k, -1, np.int32)
        slots = rng.sample(range(k), len(prev))
        for s, t in zip(slots, prev):
            slot_in[s] = t
        for cur in subsets:
            r = oracle.elastic_diff_row(prev, cur, k, slot_in)
            assert r["status"] == 0
            assert set(r["load_tok"][: r["n_load"]].tolist()) == set(cur) - set(prev)
            assert r["evict_tok"][: r["n_evict"]].tolist() == sorted(set(prev) - set(cur))
            if len(prev) == len(cur):
                assert r["n_load"] == r["n_evict"]  # fixed budget
            check_slots(prev, cur, k, slot_in, r)


def test_diff_state_error(oracle):
    slot_in = np.array([1, 7, -1], np.int32)  # 7 is not in prev
    r = oracle.elastic_diff_row([1, 2], [2, 3], 3, slot_in)
    assert r["status"] == -1


def test_diff_random_walk_slots_equal_backing(oracle):
    """10,000 elastic steps; slot contents always equal the backing rows of
    the current selection; transferred rows = n_load."""
    rng = np.random.default_rng(4)
    S, k = 400, 24
    backing = rng.standard_normal((S, 3))
    slots = np.zeros((k, 3))
    slot_tok = np.full(k, -1, np.int32)
    prev = np.zeros(0, np.int32)
    for step in range(10000):
        keep = prev[rng.random(len(prev)) < 0.8]
        pool = np.setdiff1d(np.arange(S), keep)
        n = int(rng.integers(max(1, len(keep)), k + 1)) if step % 50 else int(rng.integers(1, k + 1))
        n = max(n, len(keep)) if step % 50 else n
        add = rng.choice(pool, size=max(0, n - len(keep)), replace=False)
        cur = np.sort(np.concatenate([keep, add]).astype(np.int32))[:k]
        r = oracle.elastic_diff_row(prev, cur, k, slot_tok)
        assert r["status"] == 0
        for i in range(r["n_load"]):
            slots[r["load_slot"][i]] = backing[r["load_tok"][i]]
        slot_tok = r["slot_tok"]
        for s in range(k):
            if slot_tok[s] >= 0:
                assert np.array_equal(slots[s], backing[slot_tok[s]])
        assert sorted(slot_tok[slot_tok >= 0].tolist()) == cur.tolist()
        prev = cur
