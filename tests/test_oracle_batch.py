"""NEXT-3 batch-level retrieval oracle pins (Fig. 5(a)): the sum
over all heads of O5's weights, then top-k.  Pinned to SPEC's examples (tie toward the smaller
index; one head = head-level) and to an independent route: the per-head weights from the
group oracle with alpha = 1, summed in ascending head order with float32 adds."""
import numpy as np

import oracle


def lg_case(B, Hq, S, seed, scale=3.0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((B, Hq, S)) * scale).astype(np.float32)


def score_parts(lg, seq):
    B, Hq, S = lg.shape
    hm = np.array([[lg[b, h, :seq[b]].max() for h in range(Hq)] for b in range(B)], np.float32)
    F = oracle.norm(lg, hm, seq)
    return hm, F


def test_two_mirrored_heads_tie_to_the_smaller_index():
    """SPEC: two heads favouring positions {0} and {1} equally, B = 1 -> {0}."""
    lg = np.array([[[2.0, 0.5, -1.0], [0.5, 2.0, -1.0]]], np.float32)
    seq = [3]
    hm, F = score_parts(lg, seq)
    bs = oracle.batch_score(lg, hm, F, seq)
    assert bs[0, 0] == bs[0, 1] > bs[0, 2]
    idx, _, cnt, _ = oracle.topk(bs[:, None, :], seq, 1)
    assert idx[0, 0, 0] == 0 and cnt[0, 0] == 1


def test_single_head_equals_head_level():
    """SPEC: a single head -> identical to retrieve_head_level (the GROUP score with alpha = 1)."""
    lg = lg_case(2, 1, 777, 1)
    seq = [777, 300]
    hm, F = score_parts(lg, seq)
    bs = oracle.batch_score(lg, hm, F, seq)
    gs = oracle.group(lg, hm, F, seq, 1)[:, 0]
    assert np.array_equal(bs.view(np.uint32), gs.view(np.uint32))


def test_sum_of_head_weights_in_head_order():
    """bs equals the alpha = 1 group scores (each head's own weights) added in ascending head
    order in float32; rows past seq_len are 0; the scores of a request sum to ~Hq."""
    B, Hq, S = 2, 8, 1000
    lg = lg_case(B, Hq, S, 2)
    seq = [1000, 457]
    hm, F = score_parts(lg, seq)
    bs = oracle.batch_score(lg, hm, F, seq)
    per_head = oracle.group(lg, hm, F, seq, Hq)  # [B][Hq][S]: p_h(t)
    want = per_head[:, 0].copy()
    for h in range(1, Hq):
        want = (want + per_head[:, h]).astype(np.float32)
    assert np.array_equal(bs.view(np.uint32), want.view(np.uint32))
    assert np.all(bs[1, 457:] == 0)
    for b in range(B):
        assert abs(float(bs[b].astype(np.float64).sum()) - Hq) < Hq * seq[b] * 2.0 ** -22
