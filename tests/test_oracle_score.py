"""Pins for the oracle's scoring path O1..O6 (Eq.1 P:228 + GQA max P:328).

Each test ties the oracle to something other than itself: closed forms
(one-hot queries, uniform logits, single key), the fp64 mathematical
definition computed by torch/numpy (a library routine), the SPEC/paper worked
examples in tests/golden/, error bounds (Higham's gamma_D for the fp32 chain,
S * 2^-23 for the normaliser) and brute-force head->group mapping checks.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def bf16(a) -> np.ndarray:
    return synth.bf16_bits(torch.as_tensor(np.asarray(a, np.float32)).to(torch.bfloat16))


def from_bf16(u: np.ndarray) -> np.ndarray:
    return (u.astype(np.uint32) << 16).view(np.float32)


def rand_case(B, Hq, G, D, S, seed, scale_q=3.0):
    g = torch.Generator().manual_seed(seed)
    q = (scale_q * torch.randn(B, Hq, D, generator=g)).to(torch.bfloat16)
    kr = torch.randn(B, G, S, D, generator=g).to(torch.bfloat16)
    return synth.bf16_bits(q), synth.bf16_bits(kr)


def f32(x):
    return float(np.float32(x))


def test_logits_one_hot_query(oracle):
    """q = e_j (exact 1.0 at d=j) => s[t] = fl(K[t][j] * scale) exactly, for every head."""
    B, Hq, G, D, S = 1, 8, 2, 64, 37
    _, kr = rand_case(B, Hq, G, D, S, 1)
    q = np.zeros((B, Hq, D), np.float32)
    js = [3, 0, 63, 17, 5, 40, 22, 9]
    for h, j in enumerate(js):
        q[0, h, j] = 1.0
    scale = f32(1 / math.sqrt(D))
    lg, hm = oracle.logits(bf16(q), kr, [S], G, scale)
    kf = from_bf16(kr)
    for h, j in enumerate(js):
        g = h // (Hq // G)
        want = (kf[0, g, :, j] * np.float32(scale)).astype(np.float32)
        assert np.array_equal(lg[0, h], want), h
        assert hm[0, h] == want.max()


@pytest.mark.parametrize("alpha,G", [(1, 4), (2, 2), (4, 2), (8, 1)])
def test_logits_vs_fp64_within_higham(oracle, alpha, G):
    """|fl(chain) - exact| <= gamma_D * sum|q_d k_d| * scale + ulp(s)/2, with g = h // alpha."""
    B, D, S = 2, 128, 301
    Hq = G * alpha
    q, kr = rand_case(B, Hq, G, D, S, 2 + alpha)
    seq = np.array([S, 177], np.int32)
    scale = f32(1 / math.sqrt(D))
    lg, hm = oracle.logits(q, kr, seq, G, scale)
    qf = torch.from_numpy(from_bf16(q)).double()
    kf = torch.from_numpy(from_bf16(kr)).double()
    u = 2.0 ** -24
    gamma = D * u / (1 - D * u)
    for b in range(B):
        for h in range(Hq):
            g = h // alpha
            n = int(seq[b])
            exact = (kf[b, g, :n] @ qf[b, h]).numpy()
            absdot = (kf[b, g, :n].abs() @ qf[b, h].abs()).numpy()
            bound = gamma * absdot * scale + np.abs(exact * scale) * u + 1e-30
            assert np.all(np.abs(lg[b, h, :n] - exact * scale) <= bound * 1.0001), (b, h)
            assert hm[b, h] == lg[b, h, :n].max()
            assert np.all(lg[b, h, n:] == 0)  # beyond seq_len untouched


@pytest.mark.parametrize("case", GOLD["softmax_uniform"])
def test_uniform_logits_closed_form(oracle, case):
    """q = 0 => every logit 0 => e = 1, F = S * 2^40 exactly, p = fl(1/S)."""
    S, D, G, Hq = case["S"], 64, 1, 4
    _, kr = rand_case(1, Hq, G, D, S, 3)
    q = np.zeros((1, Hq, D), np.uint16)
    lg, hm, F, gs = oracle.score(q, kr, [S], G, 0.125)
    assert np.all(F == S * 2 ** 40)
    assert np.all(gs[0, 0, :S] == np.float32(1.0) / np.float32(S))
    assert float(gs[0, 0, 0]) == case["expect_p"]


def test_normaliser_sums_to_one(oracle):
    """sum_t p_h(t) within S * 2^-23 of 1 (fp32 weights of an exact normaliser), logits up to 1e4."""
    for scale_q, S in ((3.0, 2000), (400.0, 513)):
        B, Hq, G, D = 1, 4, 4, 64  # alpha = 1: group score == per-head weight
        q, kr = rand_case(B, Hq, G, D, S, 4, scale_q)
        lg, hm, F, gs = oracle.score(q, kr, [S], G, 1.0 / 8)
        assert np.abs(lg).max() > (1e3 if scale_q > 100 else 1)
        for h in range(Hq):
            tot = gs[0, h, :S].astype(np.float64).sum()
            assert abs(tot - 1.0) <= S * 2.0 ** -23 + 1e-6, (scale_q, h, tot)


def test_weights_match_fp64_softmax(oracle):
    """p_h(t) vs torch fp64 softmax of the oracle's own logits: relative error ~ few ulp."""
    B, Hq, G, D, S = 1, 4, 4, 128, 999
    q, kr = rand_case(B, Hq, G, D, S, 5)
    lg, hm, F, gs = oracle.score(q, kr, [S], G, f32(1 / math.sqrt(D)))
    ref = torch.softmax(torch.from_numpy(lg[0]).double(), dim=-1).numpy()
    big = ref > 1e-30
    rel = np.abs(gs[0][big] - ref[big]) / ref[big]
    # error budget: RN of (s - m) costs |s - m| * 2^-24 relative after exp; exp <= 1 ulp;
    # weight multiply, 1/l and the fixed-point truncation a few ulp more
    x = np.abs(lg[0] - hm[0][:, None])[big]
    assert np.all(rel <= (x + 8) * 2.0 ** -23), (rel / ((x + 8) * 2.0 ** -23)).max()


def test_group_max_paper_example(oracle):
    """P:328 / S:113: weight rows [0.2,0.7] and [0.9,0.1] of one group -> [0.9, 0.7].  Each row
    is completed by a padding position (0.1, 0.0) so that it is a head's softmax (Eq.1); the
    logits are log(w) (-100 for the zero weight: spc_exp returns exactly 0 below -87)."""
    case = GOLD["group_max"][0]
    w = np.concatenate([np.array(case["weights"], np.float64),
                        np.array(case["pad"], np.float64)[:, None]], axis=1)
    assert np.allclose(w.sum(axis=1), 1.0)
    lg = np.where(w > 0, np.log(np.maximum(w, 1e-300)), -100.0).astype(np.float32)[None]
    hm = lg.max(axis=-1)
    F = oracle.norm(lg, hm, [3])
    gs = oracle.group(lg, hm, F, [3], 1)  # G = 1: the two heads form one group (alpha = 2)
    assert np.allclose(gs[0, 0, :2], case["expect"], atol=1e-6)


def test_group_alpha1_identity_and_mqa(oracle):
    """alpha = 1: group score == the head's own weight.  MQA (G = 1): max of all heads."""
    B, D, S = 1, 64, 200
    q, kr1 = rand_case(B, 4, 4, D, S, 6)
    lg, hm, F, gs = oracle.score(q, kr1, [S], 4, 0.125)
    for h in range(4):
        r = np.float32(1.0) / (np.float32(float(F[0, h])) * np.float32(2.0 ** -40))
        e = np.array([oracle.spc_exp(float(np.float32(x - hm[0, h]))) for x in lg[0, h]],
                     np.float32)
        assert np.array_equal(gs[0, h], (e * r).astype(np.float32))
    # MQA: one group holding all heads sharing one key cache
    kr_mqa = np.ascontiguousarray(kr1[:, :1])
    lg2, hm2, F2, gs2 = oracle.score(q, kr_mqa, [S], 1, 0.125)
    per_head = oracle.group(lg2.reshape(1, 4, S), hm2, F2, [S], 4)  # alpha = 1 view
    assert np.array_equal(gs2[0, 0], per_head[0].max(axis=0))


def test_single_key_weight_one(oracle):
    """S = 1: p = 1 exactly."""
    q, kr = rand_case(1, 8, 2, 128, 1, 7)
    lg, hm, F, gs = oracle.score(q, kr, [1], 2, 0.088388)
    assert np.all(gs[0, :, 0] == 1.0)
    assert np.all(F == 2 ** 40)


def test_contract_faithful_to_fp64_topk(oracle):
    """The determinised top-k equals the fp64 mathematical top-k except for elements within a
    relative 1e-5 of the k-th fp64 score (faithfulness)."""
    B, Hq, G, D, S, k = 1, 16, 4, 128, 8192, 512
    kr = synth.bf16_bits(synth.retrieval_keys(B, G, S, D, seed=11))
    q = synth.bf16_bits(synth.retrieval_queries(1, B, Hq, G, D, seed=11)[0])
    scale = f32(1 / math.sqrt(D))
    _, _, _, gs = oracle.score(q, kr, [S], G, scale)
    g64 = oracle.group_score_f64(q, kr, [S], G, scale)
    assert np.allclose(gs, g64, rtol=1e-5, atol=1e-37)  # fp32 contract vs fp64 maths
    idx, _, cnt, _ = oracle.topk(gs, [S], k)
    for g in range(G):
        order = np.lexsort((np.arange(S), -g64[0, g]))
        ref = set(order[:k].tolist())
        got = set(idx[0, g, : cnt[0, g]].tolist())
        kth = g64[0, g, order[k - 1]]
        band = {int(t) for t in np.nonzero(np.abs(g64[0, g] - kth) <= 1e-5 * kth)[0]}
        assert (ref ^ got) <= band, g
