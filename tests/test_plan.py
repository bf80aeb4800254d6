"""NEXT-2 adaptive memory management (paper §6, Eq. 6-8, Algorithms 1-2): the oracle pinned to
the paper's KV-size statements and SPEC's worked examples, then the product's host functions
(libspc spc_plan_*) equal to the oracle on random configurations.  CPU only: the planner is
host code of the C ABI (no GPU work)."""
import numpy as np
import pytest

import oracle
from paper_2512_00722_b200 import spc


def ex_cfg(**kw):
    c = dict(mem_gpu=160, model_bytes=0, runtime_factor=1.3, L=2, H=1, D=1, extra_layers=2, R=1,
             B=2, bytes_per_elem=2)
    c.update(kw)
    return c


def to_prod(c):
    return spc.plan_cfg(c["mem_gpu"], c["model_bytes"], c["L"], c["H"], c["D"], c["R"], c["B"],
                        extra_layers=c["extra_layers"], runtime_factor=c["runtime_factor"],
                        bytes_per_elem=c["bytes_per_elem"])


# ------------------------------------------------------------------ oracle pins
def test_kv_bytes_match_the_paper():
    """P:154 '2GB of memory footprint' at 16K and P:225 '4GB ... with 32K context' for
    Llama3.1-8B (L=32, H=8, D=128, R=1, fp16): Eq. 6's KV term with no extra layers."""
    c = dict(model_bytes=0, L=32, H=8, D=128, extra_layers=0, R=1, B=0)
    assert oracle.plan_mem(c, 16384, 32) == 2 * 2 ** 30
    assert oracle.plan_mem(c, 32768, 32) == 4 * 2 ** 30
    assert oracle.plan_mem(c, 0, 32) == 0


def test_spec_examples():
    """SPEC m_all: M_O = M_D = 0, R = L = H = D = 1, alpha = 1 (extra 2), S = 1 -> 12 bytes;
    Algorithm 1: L = 2, alpha = 1, H = D = R = 1, B = 2, mem 160 -> S^T = [10, 12, 18];
    Algorithm 2 on those thresholds: S = 9 no action, S = 11 offloads layer L-1 only,
    S = 20 offloads both layers in one call (the inner while)."""
    assert oracle.plan_mem(dict(model_bytes=0, L=1, H=1, D=1, extra_layers=2, R=1, B=0), 1, 1) == 12
    th = oracle.plan_thresholds_search(ex_cfg())
    assert th.tolist() == [10, 12, 18]
    assert oracle.plan_step(th, 2, 9, 0) == (0, [])
    assert oracle.plan_step(th, 2, 11, 0) == (1, [1])
    assert oracle.plan_step(th, 2, 20, 0) == (2, [1, 0])
    assert oracle.plan_step(th, 2, 20, 2) == (2, [])  # idempotent once everything is offloaded


def test_eq7_boundaries():
    """Eq. 7 at l_gpu = L is Eq. 6; with B = S it equals Eq. 6 for every l_gpu (buffers as large
    as the caches); doubling S doubles the KV term (linearity)."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        c = dict(model_bytes=int(rng.integers(0, 10 ** 9)), runtime_factor=1.3,
                 L=int(rng.integers(1, 80)), H=int(rng.integers(1, 16)), D=int(rng.choice([64, 128])),
                 extra_layers=int(rng.integers(0, 9)), R=int(rng.integers(1, 64)), B=0)
        S = int(rng.integers(0, 1 << 20))
        m_model = int(1.3 * c["model_bytes"])
        c["B"] = S
        full = oracle.plan_mem(c, S, c["L"])
        for l in (0, c["L"] // 2, c["L"]):
            assert oracle.plan_mem(c, S, l) == full
        assert oracle.plan_mem(c, 2 * S, c["L"]) - m_model == 2 * (full - m_model)


# ------------------------------------------------------------------ product vs oracle
def test_product_matches_spec_example_and_oracle_random():
    p = to_prod(ex_cfg())
    assert spc.plan_thresholds(p).tolist() == [10, 12, 18]
    assert spc.plan_step([10, 12, 18], 2, 11, 0) == (1, [1])
    assert spc.plan_step([10, 12, 18], 2, 20, 0) == (2, [1, 0])
    rng = np.random.default_rng(1)
    checked = 0
    for _ in range(200):
        c = dict(mem_gpu=int(rng.integers(10 ** 9, 200 * 10 ** 9)),
                 model_bytes=int(rng.integers(0, 20 * 10 ** 9)), runtime_factor=1.3,
                 L=int(rng.integers(1, 81)), H=int(rng.integers(1, 17)),
                 D=int(rng.choice([64, 128, 192])), extra_layers=int(rng.integers(0, 10)),
                 R=int(rng.integers(1, 65)), B=int(rng.integers(0, 8193)), bytes_per_elem=2)
        p = to_prod(c)
        C = c["mem_gpu"] - int(1.3 * c["model_bytes"])
        if C <= 0:
            with pytest.raises(spc.SpcError):
                spc.plan_thresholds(p)
            continue
        th = spc.plan_thresholds(p)
        ref = oracle.plan_thresholds_search(c)
        for i in range(c["L"] + 1):
            if c["L"] + c["extra_layers"] - i == 0:
                assert th[i] == np.iinfo(np.int64).max  # no KV layer left on the GPU
            elif ref[i] >= 0:
                assert th[i] == ref[i], (c, i)
            else:
                assert th[i] < 0
        for S in (0, int(rng.integers(0, 1 << 22)), int(max(th[0], 0)), int(max(th[0], 0)) + 1,
                  int(max(th[min(1, c["L"])], 0))):
            lg, sf = spc.plan_max_resident(p, S)
            assert lg == oracle.plan_max_resident(c, S)
            assert spc.plan_mem_part(p, S, max(lg, 0)) == oracle.plan_mem(c, S, max(lg, 0))
            if lg < 0:
                assert sf == oracle.plan_mem(c, S, 0) - c["mem_gpu"] > 0
            # Algorithm 2 from L_CPU = 0 lands on Eq. 8's optimum when the thresholds increase
            # (C > c * B * (L + extra), SPEC "threshold monotonicity") -- except exactly AT a
            # threshold: Alg. 2 offloads when S >= S^T_i ("S must be smaller than
            # S^T_0") while S = S^T_i still fits Eq. 8, one layer more (reading R27)
            cc = 2 * 2 * c["R"] * c["H"] * c["D"]
            if lg >= 0 and C > cc * c["B"] * (c["L"] + c["extra_layers"]):
                assert np.all(np.diff(th[th < np.iinfo(np.int64).max]) > 0)
                l_cpu, _ = spc.plan_step(th, c["L"], S, 0)
                at = int(np.sum(th == S))
                assert c["L"] - l_cpu == lg - at, (c, S)
                checked += 1
    assert checked > 100
