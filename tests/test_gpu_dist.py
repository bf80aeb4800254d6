"""Context-sharded step (O13) through libspc with P ranks emulated on one GPU: the union of
the ranks' selections equals the single-device oracle selection bit for bit, and the
LSE-merged attention matches the oracle within 2e-3 (bf16)."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import dist as sdist
from paper_2512_00722_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_emulated_sharded_step(oracle, P):
    dev = torch.device("cuda")
    B, G, Hq, D, S, L, k = 1, 8, 32, 128, 6000, 3, 512
    kr = synth.retrieval_keys(B, G, S, D, seed=P, device=dev)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=P, device=dev)
    qr = synth.retrieval_queries(1, B, Hq, G, D, seed=P, device=dev)[0]
    ql = synth.llm_queries(1, L, B, Hq, D, seed=P, device=dev)[0]
    kl, vl = [kc[l] for l in range(L)], [vc[l] for l in range(L)]
    states = [sdist.make_shard(r, P, kr, kl, vl, qr, ql, [S], k) for r in range(P)]
    sel, out, lse = sdist.run_emulated(sdist.SpcOps(), states)
    torch.cuda.synchronize()
    scale = states[0].scale
    _, _, _, gs = oracle.score(synth.bf16_bits(qr), synth.bf16_bits(kr), [S], G, scale)
    idx, _, cnt, _ = oracle.topk(gs, [S], k, force_last=True)
    for g in range(G):
        union = sorted(int(x) * P + r for r in range(P)
                       for x in sel[r][0][0, g, :int(sel[r][1][0, g])].tolist())
        assert union == idx[0, g, :cnt[0, g]].tolist(), g
    oo, ol = oracle.sparse_attn(synth.bf16_bits(ql), [synth.bf16_bits(t) for t in kl],
                                [synth.bf16_bits(t) for t in vl], idx, cnt, scale)
    assert np.abs(out.cpu().numpy() - oo).max() <= 2e-3
    assert np.abs(lse.cpu().numpy() - ol).max() <= 1e-3
