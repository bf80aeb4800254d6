"""Algorithm 2 at run time (NEXT-2): OffloadingDecodeStep offloads the last
resident layer's KV to pinned host memory whenever the growing sequence reaches the next
threshold; resident layers are attended in place (INDEXED), offloaded ones from their HBM
budget buffers after the elastic gather (SLOTS).  Across three threshold crossings every
selection is bit-exact vs the oracle and the attention of EVERY layer (resident and
offloaded) matches the fp64 oracle within 2e-3."""
import numpy as np
import pytest
import torch

from paper_2512_00722_b200 import synth
from paper_2512_00722_b200.offload import OffloadingDecodeStep

pytestmark = pytest.mark.gpu
DEV = "cuda"


def test_offloading_step_across_thresholds(oracle):
    B, G, Hq, D, Smax, L, k = 1, 2, 8, 64, 3100, 4, 256
    S0 = 3000
    kr = synth.retrieval_keys(B, G, Smax, D, seed=41, device=DEV)
    kc, vc = synth.llm_kv(L, B, G, Smax, D, seed=41, device=DEV)
    kh, vh = synth.bf16_bits(kc), synth.bf16_bits(vc)  # the oracle's copy (before any release)
    k_layers = [kc[l].clone() for l in range(L)]  # separate allocations: offloading frees them
    v_layers = [vc[l].clone() for l in range(L)]
    del kc, vc
    qr = synth.retrieval_queries(9, B, Hq, G, D, seed=41, device=DEV)
    ql = synth.llm_queries(9, L, B, Hq, D, seed=41, device=DEV)
    seq = torch.full((B,), S0, dtype=torch.int32, device=DEV)
    th = [S0 + 2, S0 + 4, S0 + 6, 10 ** 9, 10 ** 9]  # Algorithm 1's list (explicit here)
    st = OffloadingDecodeStep(kr, k_layers, v_layers, seq, L, Hq, k, th)
    del k_layers, v_layers
    kr_h = synth.bf16_bits(kr)
    S = S0
    for s in range(8):
        S += 1
        seq.fill_(S)
        idx_d, cnt_d = st.step(qr[s], ql[s], S)
        torch.cuda.synchronize()
        expect_cpu = sum(1 for t in th[:4] if S >= t)
        assert st.l_cpu == expect_cpu, (S, st.l_cpu)
        _, _, _, gs = oracle.score(synth.bf16_bits(qr[s]), kr_h, [S], G, st.scale)
        idx, _, cnt, _ = oracle.topk(gs, [S], k, force_last=True)
        assert np.array_equal(idx_d.cpu().numpy(), idx) and np.array_equal(cnt_d.cpu().numpy(), cnt)
        oo, ol = oracle.sparse_attn(synth.bf16_bits(ql[s]), [kh[l] for l in range(L)],
                                    [vh[l] for l in range(L)], idx, cnt, st.scale)
        assert np.abs(st.out.cpu().numpy() - oo).max() <= 2e-3, (S, st.l_cpu)
        assert np.abs(st.lse.cpu().numpy() - ol).max() <= 1e-4
        # the budget slots of the offloaded layers hold exactly the slot map's rows
        slots = st.slot_tok.cpu().numpy()
        kb = synth.bf16_bits(st.kb)
        for l in range(L - st.l_cpu, L):
            for g in range(G):
                n = int(cnt[0, g])
                assert np.array_equal(kb[l, 0, g, :n], kh[l, 0, g, slots[0, g, :n]])
    assert [m[1] for m in st.migrations] == [3, 2, 1]
