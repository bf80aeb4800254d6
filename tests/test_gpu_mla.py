"""GPU parity of spc_mla_sparse_attn (NEXT-3, MLA over each head's selected latent rows) against
the fp64 select-then-expand oracle: max-abs error <= 2e-3 (the north star's bf16 tolerance),
lse within 1e-4; ragged, single-row and empty selections; several split-K chunks."""
import numpy as np
import pytest
import torch

import oracle
from paper_2512_00722_b200 import spc, synth

pytestmark = pytest.mark.gpu
DEV = "cuda"
DC, DR = 512, 64


@pytest.mark.parametrize("L,B,H,DN,DV,Smax,k", [(2, 2, 4, 128, 128, 3000, 512),
                                               (1, 1, 3, 64, 96, 700, 300)])
def test_mla_matches_oracle(L, B, H, DN, DV, Smax, k):
    rng = np.random.default_rng(B * H + DN)
    cache = synth.normal_bf16((L, B, Smax, DC + DR), 3 + H)
    w_uk = (synth.normal_bf16((L, H, DN, DC), 5 + H, dtype=torch.float32) * (1 / DC ** 0.5)).to(torch.bfloat16)
    w_uv = (synth.normal_bf16((L, H, DV, DC), 7 + H, dtype=torch.float32) * (1 / DC ** 0.5)).to(torch.bfloat16)
    q = synth.normal_bf16((L, B, H, DN + DR), 9 + H)
    idx = np.full((B, H, k), -1, np.int32)
    cnt = np.zeros((B, H), np.int32)
    sizes = [k, 1, 0, 257, 129, k // 3]
    for b in range(B):
        for h in range(H):
            n = min(sizes[(b * H + h) % len(sizes)], Smax)
            idx[b, h, :n] = np.sort(rng.choice(Smax, n, replace=False))
            cnt[b, h] = n
    out = torch.zeros((L, B, H, DV), dtype=torch.float32, device=DEV)
    lse = torch.zeros((L, B, H), dtype=torch.float32, device=DEV)
    ws = spc.alloc_workspace(spc.mla_workspace(L, B, H, k), DEV)
    scale = 1.0 / (DN + DR) ** 0.5
    cd, ud, vd = cache.to(DEV), w_uk.to(DEV), w_uv.to(DEV)
    tabs = [spc.ptr_table([t[l] for l in range(L)], DEV) for t in (cd, ud, vd)]
    for rep in range(2):  # the workspace is reusable (tickets reset)
        spc.mla_sparse_attn(q.to(DEV), *tabs, torch.from_numpy(idx).to(DEV),
                            torch.from_numpy(cnt).to(DEV), Smax, DN, DV, scale, out, lse, ws)
        torch.cuda.synchronize()
        o, lo = out.cpu().numpy(), lse.cpu().numpy()
        qb, cb = synth.bf16_bits(q), synth.bf16_bits(cache)
        ukb, uvb = synth.bf16_bits(w_uk), synth.bf16_bits(w_uv)
        for la in range(L):
            for b in range(B):
                for h in range(H):
                    oo, ol = oracle.mla_head(qb[la, b, h], cb[la, b], ukb[la, h], uvb[la, h],
                                             idx[b, h, :cnt[b, h]], DC, DR, scale)
                    assert np.abs(o[la, b, h] - oo).max() <= 2e-3, (la, b, h)
                    if cnt[b, h]:
                        assert abs(lo[la, b, h] - ol) <= 1e-4
                    else:
                        assert lo[la, b, h] == -np.inf and np.all(o[la, b, h] == 0)
