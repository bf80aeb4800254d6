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


@pytest.mark.parametrize("B,H,DN,DV,Smax,k", [(2, 4, 128, 128, 3000, 512), (1, 3, 64, 96, 700, 300)])
def test_mla_matches_oracle(B, H, DN, DV, Smax, k):
    rng = np.random.default_rng(B * H + DN)
    cache = synth.normal_bf16((B, Smax, DC + DR), 3 + H)
    w_uk = (synth.normal_bf16((H, DN, DC), 5 + H, dtype=torch.float32) * (1 / DC ** 0.5)).to(torch.bfloat16)
    w_uv = (synth.normal_bf16((H, DV, DC), 7 + H, dtype=torch.float32) * (1 / DC ** 0.5)).to(torch.bfloat16)
    q = synth.normal_bf16((B, H, DN + DR), 9 + H)
    idx = np.full((B, H, k), -1, np.int32)
    cnt = np.zeros((B, H), np.int32)
    sizes = [k, 1, 0, 257, 129, k // 3]
    for b in range(B):
        for h in range(H):
            n = min(sizes[(b * H + h) % len(sizes)], Smax)
            idx[b, h, :n] = np.sort(rng.choice(Smax, n, replace=False))
            cnt[b, h] = n
    out = torch.zeros((B, H, DV), dtype=torch.float32, device=DEV)
    lse = torch.zeros((B, H), dtype=torch.float32, device=DEV)
    ws = spc.alloc_workspace(spc.mla_workspace(B, H, k), DEV)
    scale = 1.0 / (DN + DR) ** 0.5
    for rep in range(2):  # the workspace is reusable (tickets reset)
        spc.mla_sparse_attn(q.to(DEV), cache.to(DEV), w_uk.to(DEV), w_uv.to(DEV),
                            torch.from_numpy(idx).to(DEV), torch.from_numpy(cnt).to(DEV), scale,
                            out, lse, ws)
        torch.cuda.synchronize()
        o, l = out.cpu().numpy(), lse.cpu().numpy()
        qb, cb = synth.bf16_bits(q), synth.bf16_bits(cache)
        ukb, uvb = synth.bf16_bits(w_uk), synth.bf16_bits(w_uv)
        for b in range(B):
            for h in range(H):
                oo, ol = oracle.mla_head(qb[b, h], cb[b], ukb[h], uvb[h], idx[b, h, :cnt[b, h]], DC,
                                         DR, scale)
                assert np.abs(o[b, h] - oo).max() <= 2e-3, (b, h, np.abs(o[b, h] - oo).max())
                if cnt[b, h]:
                    assert abs(l[b, h] - ol) <= 1e-4
                else:
                    assert l[b, h] == -np.inf and np.all(o[b, h] == 0)
