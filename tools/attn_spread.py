"""Attention time vs the span of the KV cache the same selected bytes are spread over (tools only).
Config-B selection sizes (32 layers x 8 groups x 2048 random rows) over caches of S rows, the TMA
gather4 kernel and the cp.async pointer-table kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

dev = torch.device("cuda")
L, B, G, Hq, D, k = 32, 1, 8, 32, 128, 2048
for S in (32768, 262144, 1048576):
    kc = torch.empty((L, B, G, S, D), dtype=torch.bfloat16, device=dev)
    vc = torch.empty_like(kc)
    kc.view(-1)[: 1 << 20].normal_()
    q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
    kt = spc.ptr_table([kc[l] for l in range(L)], dev)
    vt = spc.ptr_table([vc[l] for l in range(L)], dev)
    desc = spc.KvDesc([kc[l] for l in range(L)], [vc[l] for l in range(L)])
    out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev)
    lse = torch.zeros((L, B, Hq), dtype=torch.float32, device=dev)
    ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
    g = torch.Generator(device="cpu").manual_seed(0)
    idx = torch.stack([torch.sort(torch.randperm(S, generator=g)[:k])[0] for _ in range(G)]).view(B, G, k)
    idx = idx.to(torch.int32).to(dev)
    cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
    for tma, rep in ((True, 0), (True, 1), (False, 0), (False, 1)):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(10):
            if tma:
                spc.sparse_decode_attn_kv(desc, q, spc.KV_INDEXED, idx, cnt, k, 0.088, out, lse, ws)
            else:
                spc.sparse_decode_attn(q, kt, vt, spc.KV_INDEXED, idx, cnt, S, k, 0.088, out, lse, ws, G)
        b.record()
        torch.cuda.synchronize()
        if rep:
            print(f"S = {S:8d} ({2 * kc.numel() * 2 / 2**30:6.1f} GiB of KV) {'TMA gather4' if tma else 'cp.async'}: "
                  f"{a.elapsed_time(b) * 100:.1f} us per launch")
    del desc
    del kc, vc
    torch.cuda.empty_cache()
