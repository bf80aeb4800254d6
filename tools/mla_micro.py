"""Time spc_mla_sparse_attn at the config-M shape (tools only): python tools/mla_micro.py [--lib=...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])
L, B, H, DN, DV, DC, DR, S, k, NS = 27, 1, 16, 128, 128, 512, 64, 32768, 2048, 3
dev = torch.device("cuda")
caches = [[synth.normal_bf16((B, S, DC + DR), 97 * c + l, device=dev) for l in range(L)] for c in range(NS)]
w_uk = [synth.normal_bf16((H, DN, DC), 1000 + l, device=dev) for l in range(L)]
w_uv = [synth.normal_bf16((H, DV, DC), 2000 + l, device=dev) for l in range(L)]
q = synth.normal_bf16((L, B, H, DN + DR), 3000, device=dev)
g = torch.Generator(device="cpu").manual_seed(1)
idx = torch.stack([torch.sort(torch.randperm(S, generator=g)[:k])[0] for _ in range(B * H)])
idx = idx.view(B, H, k).to(torch.int32).to(dev)
cnt = torch.full((B, H), k, dtype=torch.int32, device=dev)
out = torch.zeros((L, B, H, DV), dtype=torch.float32, device=dev)
ws = spc.alloc_workspace(spc.mla_workspace(L, B, H, k), dev)
ct = [spc.ptr_table(caches[c], dev) for c in range(NS)]
ut, vt = spc.ptr_table(w_uk, dev), spc.ptr_table(w_uv, dev)
for rep in range(2):
    torch.cuda._sleep(20_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(12):
        spc.mla_sparse_attn(q, ct[i % NS], ut, vt, idx, cnt, S, DN, DV, 0.07, out, None, ws)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 12 * 1e3
    print(f"mla {t:7.1f} us per 27-layer step")
