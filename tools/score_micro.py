"""Time spc_score NORM and GROUP phases on a config-E-sized row set (1M tokens, 32 heads).
  python tools/score_micro.py [--lib=path]   (tools only)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])
dev = torch.device("cuda")
B, G, Hq, D, S = 1, 8, 32, 128, 1 << 20
g = torch.Generator(device=dev).manual_seed(0)
lg = torch.randn((B, Hq, S), generator=g, device=dev) * 3
hm = lg.max(-1).values.contiguous()
F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
gs = torch.zeros((B, G, S), device=dev)
seq = torch.tensor([S], dtype=torch.int32, device=dev)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
q = torch.zeros((B, Hq, D), dtype=torch.bfloat16, device=dev)
kr = torch.zeros((B, G, 8, D), dtype=torch.bfloat16, device=dev)
for name, ph in (("NORM", spc.SCORE_NORM), ("GROUP", spc.SCORE_GROUP)):
    ts = []
    for i in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        spc.score(q, kr, seq, G, 1.0, lg, hm, F, gs, ws, phases=ph)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{name:6s} {ts[len(ts) // 2]:7.1f} us   F[0]={int(F[0, 0])}")
