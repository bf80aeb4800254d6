"""spc_topk on config E's shape (8 rows x 1M tokens, k = 2048), timed in a CUDA graph (tools
only); the values are one config-E step's group scores when --real, else rand**6."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

dev = torch.device("cuda")
B, G, n, k = 1, 8, 1 << 20, 2048
if "--real" in sys.argv:
    c = synth.CONFIGS["E"]
    Hq, D = c["Hq"], c["D"]
    kr = synth.retrieval_keys(B, G, n, D, seed=7, device=dev)
    q = synth.retrieval_queries(1, B, Hq, G, D, seed=synth.BASE_SEED, device=dev)[0]
    seq0 = torch.full((B,), n, dtype=torch.int32, device=dev)
    lg = torch.zeros((B, Hq, n), device=dev)
    hm = torch.zeros((B, Hq), device=dev)
    F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
    gs = torch.zeros((B, G, n), device=dev)
    ws0 = spc.alloc_workspace(spc.score_workspace(B, Hq, n), dev)
    spc.score(q, kr, seq0, G, float(1 / math.sqrt(D)), lg, hm, F, gs, ws0)
    del kr, lg
else:
    g = torch.Generator(device=dev).manual_seed(0)
    gs = torch.rand((B, G, n), device=dev, generator=g) ** 6
seq = torch.full((B,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((B, G, k), dtype=torch.int32, device=dev)
cnt = torch.zeros((B, G), dtype=torch.int32, device=dev)
ws = spc.alloc_workspace(spc.topk_workspace(B, G, n, k), dev)
for _ in range(3):
    spc.topk(gs, seq, k, idx, cnt, ws, force_last=True)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(gr, stream=s):
        for _ in range(10):
            spc.topk(gs, seq, k, idx, cnt, ws, force_last=True, stream=s)
torch.cuda.current_stream().wait_stream(s)
gr.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    gr.replay()
b.record()
torch.cuda.synchronize()
print(f"spc_topk 8 x 1M ({'config-E scores' if '--real' in sys.argv else 'rand^6'}): "
      f"{a.elapsed_time(b) * 1e3 / 30:.1f} us")
