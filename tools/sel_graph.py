"""spc_select in a CUDA graph (tools only): config-B rows, logits of consecutive AR(1) queries
alternating, the previous selection ping-ponged; us per call.  Usage: sel_graph.py [--lib=path]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        new, old = spc.lib(), ctypes.CDLL(a[6:])
        for name in ("spc_score", "spc_score_workspace", "spc_select", "spc_status_string",
                     "spc_last_cuda_error"):
            getattr(old, name).argtypes = getattr(new, name).argtypes
            getattr(old, name).restype = getattr(new, name).restype
        spc._lib = old
c = synth.CONFIGS["B"]
B, G, Hq, D, S, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
NQ = 4
qs = synth.retrieval_queries(NQ, B, Hq, G, D, seed=1, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
f32, i32 = torch.float32, torch.int32
z = lambda *s, dt=f32: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
lgs = [z(B, Hq, S) for _ in range(NQ)]
hms = [z(B, Hq) for _ in range(NQ)]
F, gs = z(B, Hq, dt=torch.int64), z(B, G, S)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
for i in range(NQ):
    spc.score(qs[i], kr, seq, G, 0.088, lgs[i], hms[i], F, gs, ws, phases=spc.SCORE_LOGITS)
idx = [z(B, G, k, dt=i32) for _ in range(2)]
cnt = [z(B, G, dt=i32) for _ in range(2)]
lt, nl = z(B, G, k, dt=i32), z(B, G, dt=i32)


def sel(i, stream=None):
    spc.select(lgs[i % NQ], hms[i % NQ], seq, G, k, F, gs, idx[i % 2], cnt[i % 2], idx[1 - i % 2],
               cnt[1 - i % 2], lt, nl, force_last=True, stream=stream)


for i in range(4):
    sel(i)
torch.cuda.synchronize()
n = 12
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            sel(i, stream=s)
torch.cuda.current_stream().wait_stream(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
best = 1e9
for rnd in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) * 1e3 / (4 * n))
print(f"spc_select in a graph: {best:6.2f} us per call; n_load {int(nl.sum())}")
