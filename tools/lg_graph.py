"""LOGITS phase in a CUDA graph (tools only): 12 spc_score(LOGITS) calls (+ finalize) on the
config-B shape over 4 address-distinct key copies, captured once, replayed; us per call.
Usage: python tools/lg_graph.py [--lib=path] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
for a in sys.argv[1:]:
    if a.startswith("--lib="):  # another build (may predate newer exports): copy the signatures
        import ctypes
        new, old = spc.lib(), ctypes.CDLL(a[6:])
        for name in ("spc_score", "spc_score_workspace", "spc_status_string", "spc_last_cuda_error"):
            getattr(old, name).argtypes = getattr(new, name).argtypes
            getattr(old, name).restype = getattr(new, name).restype
        spc._lib = old
c = synth.CONFIGS[args[0] if args else "B"]
dev = torch.device("cuda")
B, G, Hq, D, S = c["B"], c["G"], c["Hq"], c["D"], c["S"]
ncop = 4 if B * G * S * D * 2 < 2**31 else 2
krs = [synth.retrieval_keys(B, G, S, D, seed=5 + i, device=dev) for i in range(ncop)]
q = synth.retrieval_queries(1, B, Hq, G, D, seed=1, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
f32 = torch.float32
lg, hm = torch.zeros((B, Hq, S), dtype=f32, device=dev), torch.zeros((B, Hq), dtype=f32, device=dev)
F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
gs = torch.zeros((B, G, S), dtype=f32, device=dev)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
spc.score(q, krs[0], seq, G, 0.088, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
torch.cuda.synchronize()
n = 12
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            spc.score(q, krs[i % ncop], seq, G, 0.088, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS,
                      stream=s)
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
    us = a.elapsed_time(b) * 1e3 / (4 * n)
    best = min(best, us)
print(f"LOGITS+finalize in a graph: {best:7.2f} us per call ({B * G * S * D * 2 / best / 1e3:7.1f} GB/s)")
