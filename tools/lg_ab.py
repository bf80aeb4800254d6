"""LOGITS phase timing (tools only): spc_score(LOGITS) (+ its finalize) on the config-B
shape, 4 address-distinct key copies rotated launch to launch, back to back.
Usage: python tools/lg_ab.py [--lib=path]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

for a in list(sys.argv):
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])
dev = torch.device("cuda")
B, G, Hq, D, S = 1, 8, 32, 128, 32768
krs = [synth.retrieval_keys(B, G, S, D, seed=5 + c, device=dev) for c in range(4)]
q = synth.retrieval_queries(1, B, Hq, G, D, seed=1, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
f32 = torch.float32
lg, hm = torch.zeros((B, Hq, S), dtype=f32, device=dev), torch.zeros((B, Hq), dtype=f32, device=dev)
F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
gs = torch.zeros((B, G, S), dtype=f32, device=dev)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
for rnd in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(8):
        spc.score(q, krs[i % 4], seq, G, 0.088, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
    torch.cuda.synchronize()
    a.record()
    n = 50
    for i in range(n):
        spc.score(q, krs[i % 4], seq, G, 0.088, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / n
    print(f"LOGITS+finalize {us:7.2f} us per call ({B * G * S * D * 2 / us / 1e3:7.1f} GB/s)")
