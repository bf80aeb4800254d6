"""Time spc_score(LOGITS) on config B.  Tools only.
Two timings: (1) 'cold': an L2-flushing read, then one launch between events;
(2) 'stream': 30 back-to-back launches over 16 address-distinct copies of the keys
(1 GiB, so no launch finds its keys in L2), averaged.
  python tools/logits_micro.py [--lib=path/to/libspc.so]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])
c = synth.CONFIGS["B"]
B, G, Hq, D, S = c["B"], c["G"], c["Hq"], c["D"], c["S"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=3, device=dev)
NC = 16
krs = kr.unsqueeze(0).repeat(NC, 1, 1, 1, 1)
q = synth.retrieval_queries(1, B, Hq, G, D, seed=3, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
lg = torch.zeros((B, Hq, S), device=dev)
hm = torch.zeros((B, Hq), device=dev)
F = torch.zeros((B, Hq), dtype=torch.int64, device=dev)
gs = torch.zeros((B, G, S), device=dev)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for i in range(23):
    flush.view(torch.int64).sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    spc.score(q, kr, seq, G, 0.0883883476, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1e-3)
ts.sort()
t = ts[len(ts) // 2]
ref = lg.clone()
print(f"logits cold  {t * 1e6:7.1f} us  {kr.numel() * 2 / t / 1e9:7.1f} GB/s  checksum {float(ref.sum()):.6e}")
for rep in range(2):
    torch.cuda._sleep(40_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(30):
        spc.score(q, krs[i % NC], seq, G, 0.0883883476, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) * 1e-3 / 30
    print(f"logits stream {t * 1e6:7.1f} us  {kr.numel() * 2 / t / 1e9:7.1f} GB/s")
assert torch.equal(lg, ref)
