"""Time spc_rethead_qk at the config-B retrieval-head shape (B = 1), 4 rotated weight copies,
back-to-back launches (no graph) and in a CUDA graph.  Tools only.
  python tools/rethead_micro.py [--lib=path]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import rope, spc, synth  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])
B, V, H, Hq, G, D = int(os.environ.get("RH_B", "1")), 4096, 4096, 32, 8, 128
dev = torch.device("cuda")
emb, nw, w0 = synth.retrieval_head_weights(V, H, Hq, G, D, 1, device=dev)
ws = [w0] + [w0.clone() for _ in range(3)]
inv, m = rope.yarn_inv_freq(D, factor=64.0)
inv = torch.from_numpy(inv).to(dev)
tok = synth.tokens(1, B, V, 1, device=dev)[0].contiguous()
pos = torch.full((B,), 100, dtype=torch.int32, device=dev)
q = torch.zeros((B, Hq, D), dtype=torch.bfloat16, device=dev)
kr = torch.zeros((B, G, 256, D), dtype=torch.bfloat16, device=dev)
for rep in range(3):
    torch.cuda._sleep(20_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(40):
        spc.rethead_qk(tok, emb, nw, 1e-5, ws[i % 4], inv, m, pos, Hq, G, q, kr)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 40 * 1e3
    print(f"rethead B={B}: {t:6.2f} us per launch  {w0.numel() * 2 / t / 1e3:7.1f} GB/s")
