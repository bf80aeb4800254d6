"""Run N eager decode steps of a config (for ncu launch lists / captures).  Not a bench."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="B")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--mode", default="indexed")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
qr = synth.retrieval_queries(a.steps + 1, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for i in range(a.steps):
    flush.fill_(i)
    st.step(qr[i], ql)
torch.cuda.synchronize()
print("done", st.cnt[0].sum().item())
