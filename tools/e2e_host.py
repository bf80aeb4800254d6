"""Host cost of DecodeStep.step_host (config B): wall time per call vs GPU time per step.
Tools only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
qr = synth.retrieval_queries(2, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
NSETS = int(os.environ.get("E2E_SETS", "3"))
for _ in range(NSETS - 1):
    st.add_input_set(kr.clone(), [x.clone() for x in kc], [x.clone() for x in vc])
st.step(qr[0], ql)
st.capture()
qh, lh = qr[1].cpu().pin_memory(), ql.cpu().pin_memory()
oh = torch.empty(st.out.shape, dtype=torch.float32).pin_memory()
for j in range(20):
    st.use_set(j % NSETS)
    st.step_host(qh, lh, oh)
st.sync_host()
torch.cuda.synchronize()
N = 300
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
t0 = time.perf_counter()
for j in range(N):
    st.use_set(j % NSETS)
    st.step_host(qh, lh, oh)
t1 = time.perf_counter()
st.sync_host()
b.record()
torch.cuda.synchronize()
print(f"host {1e6 * (t1 - t0) / N:.1f} us per step_host call; GPU {a.elapsed_time(b) * 1e3 / N:.1f} us per step")
a.record()
for j in range(N):
    st.use_set(j % NSETS)
    st.step(use_graph=True)
b.record()
torch.cuda.synchronize()
print(f"device-resident graph steps: {a.elapsed_time(b) * 1e3 / N:.1f} us per step")
