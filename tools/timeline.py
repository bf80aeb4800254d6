"""Kernel timeline of config-B steps inside one CUDA graph (tools only): CUPTI kernel records via
torch.profiler; prints each kernel's start / end relative to the step start, and the gaps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
NSTEP = 12
qr = synth.retrieval_queries(NSTEP, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(2, L, B, Hq, D, seed=1, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
for _ in range(2):
    kr2, kc2, vc2 = kr.clone(), kc.clone(), vc.clone()
    st.add_input_set(kr2, [kc2[l] for l in range(L)], [vc2[l] for l in range(L)])
st.step(qr[0], ql[0])
g = st.capture_sequence([(i % 3, qr[i], ql[i % 2]) for i in range(NSTEP)], bounds=[(0, NSTEP)])[0]
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.replay()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs], key=lambda x: x[0])
short = lambda n: n.split("::")[-1].split("<")[0].split("(")[0][:18]  # noqa: E731
per = 5
t_steps = []
for s in range(2, NSTEP - 1):  # steady-state steps
    ksel = ks[s * per:(s + 1) * per]
    t0 = ksel[0][0]
    t_steps.append(ks[(s + 1) * per][0] - t0)
    if s in (4, 5):
        print(f"step {s}:")
        prev_end = None
        for a, b, n in ksel:
            gap = "" if prev_end is None else f" gap {a - prev_end:6.2f}"
            print(f"  {short(n):18s} {a - t0:7.2f} .. {b - t0:7.2f}  dur {b - a:6.2f}{gap}")
            prev_end = b
print("step period (us):", " ".join(f"{t:.1f}" for t in t_steps))
