"""Kernel timeline of config-E steps (1M tokens, P = 1, one CUDA graph per step, as bench.py
--config E) from CUPTI records via torch.profiler (tools only)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2512_00722_b200 import dist as sdist  # noqa: E402
from paper_2512_00722_b200 import spc, synth  # noqa: E402

dev = torch.device("cuda")
c = synth.CONFIGS["E"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
kr = synth.retrieval_keys(B, G, S, D, seed=7, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=7, device=dev)
qr = synth.retrieval_queries(8, B, Hq, G, D, seed=synth.BASE_SEED, device=dev)
ql = synth.llm_queries(1, L, B, Hq, D, seed=synth.BASE_SEED, device=dev)[0]
scale = float(torch.tensor(1.0 / math.sqrt(D), dtype=torch.float32))
st = sdist.ShardState(0, 1, [S], kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], qr[0].clone(),
                      ql, k, scale)
ops = sdist.SpcOps()
for i in range(3):
    st.q_ret.copy_(qr[i])
    sdist.run_emulated(ops, [st])
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sdist.run_emulated(ops, [st])
torch.cuda.current_stream().wait_stream(s)
for i in range(3):
    g.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        st.q_ret.copy_(qr[3 + i])
        g.replay()
    torch.cuda.synchronize()
evs = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
              if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
short = lambda n: n.split("::")[-1].split("<")[0].split("(")[0][:22]  # noqa: E731
t0 = evs[0][0]
prev = None
for a, b, n in evs:
    print(f"{short(n):22s} {a - t0:8.2f} .. {b - t0:8.2f}  dur {b - a:7.2f}" +
          ("" if prev is None else f"  gap {a - prev:7.2f}"))
    prev = b
