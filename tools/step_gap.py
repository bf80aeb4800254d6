"""Config B: graph-replay step time with and without the per-step query copies (tools only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
qr = synth.retrieval_queries(41, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(2, L, B, Hq, D, seed=1, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
st.step(qr[0], ql[0])
st.capture()
for copies in (True, False, True, False):
    st.reset_state()
    for i in range(5):
        st.q_ret.copy_(qr[i]); st.q_llm.copy_(ql[0])
        st.graphs[(0, st.parity)].replay(); st.parity ^= 1
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(30):
        if copies:
            st.q_ret.copy_(qr[5 + i]); st.q_llm.copy_(ql[i % 2])
        st.graphs[(0, st.parity)].replay(); st.parity ^= 1
    b.record()
    torch.cuda.synchronize()
    print(f"copies={copies}: {a.elapsed_time(b) / 30 * 1e3:.1f} us/step (same K/V every step: L2-warm retrieval keys)")
