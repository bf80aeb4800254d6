"""Two eager decode steps of config A, of a 2K-context config-B shape (k = S: no cut) and of an
8K-context one (k = 1024: a cut on every row) through libspc, for compute-sanitizer (tools
only): python tools/sanitize_step.py [A|B2K|B8K|all]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda")
cases = {"A": dict(B=1, G=1, Hq=4, D=64, S=4096, L=1, k=256),
         "B2K": dict(B=1, G=8, Hq=32, D=128, S=2048, L=32, k=2048),
         "B8K": dict(B=1, G=8, Hq=32, D=128, S=8192, L=4, k=1024)}  # a cut on every row
for name, c in cases.items():
    if which not in ("all", name):
        continue
    B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
    kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
    qr = synth.retrieval_queries(2, B, Hq, G, D, seed=1, device=dev)
    ql = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
    seq = torch.full((B,), S, dtype=torch.int32, device=dev)
    for fused in (None, False):  # spc_select path and the separate calls
        st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k,
                        fused=fused)
        for s in range(2):
            st.step(qr[s], ql)
        torch.cuda.synchronize()
        print(name, "fused" if st.fused else "separate", "selected", int(st.cnt[1].sum()), flush=True)
    st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k,
                    one_launch=True)
    if st.one_launch:
        for s in range(2):
            st.step(qr[s], ql)
        torch.cuda.synchronize()
        print(name, "one_launch selected", int(st.cnt[1].sum()), flush=True)
print("launches", spc.launch_count())
