"""Config-B step cost by parts (tools only): CUDA graphs of 12 back-to-back steps over 3 rotated
input sets, each step = a prefix of LOGITS(+finalize) -> select -> attention(+merge); prints us
per step for each prefix and for select+attention and attention alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import spc, synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

for a in sys.argv[1:]:
    if a.startswith("--lib="):
        spc._lib = spc.load_library(a[6:])

c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
qr = synth.retrieval_queries(16, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(2, L, B, Hq, D, seed=1, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
st = DecodeStep(kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, L, Hq, k)
for _ in range(2):
    kr2, kc2, vc2 = kr.clone(), kc.clone(), vc.clone()
    st.add_input_set(kr2, [kc2[l] for l in range(L)], [vc2[l] for l in range(L)])
st.step(qr[0], ql[0])
torch.cuda.synchronize()


def part(i, what, s):
    st.use_set(i % 3)
    cur, prev = i % 2, 1 - i % 2
    if "L" in what:
        spc.score(qr[i], st.kr, st.seq_len, G, st.scale, st.logits, st.head_max, st.head_sumfix, st.gs,
                  st.ws_score, phases=spc.SCORE_LOGITS, stream=s)
    if "S" in what:
        spc.select(st.logits, st.head_max, st.seq_len, G, k, st.head_sumfix, st.gs, st.idx[cur],
                   st.cnt[cur], st.idx[prev], st.cnt[prev], st.load_tok, st.n_load, force_last=True,
                   stream=s)
    if "A" in what:
        spc.sparse_decode_attn_kv(st.desc, ql[i % 2], spc.KV_INDEXED, st.idx[cur], st.cnt[cur], k,
                                  st.scale, st.outs[cur], st.lses[cur], st.ws_attn, stream=s)


def timed(what, n=12):
    for i in range(n):
        part(i, what, None)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                part(i, what, s)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / (3 * n))
    st.use_set(0)
    return best


res = {w: timed(w) for w in ("L", "S", "A", "LS", "SA", "LSA")}
for w, t in res.items():
    print(f"{w:4s} {t:7.2f} us per step")
print(f"in the chain: select +{res['LS'] - res['L']:.2f}, attention +{res['LSA'] - res['LS']:.2f} us")
