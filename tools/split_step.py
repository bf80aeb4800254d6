"""Experiment: config B as two half-steps (KV groups 0-3 and 4-7, independent selections) on two
streams, so one half's latency-bound select overlaps the other half's HBM-bound kernels.
Tools only.  Prints the one-stream full step and the two-stream split step (graphs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import synth  # noqa: E402
from paper_2512_00722_b200.pipeline import DecodeStep  # noqa: E402

c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = torch.device("cuda")
NS = 3
sets = []
for si in range(NS):
    kr = synth.retrieval_keys(B, G, S, D, seed=si + 1, device=dev)
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=si + 1, device=dev)
    sets.append((kr, kc, vc))
qr = synth.retrieval_queries(2, B, Hq, G, D, seed=1, device=dev)
ql = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
H2, G2 = Hq // 2, G // 2


def half(t, h, dim):  # contiguous half along dim
    n = t.shape[dim] // 2
    return t.narrow(dim, h * n, n).contiguous()


# full step
full = DecodeStep(sets[0][0], [sets[0][1][l] for l in range(L)], [sets[0][2][l] for l in range(L)],
                  seq, L, Hq, k)
for si in range(1, NS):
    full.add_input_set(sets[si][0], [sets[si][1][l] for l in range(L)], [sets[si][2][l] for l in range(L)])
full.step(qr[0], ql)
full.capture()
# halves: views of the same caches (B = 1: group halves are contiguous)
halves = []
for h in range(2):
    kr0, kc0, vc0 = sets[0]
    st = DecodeStep(kr0[:, h * G2:(h + 1) * G2], [kc0[l][:, h * G2:(h + 1) * G2] for l in range(L)],
                    [vc0[l][:, h * G2:(h + 1) * G2] for l in range(L)], seq, L, H2, k)
    for si in range(1, NS):
        kr_, kc_, vc_ = sets[si]
        st.add_input_set(kr_[:, h * G2:(h + 1) * G2], [kc_[l][:, h * G2:(h + 1) * G2] for l in range(L)],
                         [vc_[l][:, h * G2:(h + 1) * G2] for l in range(L)])
    st.step(half(qr[0], h, 1), half(ql, h, 2))
    st.capture()
    halves.append(st)

s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
g_split = {}
for si in range(NS):
    for p in (0, 1):
        g = torch.cuda.CUDAGraph()
        s1.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=s1):
            fork = torch.cuda.Event()
            fork.record(s1)
            s2.wait_event(fork)
            halves[0].use_set(si)
            halves[0].enqueue(p, stream=s1)
            with torch.cuda.stream(s2):
                halves[1].use_set(si)
                halves[1].enqueue(p, stream=s2)
            join = torch.cuda.Event()
            join.record(s2)
            s1.wait_event(join)
        g_split[(si, p)] = g
torch.cuda.synchronize()


def time_it(run, n=60):
    for i in range(5):
        run(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        run(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


t_full = time_it(lambda i: full.graphs[(i % NS, i % 2)].replay())
t_split = time_it(lambda i: g_split[(i % NS, i % 2)].replay())
print(f"full step {t_full:.1f} us, two half-steps on two streams {t_split:.1f} us")
