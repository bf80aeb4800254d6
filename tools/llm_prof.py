"""Profile one graph-replayed LLM decode step (config L shape, resident KV) under
`ncu --profile-from-start off`: the step is bracketed by cudaProfilerStart/Stop.
Also prints CUDA-event timings of the whole step and of a GEMM-only graph."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_00722_b200 import rope, spc, synth  # noqa: E402
from paper_2512_00722_b200.llm import LlmDecoder  # noqa: E402

dev = torch.device("cuda", 0)
c = dict(synth.LLAMA8B)
L, H, Hq, G, D, F, V = (c[x] for x in ("L", "H", "Hq", "G", "D", "F", "V"))
B = int(os.environ.get("B", "4"))
S0, k = int(os.environ.get("CTX", "32768")), 2048
Smax = S0 + 64
w = synth.llm_weights(L, H, Hq, G, D, F, V, 3, device=dev)
_, nw, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, 3, device=dev)
inv_r, ms = rope.yarn_inv_freq(D, factor=64.0, orig_ctx=2048)
ret = dict(emb=w["emb"], norm_w=nw, w_qk=w_qk, inv_freq=torch.from_numpy(inv_r).to(dev), mscale=ms)
kr = synth.retrieval_keys(B, G, Smax, D, seed=3, device=dev)
kc, vc = synth.llm_kv(L, B, G, Smax, D, seed=3, device=dev)
seq = torch.full((B,), S0 + 1, dtype=torch.int32, device=dev)
tok0 = synth.tokens(1, B, V, 3, device=dev)[0]
dec = LlmDecoder(w, c, ret, kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], seq, k)
dec.reset(tok0, seq.clone())
dec.step()
dec.capture()
for _ in range(6):
    dec.step(use_graph=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    dec.step(use_graph=True)
e1.record()
torch.cuda.synchronize()
print("step ms", e0.elapsed_time(e1) / 10)

# GEMM-only graph: the same torch.mm calls
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for l in range(L):
            torch.mm(dec.xn, w["w_qkv"][l].t(), out=dec.qkv)
            torch.mm(dec.a, w["w_o"][l].t(), out=dec.o)
            torch.mm(dec.xn, w["w_gu"][l].t(), out=dec.gu)
            torch.mm(dec.y, w["w_down"][l].t(), out=dec.o)
        torch.mm(dec.xn, w["lm_head"].t(), out=dec.logits)
torch.cuda.current_stream().wait_stream(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
gm = e0.elapsed_time(e1) / 10
print("gemm-only ms", gm, "GB/s", dec.weight_bytes() / gm / 1e6)
# each GEMM shape alone
for name, Wt, x, o in (("qkv", w["w_qkv"][0], dec.xn, dec.qkv), ("o", w["w_o"][0], dec.a, dec.o),
                       ("gu", w["w_gu"][0], dec.xn, dec.gu), ("down", w["w_down"][0], dec.y, dec.o),
                       ("lm_head", w["lm_head"], dec.xn, dec.logits)):
    Ws = [w[{"qkv": "w_qkv", "o": "w_o", "gu": "w_gu", "down": "w_down"}[name]][l]
          for l in range(L)] if name != "lm_head" else [Wt]
    for _ in range(2):
        for W_ in Ws:
            torch.mm(x, W_.t(), out=o)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        for W_ in Ws:
            torch.mm(x, W_.t(), out=o)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / (3 * len(Ws))
    print(f"{name}: {t*1e3:.1f} us  {Wt.numel()*2/t/1e6:.0f} GB/s")
if os.environ.get("PROF"):
    torch.cuda.cudart().cudaProfilerStart()
    dec.step(use_graph=True)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
