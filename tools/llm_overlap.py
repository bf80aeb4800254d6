"""Offloaded-KV LLM decode (config L shape, trace queries): step time resident / serial /
prefetch, for the prefetch stream priority given in argv[1] (0 or -1).  The gather grid cap
comes from env SPC_GATHER_CTAS (read once per process)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_00722_b200 import rope, synth  # noqa: E402
from paper_2512_00722_b200.llm import LlmDecoder  # noqa: E402

prio = int(sys.argv[1]) if len(sys.argv) > 1 else -1
dev = torch.device("cuda", 0)
c = dict(synth.LLAMA8B)
L, H, Hq, G, D, F, V = (c[x] for x in ("L", "H", "Hq", "G", "D", "F", "V"))
B = int(os.environ.get("B", "4"))
S0, k = int(os.environ.get("CTX", "32768")), 2048
N = 20
Smax = S0 + 2 * N + 64
w = synth.llm_weights(L, H, Hq, G, D, F, V, 3, device=dev)
_, nw, w_qk = synth.retrieval_head_weights(V, H, Hq, G, D, 3, device=dev)
inv_r, ms = rope.yarn_inv_freq(D, factor=64.0, orig_ctx=2048)
ret = dict(emb=w["emb"], norm_w=nw, w_qk=w_qk, inv_freq=torch.from_numpy(inv_r).to(dev), mscale=ms)
kr = synth.retrieval_keys(B, G, Smax, D, seed=3, device=dev)
kh = [torch.empty((B, G, Smax, D), dtype=torch.bfloat16, pin_memory=True) for _ in range(L)]
vh = [torch.empty_like(t, pin_memory=True) for t in kh]
for l in range(L):
    kh[l].copy_(synth.normal_bf16((B, G, Smax, D), 100 + l, device=dev))
    vh[l].copy_(synth.normal_bf16((B, G, Smax, D), 200 + l, device=dev))
trace = synth.retrieval_queries(2 * N + 4, B, Hq, G, D, seed=3, device=dev)
seq = torch.full((B,), S0 + 1, dtype=torch.int32, device=dev)
tok0 = synth.tokens(1, B, V, 3, device=dev)[0]
for pf in (False, True):
    dec = LlmDecoder(w, c, ret, kr, kh, vh, seq, k, kv="offload", prefetch=pf, trace_queries=trace,
                     pf_priority=prio)
    dec.reset(tok0, torch.full((B,), S0 + 1, dtype=torch.int32, device=dev))
    dec.step()
    dec.capture()
    dec.reset(tok0, torch.full((B,), S0 + 1, dtype=torch.int32, device=dev))
    for _ in range(5):
        dec.step(use_graph=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(N):
        dec.step(use_graph=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"prio {prio} cap {os.environ.get('SPC_GATHER_CTAS', 'default')} prefetch {pf}: "
          f"{e0.elapsed_time(e1) / N:.3f} ms/step", flush=True)
    del dec
