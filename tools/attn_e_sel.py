"""Config E (1M tokens, P = 1): the attention launch timed with the step's own selection vs a
random selection of the same size on the same cache (tools only)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import dist as sdist  # noqa: E402
from paper_2512_00722_b200 import spc, synth  # noqa: E402

dev = torch.device("cuda")
c = synth.CONFIGS["E"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
kr = synth.retrieval_keys(B, G, S, D, seed=7, device=dev)
kc, vc = synth.llm_kv(L, B, G, S, D, seed=7, device=dev)
qr = synth.retrieval_queries(2, B, Hq, G, D, seed=synth.BASE_SEED, device=dev)
ql = synth.llm_queries(1, L, B, Hq, D, seed=synth.BASE_SEED, device=dev)[0]
scale = float(torch.tensor(1.0 / math.sqrt(D), dtype=torch.float32))
st = sdist.ShardState(0, 1, [S], kr, [kc[l] for l in range(L)], [vc[l] for l in range(L)], qr[0].clone(),
                      ql, k, scale)
ops = sdist.SpcOps()
sel, out, lse = sdist.run_emulated(ops, [st])
pos, cnt = sel[0][0], sel[0][1]
torch.cuda.synchronize()
p = pos.view(-1, k)[0].cpu()
print("count", cnt.view(-1).tolist()[:8], "first rows", p[:12].tolist(), "last", p[-8:].tolist())
gaps = (p[1:] - p[:-1]).float()
print(f"row gaps: median {gaps.median().item():.0f}, <= 4: {(gaps <= 4).float().mean().item() * 100:.1f}%")
g = torch.Generator(device="cpu").manual_seed(0)
rnd = torch.stack([torch.sort(torch.randperm(S, generator=g)[:k])[0] for _ in range(B * G)]).view(B, G, k)
rnd = rnd.to(torch.int32).to(dev)
desc = spc.KvDesc([kc[l] for l in range(L)], [vc[l] for l in range(L)])
o = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev)
ls = torch.zeros((L, B, Hq), dtype=torch.float32, device=dev)
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
for name, ix in (("step selection", pos), ("random rows", rnd), ("step selection", pos)):
    for rep in range(2):
        torch.cuda._sleep(20_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(10):
            spc.sparse_decode_attn_kv(desc, ql, spc.KV_INDEXED, ix, cnt, k, scale, o, ls, ws)
        b.record()
        torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) * 100:.1f} us per launch")
