"""Per-CTA timeline of the TMA attention kernel (tools only; -DSPC_TRACE build):
entry after the PDL wait, first stage landed, main loop done, exit -- relative to the
earliest entry.  Config-B shape, one launch after warm-up launches on rotated KV copies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_00722_b200 import build, spc, synth  # noqa: E402

so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspc_trace.so")
build.build(out=so, defines=["SPC_TRACE"])
spc._lib = spc.load_library(so)
import ctypes  # noqa: E402
spc.lib().spc_debug_set_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda")
L, B, G, Hq, D, S, k = 32, 1, 8, 32, 128, 32768, 2048
copies = []
for c in range(3):
    kc, vc = synth.llm_kv(L, B, G, S, D, seed=10 + c, device=dev)
    copies.append((kc, vc, spc.KvDesc([kc[l] for l in range(L)], [vc[l] for l in range(L)])))
q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
g = torch.Generator(device=dev).manual_seed(0)
idx = torch.sort(torch.rand(B, G, S, device=dev, generator=g).argsort(-1)[..., :k].to(torch.int32),
                 -1).values.contiguous()
cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev)
lse = torch.zeros((L, B, Hq), dtype=torch.float32, device=dev)
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
tr = torch.zeros(4096 + 2048 * 4, dtype=torch.int64, device=dev)
for it in range(8):
    if it == 7:
        torch.cuda.synchronize()
        spc.lib().spc_debug_set_trace(tr.data_ptr())
    spc.sparse_decode_attn_kv(copies[it % 3][2], q, spc.KV_INDEXED, idx, cnt, k, 0.088, out, lse, ws)
torch.cuda.synchronize()
spc.lib().spc_debug_set_trace(None)
t = tr[4096:].view(2048, 4).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
t = (t - t0) / 1e3
names = ["entry", "first stage", "loop done"]
for i, n in enumerate(names):
    v = t[:, i]
    print(f"{n:12s} min {v.min():7.2f}  p10 {np.percentile(v, 10):7.2f}  med {np.median(v):7.2f}  "
          f"p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f} us")
print("loop duration (done - first): med %.2f  min %.2f  max %.2f" % (
    np.median(t[:, 2] - t[:, 1]), (t[:, 2] - t[:, 1]).min(), (t[:, 2] - t[:, 1]).max()))
sm = np.arange(len(t)) % 148
