"""Per-chunk timeline of CTA 0 of the attention kernel (config B)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_00722_b200 import build, spc, synth
_so = os.environ.get("SPC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspc_trace.so")
if not os.path.exists(_so):
    build.build(out=_so, defines=["SPC_TRACE"])
spc._lib = spc.load_library(_so)
dev = torch.device("cuda")
L, B, G, Hq, D, S, k = 32, 1, 8, 32, 128, 32768, 2048
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
ktab = spc.ptr_table([kc[l] for l in range(L)], dev); vtab = spc.ptr_table([vc[l] for l in range(L)], dev)
out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev); lse = torch.zeros((L, B, Hq), device=dev)
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
g_ = torch.Generator(device=dev).manual_seed(0)
idx = torch.sort(torch.randperm(S, generator=g_, device=dev)[:k])[0].to(torch.int32).repeat(B, G, 1)
tr = torch.zeros(1024 + 1024 * 4 * 2, dtype=torch.int64, device=dev)
lib = spc.lib(); lib.spc_debug_set_trace.argtypes = [ctypes.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rep in range(3):
    flush.fill_(rep)
    lib.spc_debug_set_trace(ctypes.c_void_p(tr.data_ptr()) if rep == 2 else None)
    torch.cuda.synchronize()
    spc.sparse_decode_attn(q, ktab, vtab, spc.KV_INDEXED, idx, cnt, S, k, 0.088, out, lse, ws, G)
    torch.cuda.synchronize()
allt = tr.cpu().numpy().astype("float64")
t = allt[:1024].reshape(256, 4)
wt = allt[1024:].reshape(1024 * 4, 2)
wt = wt[wt[:, 0] > 0]
w0 = wt[:, 0].min()
st, en = (wt[:, 0] - w0) / 1e3, (wt[:, 1] - w0) / 1e3
import numpy as np  # noqa: E402
print(f"warps traced {len(wt)}: start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} us; "
      f"end min/med/p90/max {en.min():.2f}/{np.median(en):.2f}/{np.percentile(en, 90):.2f}/{en.max():.2f} us")
dur = en - st
print(f"per-warp busy time min/med/max {dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f} us")
cta_end = en.reshape(-1, 4).max(1) if len(en) % 4 == 0 else en
order = np.argsort(cta_end)[::-1][:8]
print("slowest CTAs (index: start, end):", [(int(i), round(float(st.reshape(-1, 4)[i].min()), 2), round(float(cta_end[i]), 2)) for i in order])
n = int((t[:, 0] > 0).sum())
t0 = t[0, 0]
print("chunk   issued(i+2)   landed(i)   computed(i)  flush-synced(i)  (us from the first stamp)")
for i in range(n):
    print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:10.2f}" if x > 0 else "         -" for x in t[i]))
d = t[1:n]
print("mean per chunk: wait for rows %.3f us, compute %.3f us, issue %.3f us" % (
    ((d[:, 1] - d[:, 0]) / 1e3).mean(), ((d[:, 2] - d[:, 1]) / 1e3).mean(),
    ((d[:, 0] - t[0:n - 1, 2]) / 1e3).mean()))
