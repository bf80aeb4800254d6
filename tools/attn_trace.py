"""Per-chunk timeline of CTA 0 of the attention kernel (config B)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_00722_b200 import spc, synth
dev = torch.device("cuda")
L, B, G, Hq, D, S, k = 32, 1, 8, 32, 128, 32768, 2048
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
ktab = spc.ptr_table([kc[l] for l in range(L)], dev); vtab = spc.ptr_table([vc[l] for l in range(L)], dev)
out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev); lse = torch.zeros((L, B, Hq), device=dev)
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
idx = (torch.arange(k, device=dev) * 16).to(torch.int32).repeat(B, G, 1)
tr = torch.zeros(256 * 4, dtype=torch.int64, device=dev)
lib = spc.lib(); lib.spc_debug_set_trace.argtypes = [ctypes.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rep in range(3):
    flush.fill_(rep)
    lib.spc_debug_set_trace(ctypes.c_void_p(tr.data_ptr()) if rep == 2 else None)
    torch.cuda.synchronize()
    spc.sparse_decode_attn(q, ktab, vtab, spc.KV_INDEXED, idx, cnt, S, k, 0.088, out, lse, ws, G)
    torch.cuda.synchronize()
t = tr.view(256, 4).cpu().numpy().astype("float64")
n = int((t[:, 0] > 0).sum())
t0 = t[0, 0]
print("chunk  issue_start issue_end  full_seen  released   (us from first issue)")
for i in range(n):
    print(f"{i:4d} " + " ".join(f"{(x - t0) / 1e3:10.2f}" for x in t[i]))
