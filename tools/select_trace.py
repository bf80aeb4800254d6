"""Phase timeline of spc_select (config B, row 0) from a -DSPC_TRACE build.  Not a bench."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import build, spc, synth  # noqa: E402

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspc_trace.so")
if not os.path.exists(out):
    build.build(out=out, defines=["SPC_TRACE"])
spc._lib = spc.load_library(out)
lib = spc._lib
lib.spc_debug_set_select_trace.argtypes = [ctypes.c_void_p]
cfg = sys.argv[1] if len(sys.argv) > 1 else "B"
c = synth.CONFIGS[cfg]
B, G, Hq, D, S, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["k"]
dev = torch.device("cuda")
kr = synth.retrieval_keys(B, G, S, D, seed=1, device=dev)
qs = synth.retrieval_queries(4, B, Hq, G, D, seed=1, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
f32, i32 = torch.float32, torch.int32
z = lambda *s, dt=f32: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
lg, hm, F, gs = z(B, Hq, S), z(B, Hq), z(B, Hq, dt=torch.int64), z(B, G, S)
ws = spc.alloc_workspace(spc.score_workspace(B, Hq, S), dev)
idx = [z(B, G, k, dt=i32) for _ in range(2)]
cnt = [z(B, G, dt=i32) for _ in range(2)]
lt, nl = z(B, G, k, dt=i32), z(B, G, dt=i32)
tr = torch.zeros(64 * 16 * 16, dtype=torch.int64, device=dev)
GX = int(os.environ.get("SCL", "16" if B * G <= 9 else "8"))  # CTAs per row used by the lib
names = ["start", "norm", "group", "pass0", "passes", "T", "cls_loop", "end", "cls_presync",
         "x_sync", "bitmap", "exp", "push", "h0_push", "h0_sync", "scan"]
for step in range(4):
    spc.score(qs[step], kr, seq, G, 0.088, lg, hm, F, gs, ws, phases=spc.SCORE_LOGITS)
    torch.cuda.synchronize()
    tr.zero_()
    lib.spc_debug_set_select_trace(ctypes.c_void_p(tr.data_ptr()) if step == 3 else None)
    spc.select(lg, hm, seq, G, k, F, gs, idx[step % 2], cnt[step % 2], idx[1 - step % 2],
               cnt[1 - step % 2], lt, nl, force_last=True)
    torch.cuda.synchronize()
GX = 8
t = tr[:64 * GX * 16].view(64, GX, 16).cpu().numpy().astype("float64")
order = [0, 10, 11, 12, 1, 2, 13, 14, 3, 4, 6, 8, 9, 5, 15, 7]
print("clock64 marks, us from each CTA's own start (1.965 GHz); row 0 and row 1")
print("rank " + " ".join(f"{names[i]:>8s}" for i in order))
for row in range(2):
    for r in range(GX):
        st = t[row, r, 0]
        print(f"{row}.{r:2d} " + " ".join(f"{(t[row, r, i] - st) / 1965.0:8.2f}" if t[row, r, i] > 0 else "       -"
                                       for i in order))
