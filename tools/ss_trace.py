"""Phase timeline of spc_score_select (tools only): %globaltimer per CTA at each phase mark,
config-B shape, one launch after warm-up launches.  Marks: 1 entry, 2 LOGITS done,
3 barrier 1 passed, 4 NORM done, 5 barrier 2, 6 GROUP done, 7 barrier 3, 10 candidates
pushed, 8 leaders done, 11 row released, 9 writes done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2512_00722_b200 import spc, synth
c = synth.CONFIGS["B"]
B, G, Hq, D, S, L, k = c["B"], c["G"], c["Hq"], c["D"], c["S"], c["L"], c["k"]
dev = "cuda"
spc.lib().spc_debug_set_ss_time.argtypes = [ctypes.c_void_p]
krs = [synth.retrieval_keys(B, G, S, D, seed=3 + i, device=dev) for i in range(3)]
qr = synth.retrieval_queries(8, B, Hq, G, D, seed=3, device=dev)
seq = torch.full((B,), S, dtype=torch.int32, device=dev)
f32, i32 = torch.float32, torch.int32
z = lambda *s, dt=f32, fill=0: torch.full(s, fill, dtype=dt, device=dev)
ws = spc.alloc_workspace(spc.score_select_workspace(B, Hq, G, S), dev)
hm, F, gs = z(B, Hq), z(B, Hq, dt=torch.int64), z(B, G, S)
idx = [z(B, G, k, dt=i32, fill=-1) for _ in range(2)]
cnt = [z(B, G, dt=i32) for _ in range(2)]
lt, nl = z(B, G, k, dt=i32), z(B, G, dt=i32)
tt = torch.zeros(256 * 16, dtype=torch.int64, device=dev)
for s in range(8):
    cur, prev = s % 2, 1 - s % 2
    if s == 7:
        torch.cuda.synchronize()
        spc.lib().spc_debug_set_ss_time(tt.data_ptr())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    spc.score_select(qr[s], krs[s % 3], seq, 0.088, k, hm, F, gs, idx[cur], cnt[cur], idx[prev], cnt[prev],
                     lt, nl, ws, force_last=True)
    b.record()
    torch.cuda.synchronize()
    print(f"launch {s}: {a.elapsed_time(b) * 1e3:.1f} us")
spc.lib().spc_debug_set_ss_time(None)
t = tt.view(256, 16).cpu().numpy().astype(np.float64)[:148]
t0 = t[:, 1].min()
for m, name in [(1, "entry"), (2, "LOGITS done"), (3, "barrier 1"), (4, "NORM done"), (5, "barrier 2"),
                (6, "GROUP done"), (7, "barrier 3"), (10, "cands pushed"), (8, "leaders done"),
                (11, "row released"), (9, "writes done")]:
    v = (t[:, m] - t0) / 1e3
    print(f"{name:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
