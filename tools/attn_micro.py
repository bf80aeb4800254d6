"""Microbenchmark: spc_sparse_decode_attn bandwidth vs the access pattern of the selected rows
(contiguous rows, scattered top-k-like rows at various densities), plus library references
(torch copy, torch index_select of the same rows).  Prints one line per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_00722_b200 import build, spc, synth  # noqa: E402

_lib_arg = [a for a in sys.argv if a.startswith("--lib=")]
if _lib_arg:  # a debug build of libspc (tools/ only)
    spc._lib = spc.load_library(_lib_arg[0][6:])
elif "--nomath" in sys.argv:  # the kernel's load pipeline alone (debug build, tools/ only)
    _so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspc_nomath.so")
    if not os.path.exists(_so):
        build.build(out=_so, defines=["SPC_ATTN_NOMATH"])
    spc._lib = spc.load_library(_so)

dev = torch.device("cuda")
L, B, G, Hq, D, S, k = 32, 1, 8, 32, 128, 32768, 2048
kc, vc = synth.llm_kv(L, B, G, S, D, seed=1, device=dev)
q = synth.llm_queries(1, L, B, Hq, D, seed=1, device=dev)[0]
ktab = spc.ptr_table([kc[l] for l in range(L)], dev)
vtab = spc.ptr_table([vc[l] for l in range(L)], dev)
out = torch.zeros((L, B, Hq, D), dtype=torch.float32, device=dev)
lse = torch.zeros((L, B, Hq), dtype=torch.float32, device=dev)
ws = spc.alloc_workspace(spc.attn_workspace(L, B, Hq, D, k), dev)
cnt = torch.full((B, G), k, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
nbytes = L * B * G * k * D * 2 * 2


def timeit(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        flush.view(torch.int64).sum()  # evict by reading: leaves no dirty lines in L2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] * 1e-3


def run(idx):
    return lambda: spc.sparse_decode_attn(q, ktab, vtab, spc.KV_INDEXED, idx, cnt, S, k, 0.088,
                                          out, lse, ws, G)


cases = {}
cases["contiguous rows 0..k-1"] = torch.arange(k, dtype=torch.int32, device=dev).repeat(B, G, 1)
for stride in (2, 4, 16):
    cases[f"strided rows (every {stride})"] = (torch.arange(k, device=dev) * stride).to(
        torch.int32).repeat(B, G, 1)
g = torch.Generator(device=dev).manual_seed(0)
for dens in (0.0625, 0.25):
    n = int(k / dens)
    r = torch.stack([torch.sort(torch.randperm(n, generator=g, device=dev)[:k])[0]
                     for _ in range(B * G)]).view(B, G, k).to(torch.int32)
    cases[f"random sorted rows, density {dens}"] = r
for name, idx in cases.items():
    t = timeit(run(idx))
    print(f"attn  {name:36s} {t*1e6:8.1f} us  {nbytes/t/1e9:8.1f} GB/s")
# library references
src = kc.view(-1, D)
rows = cases["random sorted rows, density 0.0625"]
flat = (rows.view(B * G, k).long() + torch.arange(B * G, device=dev)[:, None] * S).view(-1)
dst = torch.empty((flat.numel(), D), dtype=kc.dtype, device=dev)
t = timeit(lambda: torch.index_select(src[: B * G * S], 0, flat, out=dst))
print(f"torch index_select same rows (1 layer K)   {t*1e6:8.1f} us  {flat.numel()*D*2*2/t/1e9:8.1f} GB/s (r+w)")
a = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
bb = torch.empty_like(a)
t = timeit(lambda: bb.copy_(a))
print(f"torch copy 1 GiB                           {t*1e6:8.1f} us  {2*a.numel()/t/1e9:8.1f} GB/s (r+w)")
t = timeit(lambda: a.sum(dtype=torch.int64) if False else torch.sum(a.view(torch.int64)))
print(f"torch sum 1 GiB (read only)                {t*1e6:8.1f} us  {a.numel()/t/1e9:8.1f} GB/s")
# V allocation shifted by an odd multiple of 256 B relative to K (HBM channel/bank aliasing test)
for shift_bytes in (0, 256 * 4099, (1 << 20) + 256 * 3):
    big = torch.empty(vc.numel() + shift_bytes // 2 + 64, dtype=vc.dtype, device=dev)
    vs = big[shift_bytes // 2: shift_bytes // 2 + vc.numel()].view_as(vc)
    vs.copy_(vc)
    vtab_s = spc.ptr_table([vs[l] for l in range(L)], dev)
    idx = cases["random sorted rows, density 0.0625"]
    t = timeit(lambda: spc.sparse_decode_attn(q, ktab, vtab_s, spc.KV_INDEXED, idx, cnt, S, k, 0.088,
                                              out, lse, ws, G))
    print(f"attn  V shifted by {shift_bytes:9d} B, dens 1/16      {t*1e6:8.1f} us  {nbytes/t/1e9:8.1f} GB/s"
          f"  (K-V offset mod 2 MiB = {(vs.data_ptr() - kc.data_ptr()) % (2 << 20)})")
    del big, vs
# back-to-back launches (no flush in between: each launch still reads 268 MB > L2)
idx = cases["random sorted rows, density 0.0625"]
fn = run(idx)
for _ in range(3):
    fn()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    fn()
b.record()
torch.cuda.synchronize()
t = a.elapsed_time(b) * 1e-3 / 10
print(f"attn  10 back-to-back launches, dens 1/16     {t*1e6:8.1f} us  {nbytes/t/1e9:8.1f} GB/s")
