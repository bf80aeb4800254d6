"""Row-gather bandwidth microbenchmarks (tools/membench.cu).  Reads 2048*256 rows of 256 B
(config-B-sized: 128 MiB) at random sorted positions of a 4 GiB table."""
import ctypes
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmembench.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "membench.cu")):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-shared", "-Xcompiler", "-fPIC", "-O3",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-o", SO,
                           os.path.join(HERE, "membench.cu")])
lib = ctypes.CDLL(SO)
lib.membench.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 2 + [ctypes.c_int] + [ctypes.c_void_p] * 2
dev = torch.device("cuda")
table_rows = 34 << 20  # 8.5 GiB of 256-B rows (hashed rows reach 32 x n_rows)
src = torch.empty((table_rows, 128), dtype=torch.bfloat16, device=dev)
n_rows = 2048 * 256 * (1 if "--sweep1" in sys.argv else 2)
g = torch.Generator(device=dev).manual_seed(0)
rows = torch.sort(torch.randperm(table_rows, generator=g, device=dev)[:n_rows])[0].to(torch.int32)
rows_seq = torch.arange(n_rows, dtype=torch.int32, device=dev)
sink = torch.zeros(4, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
nbytes = n_rows * 256


def run(mode, depth, ctas, threads, r):
    ts = []
    for i in range(8):
        flush.view(torch.int64).sum()  # read-based: leaves no dirty lines
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.membench(mode, depth, ctas, threads, src.data_ptr(), r.data_ptr(), n_rows,
                          sink.data_ptr(), torch.cuda.current_stream().cuda_stream)
        b.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        if i >= 2:
            ts.append(a.elapsed_time(b) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    return nbytes / t / 1e9


names = {0: "LDGSTS ring", 1: "LDG regs", 2: "TMA bulk/row", 3: "LDGSTS hashrow", 4: "LDG hashrow",
         5: "LDGSTS hash+contig", 6: "K+V stage pad272", 7: "K+V stage dense",
         8: "K+V pad272 + meta.ca"}
CASES = [(0, 3, 2, 128), (0, 3, 4, 128), (0, 4, 2, 256), (0, 6, 1, 256),
                                  (0, 3, 8, 64), (1, 4, 4, 256), (1, 8, 4, 256), (1, 16, 2, 256),
                                  (1, 8, 8, 256), (2, 2, 2, 128), (2, 4, 2, 128), (2, 4, 4, 64)]
if "--sweep5" in sys.argv:  # attention-shaped 8 KiB stages
    CASES = [(6, 3, 2, 128), (8, 3, 2, 128), (7, 3, 2, 128), (6, 2, 2, 128), (8, 2, 2, 128),
             (3, 3, 2, 128)]
if "--sweep4" in sys.argv:  # interleaved vs contiguous per-warp block ranges
    CASES = [(3, 3, 2, 128), (5, 3, 2, 128), (3, 6, 2, 128), (5, 6, 2, 128), (5, 3, 4, 128)]
if "--sweep3" in sys.argv:  # no index loads: rows computed in-kernel (density 1/32)
    CASES = [(3, d, c, t) for (d, c, t) in [(2, 2, 128), (3, 2, 128), (4, 2, 128), (6, 2, 128),
                                             (3, 1, 128), (6, 1, 128), (3, 4, 128), (2, 4, 128)]] + [
        (4, 4, 2, 128), (4, 8, 2, 128), (4, 16, 2, 128), (4, 8, 4, 128), (4, 16, 1, 128)]
if "--sweep2" in sys.argv:  # LDGSTS in-flight depth sweep (warps/SM x stages of 4 KiB)
    CASES = [(0, d, c, t) for (d, c, t) in [(3, 2, 128), (4, 2, 128), (6, 2, 128), (2, 4, 128),
                                             (3, 4, 128), (2, 6, 128), (4, 3, 128), (12, 1, 128),
                                             (6, 1, 256), (3, 2, 256), (2, 3, 256)]] + [
        (1, 4, 2, 128), (1, 8, 2, 128), (1, 16, 2, 128), (1, 4, 4, 128), (1, 8, 4, 128),
        (1, 4, 4, 256), (1, 8, 4, 256), (1, 4, 8, 256)]
for mode, depth, cps, threads in CASES:
    for label, r in ((("hash", rows),) if mode >= 3 else (("random", rows), ("seq", rows_seq))):
        try:
            bw = run(mode, depth, 148 * cps, threads, r)
            print(f"{names[mode]:14s} depth={depth:2d} ctas/SM={cps} thr={threads:3d} {label:6s} "
                  f"{bw:8.1f} GB/s")
        except AssertionError as e:
            print(names[mode], depth, cps, threads, "launch failed", e)
