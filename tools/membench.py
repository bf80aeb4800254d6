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
table_rows = 16 << 20  # 4 GiB of 256-B rows
src = torch.empty((table_rows, 128), dtype=torch.bfloat16, device=dev)
n_rows = 2048 * 256
g = torch.Generator(device=dev).manual_seed(0)
rows = torch.sort(torch.randperm(table_rows, generator=g, device=dev)[:n_rows])[0].to(torch.int32)
rows_seq = torch.arange(n_rows, dtype=torch.int32, device=dev)
sink = torch.zeros(4, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
nbytes = n_rows * 256


def run(mode, depth, ctas, threads, r):
    ts = []
    for i in range(8):
        flush.fill_(i)
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


names = {0: "LDGSTS ring", 1: "LDG regs", 2: "TMA bulk/row"}
for mode, depth, cps, threads in [(0, 3, 2, 128), (0, 3, 4, 128), (0, 4, 2, 256), (0, 6, 1, 256),
                                  (0, 3, 8, 64), (1, 4, 4, 256), (1, 8, 4, 256), (1, 16, 2, 256),
                                  (1, 8, 8, 256), (2, 2, 2, 128), (2, 4, 2, 128), (2, 4, 4, 64)]:
    for label, r in (("random", rows), ("seq", rows_seq)):
        try:
            bw = run(mode, depth, 148 * cps, threads, r)
            print(f"{names[mode]:14s} depth={depth:2d} ctas/SM={cps} thr={threads:3d} {label:6s} "
                  f"{bw:8.1f} GB/s")
        except AssertionError as e:
            print(names[mode], depth, cps, threads, "launch failed", e)
