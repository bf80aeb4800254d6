"""FMA throughput of the LOGITS inner-loop mix per SM (tools/ffma_bench.cu)."""
import ctypes, os, subprocess, torch
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libffma.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-shared", "-Xcompiler", "-fPIC", "-O3", "-gencode",
                       "arch=compute_100a,code=sm_100a", "-o", SO, os.path.join(HERE, "ffma_bench.cu")])
lib = ctypes.CDLL(SO)
lib.ffma_bench.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 2
out = torch.zeros(148 * 1024, device="cuda")
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
iters = 4096
for rpt, mode in ((2, 0), (4, 0), (8, 0), (4, 1)):
    for warps in (1, 2, 4, 8, 16):
        lib.ffma_bench(rpt, mode, warps, iters, out.data_ptr(), cyc.data_ptr())
        torch.cuda.synchronize()
        c = cyc.float().mean().item()
        fma = iters * 8 * 4 * rpt * 32 * warps  # per SM (one CTA per SM)
        print(f"rpt={rpt} mode={'FFMA2' if mode == 0 else 'FFMA '} warps/SM={warps:2d}  "
              f"{fma / c:7.1f} FMA/clk/SM")
