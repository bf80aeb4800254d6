"""Where the packed device exp (spc_exp2_dev) differs from the oracle's O3 (tools only)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2512_00722_b200 import spc
L = spc.lib()
L.spc_debug_exp.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_void_p]
lo, hi = 0x80000000, int(np.frombuffer(np.float32(-87.5).tobytes(), np.uint32)[0])
chunk = 1 << 24
x_d = torch.empty(chunk, dtype=torch.float32, device="cuda")
y = torch.empty(chunk, dtype=torch.float32, device="cuda")
nd = 0
for start in range(lo, hi + 1, chunk):
    n = min(chunk, hi + 1 - start)
    x = np.arange(start, start + n, dtype=np.uint64).astype(np.uint32).view(np.float32)
    x_d[:n].copy_(torch.from_numpy(x))
    L.spc_debug_exp(x_d.data_ptr(), y.data_ptr(), n, 1, None)
    want = oracle.exp_array(x).view(np.uint32)
    got = y[:n].cpu().numpy().view(np.uint32)
    bad = np.nonzero(got != want)[0]
    nd += len(bad)
    if len(bad):
        print(hex(start), len(bad), [(float(x[i]), hex(got[i]), hex(want[i]), int(i % 2)) for i in bad[:4]])
print("total differing", nd)
