import sys; sys.argv=['x']
exec(open('/root/repo/tools/membench.py').read().split('names = {')[0])
big = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
def run2(mode, depth, ctas, threads, r, nr, flush_mode):
    ts = []
    for i in range(8):
        if flush_mode == 'write': flush.fill_(i)
        elif flush_mode == 'read': big.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.membench(mode, depth, ctas, threads, src.data_ptr(), r.data_ptr(), nr, sink.data_ptr(), torch.cuda.current_stream().cuda_stream)
        b.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b) * 1e-3)
    t = sorted(ts)[len(ts)//2]
    return nr * 256 / t / 1e9, t
big_rows = torch.sort(torch.randperm(table_rows, generator=g, device=dev)[:8*n_rows])[0].to(torch.int32)
for fm in ('write', 'read', 'none'):
    for nr, r in ((n_rows, rows), (8*n_rows, big_rows)):
        for mode, depth, cps, thr in ((0, 3, 4, 128), (1, 8, 4, 256), (2, 2, 2, 128)):
            bw, t = run2(mode, depth, 148*cps, thr, r, nr, fm)
            print(f"flush={fm:5s} rows={nr:8d} mode={mode} {bw:8.1f} GB/s  {t*1e6:8.1f} us")
# read-only streaming reference
x = torch.empty(2 << 30, dtype=torch.uint8, device=dev)
for i in range(3): x.view(torch.int64).sum()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); x.view(torch.int64).sum(); b.record(); torch.cuda.synchronize()
print("torch sum 2GiB", 2*2**30/(a.elapsed_time(b)*1e-3)/1e9, "GB/s")
