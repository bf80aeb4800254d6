"""Per-CUDA-line warp-stall samples and executed instructions from an ncu report (tools only):
python tools/ncu_lines.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    try:
        smp = float(r[4] or 0)
        ins = float(r[7] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, r[1].strip()])
    a[0] += smp
    a[1] += ins
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts:.0f}  warp-instructions {ti:.0f}")
for (f, ln), (smp, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{smp / ts * 100:5.1f}% smp {ins / ti * 100:5.1f}% ins  {f}:{ln:<4d} {src[:90]}")
