"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv
--print-source sass` export (tools only): python tools/sass_hot.py file.csv [N]."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
# per-reason columns (ncu names them after the reason) -- print the ones present
reason_cols = [h for h in hdr if h not in ("Address", "Source") and h.lower().replace(" ", "_") in hdr]
top = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:n]
for r in top:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{s / tot * 100:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")
