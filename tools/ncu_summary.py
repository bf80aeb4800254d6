"""Summarise ncu output for profiles/: a launch list CSV (gpu__time_duration.sum) -> a markdown
table of per-kernel shares, and a --set full report -> a JSON of key metrics per kernel plus
the DRAM traffic per launch (profiles/traffic.json).  Tools only.

  python tools/ncu_summary.py launches <launches.csv> <out.md> "<title>"
  python tools/ncu_summary.py full <report.ncu-rep> <out.json> [traffic.json]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


LIBSPC = re.compile(r"spc::|unnamed>::|anonymous namespace")


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("spc::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")


def launches(path, out, title):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    acc = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        if not LIBSPC.search(r[ki]):  # libspc kernels only (not torch set-up / spin kernels)
            continue
        acc.setdefault(short(r[ki]), []).append(float(r[vi].replace(",", "")) / 1e3)
    total = sum(sum(v) / len(v) for v in acc.values())
    lines = [f"# {title}", "",
             "ncu serialises launches and runs them cold; compare SHARES, not absolute times.", "",
             "| kernel | launches | mean us | share of step |", "|---|---|---|---|"]
    for k, v in acc.items():
        m = sum(v) / len(v)
        lines.append(f"| {k} | {len(v)} | {m:.2f} | {100 * m / total:.1f}% |")
    lines.append(f"| **sum of means** | | {total:.2f} | 100% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kern = []
    per = defaultdict(list)
    for r in rows[2:]:
        d = {"Kernel Name": short(r[hdr.index("Kernel Name")])}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)]
        kern.append(d)
        rb = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
        wb = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        scale = {"Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Gbyte": 1e9}
        ur = units[hdr.index("dram__bytes_read.sum")]
        uw = units[hdr.index("dram__bytes_write.sum")]
        per[d["Kernel Name"]].append(rb * scale.get(ur, 1) + wb * scale.get(uw, 1))
    json.dump({"source": rep, "units": {k: units[hdr.index(k)] for k in KEYS if k in hdr},
               "kernels": kern}, open(out, "w"), indent=1)
    print(json.dumps({k: [round(x) for x in v] for k, v in per.items()}, indent=1))
    if traffic:
        t = json.load(open(traffic))
        for k, v in per.items():
            if "attn_bf16" in k:
                t["attn"] = round(sum(v) / len(v))
            elif "logits_kernel" in k:
                t["logits"] = round(sum(v) / len(v))
            elif "select_kernel" in k:
                t["select"] = round(sum(v) / len(v))
        t["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one "
                       f"`ncu --set full --clock-control none` capture ({rep}); see {out}")
        json.dump(t, open(traffic, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
