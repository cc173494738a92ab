"""Summarize ncu outputs into profiles/ (markdown).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv --out profiles/x.md
"""

import argparse
import csv
import io
import subprocess
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps act %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def short(name):
    return name.split("(")[0].replace("void ", "")[:48]


def rep_table(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    out = ["| kernel | " + " | ".join(f"{lab} ({units[idx[m]]})" for m, lab in METRICS if m in idx) + " |",
           "|---|" + "---|" * len(idx)]
    for r in rows[2:]:
        out.append(f"| {short(r[hdr.index('Kernel Name')])} | " +
                   " | ".join(r[idx[m]] for m, _ in METRICS if m in idx) + " |")
    return "\n".join(out)


def launch_table(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rdr = csv.reader(lines)
    hdr = next(rdr)
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    for r in rdr:
        if r[mn] != "gpu__time_duration.sum":
            continue
        k = short(r[kn])
        tot[k] += float(r[mv].replace(",", ""))
        cnt[k] += 1
    all_t = sum(tot.values()) or 1.0
    out = ["| kernel | launches | total | share |", "|---|---|---|---|"]
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| {k} | {cnt[k]} | {t:,.0f} | {100 * t / all_t:.1f}% |")
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--title", default="")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    parts = [f"# {a.title}\n"]
    if a.launches:
        parts.append("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, "
                     "serialized: compare shares)\n\n" + launch_table(a.launches) + "\n")
    if a.rep:
        parts.append("## ncu --set full (per captured launch)\n\n" + rep_table(a.rep) + "\n")
    with open(a.out, "w") as fh:
        fh.write("\n".join(parts))


if __name__ == "__main__":
    main()
