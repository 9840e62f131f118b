"""Summarise an ncu --csv launch list of scripts/ncu_ab_decode.py: mean/min duration of the
dual-GEMM kernel per (shape, csplit) block, in the script's launch order."""
import csv
import sys
from statistics import mean

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6}
durs = [float(r[vi].replace(",", "")) * scale[r[ui]] for r in rows[1:] if "ffn_dual_gemm" in r[ki]]
labels = [ln.split()[1:] for ln in open(sys.argv[2]) if ln.startswith("MARK")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
per = len(durs) // len(labels)
for i, lab in enumerate(labels):
    blk = durs[i * per:(i + 1) * per][-reps:]
    print(" ".join(lab), "n", len(blk), "mean_us", round(mean(blk) / 1e3, 2), "min_us", round(min(blk) / 1e3, 2))
