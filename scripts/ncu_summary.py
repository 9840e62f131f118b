"""Summarise ncu captures for profiles/ (run here, on the CPU host).

    python scripts/ncu_summary.py gpurun_out/prof_gemm_r01.ncu-rep [--launches gpurun_out/launches_r01.csv]

Prints a JSON object with the metrics the roofline and DESIGN.md cite:
duration, SM clock, DRAM bytes read/written, tensor-pipe (UTCHMMA) utilisation,
SM-active vs elapsed cycles, L2 hit rate, registers, and -- with --launches --
each kernel's share of the per-step device time from the launch list.
"""
import argparse
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed":
        "tensor_utchmma_bf16_pct_of_peak_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed":
        "tensor_utchmma_tf32_pct_of_peak_elapsed",
    "sm__cycles_active.avg": "sm_active_cycles_avg",
    "sm__cycles_elapsed.avg": "sm_elapsed_cycles_avg",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__cluster_dim_x": "cluster_x",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_bytes",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct": "stall_long_scoreboard_pct",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
              "ms": 1e-3, "s": 1.0, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "cycle": 1, "%": 1, "": 1,
              "register/thread": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for i, name in enumerate(hdr):
            if name in KEYS:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[KEYS[name]] = v * UNIT_SCALE.get(units[i], 1)
                d[KEYS[name] + "_unit_raw"] = units[i]
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(list)
    for r in rows[i + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name].append(float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1))
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches")
    a = ap.parse_args()
    out = {"captures": []}
    for rep in a.reps:
        for d in raw(rep):
            d = {k: v for k, v in d.items() if not k.endswith("_unit_raw")}
            if "sm_active_cycles_avg" in d and "sm_elapsed_cycles_avg" in d:
                d["sm_active_frac"] = d["sm_active_cycles_avg"] / d["sm_elapsed_cycles_avg"]
            if "dram_read" in d and "dram_write" in d:
                d["dram_traffic_bytes"] = d["dram_read"] + d["dram_write"]
            d["source"] = rep
            out["captures"].append(d)
    if a.launches:
        tot = launches(a.launches)
        ours = {k: v for k, v in tot.items() if "cuasm::" in k}
        # per-step share among our kernels (skip the one-time pack)
        step = {k: v for k, v in ours.items() if "pack" not in k}
        per = {k: sum(v) / len(v) for k, v in step.items()}
        s = sum(per.values())
        out["launch_list"] = {k: {"launches": len(tot[k]), "mean_ns": per[k] * 1e9, "share_of_step": per[k] / s}
                              for k in per}
        out["launch_list_source"] = a.launches
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
