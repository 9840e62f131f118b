"""Per-CTA timeline of the dual-GEMM kernel (CUASM_OPT_TRACE) for a few shapes.

Prints, relative to the earliest CTA entry of the launch (microseconds):
entry spread, first TMA issue, last TMA issue, last MMA issue, epilogue start
(after griddepcontrol.wait, i.e. after the pre-pass finished if PDL overlapped),
epilogue done and exit -- min / median / max over CTAs.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

SLOTS = ["entry", "first_tma", "last_tma", "last_mma", "epi_start", "epi_done", "exit", "last_tfull",
         "first_tfull", "first_epi_done", "last_flags", "last_epi_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="2048x4096x11008,16x4096x11008")
    ap.add_argument("--json", default=None)
    ap.add_argument("--op", default="ffn", choices=["ffn", "gemm"], help="gemm: cuasm_gemm_act (identity)")
    ap.add_argument("--scheds", default="0,1")
    ap.add_argument("--bns", default="0", help="SwiGLU tile widths (CUASM_OPT_TILE_BN), 0 = auto")
    ap.add_argument("--talls", default="0", help="CUASM_OPT_TALL values (0 auto, 1 off, 2 on)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    wbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rbuf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    report = {}
    for shp in a.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 1, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        for sched, bn, tall in [(s_, b_, t_) for s_ in map(int, a.scheds.split(",")) for b_ in map(int, a.bns.split(","))
                                for t_ in map(int, a.talls.split(","))]:
            pdl = 1
            h = ffn.FusedFFN(dev)
            h.set_option(ffn.OPT_PDL, pdl)
            h.set_option(ffn.OPT_SCHEDULE, sched)
            h.set_option(ffn.OPT_TILE_BN, bn)
            h.set_option(ffn.OPT_TALL, tall)
            is_tall = tall == 2 or (tall == 0 and ffn.plan_config(M, K, N)[0] == "tall")
            floor = (4 * (bn or ffn.plan_config(M, K, N)[4]) * (1.5 if is_tall else 1.0) if a.op == "ffn" else 512)
            def run():
                if a.op == "ffn":
                    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
                else:
                    h.gemm_act(t["x"], t["w1"], "identity", 0.0, out=out)
            for _ in range(3):
                run()
            h.set_option(ffn.OPT_TRACE, 1)
            if not os.environ.get("NOFLUSH"):  # NOFLUSH=1: code and operands stay in L2 (cold-code A/B)
                wbuf.zero_()
                rbuf.sum()
            torch.cuda.synchronize()
            torch.cuda._sleep(int(1e8))
            run()
            tr = h.trace_read().double()
            h.close()
            t0 = tr[:, 0][tr[:, 0] > 0].min()
            rows = {}
            if os.environ.get("EPI_DIAG"):  # library built with -DCUASM_DIAG=1: final-tile epilogue phases
                e = tr[:, 12:15]
                e = e[e[:, 0] > 0]
                print(f"   epilogue cycles after tfull (flags, pair 0 done, pair 1 done): med "
                      f"{e.median(0).values.tolist()} max {e.max(0).values.tolist()}")
                tr[:, 12:16] = 0
            cyc, kbs = tr[:, 12], tr[:, 13]
            sel = kbs > 1
            if sel.any():
                cpk = cyc[sel] / (kbs[sel] - 1)
                span_ns = (tr[:, 3] - tr[:, 1])[sel]
                ghz = cyc[sel] / span_ns.clamp(min=1)
                print(f"   cycles per k-block (MMA issue, leader CTAs): min {cpk.min():.0f} med {cpk.median():.0f} "
                      f"max {cpk.max():.0f}  (tcgen05 floor: {floor}); implied SM clock med {ghz.median():.3f} GHz")
                wf = tr[:, 14][sel] / (kbs[sel] - 1)
                wt = tr[:, 15][sel] / (kbs[sel] - 1)
                print(f"   MMA-thread wait per k-block: full (data) med {wf.median():.0f} cyc, "
                      f"tempty (accumulator) med {wt.median():.0f} cyc")
                rows["wait_full_per_kblock_med"] = round(wf.median().item(), 1)
                rows["cycles_per_kblock_med"] = round(cpk.median().item(), 1)
                rows["sm_ghz_med"] = round(ghz.median().item(), 3)
            for i, name in enumerate(SLOTS):
                col = tr[:, i]
                col = col[col > 0]
                if col.numel() == 0:
                    continue
                rel = (col - t0) / 1e3
                rows[name] = {"min": round(rel.min().item(), 2), "med": round(rel.median().item(), 2),
                              "max": round(rel.max().item(), 2)}
            key = (f"{a.op} {shp} schedule={['auto', 'data-parallel', 'stream-k-all', 'stream-k-tail'][sched]}"
                   f" bn={bn or 'auto'}" + (f" tall={tall}" if tall else ""))
            report[key] = rows
            print(key)
            for name, r in rows.items():
                if isinstance(r, dict):
                    print(f"   {name:10s} min {r['min']:8.2f}  med {r['med']:8.2f}  max {r['max']:8.2f} us")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
