"""Reading R4 statistics (SURVEY §8(c) "Full-entropy data ... reported against the
plain mode as statistics (not a gate)"): the GPU output on full-entropy inputs
against (a) the fold-aware oracle -- the gate every parity test applies -- and
(b) the plain fp64 definition (g applied to x, not folded into bf16 weights).

    python scripts/plain_vs_fold_stats.py [--out profiles/r01/plain_vs_fold.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs

CASES = [("C", 2048, 4096, 11008, 64), ("C", 16, 4096, 11008, 16), ("L", 2048, 4096, 11008, 64),
         ("C", 4096, 8192, 3584, 32), ("A", 2048, 4096, 11008, 64), ("B", 2048, 4096, 11008, 64)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows_out = []
    for fam, M, K, N, nrows in CASES:
        d = make_inputs(M, K, N, family=fam, seed=9100 + M, dtype="bf16")
        t = {k: v.to(dev) for k, v in d.items()}
        out = ffn.FusedFFN(dev).forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
        torch.cuda.synchronize()
        rows = sorted(set(np.linspace(0, M - 1, nrows).astype(int).tolist()))
        got = out[rows].double().cpu().numpy()
        rec = {"family": fam, "M": M, "K": K, "N": N, "rows_checked": len(rows), "elements": got.size}
        for mode in ("fold_bf16", "plain"):
            ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode=mode, rows=rows)
            worst, nbad, maxerr = oracle.tolerance_ratio(got, ref)
            rec[mode] = {"worst_err_over_tol": round(worst, 4), "violations": nbad,
                         "violation_frac": nbad / got.size, "max_abs_err": maxerr}
        rows_out.append(rec)
        print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"note": "fold_bf16 is the parity gate (reading R4); plain is statistics only",
                       "tolerance": "|gpu - ref| <= 2e-2 |ref| + 1e-3", "rows": rows_out}, f, indent=1)


if __name__ == "__main__":
    main()
