"""bench.py's JSON-line contract, run end to end on the GPU (short runs).

The driver parses one JSON line per run; these tests pin the keys it reads
(metric/value/unit/n_gpus/steps/warmup/ms_per_step/higher_is_better/scaling/
vs_baseline/dtype/data/config, roofline, cpu_baseline, e2e, gpu_launches,
clocks) for the default workload and for the reference arm.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_default_line_carries_the_contract_keys():
    d = run_bench("--steps", "5", "--warmup", "3", "--cpu-budget-s", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["unit"] == "TFLOP/s" and d["value"] > 0
    assert d["config"]["workload"] == "llama7b_prefill"
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.5
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2048 * 4096 * 2
    assert e["d2h_bytes_per_step"] == 2048 * 11008 * 2
    assert d["gpu_launches"] >= 5
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["back_to_back"]["value"] > 0
    # a1 runs inside the GEMM by default: no field may be derived from an empty pre-pass span
    assert "prepass_GBps" not in r and "gemm_share_of_step" not in r and "prepass" in r
    ps = d["prepass_standalone"]
    assert ps["kernel"] == "ffn_rms_prepass_kernel" and 0 < ps["frac_of_hbm"] < 1.2
    pr = d["protocol_5x100"]
    assert pr["runs"] == 5 and len(pr["ms_per_step_runs"]) == 5 and pr["value_mean"] > 0


def test_fp32_e2e_bytes_use_the_element_size():
    d = run_bench("--workload", "tiny_fp32", "--steps", "5", "--warmup", "3", "--skip-cpu-baseline",
                  "--skip-b2b", "--protocol-runs", "0")
    assert d["e2e"]["h2d_bytes_per_step"] == 16 * 64 * 4 and d["e2e"]["d2h_bytes_per_step"] == 16 * 128 * 4


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-budget-s", "4")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["e2e"] == {"value": d["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]


def test_decode_roofline_is_hbm_bound():
    d = run_bench("--workload", "llama7b_decode", "--steps", "5", "--warmup", "3", "--skip-cpu-baseline",
                  "--skip-e2e", "--skip-b2b")
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["unit"] == "GB/s"


def test_tuned_bench_line_records_the_search():
    d = run_bench("--workload", "llama7b_decode", "--steps", "5", "--warmup", "3", "--skip-cpu-baseline",
                  "--skip-e2e", "--skip-b2b", "--protocol-runs", "0", "--tune")
    t = d["config"]["tuned"]
    assert t["plan"][0] in ("1sm", "2sm", "tall") and t["us_per_forward"] > 0 and t["candidates"] >= 10
    assert d["value"] > 0
