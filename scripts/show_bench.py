"""Print one line per bench JSON file: value, step, roofline fraction, back-to-back."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f"{path}: unreadable ({e})")
        continue
    r = d.get("roofline") or {}
    b = d.get("back_to_back") or {}
    c = d.get("clocks") or {}
    print(f"{path.split('/')[-1]:30s} {d['value']:9.2f} {d['unit']:8s} step {d['ms_per_step'] * 1e3:8.2f} us "
          f"frac {r.get('frac', 0):.3f} | b2b {b.get('value')} step {b.get('ms_per_step')} "
          f"sus {b.get('frac_of_sustained_peak')} L={b.get('layer_copies')} | {c.get('sm_mhz')} {c.get('reasons')}")
