"""Print DESIGN.md §7's measurement numbers from profiles/r01 (bench JSON lines, ncu summary)
so the tables are regenerated from the committed evidence instead of retyped."""
import json
import os

R = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r01")


def L(f):
    with open(os.path.join(R, f)) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def main():
    for f in sorted(os.listdir(R)):
        if f.startswith("bench_") and f.endswith(".json") and "reference" not in f:
            d = L(f)
            r = d.get("roofline") or {}
            b = d.get("back_to_back") or {}
            print(f"{f:55s} iso {d['ms_per_step'] * 1e3:9.1f} us  {d['value']:10.2f} {d['unit']:8s} "
                  f"roof {r.get('achieved')} ({r.get('frac')})  b2b {b.get('value')} @ {b.get('ms_per_step')} ms "
                  f"sus {b.get('frac_of_sustained_peak')}  clk {(d.get('clocks') or {}).get('sm_mhz')}")
    for w in ("llama7b_prefill", "llama70b", "llama7b_decode"):
        base = L(f"bench_{w}.json")["ms_per_step"]
        row = []
        for P in (2, 4, 8):
            t = L(f"bench_{w}_shard{P}.json")["ms_per_step"]
            row.append(f"P={P}: {t * 1e3:.1f} us, eff {base / (P * t):.2f}")
        print(w, " | ".join(row))


if __name__ == "__main__":
    main()
