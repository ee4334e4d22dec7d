"""Print a markdown table from a bench.py JSON line or a .jsonl sweep."""
import json
import sys


def row(name, v):
    r = v.get("roofline") or {}
    b = v.get("baseline_atomic") or {}
    p = v.get("parity") or {}
    sl = b.get("slowdown_repro_vs_atomic")
    return (f"| {name} | {v.get('ms_per_step', 0):.3f} | {v.get('value', 0):.3e} | {r.get('kernel')} {r.get('kernel_ms') or 0:.3f} ms = "
            f"{100 * (r.get('frac') or 0):.1f}% | {100 * (v.get('step_roofline_frac') or 0):.1f}% | "
            f"{'%.2fx (%s)' % (sl, b.get('variant')) if sl else '-'} | {p.get('vs_oracle')} ({p.get('groups')} groups) |")


print("| Workload | ms/step | rows/s | dominant kernel vs HBM peak | step vs HBM roofline | repro / atomicAdd time | parity |")
print("|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    c = d.get("config", {})
    print(row(f"config {c.get('workload', '?').split(':')[0].replace('config', '')} G={c.get('n_groups')}", d))
    for k, v in (d.get("configs") or {}).items():
        print(row(k, v))
