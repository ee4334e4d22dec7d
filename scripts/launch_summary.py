"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, mean duration (us) and share of the reproducible step
(the non-reproducible atomicAdd baseline kernels k_base_* listed apart)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "").replace("repro::", "").replace("<unnamed>::", "")
        name = name.replace("unnamed>::", "").lstrip("<")
        agg[name].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
def aside(k):  # not part of the timed step: the atomicAdd baseline, input generation, the FP-rate probe, torch fills
    return "k_base" in k or "k_synth" in k or "k_fp_add_peak" in k or k.startswith("at::")


step = {k: v for k, v in agg.items() if not aside(k)}
total = sum(sum(v) for v in step.values())
print(f"{'kernel':48s} {'launches':>8s} {'avg_us':>10s} {'share_of_step':>13s}")
for k, v in sorted(step.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:48]:48s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v) / total:13.3f}")
base = {k: v for k, v in agg.items() if aside(k)}
if base:
    print("# not part of the step (atomicAdd baseline, input generator, FP add-rate probe, torch fills):")
    for k, v in base.items():
        print(f"{k[:48]:48s} {len(v):8d} {sum(v) / len(v):10.2f}")
