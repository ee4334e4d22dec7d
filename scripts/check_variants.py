"""Bit-compare every variant library in scripts/variants/ with the oracle on
config-1-shaped and config-0 inputs (one subprocess per library)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O, paper_1802_09883_b200 as R
from inputs import synth
res = []
for cfg, n, G in ((0, 1 << 16, 16), (1, 1 << 22, 1024), (1, 1 << 24, 1024), (1, 1 << 22, 3000),
                  ("hot", 1 << 22, 1024), ("hot", 1 << 22, 16), ("hotneg", 1 << 22, 1024)):
    if cfg == 0:
        k, v = synth.generate(0, n=n)
    elif cfg in ("hot", "hotneg"):  # every row in one group, same-sign values: counters grow linearly
        k, v = synth.generate(1, n=n, n_groups=G)
        k[:] = 7
        v = np.abs(v) * (1 if cfg == "hot" else -1)
    else:
        k, v = synth.generate(1, n=n, n_groups=G)
    out = R.groupby_sum(torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda(), G, 3).cpu().numpy()
    rc, ref = O.groupby_sum(k, v, G, 3)
    bad = int((out.view(np.uint64) != ref.view(np.uint64)).sum())
    res.append(f"cfg{cfg} n={n} G={G}: {bad} mismatching groups")
print("; ".join(res))
''' % ROOT
for lib in sorted(glob.glob(os.path.join(ROOT, "scripts", "variants", "lib_*.so"))) + [None]:
    env = dict(os.environ)
    if lib:
        env["REPRO_B200_LIB"] = lib
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(os.path.basename(lib) if lib else "default", "->", r.stdout.strip() or r.stderr[-600:], flush=True)
