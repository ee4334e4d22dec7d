"""Repeat one GroupBy many times and count distinct outputs / oracle mismatches
(race detector for kernel variants).  REPRO_B200_LIB selects the library."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_1802_09883_b200 as R
from inputs import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
k, v = synth.generate(1, n=n, n_groups=G)
rc, ref = O.groupby_sum(k, v, G, 3)
kd, vd = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
outs = set()
bad = []
for it in range(20):
    o = R.groupby_sum(kd, vd, G, 3).cpu().numpy()
    outs.add(o.tobytes())
    bad.append(int((o.view(np.uint64) != ref.view(np.uint64)).sum()))
print(f"n={n} G={G}: {len(outs)} distinct outputs over 20 runs; mismatches per run {bad}")
