"""Debug: dynamic-fold data loss (round-2 edge tests)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O
import paper_1802_09883_b200 as R
import edge_values as EV

def run(keys, vals, G, K):
    try:
        out = R.groupby_sum(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), G, K)
        return 0, out.cpu().numpy()
    except R.ReproError as e:
        return e.status, None

b = np.float32(EV.below(2.0 ** -6, 32))
for n in (1 << 20, 1 << 24, (1 << 28) - 16, 1 << 28):
    keys = np.zeros(n, np.int32); vals = np.full(n, b, np.float32)
    for v in (0, 1, 3):
        R.set_kernel_variant(v)
        st, out = run(keys, vals, 40, 2)
        print("f32 n", n, "variant", v, "status", st, "out0", None if out is None else out[0], "expect", float(n) * float(b), flush=True)
    R.set_kernel_variant(0)
rng = np.random.default_rng(33)
for G in (33, 1024):
    n = 1 << 22
    keys = rng.choice(np.array([0, 1, G - 1], np.int32), n)
    vals = np.full(n, EV.below(EV.threshold(1, 64), 64), np.float64) * rng.uniform(0.9, 1.0, n)
    for big in (False, True):
        v2 = vals.copy()
        if big:
            v2[rng.integers(n // 2, n, 24)] = 2.0 ** 60
        rc, ref = O.groupby_sum(keys, v2, G, 3)
        for var in (1, 3):
            R.set_kernel_variant(var)
            st, out = run(keys, v2, G, 3)
            d = np.nonzero(out != ref)[0]
            print("f64 G", G, "big", big, "var", var, "status", st, "ndiff", d.size, [(int(g), out[g] - ref[g]) for g in d[:3]], flush=True)
        R.set_kernel_variant(0)
