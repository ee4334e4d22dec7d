"""Time the keyless SUM / dot kernels (repro_dot_async) on 2^27 elements."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1802_09883_b200 as R
from inputs import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
keys = torch.empty(n, dtype=torch.int32, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
x.uniform_(-1, 1); y.uniform_(-1, 1)
x.mul_(torch.exp2(torch.randint(-20, 21, (n,), device="cuda").double()))
ws = torch.empty(R.dot_workspace_bytes(3, R.F64) + 256, dtype=torch.uint8, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.empty(1, dtype=torch.float64, device="cuda")
for name, yy, nb in (("sum", None, 8), ("dot", y, 16)):
    for _ in range(5):
        R.dot_async(x, yy, 3, out, ws, st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(50):
        R.dot_async(x, yy, 3, out, ws, st)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 50
    print(f"{name}: {ms:.4f} ms/call  {n * nb / ms / 1e6:.0f} GB/s  status={st.item()}")
    # plain torch reference speed
    a.record()
    for _ in range(50):
        (x.sum() if yy is None else torch.dot(x, yy))
    b.record()
    torch.cuda.synchronize()
    print(f"  torch {name}: {a.elapsed_time(b) / 50:.4f} ms")
