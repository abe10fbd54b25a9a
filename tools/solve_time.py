"""Time the FFT solve at one size: python tools/solve_time.py H W."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1812_07122_b200 as P  # noqa: E402

h, w = int(sys.argv[1]), int(sys.argv[2])
g = torch.rand(3, h, w, device="cuda")
tx = torch.rand(3, h, w, device="cuda") - 0.5
ty = torch.rand(3, h, w, device="cuda") - 0.5
sp = P.SolveParams(1000.0, 0)
for _ in range(3):
    P.lsgrad_solve_fft(g, (tx, ty), sp)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    P.lsgrad_solve_fft(g, (tx, ty), sp)
b.record()
torch.cuda.synchronize()
print(f"solve {h}x{w}x3: {a.elapsed_time(b) / 10:.3f} ms")
