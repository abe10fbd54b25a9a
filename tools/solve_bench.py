"""Time the FFT solve (blfls_solve through lsgrad_solve_fft) on device tensors:
python tools/solve_bench.py H W C B [reps]  -> ms per solve, effective GB/s (fold form)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1812_07122_b200 as P  # noqa: E402

h, w, c, b = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
g = torch.rand(b, c, h, w, device="cuda")
tx = torch.rand(b, c, h, w, device="cuda") - 0.5
ty = torch.rand(b, c, h, w, device="cuda") - 0.5
sp = P.SolveParams(1000.0, 0)
for _ in range(3):
    P.lsgrad_solve_fft(g, (tx, ty), sp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    P.lsgrad_solve_fft(g, (tx, ty), sp)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
planes = b * c
byts = planes * (16 * h * w + 4 * 8 * h * (w // 2 + 1))
print(f"solve {b}x{c}x{h}x{w}: {ms:.3f} ms, {byts / ms / 1e6:.0f} GB/s (fold-form algorithmic bytes)")
