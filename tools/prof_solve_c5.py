"""c5-shaped solve (24 planes of 2048^2: 8 RGB images), twice: the target of
an ncu capture of the row r2c / column / row c2r passes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1812_07122_b200 as P  # noqa: E402

n, h, w = (int(sys.argv[1]) if len(sys.argv) > 1 else 8), 2048, 2048
g = torch.rand((n, 3, h, w), device="cuda")
tx = (torch.rand_like(g) - 0.5) * 0.1
ty = (torch.rand_like(g) - 0.5) * 0.1
for _ in range(2):
    u = P.lsgrad_solve_fft(g, (tx, ty), P.SolveParams(1000.0, 0))
torch.cuda.synchronize()
print("ok", float(u.mean()))
