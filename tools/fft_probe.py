"""Per-phase times of one configuration (dev tool).
usage: python tools/fft_probe.py [T] [nfld] [pairs] [recompute]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1908_06097_b200 import SHTransform  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 639
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 548
pairs = int(sys.argv[3]) if len(sys.argv) > 3 else 5
recompute = len(sys.argv) > 4 and sys.argv[4] == "recompute"
sh = SHTransform(T, nfld=nf, profile=True, recompute_legendre=recompute)
spec = torch.randn(nf, sh.nspec_local, dtype=torch.float64, device="cuda")
grid = torch.empty(nf, sh.npts_local, dtype=torch.float64, device="cuda")
for _ in range(pairs):
    sh.inv_trans(spec, out=grid)
    sh.dir_trans(grid, out=spec)
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in sh.phase_ms(pairs).items()})
