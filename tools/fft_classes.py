"""FFT phase time by ring class (dev tool): TCo639's ring lengths split into direct
(prime factors <= 16), DMMA-prime (one prime 17..127) and whole-ring Bluestein, each run as a
custom grid of just those rings (same T, same field count), FFT ms per direction and ns per point.
usage: python tools/fft_classes.py [T] [nfld]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1908_06097_b200 import SHTransform, fft_plan_info  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 639
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 548
north = [4 * i + 16 for i in range(1, T + 2)]
cls = {"direct": [], "dprime": [], "bluestein": []}
for n in north:
    M = min(T, (n - 1) // 2)
    info = fft_plan_info(n)
    if info["bluestein"]:
        cls["bluestein"].append(n)
    elif any(r > 16 for r in info["radices"]):
        cls["dprime"].append(n)
    else:
        cls["direct"].append(n)
for name, rings in cls.items():
    nl = np.array(rings + rings[::-1], dtype=np.int32)
    sh = SHTransform(T, grid=nl, nfld=nf, profile=True)
    spec = torch.randn(nf, sh.nspec_local, dtype=torch.float64, device="cuda")
    grid = torch.empty(nf, sh.npts_local, dtype=torch.float64, device="cuda")
    for _ in range(5):
        sh.inv_trans(spec, out=grid)
        sh.dir_trans(grid, out=spec)
    torch.cuda.synchronize()
    ph = sh.phase_ms(5)
    pts = 2 * sum(rings) * nf
    print(f"{name:10s} rings {len(rings):4d} points/field {2 * sum(rings):8d}  f2g {ph['inv_fft']:7.3f} ms "
          f"g2f {ph['dir_fft']:7.3f} ms  ns/point f2g {ph['inv_fft'] * 1e6 / pts:.4f} g2f {ph['dir_fft'] * 1e6 / pts:.4f}",
          flush=True)
    sh.close()
