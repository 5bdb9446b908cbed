"""Developer parity check on a GPU box: SHTransform vs the CPU oracle.

usage: python tools/dev_check.py T nfld [T nfld ...]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.sht_oracle import SHTransformOracle, random_grid, random_spectral  # noqa: E402
from paper_1908_06097_b200 import SHTransform  # noqa: E402


def relerr(x, ref):
    return float(np.max(np.max(np.abs(x - ref), axis=1) / np.max(np.abs(ref), axis=1)))


def run(T, nfld):
    t0 = time.time()
    o = SHTransformOracle(T, nfld=nfld)
    t1 = time.time()
    sh = SHTransform(T, nfld=nfld, profile=True)
    torch.cuda.synchronize()
    t2 = time.time()
    a = random_spectral(T, nfld)
    g = random_grid(T, nfld, o.npts)
    ga = o.inv_trans(a)
    ad = o.dir_trans(g)
    t3 = time.time()
    da = torch.from_numpy(a).cuda()
    dg = torch.from_numpy(g).cuda()
    gg = sh.inv_trans(da)
    sa = sh.dir_trans(dg)
    rt = sh.dir_trans(gg)
    torch.cuda.synchronize()
    e_inv = relerr(gg.cpu().numpy(), ga)
    e_dir = relerr(sa.cpu().numpy(), ad)
    e_rt = relerr(rt.cpu().numpy(), a)
    print(f"T={T} nfld={nfld}: inv {e_inv:.3e} dir {e_dir:.3e} roundtrip {e_rt:.3e} | oracle setup {t1-t0:.2f}s"
          f" gpu setup {t2-t1:.2f}s oracle run {t3-t2:.2f}s  phases {sh.phase_ms()}", flush=True)
    return max(e_inv, e_dir, e_rt)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [79, 10]
    worst = 0.0
    for T, n in zip(args[0::2], args[1::2]):
        worst = max(worst, run(T, n))
    print("WORST", worst)
    sys.exit(0 if worst < 1e-10 else 1)
