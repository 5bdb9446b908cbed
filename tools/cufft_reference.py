"""Out-of-product speed sanity check: cuFFT (torch.fft) on the TCo639 rings.

Times rfft (grid -> Fourier) and irfft over every ring pair for 548 fields,
i.e. the FLOP work of the ring-FFT phase without the hemispheric fusion,
transposed layouts or Fourier-row packing.  Reported only for context
(profiles/); the product never calls cuFFT.
"""
import sys

import torch

T = int(sys.argv[1]) if len(sys.argv) > 1 else 639
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 548
rings = [4 * i + 16 for i in range(1, T + 2)]
xs = [torch.randn(2 * nf, n, dtype=torch.float64, device="cuda") for n in rings]
mcap = [min(T, (n - 1) // 2) for n in rings]
cs = [torch.fft.rfft(x, dim=1)[:, : m + 1].contiguous() for x, m in zip(xs, mcap)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("rfft (g2f)", lambda: [torch.fft.rfft(x, dim=1) for x in xs]),
                 ("irfft (f2g)", lambda: [torch.fft.irfft(c, n=n, dim=1) for c, n in zip(cs, rings)])):
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"cuFFT {name}: {e0.elapsed_time(e1) / 3:.2f} ms for TCo{T} x {nf} fields (both hemispheres)")
