"""cuBLAS DGEMM (torch.matmul float64) throughput probe: the library FP64 reference point."""
import json
import torch

def main():
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(5):
            e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_tflops"] = 2 * n ** 3 / (best * 1e-3) / 1e12
    # sustained: back to back for ~4 s
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    k = 0
    while True:
        torch.matmul(a, b); k += 1
        if k % 10 == 0:
            e1.record(); torch.cuda.synchronize()
            if e0.elapsed_time(e1) > 4000:
                break
    out["dgemm_8192_sustained_tflops"] = 2 * n ** 3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps(out))

if __name__ == "__main__":
    main()
