"""cuBLAS DGEMM ceiling (torch.matmul on float64) -- practical FP64 reference.

Measurement-only; never on the product path.  Prints TFLOP/s (dense 2*d^3) for a
few sizes, best of N with CUDA events, plus nvidia-smi clocks.
"""
import subprocess
import sys

import torch


def main():
    dev = torch.device("cuda:0")
    torch.backends.cuda.matmul.allow_tf32 = False
    for d in [4096, 8192, 16384]:
        a = torch.randn(d, d, dtype=torch.float64, device=dev)
        b = torch.randn(d, d, dtype=torch.float64, device=dev)
        c = a @ b
        torch.cuda.synchronize()
        best = 1e30
        reps = 5 if d <= 8192 else 3
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b, out=c)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        tf = 2.0 * d ** 3 / (best * 1e-3) / 1e12
        print(f"cuBLAS DGEMM d={d}: {best:.2f} ms  {tf:.2f} TFLOP/s", flush=True)
        del a, b, c
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                          "--format=csv"], capture_output=True, text=True).stdout
    print(out)


if __name__ == "__main__":
    sys.exit(main())
