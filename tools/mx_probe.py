"""Quick timing probe of the two contraction cores through ns_symm_product (includes padding/copies)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr  # noqa: E402


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    dev = torch.device("cuda:0")
    A = torch.randn(d, d, dtype=torch.float64, device=dev)
    A = (A + A.T) * (0.5 / d ** 0.5)
    for prec, name in ((nsr.NS_PREC_FP64_OZAKI, "ozaki_i8"), (nsr.NS_PREC_MIXED_BF16X3, "bf16x3"),
                       (nsr.NS_PREC_FP64, "fp64")):
        ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(d, prec), dev)
        C = torch.empty_like(A)
        for mode in (0, 2):
            nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=prec)
            torch.cuda.synchronize()
            t = time.perf_counter()
            n = 3
            for _ in range(n):
                nsr.ns_symm_product(A, A, mode=mode, C=C, ws=ws, prec=prec)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t) / n * 1e3
            flops = d ** 3 * (1 if mode == 0 else 2)
            print(f"{name} mode {mode} d={d}: {ms:.2f} ms/call  ({flops / ms / 1e9:.1f} TFLOP/s algorithmic incl. "
                  f"overheads; x3 split GEMMs = {3 * flops / ms / 1e9:.1f} TFLOP/s bf16 executed)", flush=True)
        ref = A @ A
        print(name, "max rel err", float((C - ref).abs().max() / ref.abs().max()))


if __name__ == "__main__":
    main()
