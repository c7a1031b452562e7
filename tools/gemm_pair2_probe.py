"""GEMM variant 5 (two CTA pairs per cluster sharing B) against variant 4 (one
CTA pair) bitwise and against fp32 torch, on ragged shapes (M not a multiple
of the 512-row cluster unit).  python tools/gemm_pair2_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_variants_probe import gemm  # noqa: E402


def main():
    torch.manual_seed(1)
    for (M, N, K) in [(512, 256, 128), (1024, 512, 192), (640, 288, 512), (200, 768, 256), (2048, 1024, 1024)]:
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.5).to(torch.bfloat16)
        ref = A.float() @ B.float().t()
        out = {}
        for variant in (4, 5):
            c = torch.zeros(M, N, device="cuda")
            gemm(M, N, K, A, K, 0, B, K, 0, c, variant)
            torch.cuda.synchronize()
            out[variant] = c
        err = ((out[5] - ref).abs().max() / (1 + ref.abs().max())).item()
        print(M, N, K, "bitwise equal to pair:", torch.equal(out[4], out[5]), "rel err", f"{err:.2e}", flush=True)
        assert err < 1e-3


if __name__ == "__main__":
    main()
