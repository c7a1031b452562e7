"""Runs every GEMM kernel variant (memo_gemm_args.variant 1-5: single CTA,
2-CTA B-multicast cluster, 2x2 cluster, CTA pair) on the three operand layouts
at small ragged shapes and checks each against torch fp32.  Meant to run under
compute-sanitizer (tools/sanitize.sh): the clustered kernels' multicast TMA and
remote mbarrier arrivals are exercised on every layout."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def gemm(M, N, K, a, lda, amn, b, ldb, bmn, c, variant):
    args = _abi.GemmArgsC()
    args.M, args.N, args.K = M, N, K
    args.a, args.lda, args.a_mn_major = a.data_ptr(), lda, amn
    args.b, args.ldb, args.b_mn_major = b.data_ptr(), ldb, bmn
    args.epilogue = 1
    args.c, args.ldc = c.data_ptr(), N
    args.variant = variant
    _abi.check(_abi.lib.memo_gemm(C.byref(args), None))


def main():
    torch.manual_seed(0)
    worst = 0.0
    import hashlib
    h = hashlib.sha256()
    for (M, N, K) in [(200, 512, 192), (384, 768, 256), (640, 288, 512)]:
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.5).to(torch.bfloat16)
        At, Bt = A.t().contiguous(), B.t().contiguous()
        ref = A.float() @ B.float().t()
        for variant in (1, 2, 3, 4, 5):
            for lay, (a, lda, amn, b, ldb, bmn) in {"fwd": (A, K, 0, B, K, 0), "dgrad": (A, K, 0, Bt, N, 1),
                                                    "wgrad": (At, M, 1, Bt, N, 1)}.items():
                c = torch.zeros(M, N, device="cuda")
                gemm(M, N, K, a, lda, amn, b, ldb, bmn, c, variant)
                torch.cuda.synchronize()
                h.update(c.cpu().numpy().tobytes())
                err = ((c - ref).abs().max() / (1 + ref.abs().max())).item()
                worst = max(worst, err)
                assert err < 1e-3, (M, N, K, variant, lay, err)
    print(f"gemm variants ok, worst rel err {worst:.2e}")
    print(f"outputs sha256 {h.hexdigest()}")


if __name__ == "__main__":
    main()
