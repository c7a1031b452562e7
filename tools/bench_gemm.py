"""Micro-benchmark of the tcgen05 GEMM at the cfg2 layer shapes (CUDA events)."""
import ctypes as C
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def run(M, N, K, layout, iters=10):
    if layout == "fwd":
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16); B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        lda, amn, ldb, bmn = K, 0, K, 0
    elif layout == "dgrad":
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16); B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        lda, amn, ldb, bmn = K, 0, N, 1
    else:
        A = torch.randn(K, M, device="cuda").to(torch.bfloat16); B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        lda, amn, ldb, bmn = M, 1, N, 1
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if layout != "wgrad" else torch.float32)
    args = _abi.GemmArgsC()
    args.M, args.N, args.K = M, N, K
    args.a, args.lda, args.a_mn_major = A.data_ptr(), lda, amn
    args.b, args.ldb, args.b_mn_major = B.data_ptr(), ldb, bmn
    args.epilogue = 0 if layout != "wgrad" else 1
    args.c, args.ldc = out.data_ptr(), N
    # GEMM_VARIANT (this tool's switch): 0 product choice, 1 single CTA, 2 B-multicast
    # cluster, 3 2x2 cluster, 4 CTA pair (memo_gemm_args.variant)
    args.variant = int(os.environ.get("GEMM_VARIANT", "0"))
    args.raster = int(os.environ.get("GEMM_RASTER", "0"))  # 1: the round-1 tile order
    for _ in range(3):
        _abi.check(_abi.lib.memo_gemm(C.byref(args), None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        _abi.lib.memo_gemm(C.byref(args), None)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2.0 * M * N * K / ms / 1e9
    # torch/cuBLAS reference for context
    if layout == "fwd":
        f = lambda: torch.matmul(A, B.t())
    elif layout == "dgrad":
        f = lambda: torch.matmul(A, B)
    else:
        f = lambda: torch.matmul(A.t(), B)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms_ref = e0.elapsed_time(e1) / iters
    return {"M": M, "N": N, "K": K, "layout": layout, "ms": ms, "tflops": tf,
            "cublas_ms": ms_ref, "cublas_tflops": 2.0 * M * N * K / ms_ref / 1e9}


if __name__ == "__main__":
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    only = os.environ.get("GEMM_ONLY")  # comma-separated shape indices
    # GEMM_MODEL=13b: the Llama-13B layer shapes (h 5120, f 13824) instead of 7B's
    h, f = (5120, 13824) if os.environ.get("GEMM_MODEL") == "13b" else (4096, 11008)
    shapes = [(S, 3 * h, h, "fwd"), (S, 2 * f, h, "fwd"), (S, h, f, "fwd"),
              (S, h, 3 * h, "dgrad"), (S, h, 2 * f, "dgrad"),
              (h, f, S, "wgrad"), (3 * h, h, S, "wgrad")]
    for i, (M, N, K, lay) in enumerate(shapes):
        if only and str(i) not in only.split(","):
            continue
        print(json.dumps(run(M, N, K, lay)), flush=True)
