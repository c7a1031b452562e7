"""Micro-benchmark of the RMSNorm backward (memo_rmsnorm_bwd) at the bench's row
count, CUDA events; HBM bytes per call = x f32 + a bf16 + dy f32 + dres f32 in,
dx f32 + dx bf16 out (the executor's use), plus the dg partials.
  python tools/bench_norm.py [S] [h ...]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def run(S, h, iters=20):
    x, dy, dres = (torch.randn(S, h, device="cuda") for _ in range(3))
    a = torch.randn(S, h, device="cuda").to(torch.bfloat16)
    g = torch.randn(h, device="cuda").to(torch.bfloat16)
    dx = torch.empty(S, h, device="cuda")
    dxb = torch.empty(S, h, device="cuda", dtype=torch.bfloat16)
    part = torch.empty(_abi.lib.memo_rmsnorm_bwd_partials(S) * h, device="cuda")
    dg = torch.zeros(h, device="cuda")
    P = lambda t: C.c_void_p(t.data_ptr())
    f = lambda: _abi.lib.memo_rmsnorm_bwd(P(x), P(a), P(g), P(dy), P(dres), P(dx), P(dxb), P(part), P(dg), S, h,
                                          C.c_float(1e-5), 0, None)
    for _ in range(3):
        _abi.check(f())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    byts = S * h * (4 + 2 + 4 + 4 + 4 + 2)
    return {"S": S, "h": h, "ms": round(ms, 3), "TBps": round(byts / ms / 1e9, 2)}


if __name__ == "__main__":
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    for h in [int(v) for v in (sys.argv[2:] or ["4096", "5120"])]:
        print(json.dumps(run(S, h)), flush=True)
