"""Attention fwd/bwd on fixed inputs, saved (mode save) or compared bitwise
against the saved outputs (mode check) -- for finding kernels whose results
change under a tool that perturbs timing (compute-sanitizer).
  python tools/attn_golden_probe.py save|check S H D out.pt"""
import ctypes as C
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def run(S, H, D):
    torch.manual_seed(0)
    h = H * D
    q, k, v, do = (torch.randn(S, h, device="cuda").to(torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda")
    sc = C.c_float(1.0 / math.sqrt(D))
    ws = torch.empty((_abi.lib.memo_attn_bwd_workspace_bytes(S, H, D) + 3) // 4, device="cuda")
    dqkv = torch.zeros(S, 3 * h, device="cuda", dtype=torch.bfloat16)
    P = lambda t: C.c_void_p(t.data_ptr())
    _abi.check(_abi.lib.memo_attn_fwd(P(q), P(k), P(v), P(o), P(lse), S, H, D, sc, None))
    b = dqkv.data_ptr()
    _abi.check(_abi.lib.memo_attn_bwd(P(q), P(k), P(v), P(o), P(lse), P(do), P(ws), C.c_void_p(b),
                                      C.c_void_p(b + 2 * h), C.c_void_p(b + 4 * h), C.c_int64(3 * h),
                                      None, C.c_int64(0), S, H, D, sc, None))
    torch.cuda.synchronize()
    return {"o": o.cpu(), "lse": lse.cpu(), "dqkv": dqkv.cpu()}


if __name__ == "__main__":
    mode, S, H, D, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    out = run(S, H, D)
    if mode == "save":
        torch.save(out, path)
    else:
        ref = torch.load(path)
        h = H * D
        for k in out:
            same = torch.equal(out[k], ref[k])
            msg = ""
            if not same:
                d = (out[k].float() - ref[k].float()).abs()
                if k == "dqkv":
                    msg = f" max|diff| dq/dk/dv {[round(x, 4) for x in d.view(S, 3, h).amax(dim=(0, 2)).tolist()]}"
                else:
                    msg = f" max|diff| {d.max().item():.4g}, rows differing {int((d.view(d.shape[0], -1).amax(1) > 0).sum())}"
            print(f"{k}: {'equal' if same else 'DIFFERS'}{msg}")
