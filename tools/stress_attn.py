"""Repeat attention fwd/bwd on fixed inputs; report bitwise run-to-run mismatches
(races show up as nondeterminism).  python tools/stress_attn.py S H D [reps]"""
import ctypes as C
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def main(S, H, D, reps=30):
    torch.manual_seed(0)
    h = H * D
    q, k, v, do = (torch.randn(S, h, device="cuda").to(torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda")
    sc = C.c_float(1.0 / math.sqrt(D))
    ws = torch.empty((_abi.lib.memo_attn_bwd_workspace_bytes(S, H, D) + 3) // 4, device="cuda")
    dqkv = torch.empty(S, 3 * h, device="cuda", dtype=torch.bfloat16)
    P = lambda t: C.c_void_p(t.data_ptr())
    ref_o = ref_g = None
    bad_f = bad_b = 0
    for _ in range(reps):
        _abi.check(_abi.lib.memo_attn_fwd(P(q), P(k), P(v), P(o), P(lse), S, H, D, sc, None))
        dqkv.zero_()
        b = dqkv.data_ptr()
        _abi.check(_abi.lib.memo_attn_bwd(P(q), P(k), P(v), P(o), P(lse), P(do), P(ws), C.c_void_p(b),
                                          C.c_void_p(b + 2 * h), C.c_void_p(b + 4 * h), C.c_int64(3 * h),
                                          None, C.c_int64(0), S, H, D, sc, None))
        torch.cuda.synchronize()
        if ref_o is None:
            ref_o, ref_g = o.clone(), dqkv.clone()
            continue
        bad_f += int(not torch.equal(o, ref_o))
        if not torch.equal(dqkv, ref_g):
            bad_b += 1
            d = (dqkv.float() - ref_g.float()).abs().view(S, 3, h).amax(dim=(0, 2))
            print("  bwd mismatch max|diff| dq/dk/dv:", [round(x, 4) for x in d.tolist()])
    print(f"S={S} H={H} D={D}: fwd mismatches {bad_f}/{reps - 1}, bwd mismatches {bad_b}/{reps - 1}", flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
