"""Cycle accounting of the ping-pong attention forward from the MEMO_FWD_PROF build
(make -C paper_2407_12117_b200/csrc prof; MEMO_LIB_PATH=paper_2407_12117_b200/_lib_prof/libmemo.so),
per 128x128 tile and softmax group: cycles waiting for S, S ready -> first P release, S ready -> last
P release, release -> end of tile; and the MMA warp's waits for P and for K/V, per tile pair.
Variants of the ablation build are selected with MEMO_ATTN_FWD_VARIANT.
  python tools/fwd_prof.py S H"""
import ctypes as C
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def main(S, H, D=128):
    torch.manual_seed(0)
    h = H * D
    q, k, v = (torch.randn(S, h, device="cuda").to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda")
    sc = C.c_float(1.0 / math.sqrt(D))
    P = lambda t: C.c_void_p(t.data_ptr())
    buf = (C.c_ulonglong * 24)()
    _abi.check(_abi.lib.memo_attn_fwd(P(q), P(k), P(v), P(o), P(lse), S, H, D, sc, None))
    _abi.lib.memo_debug_fwd_prof(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _abi.check(_abi.lib.memo_attn_fwd(P(q), P(k), P(v), P(o), P(lse), S, H, D, sc, None))
    e1.record()
    torch.cuda.synchronize()
    _abi.lib.memo_debug_fwd_prof(buf, 0)
    out = {"variant": os.environ.get("MEMO_ATTN_FWD_VARIANT", "8"), "S": S, "H": H,
           "ms": round(e0.elapsed_time(e1), 2)}
    for g in (0, 1):
        n = max(buf[8 * g + 4], 1)
        out[f"g{g}"] = {"wait_S": round(buf[8 * g] / n, 1), "to_release0": round(buf[8 * g + 1] / n, 1),
                        "to_release": round(buf[8 * g + 2] / n, 1), "after_release": round(buf[8 * g + 3] / n, 1),
                        "tiles": n}
    pairs = max(buf[12], 1)  # tiles of group B = key-tile steps of the MMA warp
    out["mma"] = {"wait_P": round(buf[16] / pairs, 1), "wait_KV": round(buf[17] / pairs, 1),
                  "total": round(buf[18] / pairs, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 32768, int(sys.argv[2]) if len(sys.argv) > 2 else 32)
