"""Stall accounting of the dK/dV kernel from the MEMO_DKDV_PROF build
(MEMO_LIB_PATH=.../prof/libmemo.so): per 32-query step, cycles the MMA warp
waits for Q/dO tiles and for P/dS, and cycles compute warp 4 waits for S/dP and
spends producing P/dS.  python tools/dkdv_prof.py S H D"""
import ctypes as C
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def main(S, H, D):
    torch.manual_seed(0)
    h = H * D
    q, k, v, do = (torch.randn(S, h, device="cuda").to(torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda")
    sc = C.c_float(1.0 / math.sqrt(D))
    ws = torch.empty((_abi.lib.memo_attn_bwd_workspace_bytes(S, H, D) + 3) // 4, device="cuda")
    dqkv = torch.empty(S, 3 * h, device="cuda", dtype=torch.bfloat16)
    P = lambda t: C.c_void_p(t.data_ptr())
    buf = (C.c_ulonglong * 16)()
    _abi.check(_abi.lib.memo_attn_fwd(P(q), P(k), P(v), P(o), P(lse), S, H, D, sc, None))
    for it in range(2):
        _abi.lib.memo_debug_dkdv_prof(buf, 1)
        b = dqkv.data_ptr()
        _abi.check(_abi.lib.memo_attn_bwd(P(q), P(k), P(v), P(o), P(lse), P(do), P(ws), C.c_void_p(b),
                                          C.c_void_p(b + 2 * h), C.c_void_p(b + 4 * h), C.c_int64(3 * h),
                                          None, C.c_int64(0), S, H, D, sc, None))
        torch.cuda.synchronize()
    _abi.lib.memo_debug_dkdv_prof(buf, 0)
    steps = buf[4]
    names = ["mma_wait_qdo", "mma_wait_pds", "cmp_wait_sdp", "cmp_busy", "steps", "mma_total"]
    print({n: buf[i] for i, n in enumerate(names)})
    print("per step (cycles): MMA waits tiles %.1f, MMA waits P/dS %.1f, compute waits S/dP %.1f, "
          "compute busy %.1f (TMEM load+wait %.1f, tcgen05.st wait %.1f), MMA-warp total %.1f "
          "(ideal tensor time 512)" % (buf[0] / steps, buf[1] / steps, buf[2] / steps, buf[3] / steps,
                                        buf[6] / steps, buf[7] / steps, buf[5] / steps))
    tile_waits(buf)


def tile_waits(buf):
    print("Q/dO tile waits: first tile of each CTA %.0f cycles total (%.2f per step); later tiles: %d of %d waits "
          "over 200 cycles, %.0f cycles each on average" % (buf[8], buf[8] / max(buf[4], 1), buf[10], buf[11],
                                                            buf[9] / max(buf[10], 1)))
    print("  for those waits, issue -> arrival %.0f cycles on average; TMA producer waited %.0f cycles per tile "
          "for a free stage" % (buf[12] / max(buf[10], 1), buf[14] / max(buf[11], 1)))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
