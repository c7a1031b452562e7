"""Vendor yardstick for the attention kernels: torch SDPA (cuDNN / flash backends) and FlashAttention-4
(vllm's CuTe-DSL build, deterministic and not) causal fwd+bwd at the bench shapes, timed with CUDA
events.  Library kernels, measured only to place ours.

usage: python tools/bench_sdpa.py S [S...]   (H=32, D=128, bf16)
"""
import json
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel


def run(S, H=32, D=128, iters=3):
    q, k, v = (torch.randn(1, H, S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3))
    do = torch.randn(1, H, S, D, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * S * S * H * D
    out = {"S": S, "H": H, "D": D}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                o.backward(do)
                torch.cuda.synchronize()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                tf = tb = 0.0
                for _ in range(iters):
                    e[0].record()
                    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                    e[1].record()
                    o.backward(do)
                    e[2].record()
                    torch.cuda.synchronize()
                    tf += e[0].elapsed_time(e[1])
                    tb += e[1].elapsed_time(e[2])
                tf /= iters
                tb /= iters
            out[name] = {"fwd_ms": tf, "fwd_tflops": fl / tf / 1e9, "bwd_ms": tb, "bwd_tflops_4units": 2 * fl / tb / 1e9}
        except Exception as ex:  # noqa: BLE001
            out[name] = str(ex)[:120]
        q.grad = k.grad = v.grad = None
    qq, kk, vv = (t.detach().transpose(1, 2).contiguous().requires_grad_(True) for t in (q, k, v))
    dd = do.transpose(1, 2).contiguous()
    for det in (False, True):
        name = "fa4_det" if det else "fa4"
        try:
            from vllm.vllm_flash_attn.cute import flash_attn_func as fa4
            o = fa4(qq, kk, vv, causal=True, deterministic=det)
            o = o[0] if isinstance(o, tuple) else o
            o.backward(dd)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            tf = tb = 0.0
            for _ in range(iters):
                e[0].record()
                o = fa4(qq, kk, vv, causal=True, deterministic=det)
                o = o[0] if isinstance(o, tuple) else o
                e[1].record()
                o.backward(dd)
                e[2].record()
                torch.cuda.synchronize()
                tf += e[0].elapsed_time(e[1])
                tb += e[1].elapsed_time(e[2])
            tf /= iters
            tb /= iters
            out[name] = {"fwd_ms": tf, "fwd_tflops": fl / tf / 1e9, "bwd_ms": tb, "bwd_tflops_4units": 2 * fl / tb / 1e9}
        except Exception as ex:  # noqa: BLE001
            out[name] = (type(ex).__name__ + ": " + str(ex))[:200]
        qq.grad = kk.grad = vv.grad = None
    return out


if __name__ == "__main__":
    for s in sys.argv[1:] or ["32768"]:
        print(json.dumps(run(int(s))), flush=True)
