"""Micro-benchmark of the tcgen05 attention kernels (CUDA events); causal FLOPs = 2*S^2*h (fwd)."""
import ctypes as C
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import _abi  # noqa: E402


def bench(S, H, D, iters=5, bwd=False):
    q = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    k = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    v = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda")
    sc = C.c_float(1.0 / math.sqrt(D))
    f = lambda: _abi.lib.memo_attn_fwd(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                       C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), S, H, D, sc, None)
    _abi.check(f())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = 2.0 * S * S * H * D  # causal half of 4*S^2*h
    out = {"S": S, "H": H, "D": D, "fwd_ms": ms, "fwd_tflops": flops / ms / 1e9}
    try:
        if os.environ.get("MEMO_NO_FA2"):
            raise RuntimeError("skipped (MEMO_NO_FA2)")
        from flash_attn import flash_attn_func
        qq, kk, vv = (t.view(1, S, H, D) for t in (q, k, v))
        flash_attn_func(qq, kk, vv, causal=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            flash_attn_func(qq, kk, vv, causal=True)
        e1.record()
        torch.cuda.synchronize()
        out["flash_attn2_tflops"] = flops / (e0.elapsed_time(e1) / iters) / 1e9
    except Exception as ex:  # noqa: BLE001
        out["flash_attn2"] = str(ex)[:80]
    if bwd and hasattr(_abi.lib, "memo_attn_bwd"):
        do = torch.randn_like(q)
        delta = torch.empty((_abi.lib.memo_attn_bwd_workspace_bytes(S, H, D) + 3) // 4, device="cuda")
        dqkv = torch.empty(S, 3 * H * D, device="cuda", dtype=torch.bfloat16)
        g = lambda: _abi.lib.memo_attn_bwd(
            C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()),
            C.c_void_p(lse.data_ptr()), C.c_void_p(do.data_ptr()), C.c_void_p(delta.data_ptr()),
            C.c_void_p(dqkv.data_ptr()), C.c_void_p(dqkv.data_ptr() + 2 * H * D),
            C.c_void_p(dqkv.data_ptr() + 4 * H * D), C.c_int64(3 * H * D), None, C.c_int64(0), S, H, D, sc, None)
        _abi.check(g())
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            g()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        out["bwd_ms"] = ms
        out["bwd_tflops_algo"] = 2.5 * flops / ms / 1e9
        ms3 = (C.c_float * 3)()
        _abi.check(_abi.lib.memo_attn_bwd_timed(
            C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()),
            C.c_void_p(lse.data_ptr()), C.c_void_p(do.data_ptr()), C.c_void_p(delta.data_ptr()),
            C.c_void_p(dqkv.data_ptr()), C.c_void_p(dqkv.data_ptr() + 2 * H * D),
            C.c_void_p(dqkv.data_ptr() + 4 * H * D), C.c_int64(3 * H * D), None, C.c_int64(0), S, H, D, sc, None, ms3))
        out["prep_ms"], out["dkdv_ms"], out["dq_ms"] = list(ms3)
        if D == 128 and os.environ.get("MEMO_ATTN_BWD") == "fused":
            out["fused_tflops_algo"] = 2 * flops / ms3[1] / 1e9  # model bwd FLOPs (4 S^2 h)
            out["fused_tflops_exec"] = 2.5 * flops / ms3[1] / 1e9  # 5 GEMM units executed
        else:
            out["dkdv_tflops"] = 2 * flops / ms3[1] / 1e9
            out["dq_tflops"] = 1.5 * flops / ms3[2] / 1e9
    return out


if __name__ == "__main__":
    for S in [int(x) for x in (sys.argv[1:] or ["8192", "32768"])]:
        print(json.dumps(bench(S, 32, 128, bwd=True)), flush=True)
    # variant sweeps run on the ablation library (make -C paper_2407_12117_b200/csrc ablations)
    abl = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2407_12117_b200",
                       "_lib_ablations", "libmemo.so")
    if os.environ.get("MEMO_FWD_SWEEP"):
        import subprocess
        for v in range(4):
            env = dict(os.environ, MEMO_ATTN_FWD_VARIANT=str(v), MEMO_LIB_PATH=abl)
            env.pop("MEMO_FWD_SWEEP")
            out = subprocess.check_output([sys.executable, __file__, sys.argv[-1]], env=env, text=True)
            r = json.loads(out.strip().splitlines()[0])
            print(json.dumps({"variant": v, "S": r["S"], "fwd_tflops": r["fwd_tflops"]}), flush=True)
    if os.environ.get("MEMO_DQ_SWEEP"):
        import subprocess
        for v in range(2):
            env = dict(os.environ, MEMO_ATTN_DQ_TMEM_A=str(v), MEMO_LIB_PATH=abl)
            env.pop("MEMO_DQ_SWEEP")
            out = subprocess.check_output([sys.executable, __file__, sys.argv[-1]], env=env, text=True)
            r = json.loads(out.strip().splitlines()[0])
            print(json.dumps({"dq_tmem_a": v, "S": r["S"], "dq_ms": r["dq_ms"], "dq_tflops": r["dq_tflops"]}), flush=True)
