"""fragmentation of a caching allocator vs the static plan
(paper Fig. 1, reference allocator.hpp), on the executor's OWN request trace.

  python tools/frag_compare.py [cfg2|cfg1p] > profiles/frag_r01.json

Three numbers for the same tensor sequence (transients, carries and the
skeletal activations, each malloc'ed / freed in trace order):
  * reference simulator: `ref_probe frag <trace> 0` = the reference CLI's
    `frag` (actmem.cpp:194-225) with an unbounded capacity: caching-allocator
    peak reserved / allocated / fragmentation vs the planned arena;
  * real allocator: the same sequence replayed through PyTorch's CUDA caching
    allocator on this GPU (torch.empty / del), peak reserved and allocated;
  * MEMO as executed: arena (bi-level plan of the trace) + the two rounding
    buffers that hold the skeletal activations of the layers on device (the
    rest live in pinned host memory), i.e. the activation part of the single
    cudaMalloc.
The trace keeps every layer's skeletal tensors resident from forward to
backward (no offload), so the caching numbers are what the same step costs
without MEMO's swap; the arena alone is the transient part.
"""
import json
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200.executor import Executor  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = {
    "cfg2": (4, 4096, 32, 11008, 32000, 131072),
    "cfg1p": (4, 256, 4, 768, 512, 4096),
}


def torch_replay(trace_text):
    import torch
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    base_res = torch.cuda.memory_reserved()
    live = {}
    for line in trace_text.splitlines():
        if not line or line.startswith("#"):
            continue
        op, tid, nbytes = line.split()
        if op == "malloc":
            live[tid] = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        else:
            del live[tid]
    torch.cuda.synchronize()
    out = {"peak_reserved": torch.cuda.max_memory_reserved() - base_res,
           "peak_allocated": torch.cuda.max_memory_allocated(),
           "allocator": "torch " + torch.__version__ + " CUDA caching allocator (default settings)"}
    live.clear()
    torch.cuda.empty_cache()
    return out


def main(name="cfg2"):
    n, h, H, inter, V, S = CONFIGS[name]
    cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=inter * 3 // 2, n_heads=H, vocab=V, seq_len=S,
                        untied_classifier=True)
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=126 * P.GiB, gpu_mem=180 * 10 ** 9, peak_flops=2.25e15)
    ex = Executor(cfg, hw, dry_run=1, alpha=0.5)
    info = ex.info()
    trace = ex.trace_text()
    res = {"config": name, "arena_bytes": info["arena_bytes"], "rounding_buffer_bytes": info["rb_bytes"],
           "memo_activation_bytes": info["arena_bytes"] + 2 * info["rb_bytes"]}
    probe = os.path.join(ROOT, "oracle", "_ref", "ref_probe")
    if os.path.exists(probe):
        with tempfile.NamedTemporaryFile("w", suffix=".trace", delete=False) as f:
            f.write(trace)
        try:
            res["reference_simulator"] = json.loads(
                subprocess.check_output([probe, "frag", f.name, "0"], text=True))
        finally:
            os.unlink(f.name)
    try:
        import torch
        if torch.cuda.is_available():
            res["torch_caching_allocator"] = torch_replay(trace)
    except ImportError:
        pass
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))
