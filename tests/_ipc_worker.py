"""One rank of the CUDA-IPC peer-memory SP+TP step (kind 2), launched by
tests/test_tp_ipc_gpu.py as a separate process.  Handles are exchanged over a
gloo process group; the step's loss and gradients are written to an .npz."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port, outdir, spec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    spec = json.loads(spec)
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2407_12117_b200 import planner as P
    from paper_2407_12117_b200.executor import KIND_IPC, Executor

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n, h, H, F, V, S = spec["dims"]
    cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=F * 3 // 2, n_heads=H, vocab=V, batch=1, seq_len=S,
                        dtype_bytes=2, tp_degree=world, untied_classifier=True)
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=64 * P.GiB, gpu_mem=180 * 10 ** 9, peak_flops=2.25e15,
                          efficiency=0.5)
    toks, labels = O.tokens(spec["data_seed"], V, S)
    ocfg = O.make_cfg(n, h, H, F, V, S)
    with Executor(cfg, hw, tp=(KIND_IPC, None, rank), **spec["opts"]) as ex:
        handles = [None] * world
        dist.all_gather_object(handles, ex.peer_handle())
        ex.peer_connect(handles)
        losses = [ex.step(toks, labels) for _ in range(spec.get("steps", 1))]
        out = {"loss": np.array(losses, dtype=np.float32), "peer_flags": np.array(ex.peer_flags(), dtype=np.uint64)}
        for name, layer, _, _ in O.layout(ocfg):
            out[f"{name}:{layer}"] = ex.read("grad/" + name, layer)
    dist.barrier()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
