"""Per-tensor gradient error at the bench's layer widths (the fullwidth fixture,
tests/golden/fullwidth_7b_s2048.npz) for two bf16 steps against the fp32 CPU
oracle: this repo's step (libmemo) and PyTorch's standard bf16 AMP step
(tests/torch_ref.amp_loss_and_grads).  Prints one JSON line per tensor."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200.executor import Executor  # noqa: E402
from tests import torch_ref  # noqa: E402
from tests.golden.make_fullwidth_fixture import F, H_, HEADS, N, S, SEED, V, sample_indices  # noqa: E402


def main():
    fx = np.load(os.path.join(ROOT, "tests", "golden", "fullwidth_7b_s2048.npz"))
    ocfg = O.make_cfg(N, H_, HEADS, F, V, S)
    params = O.init_params(ocfg, SEED)
    toks, labels = O.tokens(SEED, V, S)
    cfg = P.ModelConfig(n_layers=N, hidden=H_, ffn_hidden=F * 3 // 2, n_heads=HEADS, vocab=V, batch=1,
                        seq_len=S, dtype_bytes=2, untied_classifier=True)
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=64 * P.GiB, gpu_mem=180 * 10 ** 9, peak_flops=2.25e15,
                          efficiency=0.5)
    with Executor(cfg, hw, seed=SEED, alpha=0.5, optimizer=0, ce_chunk=1024) as ex:
        loss = ex.step(toks, labels)
        ours = ex.read("grad/all")
    amp_loss, amp = torch_ref.amp_loss_and_grads(ocfg, params, toks, labels)
    print(json.dumps({"loss_oracle": float(fx["loss"]), "loss_ours": loss, "loss_amp": amp_loss}))
    for name, layer, off, cnt in O.layout(ocfg):
        key = f"{name}/{layer}"
        idx = sample_indices(name, layer, cnt)
        r = fx[key + "/sample"]
        out = {"tensor": key}
        for arm, g in (("ours", ours), ("amp", amp)):
            gs = g[off:off + cnt][idx]
            out[arm] = float(np.linalg.norm(gs - r) / np.linalg.norm(r))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
