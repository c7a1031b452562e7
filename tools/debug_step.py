"""Debug helper: per-tensor gradient error of the GPU step vs the CPU oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200.executor import Executor  # noqa: E402

n, h, H, F, V, S = [int(x) for x in (sys.argv[1:7] if len(sys.argv) > 6 else (4, 256, 2, 768, 512, 512))]
alpha = float(sys.argv[7]) if len(sys.argv) > 7 else 0.5
swap = int(sys.argv[8]) if len(sys.argv) > 8 else 1
cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=F * 3 // 2, n_heads=H, vocab=V, seq_len=S,
                    untied_classifier=True)
hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=64 * P.GiB, gpu_mem=180 * 10 ** 9, peak_flops=2.25e15)
ocfg = O.make_cfg(n, h, H, F, V, S)
params = O.init_params(ocfg, 1234)
toks, labels = O.tokens(1234, V, S)
with Executor(cfg, hw, seed=1234, alpha=alpha, optimizer=0, ce_chunk=256, swap_enabled=swap) as ex:
    loss = ex.step(toks, labels)
    grads = ex.read("grad/all")
    acts = {c: ex.read("act/" + c, 0, dtype="bf16" if c not in ("layer_input",) else np.float32)
            for c in ("layer_input",)}
    print("info", {k: v for k, v in ex.info().items() if k in ("split", "arena_bytes")})
ref_loss, ref = O.step(ocfg, params, toks, labels)
print("loss", loss, ref_loss)
for name, layer, off, cnt in O.layout(ocfg):
    g, r = grads[off:off + cnt], ref[off:off + cnt]
    nan = int(np.isnan(g).sum())
    rel = float(np.linalg.norm(np.nan_to_num(g) - r) / max(np.linalg.norm(r), 1e-30))
    print(f"{name:10s} {layer:3d} rel={rel:.3e} nan={nan} |g|={np.linalg.norm(np.nan_to_num(g)):.3e} |ref|={np.linalg.norm(r):.3e}")
