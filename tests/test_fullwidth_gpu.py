"""The training step at the bench's LAYER WIDTHS against the CPU oracle.

Llama-7B layer shapes (h=4096, 32 heads of D=128, SwiGLU f=11008, V=32000 --
the GEMM epilogues, the V=32000 cross-entropy chunks and the D=128 attention
the cfg2 bench runs) in a 3-layer model at S=2048, with layer 0 swapped and
half of its tokens recomputed (alpha = 0.5).  The oracle's output is the
committed fixture tests/golden/fullwidth_7b_s2048.npz (generator:
tests/golden/make_fullwidth_fixture.py): loss, each gradient tensor's exact
squared norm and 16384 sampled entries per tensor.

Bar: loss within 5e-3 relative.  Per gradient tensor, relative L2
on the sampled entries within max(2e-2, 1.1 x the error of PyTorch's own bf16
AMP step on the same weights and tokens) and below 3e-2 outright, and the full
norm within 5e-3.  The yardstick is measured in the test
(tests/torch_ref.amp_loss_and_grads: fp32 masters, autocast bf16 GEMMs,
flash SDPA): at these widths bf16 training itself is 1.4-2.5 % away from the
fp32 oracle on the attention-side tensors of the last layers (measured r02,
profiles/fullwidth_errors_r02.jsonl), so the survey's flat 2e-2 is below what
any bf16 step reaches there.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_12117_b200 import planner as P
from paper_2407_12117_b200.executor import Executor
from tests.golden.make_fullwidth_fixture import F, H_, HEADS, N, S, SEED, V, sample_indices

pytestmark = pytest.mark.gpu

FIXTURE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullwidth_7b_s2048.npz")
HW = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=64 * P.GiB, gpu_mem=180 * 10 ** 9,
                      peak_flops=2.25e15, efficiency=0.5)


def test_fullwidth_step_matches_cpu_oracle_fixture():
    fx = np.load(FIXTURE)
    assert list(fx["shape"]) == [N, H_, HEADS, F, V, S, SEED]
    cfg = P.ModelConfig(n_layers=N, hidden=H_, ffn_hidden=F * 3 // 2, n_heads=HEADS, vocab=V, batch=1,
                        seq_len=S, dtype_bytes=2, untied_classifier=True)
    toks, labels = O.tokens(SEED, V, S)
    with Executor(cfg, HW, seed=SEED, alpha=0.5, optimizer=0, ce_chunk=1024) as ex:
        loss = ex.step(toks, labels)
        grads = ex.read("grad/all")
        info = ex.info()
        tl = ex.timeline()
    assert info["split"] == (1024, 1024)
    assert sum(e.kind == "recompute" for e in tl) == 1
    ref_loss = float(fx["loss"])
    assert abs(loss - ref_loss) <= 5e-3 * abs(ref_loss), (loss, ref_loss)
    from tests import torch_ref
    ocfg = O.make_cfg(N, H_, HEADS, F, V, S)
    amp_loss, amp = torch_ref.amp_loss_and_grads(ocfg, O.init_params(ocfg, SEED), toks, labels)
    rows = []
    for name, layer, off, cnt in O.layout(ocfg):
        key = f"{name}/{layer}"
        idx = sample_indices(name, layer, cnt)
        r = fx[key + "/sample"]
        g = grads[off:off + cnt]
        rel = float(np.linalg.norm(g[idx] - r) / max(np.linalg.norm(r), 1e-30))
        rel_amp = float(np.linalg.norm(amp[off:off + cnt][idx] - r) / max(np.linalg.norm(r), 1e-30))
        n_ratio = float(np.sqrt(np.dot(g.astype(np.float64), g.astype(np.float64)) / fx[key + "/norm2"]))
        rows.append((key, cnt, rel, rel_amp, n_ratio))
    for key, cnt, rel, rel_amp, n_ratio in rows:
        print(f"fullwidth {key:14s} n={cnt:>10d} rel-L2 {rel:.3e} (torch AMP {rel_amp:.3e}) norm ratio {n_ratio:.5f}")
    print(f"fullwidth: loss {loss:.6f} vs {ref_loss:.6f} (torch AMP {amp_loss:.6f})")
    for key, cnt, rel, rel_amp, n_ratio in rows:
        assert rel < max(2e-2, 1.1 * rel_amp), (key, rel, rel_amp)
        assert rel < 3e-2, (key, rel)
        assert abs(n_ratio - 1) < 5e-3, (key, n_ratio)
