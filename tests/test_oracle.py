"""Pins the CPU numeric oracle (oracle/llama_cpu.c) against an independent torch
fp64 autograd restatement (tests/torch_ref.py).  The reference has no model math
(SURVEY discovery 1), so this is the oracle's only pin for loss/gradients."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import torch_ref


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("n_layers,hidden,heads,ffn,vocab,seq", [
    (2, 64, 2, 96, 64, 48),
    (1, 128, 2, 128, 96, 40),
])
def test_oracle_matches_torch_fp64(n_layers, hidden, heads, ffn, vocab, seq):
    cfg = O.make_cfg(n_layers, hidden, heads, ffn, vocab, seq)
    p = O.init_params(cfg, seed=7)
    toks, labels = O.tokens(1234, vocab, seq)
    loss, g = O.step(cfg, p, toks, labels)
    tloss, tg = torch_ref.loss_and_grads(cfg, p, toks, labels)
    assert abs(loss - tloss) < 1e-4 * abs(tloss)
    for name, layer, off, cnt in O.layout(cfg):
        r = _rel(g[off:off + cnt], tg[off:off + cnt])
        assert r < 1e-3, (name, layer, r)


def test_init_is_deterministic_and_bf16():
    cfg = O.make_cfg(2, 64, 2, 96, 64, 48)
    a = O.init_params(cfg, 1)
    b = O.init_params(cfg, 1)
    c = O.init_params(cfg, 2)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # every value is exactly representable in bf16
    assert np.all((a.view(np.uint32) & 0xFFFF) == 0)
    # norm weights near 1, matrices within +-sqrt(3)*0.02
    for name, layer, off, cnt in O.layout(cfg):
        v = a[off:off + cnt]
        if name in ("g1", "g2", "gf"):
            assert np.all(np.abs(v - 1) <= 0.105)  # 0.1 + half a bf16 ulp at 1
        else:
            assert np.all(np.abs(v) <= 0.0347)


def test_tokens_shifted_labels():
    t, l = O.tokens(1234, 512, 100)
    assert np.array_equal(l[:-1], t[1:]) and l[-1] == -1
    assert t.min() >= 0 and t.max() < 512
