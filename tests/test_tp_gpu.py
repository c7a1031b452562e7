"""Megatron SP+TP executor (tp_degree = 2) on one B200 through the loopback
communicator (2 ranks = 2 host threads sharing the GPU): parameter shards
initialise to exact slices of the full model, the sharded step matches the
CPU oracle, replicas agree, and swap+recompute stays bitwise equal to the
no-swap sharded path."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_12117_b200 import planner as P
from paper_2407_12117_b200.executor import (KIND_LOOPBACK, KIND_PEER_LOCAL, Executor, LoopbackGroup,
                                            run_ranks)

pytestmark = pytest.mark.gpu

HW = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=64 * P.GiB, gpu_mem=180 * 10 ** 9,
                      peak_flops=2.25e15, efficiency=0.5)


def model(n, h, H, F, V, S, t):
    return P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=F * 3 // 2, n_heads=H, vocab=V, batch=1,
                         seq_len=S, dtype_bytes=2, tp_degree=t, untied_classifier=True)


def assemble(ocfg, shards, t, get):
    """Full tensor layout (oracle order) from per-rank shards."""
    h, F, V = ocfg.hidden, ocfg.ffn, ocfg.vocab
    H = ocfg.n_heads
    hl, Fl, Vl = h // t, F // t, V // t
    parts = []
    for name, layer, off, cnt in O.layout(ocfg):
        loc = [get(r, name, layer) for r in range(t)]
        if name in ("embedding", "g1", "g2", "gf"):
            full = loc[0]
        elif name == "wqkv":
            full = np.concatenate([np.concatenate([l.reshape(3, hl, h)[k] for l in loc], 0) for k in range(3)], 0)
        elif name == "wo":
            full = np.concatenate([l.reshape(h, hl) for l in loc], 1)
        elif name == "wgu":
            full = np.concatenate([np.concatenate([l.reshape(2, Fl, h)[k] for l in loc], 0) for k in range(2)], 0)
        elif name == "wd":
            full = np.concatenate([l.reshape(h, Fl) for l in loc], 1)
        else:  # wcls
            full = np.concatenate([l.reshape(Vl, h) for l in loc], 0)
        parts.append(full.reshape(-1))
    return np.concatenate(parts)


def run_tp(cfg, t, toks, labels, kind=KIND_LOOPBACK, **opts):
    g = LoopbackGroup(t)

    def rank(r):
        with Executor(cfg, HW, tp=(kind, g, r), **opts) as ex:
            params = {(n, l): ex.read(n, l, dtype="bf16") for n, l, _, _ in O.layout(ocfg_of(cfg))}
            loss = ex.step(toks, labels)
            grads = {(n, l): ex.read("grad/" + n, l) for n, l, _, _ in O.layout(ocfg_of(cfg))}
            tl = ex.timeline()
            return loss, params, grads, tl, ex.info()
    return run_ranks(t, rank)


def ocfg_of(cfg):
    return O.make_cfg(cfg.n_layers, cfg.hidden, cfg.n_heads, cfg.ffn_hidden * 2 // 3, cfg.vocab,
                      cfg.seq_len)


@pytest.mark.parametrize("t,kind,dims", [(2, KIND_LOOPBACK, None), (2, KIND_PEER_LOCAL, None),
                                         (4, KIND_PEER_LOCAL, None),
                                         (8, KIND_PEER_LOCAL, (4, 512, 8, 768, 512, 2048))])
def test_tp_matches_oracle(t, kind, dims):
    n, h, H, F, V, S = dims or (4, 256, 4, 768, 512, 1024)
    cfg = model(n, h, H, F, V, S, t)
    ocfg = ocfg_of(cfg)
    params = O.init_params(ocfg, 1234)
    toks, labels = O.tokens(1234, V, S)
    res = run_tp(cfg, t, toks, labels, kind=kind, seed=1234, alpha=0.5, optimizer=0, ce_chunk=256)
    full_params = assemble(ocfg, None, t, lambda r, n_, l_: res[r][1][(n_, l_)])
    assert np.array_equal(full_params, params), "sharded init differs from slices of the full model"
    losses = [r[0] for r in res]
    assert all(x == losses[0] for x in losses)
    ref_loss, ref = O.step(ocfg, params, toks, labels)
    assert abs(losses[0] - ref_loss) <= 5e-3 * abs(ref_loss), (losses, ref_loss)
    grads = assemble(ocfg, None, t, lambda r, n_, l_: res[r][2][(n_, l_)])
    for name, layer, off, cnt in O.layout(ocfg):
        g, rr = grads[off:off + cnt], ref[off:off + cnt]
        rel = float(np.linalg.norm(g - rr) / max(np.linalg.norm(rr), 1e-30))
        assert rel < 2e-2, (name, layer, rel)
    for r in range(t):  # replicated grads identical on every rank
        assert np.array_equal(res[r][2][("embedding", -1)], res[0][2][("embedding", -1)])
        assert P.validate_schedule(res[r][3], n, res[r][4]["swap"]) == []


@pytest.mark.parametrize("t,kind", [(2, KIND_LOOPBACK), (4, KIND_PEER_LOCAL)])
def test_tp_swap_bitwise_equals_no_swap(t, kind):
    n, h, H, F, V, S = 4, 256, 4, 768, 512, 1024
    cfg = model(n, h, H, F, V, S, t)
    toks, labels = O.tokens(77, V, S)
    on = run_tp(cfg, t, toks, labels, kind=kind, seed=9, alpha=0.5, optimizer=0, ce_chunk=512, swap_enabled=1)
    off = run_tp(cfg, t, toks, labels, kind=kind, seed=9, alpha=0.5, optimizer=0, ce_chunk=512, swap_enabled=0)
    for r in range(t):
        assert on[r][0] == off[r][0]
        for k in on[r][2]:
            assert np.array_equal(on[r][2][k], off[r][2][k]), k


def test_tp2_peer_paths_bitwise_equal_loopback():
    """For t = 2 the staggered reduce-scatter sums p_{r+1} + p_r, the loopback
    reduce p_0 + p_1: the same IEEE sums, so every result is bitwise equal."""
    n, h, H, F, V, S, t = 4, 256, 4, 768, 512, 1024, 2
    cfg = model(n, h, H, F, V, S, t)
    toks, labels = O.tokens(5, V, S)
    a = run_tp(cfg, t, toks, labels, kind=KIND_LOOPBACK, seed=3, alpha=0.5, optimizer=0, ce_chunk=512)
    b = run_tp(cfg, t, toks, labels, kind=KIND_PEER_LOCAL, seed=3, alpha=0.5, optimizer=0, ce_chunk=512)
    for r in range(t):
        assert a[r][0] == b[r][0]
        for k in a[r][2]:
            assert np.array_equal(a[r][2][k], b[r][2][k]), (r, k)


def test_solo_rank_step_runs_with_valid_timeline():
    """Communicator kind 4 (tools/project_rank.py): one rank of a t = 4 group
    runs its whole step alone -- finite loss, a timeline that passes the
    reference validator, and the device allocation of the group rank's plan."""
    from paper_2407_12117_b200.executor import KIND_SOLO
    n, h, H, F, V, S, t = 4, 256, 4, 768, 512, 1024, 4
    cfg = model(n, h, H, F, V, S, t)
    toks, labels = O.tokens(5, V, S)
    planned = Executor(cfg, HW, alpha=0.5, dry_run=1, ce_chunk=512).info()["device_bytes"]
    with Executor(cfg, HW, tp=(KIND_SOLO, None, 0), seed=3, alpha=0.5, optimizer=1, ce_chunk=512) as ex:
        losses = [ex.step(toks, labels) for _ in range(2)]
        tl, info = ex.timeline(), ex.info()
    assert all(np.isfinite(losses))
    assert P.validate_schedule(tl, n, info["swap"]) == []
    assert info["device_bytes"] == planned
