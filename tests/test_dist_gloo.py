"""N>1 host-side coverage on CPU with torch.distributed (gloo, world_size 2).

* Every rank plans the same SP+TP arena (SPMD consistency: collectives pair
  buffers by offset, so all ranks must bind byte-identical plans).
* The shard maps the executor uses (column-parallel Wqkv/Wgu, row-parallel
  Wo/Wd, vocab-parallel Wcls, replicated embedding/norms) partition the full
  parameter vector exactly once.
* The SP+TP schedule of one Llama layer forward (norm on the local token shard
  -> all-gather -> column-parallel QKV/attention on local heads -> row-parallel
  out-projection -> reduce-scatter -> residual -> norm -> all-gather ->
  column-parallel gate/up -> SwiGLU -> row-parallel down -> reduce-scatter)
  reproduces the unsharded layer (fp64), with real gloo collectives.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_params(ocfg, full, t, r):
    """Local shard of every parameter tensor, exactly as Executor::init_weights slices it."""
    h, F, V = ocfg.hidden, ocfg.ffn, ocfg.vocab
    hl, Fl, Vl = h // t, F // t, V // t
    out = {}
    for name, layer, off, cnt in O.layout(ocfg):
        x = full[off:off + cnt]
        if name in ("embedding", "g1", "g2", "gf"):
            out[(name, layer)] = x.copy()
        elif name == "wqkv":
            m = x.reshape(3, h, h)
            out[(name, layer)] = np.concatenate([m[k, r * hl:(r + 1) * hl] for k in range(3)], 0).reshape(-1)
        elif name == "wo":
            out[(name, layer)] = x.reshape(h, h)[:, r * hl:(r + 1) * hl].reshape(-1)
        elif name == "wgu":
            m = x.reshape(2, F, h)
            out[(name, layer)] = np.concatenate([m[k, r * Fl:(r + 1) * Fl] for k in range(2)], 0).reshape(-1)
        elif name == "wd":
            out[(name, layer)] = x.reshape(h, F)[:, r * Fl:(r + 1) * Fl].reshape(-1)
        else:
            out[(name, layer)] = x.reshape(V, h)[r * Vl:(r + 1) * Vl].reshape(-1)
    return out


def _rmsnorm(x, g, eps=1e-5):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps) * g


def _attn(q, k, v, H, D):
    S = q.shape[0]
    qh, kh, vh = (a.view(S, H, D).transpose(0, 1) for a in (q, k, v))
    s = qh @ kh.transpose(1, 2) / D ** 0.5
    s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    return (torch.softmax(s, -1) @ vh).transpose(0, 1).reshape(S, H * D)


def _layer_full(x, L, H, D, F):
    h = x.shape[1]
    xn = _rmsnorm(x, L["g1"])
    qkv = xn @ L["wqkv"].t()
    o = _attn(qkv[:, :h], qkv[:, h:2 * h], qkv[:, 2 * h:], H, D)
    x1 = x + o @ L["wo"].t()
    gu = _rmsnorm(x1, L["g2"]) @ L["wgu"].t()
    return x1 + (torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]) @ L["wd"].t()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        from paper_2407_12117_b200 import planner as P
        from paper_2407_12117_b200.executor import Executor
        # 1) SPMD plan consistency
        hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=96 * P.GiB, gpu_mem=180 * 10 ** 9,
                              peak_flops=2.25e15)
        cfg = P.ModelConfig(n_layers=4, hidden=4096, ffn_hidden=16512, n_heads=32, vocab=32000,
                            seq_len=131072, tp_degree=world, untied_classifier=True)
        plan = Executor(cfg, hw, alpha=0.5, dry_run=1).plan_json()
        digest = torch.tensor([int(P.fnv1a_hex(plan), 16) & ((1 << 62) - 1)], dtype=torch.int64)
        allp = [torch.zeros_like(digest) for _ in range(world)]
        dist.all_gather(allp, digest)
        assert all(int(d) == int(digest) for d in allp)
        # 2) shard maps partition the parameters
        ocfg = O.make_cfg(2, 64, 2, 96, 64, 48)
        full = O.init_params(ocfg, 5)
        mine = shard_params(ocfg, full, world, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        h, F, V = ocfg.hidden, ocfg.ffn, ocfg.vocab
        hl, Fl, Vl = h // world, F // world, V // world
        rebuilt = []
        for name, layer, off, cnt in O.layout(ocfg):
            loc = [g[(name, layer)] for g in gathered]
            if name in ("embedding", "g1", "g2", "gf"):
                rebuilt.append(loc[0])
            elif name == "wqkv":
                rebuilt.append(np.concatenate([np.concatenate([l.reshape(3, hl, h)[k] for l in loc]) for k in range(3)]).reshape(-1))
            elif name == "wo":
                rebuilt.append(np.concatenate([l.reshape(h, hl) for l in loc], 1).reshape(-1))
            elif name == "wgu":
                rebuilt.append(np.concatenate([np.concatenate([l.reshape(2, Fl, h)[k] for l in loc]) for k in range(2)]).reshape(-1))
            elif name == "wd":
                rebuilt.append(np.concatenate([l.reshape(h, Fl) for l in loc], 1).reshape(-1))
            else:
                rebuilt.append(np.concatenate([l.reshape(Vl, h) for l in loc]).reshape(-1))
        assert np.array_equal(np.concatenate(rebuilt), full)
        # 3) SP+TP layer forward with gloo collectives == unsharded layer
        torch.manual_seed(0)
        S, h, H, F = 32, 64, 4, 96
        D, Sl, Hl, Fl = h // H, S // world, H // world, F // world
        hl = Hl * D
        L = {"g1": 1 + 0.1 * torch.randn(h, dtype=torch.float64),
             "wqkv": 0.05 * torch.randn(3 * h, h, dtype=torch.float64),
             "wo": 0.05 * torch.randn(h, h, dtype=torch.float64),
             "g2": 1 + 0.1 * torch.randn(h, dtype=torch.float64),
             "wgu": 0.05 * torch.randn(2 * F, h, dtype=torch.float64),
             "wd": 0.05 * torch.randn(h, F, dtype=torch.float64)}
        x = torch.randn(S, h, dtype=torch.float64)
        ref = _layer_full(x, L, H, D, F)
        xl = x[rank * Sl:(rank + 1) * Sl]
        wq = torch.cat([L["wqkv"][k * h + rank * hl:k * h + (rank + 1) * hl] for k in range(3)])
        wo = L["wo"][:, rank * hl:(rank + 1) * hl]
        wgu = torch.cat([L["wgu"][k * F + rank * Fl:k * F + (rank + 1) * Fl] for k in range(2)])
        wd = L["wd"][:, rank * Fl:(rank + 1) * Fl]

        def ag(t):
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t.contiguous())
            return torch.cat(parts)

        def rs(t):
            out = torch.empty(Sl, t.shape[1], dtype=t.dtype)
            chunks = list(t.chunk(world))
            red = [c.clone() for c in chunks]
            for c in red:
                dist.all_reduce(c)
            out.copy_(red[rank])
            return out
        xn_full = ag(_rmsnorm(xl, L["g1"]))
        qkv = xn_full @ wq.t()
        o = _attn(qkv[:, :hl], qkv[:, hl:2 * hl], qkv[:, 2 * hl:], Hl, D)
        x1 = xl + rs(o @ wo.t())
        gu = ag(_rmsnorm(x1, L["g2"])) @ wgu.t()
        y = x1 + rs((torch.nn.functional.silu(gu[:, :Fl]) * gu[:, Fl:]) @ wd.t())
        err = (y - ref[rank * Sl:(rank + 1) * Sl]).abs().max().item()
        assert err < 1e-10, err
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sp_tp_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
