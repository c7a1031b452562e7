"""ctypes wrapper of the CPU numeric oracle (oracle/llama_cpu.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, bench.py's CPU-baseline leg and
__graft_entry__.smoke() as the checker; the product never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libllama_cpu.so")


class OcCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layers", "hidden", "n_heads", "head_dim", "ffn",
                                       "vocab", "seq")] + [("eps", C.c_float),
                                                           ("rope_theta", C.c_float)]


def _load():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-C", HERE, "cpu"])
    lib = C.CDLL(LIB)
    lib.oc_param_count.restype = C.c_longlong
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def make_cfg(n_layers, hidden, n_heads, ffn, vocab, seq, eps=1e-5, rope_theta=10000.0):
    return OcCfg(n_layers, hidden, n_heads, hidden // n_heads, ffn, vocab, seq, eps, rope_theta)


def param_count(cfg: OcCfg) -> int:
    return lib().oc_param_count(C.byref(cfg))


def init_params(cfg: OcCfg, seed: int) -> np.ndarray:
    p = np.empty(param_count(cfg), dtype=np.float32)
    lib().oc_init(C.byref(cfg), C.c_uint64(seed), p.ctypes.data_as(C.c_void_p))
    return p


def tokens(seed: int, vocab: int, seq: int):
    t = np.empty(seq, dtype=np.int32)
    l = np.empty(seq, dtype=np.int32)
    lib().oc_tokens(C.c_uint64(seed), vocab, seq, t.ctypes.data_as(C.c_void_p),
                    l.ctypes.data_as(C.c_void_p))
    return t, l


def step(cfg: OcCfg, params: np.ndarray, toks: np.ndarray, labels: np.ndarray):
    """Forward + backward on the CPU; returns (loss, grads[float32, same layout])."""
    g = np.empty_like(params)
    loss = C.c_double()
    rc = lib().oc_step(C.byref(cfg), params.ctypes.data_as(C.c_void_p),
                       np.ascontiguousarray(toks, np.int32).ctypes.data_as(C.c_void_p),
                       np.ascontiguousarray(labels, np.int32).ctypes.data_as(C.c_void_p),
                       g.ctypes.data_as(C.c_void_p), C.byref(loss), None)
    assert rc == 0
    return loss.value, g


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, dout: np.ndarray, H: int):
    """Causal attention forward + backward of [S, H*D] f32 arrays on the CPU;
    returns (o, lse, dq, dk, dv).  bench.py times it for the CPU baseline."""
    q, k, v, dout = (np.ascontiguousarray(a, np.float32) for a in (q, k, v, dout))
    S, h = q.shape
    D = h // H
    o, dq, dk, dv = (np.empty_like(q) for _ in range(4))
    lse = np.empty((H, S), np.float32)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = lib().oc_attention(S, H, D, ptr(q), ptr(k), ptr(v), ptr(dout), ptr(o), ptr(lse), ptr(dq), ptr(dk),
                            ptr(dv))
    assert rc == 0
    return o, lse, dq, dk, dv


def layout(cfg: OcCfg):
    """[(name, layer, offset, count)] in the shared parameter layout."""
    h, F, V = cfg.hidden, cfg.ffn, cfg.vocab
    out, off = [], 0

    def add(n, l, c):
        nonlocal off
        out.append((n, l, off, c))
        off += c
    add("embedding", -1, V * h)
    for l in range(cfg.n_layers):
        add("g1", l, h)
        add("wqkv", l, 3 * h * h)
        add("wo", l, h * h)
        add("g2", l, h)
        add("wgu", l, 2 * F * h)
        add("wd", l, h * F)
    add("gf", -1, h)
    add("wcls", -1, V * h)
    return out
