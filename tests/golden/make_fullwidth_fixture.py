"""Generate tests/golden/fullwidth_7b_s2048.npz: the CPU oracle (oracle/llama_cpu.c)
on a 3-layer step at the bench's layer widths (Llama-7B: h=4096, 32 heads of
D=128, SwiGLU f=11008, V=32000) at S=2048, seed 1234.

The full gradient is 3.5 GB, so the fixture keeps, per parameter tensor, its
exact squared L2 norm and SAMPLE values at indices drawn by
`sample_indices(name, layer, count)` (numpy PCG64, seeded from the tensor name),
which tests/test_fullwidth_gpu.py regenerates.  Relative L2 is then estimated on
the sample (Σ(g-r)² / Σr² over the sampled entries), and the full norms are
compared exactly.

TEST INFRASTRUCTURE: the oracle is the checker; run here (CPU, ~5 min on 8 cores):
    python tests/golden/make_fullwidth_fixture.py
"""
from __future__ import annotations

import os
import sys
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

N, H_, HEADS, F, V, S, SEED = 3, 4096, 32, 11008, 32000, 2048, 1234
N_SAMPLE = 16384
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fullwidth_7b_s2048.npz")


def sample_indices(name: str, layer: int, count: int, k: int = N_SAMPLE) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(zlib.crc32(f"{name}/{layer}".encode())))
    if count <= k:
        return np.arange(count, dtype=np.int64)
    return np.sort(rng.choice(count, size=k, replace=False)).astype(np.int64)


def main():
    from oracle import oracle as O
    ocfg = O.make_cfg(N, H_, HEADS, F, V, S)
    t0 = time.time()
    params = O.init_params(ocfg, SEED)
    toks, labels = O.tokens(SEED, V, S)
    loss, g = O.step(ocfg, params, toks, labels)
    print(f"oracle step {time.time() - t0:.1f} s, loss {loss:.6f}", flush=True)
    out = {"loss": np.float64(loss), "shape": np.array([N, H_, HEADS, F, V, S, SEED], np.int64)}
    for name, layer, off, cnt in O.layout(ocfg):
        gi = g[off:off + cnt]
        key = f"{name}/{layer}"
        out[key + "/norm2"] = np.float64(np.dot(gi.astype(np.float64), gi.astype(np.float64)))
        out[key + "/sample"] = gi[sample_indices(name, layer, cnt)].copy()
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
