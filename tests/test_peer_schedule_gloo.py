"""Host-side schedule of the peer-memory SP+TP collectives (executor.cu:
Executor::gemm_reduce_rows / Executor::gather_gemm), replayed on CPU with real
point-to-point messages over gloo at world sizes 2 and 4.

Staggered reduce-scatter: at step j rank r produces the partial of row block
b = r-j-1 (mod t) and, as owner of block r, pulls the partial of producer
p = r+j+1; its own partial comes last (added in the GEMM epilogue).  The test
checks that every step is a permutation (each rank sends one block and
receives one, so every link is busy), that the result is the fixed-order sum
p_{r+1} + ... + p_{r-1} + p_r bitwise (== loopback's p_0 + p_1 for t = 2),
and that the all-gather pull order (k = r+j) is a permutation per step too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rs_schedule(t):
    """[(step, producer, owner)] of the staggered reduce-scatter (pulls only)."""
    out = []
    for j in range(t - 1):
        for r in range(t):
            out.append((j, (r + j + 1) % t, r))  # owner r pulls from p = r+j+1
    return out


def partials(t, rows, cols, seed=7):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((t, t, rows, cols)).astype(np.float32)  # [producer][block]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t, r = world, rank
    P = partials(t, 8, 16)
    acc = None
    for j in range(t):
        b = ((r - j - 1) % t + t) % t           # block this rank produces at step j
        p = (r + j + 1) % t                     # producer this rank (owner of block r) pulls from
        reqs = []
        if b != r:
            reqs.append(dist.isend(torch.from_numpy(P[r, b].copy()), dst=b, tag=j))
        if p != r:
            buf = torch.empty(P.shape[2:], dtype=torch.float32)
            dist.irecv(buf, src=p, tag=j).wait()
            x = buf.numpy()
            acc = x.copy() if j == 0 else (acc + x).astype(np.float32)
        for rq in reqs:
            rq.wait()
    acc = (acc + P[r, r]).astype(np.float32)    # own block in the GEMM epilogue (F32_ACC)
    q.put((r, acc))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_staggered_reduce_scatter_gloo(world):
    for j in range(world - 1):  # every pull step is a permutation: all links busy
        pulls = [(p, o) for (s, p, o) in rs_schedule(world) if s == j]
        assert sorted(p for p, _ in pulls) == list(range(world))
        assert sorted(o for _, o in pulls) == list(range(world))
        assert all(p != o for p, o in pulls)
    for j in range(world):  # all-gather pull order k = r + j
        assert sorted((r + j) % world for r in range(world)) == list(range(world))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = partials(world, 8, 16)
    for r in range(world):
        ref = None
        for k in list(range(r + 1, world)) + list(range(0, r)) + [r]:  # p_{r+1} .. p_{r-1}, p_r
            ref = P[k, r].copy() if ref is None else (ref + P[k, r]).astype(np.float32)
        assert np.array_equal(got[r], ref)
        if world == 2:  # same IEEE sums as the loopback/NCCL-order p_0 + p_1
            assert np.array_equal(got[r], (P[0, r] + P[1, r]).astype(np.float32))
        np.testing.assert_allclose(got[r], P[:, r].sum(0), rtol=1e-5, atol=1e-5)
