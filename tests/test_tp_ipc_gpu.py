"""Peer-memory SP+TP over CUDA IPC (communicator kind 2) with two real
processes: each maps the other's single device allocation and flag page
(cudaIpcOpenMemHandle), synchronises with cuStreamWriteValue64 /
cuStreamWaitValue64, and runs the fused all-gather->GEMM and staggered
GEMM->reduce-scatter paths.  This pool's boxes have one GPU, so both
processes share it (the driver time-slices their contexts); the protocol is
the one a multi-GPU box runs.  Result: bitwise equal to the in-process
loopback backend (t = 2 sums are order-free)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from tests.test_tp_gpu import model, run_tp
from paper_2407_12117_b200.executor import KIND_LOOPBACK

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ipc_two_processes_bitwise_equal_loopback(tmp_path):
    n, h, H, F, V, S, t = 4, 256, 4, 768, 512, 1024, 2
    opts = dict(seed=3, alpha=0.5, optimizer=0, ce_chunk=512)
    spec = json.dumps({"dims": [n, h, H, F, V, S], "data_seed": 5, "opts": opts})
    port = free_port()
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_ipc_worker.py"), str(r), str(t),
                               str(port), str(tmp_path), spec], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(t)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=400)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace")[-3000:])
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    toks, labels = O.tokens(5, V, S)
    ref = run_tp(model(n, h, H, F, V, S, t), t, toks, labels, kind=KIND_LOOPBACK, **opts)
    for r in range(t):
        got = np.load(tmp_path / f"rank{r}.npz")
        assert float(got["loss"][0]) == ref[r][0]
        for (name, layer), g in ref[r][2].items():
            assert np.array_equal(got[f"{name}:{layer}"], g), (r, name, layer)


def _run_workers(tmp_path, t, spec):
    port = free_port()
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_ipc_worker.py"), str(r), str(t),
                               str(port), str(tmp_path), json.dumps(spec)], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT) for r in range(t)]
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=400)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(out.decode(errors="replace")[-3000:])
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(t)]


def test_ipc_cuda_graph_replays_bitwise_equal_eager(tmp_path):
    """cuda_graph=1 at tp=2 over CUDA IPC: the second step is captured and
    replayed; every replay rebases the captured signal values and stream-wait
    thresholds (IpcComm::before_replay).  Four steps with the graph (one eager,
    three replays) equal four eager steps bitwise on both ranks, loss and every
    gradient tensor."""
    n, h, H, F, V, S, t = 4, 256, 4, 768, 512, 1024, 2
    base = {"dims": [n, h, H, F, V, S], "data_seed": 5, "steps": 4}
    (tmp_path / "eager").mkdir()
    (tmp_path / "graph").mkdir()
    eager = _run_workers(tmp_path / "eager", t,
                         dict(base, opts=dict(seed=3, alpha=0.5, optimizer=1, ce_chunk=512)))
    graph = _run_workers(tmp_path / "graph", t,
                         dict(base, opts=dict(seed=3, alpha=0.5, optimizer=1, ce_chunk=512, cuda_graph=1)))
    for r in range(t):
        # every replay posted its signals with rebased values: the flag pages
        # hold the same signal counts as after four eager steps
        assert graph[r]["peer_flags"].sum() > 0
        assert np.array_equal(graph[r]["peer_flags"], eager[r]["peer_flags"]), (r, graph[r]["peer_flags"])
        assert len(graph[r]["loss"]) == 4
        assert np.array_equal(graph[r]["loss"], eager[r]["loss"]), (r, graph[r]["loss"], eager[r]["loss"])
        for k in eager[r]:
            assert np.array_equal(graph[r][k], eager[r][k]), (r, k)
