"""Two tiny training steps (t ranks as threads on one GPU; t = 1 is the plain
single-GPU executor) through a chosen communicator kind, printing the losses
and a hash of every rank's gradients -- for compute-sanitizer runs and for
bitwise comparison of a normal run against a perturbed one.
Usage: python tools/tp_peer_smoke.py [kind=3] [t=2] [heads=4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402
from paper_2407_12117_b200 import planner as P  # noqa: E402
from paper_2407_12117_b200.executor import Executor, LoopbackGroup, run_ranks  # noqa: E402


def main():
    kind = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    t = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    H = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    n, h, F, V, S = 4, 256, 768, 512, 1024
    cfg = P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=F * 3 // 2, n_heads=H, vocab=V, batch=1, seq_len=S,
                        dtype_bytes=2, tp_degree=t, untied_classifier=True)
    hw = P.HardwareConfig(pcie_bandwidth=50e9, cpu_mem=16 * P.GiB, gpu_mem=180 * 10 ** 9, peak_flops=2.25e15,
                          efficiency=0.5)
    toks, labels = O.tokens(5, V, S)
    import hashlib
    g = LoopbackGroup(t) if t > 1 else None

    def rank(r):
        tp = (kind, g, r) if t > 1 else None
        with Executor(cfg, hw, tp=tp, seed=3, alpha=0.5, optimizer=1, ce_chunk=512) as ex:
            losses = [ex.step(toks, labels) for _ in range(2)]
            return losses, hashlib.sha256(ex.read("grad/all").tobytes()).hexdigest()[:16]
    print("losses+grad hash", run_ranks(t, rank))


if __name__ == "__main__":
    main()
