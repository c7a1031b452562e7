#!/usr/bin/env python
"""bench.py — MEMO training-step throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

N=1 workload (BASELINE configs[1]): Llama-7B architecture, 4 layers, seq 131072,
one B200, alpha tuned by the planner (solve_alpha with the MEASURED host-link
bandwidth and MEASURED forward-layer time).  A step = embedding -> 4 layers fwd
(offload of the swapped layers' activations) -> classifier + CE -> 4 layers bwd
(prefetch + suffix recompute) -> embedding grad -> AdamW.  Synthetic tokens,
random-init weights (counter hash).  N>1 under torchrun: Megatron SP+TP of the
same cfg2 sequence across the N GPUs over NCCL (tp_degree = N; strong scaling:
`value` = tokens of the one sequence / step time, max over ranks); if the NCCL
communicator cannot start, every rank runs an independent replica instead
(weak scaling) and `config.parallelism` says which ran.

Prints ONE JSON line (rank 0).  `value` is device-resident tokens/s over all
ranks; `e2e` is the same metric through the C-ABI step with host token buffers
(H2D of the batch and D2H of the loss inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MFU and tokens/sec/GPU, 7B train step at 128K–1M seq, 1/2/4/8 B200"
B200_SPEC_BF16 = 2.25e15

CONFIGS = {
    # name: (n_layers, hidden, heads, intermediate, vocab, seq, description)
    "cfg2": (4, 4096, 32, 11008, 32000, 131072,
             "Llama-7B arch, 4 layers, seq 131072, 1xB200, alpha tuned by planner"),
    "cfg1p": (4, 256, 4, 768, 512, 4096, "tiny 4-layer (h256, 4 heads, seq 4096), alpha=0.5"),
    "cfg5": (32, 4096, 32, 11008, 32000, 262144, "Llama-7B arch, 32 layers, seq 262144, 1xB200"),
    # cfg5 at 32 layers needs 6.5 GB/layer of mandatory offload, more pinned memory than this
    # host has (status 4); 20 layers is the deepest 256K stack that fits it
    "cfg5s": (20, 4096, 32, 11008, 32000, 262144, "Llama-7B arch, 20 layers, seq 262144, 1xB200"),
    # the model family of BASELINE configs[3] (13B, 40 heads), sliced to 4 layers on one GPU
    "cfg4s": (4, 5120, 40, 13824, 32000, 131072,
              "Llama-13B arch, 4 layers, seq 131072, 1xB200, alpha tuned by planner"),
}


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


def synthetic_batch(seed, vocab, seq):
    import numpy as np
    idx = np.arange(seq, dtype=np.uint64) + np.uint64(seed)
    with np.errstate(over="ignore"):
        x = idx + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    toks = (x % np.uint64(vocab)).astype(np.int32)
    labels = np.empty_like(toks)
    labels[:-1] = toks[1:]
    labels[-1] = -1
    return toks, labels


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, name in enumerate(names):
                if r[4 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1678.8), d.get("bf16_tflops_sustained", 1409.0), d.get("hbm_gbs", 6459.0), "measured"
    except OSError:
        return 1590.0, 1400.0, 6650.0, "fallback"


def host_link_bandwidth(torch, nbytes=1 << 31):
    """Pinned D2H and H2D GB/s on this GPU (CUDA events)."""
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    out = {}
    for name, fn in (("d2h", lambda: host.copy_(dev, non_blocking=True)),
                     ("h2d", lambda: dev.copy_(host, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name] = 3 * nbytes / (e0.elapsed_time(e1) * 1e-3)
    del dev, host
    return out


def flop_terms(n, h, H, inter, V, S):
    """The reference FLOP model in plain Python (schedule.hpp:44-61): params
    P = V*h + n*(4h^2 + 2h*ffn + 4h) + 2h (+ V*h untied, ffn = the reference's
    ffn_hidden = 3/2 of the SwiGLU width); FLOPs per sample = 6*s*P (dense)
    + 6*n*h*s^2 (causal attention).  Returns (dense, attention)."""
    ffn = inter * 3 // 2
    p = V * h + n * (4 * h * h + 2 * h * ffn + 4 * h) + 2 * h + V * h
    return 6.0 * S * p, 6.0 * n * h * float(S) * S


def cpu_baseline(n_cfg, s_dense=128, v_dense=4096, s_attn=8192, h_attn=1):
    """CPU oracle (oracle/llama_cpu.c, OpenMP on all host cores) on a bounded
    sample, each FLOP term of the workload timed on its own:
      * dense: one full-width layer (+ embedding/classifier over a `v_dense`
        vocabulary) fwd+bwd at `s_dense` tokens, the sample's small attention
        share removed with the attention rate below;
      * attention: causal attention fwd+bwd of `h_attn` heads (D = the
        workload's head dim) at `s_attn` tokens.
    The workload step time is dense/rate_dense + attention/rate_attention
    (reference FLOP model, flop_terms); value = tokens of the step / that time."""
    import numpy as np
    from oracle import oracle as O
    n, h, H, inter, V, S, _ = n_cfg
    D = h // H
    # attention rate
    rng = np.random.default_rng(7)
    qa, ka, va, da = (rng.standard_normal((s_attn, h_attn * D), dtype=np.float32) for _ in range(4))
    t0 = time.perf_counter()
    O.attention(qa, ka, va, da, h_attn)
    t_attn = time.perf_counter() - t0
    _, f_attn_sample = flop_terms(1, h_attn * D, h_attn, 0, 0, s_attn)
    rate_attn = f_attn_sample / t_attn
    # dense rate
    vs = min(V, v_dense)
    ocfg = O.make_cfg(1, h, H, inter, vs, s_dense)
    params = O.init_params(ocfg, 1234)
    toks, labels = synthetic_batch(1234, vs, s_dense)
    t0 = time.perf_counter()
    O.step(ocfg, params, toks, labels)
    t_dense_all = time.perf_counter() - t0
    f_dense_s, f_attn_s = flop_terms(1, h, H, inter, vs, s_dense)
    t_dense = max(t_dense_all - f_attn_s / rate_attn, 1e-9)
    rate_dense = f_dense_s / t_dense
    f_dense_w, f_attn_w = flop_terms(n, h, H, inter, V, S)
    t_work = f_dense_w / rate_dense + f_attn_w / rate_attn
    cores = os.cpu_count()
    return {"value": S / t_work, "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": (f"oracle/llama_cpu.c on {cores} OpenMP threads: dense part = 1 layer (h={h}, heads={H}, "
                       f"f={inter}, V={vs}) fwd+bwd at {s_dense} tokens, {t_dense_all:.2f} s "
                       f"({rate_dense / 1e9:.1f} GFLOP/s); attention part = causal attention fwd+bwd of "
                       f"{h_attn} heads (D={D}) at {s_attn} tokens, {t_attn:.2f} s ({rate_attn / 1e9:.1f} "
                       f"GFLOP/s); workload step = dense {f_dense_w:.3e} / dense rate + attention "
                       f"{f_attn_w:.3e} / attention rate (reference FLOP model, schedule.hpp:57-61) = "
                       f"{t_work:.0f} s"),
            "sample_seconds": t_dense_all + t_attn,
            "workload_step_s_extrapolated": t_work,
            "dense_gflops": rate_dense / 1e9, "attention_gflops": rate_attn / 1e9}


def reference_planner_ms(name):
    """The reference's own CPU path (actmem report pipeline) on this config, if built."""
    probe = os.path.join(ROOT, "oracle", "_ref", "ref_probe")
    if not os.path.exists(probe):
        return None
    n, h, H, inter, V, S, _ = CONFIGS[name]
    cfg = {"model": {"n_layers": n, "hidden": h, "ffn_hidden": inter * 3 // 2, "n_heads": H,
                     "vocab": V, "batch": 1, "seq_len": S, "dtype_bytes": 2, "tp_degree": 1,
                     "sp_or_cp_degree": 1, "untied_classifier": True},
           "hardware": {"pcie_bandwidth": 50e9, "cpu_mem": 96 * 2 ** 30, "gpu_mem": 180 * 10 ** 9,
                        "peak_flops": 2.25e15, "efficiency": 0.5}}
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump(cfg, f)
    try:
        out = subprocess.check_output([probe, "bench_report", f.name, "20"], text=True, timeout=120)
        return json.loads(out)["per_iter_s"] * 1e3
    except Exception:  # noqa: BLE001
        return None
    finally:
        os.unlink(f.name)


def workload_config(name):
    """The config keys both arms report for a workload (no run-dependent keys)."""
    n, h, H, inter, V, S, desc = CONFIGS[name]
    return {"workload": desc, "model": "llama-13b-arch" if h == 5120 else "llama-7b-arch", "n_layers": n,
            "global_batch": 1, "seq_len": S}


def run_reference(args, rank):
    """The reference's CPU implementation of the step (the oracle port; the
    reference itself has no model math) on this box's host cores.  Each step is
    one bounded sample (cpu_baseline); the workload's tokens/s is extrapolated
    per FLOP term.  Imports nothing from the product package."""
    if rank != 0:
        return
    n_cfg = CONFIGS[args.config]
    for _ in range(min(args.warmup, 1)):
        cpu_baseline(n_cfg)
    t0 = time.perf_counter()
    samples = [cpu_baseline(n_cfg) for _ in range(max(1, args.steps))]
    wall = time.perf_counter() - t0
    base = samples[-1]
    v = statistics.median(x["value"] for x in samples)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # measured wall of one step (= one bounded sample); the workload step it
            # stands for is reported separately, extrapolated
            "ms_per_step": wall / len(samples) * 1e3,
            "workload_ms_per_step_extrapolated": n_cfg[5] / v * 1e3 if v else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {**workload_config(args.config), "parallelism": "cpu"},
            "cpu_baseline": {**base, "value": v},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    rp = reference_planner_ms(args.config)
    if rp is not None:
        line["reference_planner_ms"] = rp
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step kernel by kernel (no CUDA graph)")
    ap.add_argument("--no-swap-delta", action="store_true", help="skip the swap-disabled reference step")
    ap.add_argument("--watchdog", type=float, default=1800.0, help="abort the run after this many seconds")
    ap.add_argument("--comm", default="peer", choices=["peer", "nccl"],
                    help="SP+TP collectives: peer memory over CUDA IPC (fused AG->GEMM / GEMM->RS) or NCCL")
    ap.add_argument("--parallel", default="tp", choices=["tp", "replicas"],
                    help="N>1: Megatron SP+TP over NCCL (strong scaling of one sequence) or "
                         "independent replicas (weak scaling)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    # A collective that never completes (e.g. a peer that died) must not hang the
    # driver: after --watchdog seconds the process reports and exits.
    import threading

    def _watchdog():
        print(f"[bench] rank {rank}: watchdog fired after {args.watchdog} s; aborting", file=sys.stderr, flush=True)
        os._exit(3)
    wd = threading.Timer(args.watchdog, _watchdog)
    wd.daemon = True
    wd.start()

    import numpy as np
    import torch
    # more ranks than GPUs (a test of the multi-process path on a one-GPU box):
    # ranks share devices, the process group runs on gloo, and only the
    # peer-memory (CUDA IPC) communicator works -- NCCL rejects shared devices
    shared_gpu = world > torch.cuda.device_count()
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist = None
    ddev = "cpu" if shared_gpu else "cuda"  # device of the small control tensors
    if world > 1:
        import torch.distributed as dist
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2407_12117_b200 import planner as P
    from paper_2407_12117_b200.executor import Executor

    n, h, H, inter, V, S, desc = CONFIGS[args.config]
    mode = "single" if world == 1 else args.parallel
    tp_spec = None
    from paper_2407_12117_b200.executor import KIND_IPC, KIND_NCCL
    comm = args.comm

    def nccl_spec():
        from paper_2407_12117_b200.executor import nccl_unique_id
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        return (KIND_NCCL, uid[0], rank)

    if mode == "tp":
        # peer memory over CUDA IPC (default) or one NCCL communicator for the SP+TP
        # group; fall back to NCCL, then to replicas, if it cannot start
        try:
            tp_spec = (KIND_IPC, None, rank) if comm == "peer" else nccl_spec()
        except Exception as ex:  # noqa: BLE001
            print(f"[bench] SP+TP unavailable ({ex}); running replicas", file=sys.stderr)
            mode = "replicas"

    def connect(e):
        """kind 2: exchange the CUDA IPC handles and map every rank's allocation."""
        if tp_spec is not None and tp_spec[0] == KIND_IPC:
            hs = [None] * world
            dist.all_gather_object(hs, e.peer_handle())
            e.peer_connect(hs)
    def model_cfg():
        return P.ModelConfig(n_layers=n, hidden=h, ffn_hidden=inter * 3 // 2, n_heads=H, vocab=V,
                             batch=1, seq_len=S, dtype_bytes=2, untied_classifier=True,
                             tp_degree=world if mode == "tp" else 1)
    cfg = model_cfg()
    link = host_link_bandwidth(torch)
    host_mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    gpus_on_node = max(torch.cuda.device_count(), world)
    cpu_mem = int(min(host_mem * 0.6 / gpus_on_node, 2 ** 40))  # per-GPU pinned budget
    hw = P.HardwareConfig(pcie_bandwidth=link["d2h"], cpu_mem=cpu_mem,
                          gpu_mem=torch.cuda.get_device_properties(local % torch.cuda.device_count()).total_memory,
                          peak_flops=B200_SPEC_BF16, efficiency=0.5)
    toks, labels = synthetic_batch(1234 + (rank if mode == "replicas" else 0), V, S)
    forced_alpha = 0.5 if args.config == "cfg1p" else -1.0

    # Calibrate: one step with the analytic layer time, then re-solve alpha with
    # the measured forward-layer time (swap.hpp:105 with SwapOptions.t_layer).
    ex, err = None, None
    try:
        ex = Executor(cfg, hw, tp=tp_spec, alpha=forced_alpha, op_timing=0)
    except Exception as e:  # noqa: BLE001
        err = e
    if mode == "tp" and tp_spec[0] == KIND_IPC:  # collective decision: IPC, else NCCL
        ok = torch.tensor([0 if err else 1], device=ddev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 1:
            try:
                connect(ex)
            except Exception as e:  # noqa: BLE001
                err = e
            ok = torch.tensor([0 if err else 1], device=ddev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            print(f"[bench] peer-memory SP+TP unavailable ({err}); using NCCL", file=sys.stderr)
            if ex is not None:
                ex.close()
            comm, err, ex = "nccl", None, None
            tp_spec = nccl_spec()
            try:
                ex = Executor(cfg, hw, tp=tp_spec, alpha=forced_alpha, op_timing=0)
            except Exception as e:  # noqa: BLE001
                err = e
    if mode == "tp":  # every rank must agree before falling back (collective decision)
        ok = torch.tensor([0 if err else 1], device=ddev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            print(f"[bench] SP+TP executor unavailable ({err}); running replicas", file=sys.stderr)
            if ex is not None:
                ex.close()
            mode, tp_spec = "replicas", None
            cfg = model_cfg()
            toks, labels = synthetic_batch(1234 + rank, V, S)
            ex, err = Executor(cfg, hw, alpha=forced_alpha, op_timing=0), None
    if err is not None:
        raise err
    with ex:
        ex.step(toks, labels)
        tl = ex.timeline()
    t_fwd = [e.end - e.start for e in tl if e.kind == "layer_fwd"]
    t_layer = float(np.median(t_fwd))
    if dist:  # SPMD: every rank solves alpha from the same (slowest) layer time
        tt = torch.tensor([t_layer], device=ddev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_layer = tt.item()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    # the step as one CUDA graph (captured on the second step, replayed after): single GPU,
    # and SP+TP over CUDA-IPC peer memory, whose signals the executor rebases per replay
    use_graph = 1 if (not args.no_graph and (cfg.tp_degree == 1 or (tp_spec is not None and tp_spec[0] == KIND_IPC))) else 0
    ex = Executor(cfg, hw, tp=tp_spec, alpha=forced_alpha, t_layer=t_layer, op_timing=1, cuda_graph=use_graph)
    connect(ex)
    free1, _ = torch.cuda.mem_get_info()
    info0 = ex.info()
    stream = torch.cuda.ExternalStream(ex.stream)

    # ---- device-resident timing
    ex.load_batch(toks, labels)
    for _ in range(args.warmup):
        ex.step_resident()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    free_before, _ = torch.cuda.mem_get_info()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            ex.step_resident()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # MEMO's planned allocator never reorganises (allocator.hpp:264-285): device
    # memory is the same before and after the timed steps
    free_after, _ = torch.cuda.mem_get_info()
    tl = ex.timeline()  # last step
    info = ex.info()
    launches = info["kernel_launches"] * args.steps
    t_max = ms
    if dist:
        t = torch.tensor([ms], device=ddev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = t.item()
    seqs = world if mode == "replicas" else 1  # sequences processed by the job per step
    value = seqs * S / (t_max * 1e-3)

    # ---- end to end through the C ABI with host buffers
    e2e_ms = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ex.step(toks, labels)
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e = statistics.mean(e2e_ms)
    info_e2e = ex.info()  # byte counts of the last end-to-end step (H2D batch, D2H loss)
    if dist:
        t = torch.tensor([e2e], device=ddev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = t.item()

    # ---- the same step with swapping disabled (one rounding buffer per layer),
    # when it fits: exposed swap as a step-time difference, T(swap) - T(no swap)
    nosw_ms = None
    if world == 1 and not args.no_swap_delta:
        ex.close()
        try:
            exn = Executor(cfg, hw, alpha=forced_alpha, t_layer=t_layer, op_timing=0, cuda_graph=use_graph,
                           swap_enabled=0)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] no-swap reference step does not fit ({e})", file=sys.stderr)
            exn = None
        if exn is not None:
            with exn:
                sn = torch.cuda.ExternalStream(exn.stream)
                exn.load_batch(toks, labels)
                for _ in range(3):
                    exn.step_resident()
                torch.cuda.synchronize()
                k = max(1, min(args.steps, 5))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(sn)
                for _ in range(k):
                    exn.step_resident()
                b.record(sn)
                torch.cuda.synchronize()
                nosw_ms = a.elapsed_time(b) / k

    # ---- MEMO report on the measured timeline (reference validator + simulator)
    swap = info0["swap"]
    violations = P.validate_schedule(tl, n, swap)
    p_total = P.count_params(cfg)["total"]
    sim = P.simulate(tl, cfg, hw, p_total)
    flops = P.estimate_flops_per_sample(cfg, p_total)
    n_rec = sum(e.kind == "recompute" for e in tl)
    rec_s = sum(e.end - e.start for e in tl if e.kind == "recompute")
    f_int = inter  # SwiGLU width
    recompute_flops = n_rec * 2.0 * info0["split"][1] * (4.0 * h * h + 2.0 * h * f_int)  # whole job
    mfu = seqs * flops / (t_max * 1e-3) / (world * B200_SPEC_BF16)
    burst, sustained, hbm, peak_src = measured_peaks()
    off = [e for e in tl if e.kind == "offload"]
    pre = [e for e in tl if e.kind == "prefetch"]
    off_s = sum(e.end - e.start for e in off)
    pre_s = sum(e.end - e.start for e in pre)
    ops = info["ops"]
    dk = ops["attn_bwd_dkdv"]
    achieved = dk["flops"] / dk["count"] / (dk["ms"] / dk["count"] * 1e-3) / 1e12 if dk["count"] else None
    traffic = None
    try:
        # DRAM bytes of one launch at the bench shape, from the committed `ncu --set full` capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("attn_bwd_dkdv", {}).get("dram_bytes_per_launch")
    except OSError:
        pass
    kernels = {k: {"ms_per_step": v["ms"], "launches": v["count"],
                   "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] and v["flops"] else None}
               for k, v in ops.items()}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max,
        "higher_is_better": True, "scaling": "strong" if mode == "tp" else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (splitmix64 tokens, counter-hash random-init weights)",
        "config": {**workload_config(args.config), "global_batch": world if mode == "replicas" else 1,
                   "parallelism": {"single": "single", "tp": f"sp+tp{world} ({comm})",
                                                 "replicas": f"replicas{world}"}[mode],
                   "l2": "working set (GB of activations) >> 126 MB L2; no flush needed",
                   "alpha": swap.alpha, "swap_tokens": info0["split"][0],
                   "recompute_tokens": info0["split"][1], "t_layer_measured_s": t_layer,
                   "host_link_d2h_GBps": link["d2h"] / 1e9, "host_link_h2d_GBps": link["h2d"] / 1e9,
                   "cpu_mem_budget": cpu_mem, "cuda_graph": bool(use_graph)},
        "tokens_per_s_per_gpu": value / world,
        "mfu": mfu, "mfu_vs_measured_peak": mfu * B200_SPEC_BF16 / (burst * 1e12),
        # HFU adds the recomputed suffix rows of every swapped layer: QKV, out-projection
        # and gate/up GEMMs (the attention output itself is swapped, not recomputed)
        "hfu": (seqs * flops + seqs * recompute_flops) / (t_max * 1e-3) / (world * B200_SPEC_BF16),
        "e2e": {"value": seqs * S / (e2e * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(info_e2e["h2d_bytes"]), "d2h_bytes_per_step": int(info_e2e["d2h_bytes"])},
        "roofline": {"kernel": "attn_bwd_dkdv (causal FlashAttention dK/dV, tcgen05)",
                     "bound": "tensor", "achieved": achieved, "peak": sustained,
                     "unit": "TFLOP/s", "frac": (achieved / sustained) if achieved else None,
                     "traffic": traffic, "peak_source": f"{peak_src} bf16_tflops_sustained",
                     "algorithmic_flops_per_launch": dk["flops"] / dk["count"] if dk["count"] else None},
        "kernels": kernels,
        "memo": {"schedule_violations": violations, "sim": sim,
                 # compute-stream gaps waiting on copy events (simulate, schedule.hpp:250-297)
                 # + stalls on the copy event waited inside a layer (copy_wait_ms)
                 "exposed_swap_s": sim["compute_blocked"] + info["copy_wait_ms"] * 1e-3,
                 "exposed_swap_frac": ((sim["compute_blocked"] + info["copy_wait_ms"] * 1e-3) / sim["iteration_time"]
                                       if sim["iteration_time"] else None),
                 "in_layer_copy_wait_s": info["copy_wait_ms"] * 1e-3,
                 "no_swap_ms_per_step": nosw_ms,
                 # T(swap) - T(swap disabled): recompute (MEMO's price for the swapped
                 # tokens' skeletal activations) + any exposed copy time
                 "swap_vs_no_swap_delta_s": (t_max - nosw_ms) * 1e-3 if nosw_ms else None,
                 "recompute_s": rec_s,
                 "exposed_swap_delta_s": (t_max - nosw_ms) * 1e-3 - rec_s if nosw_ms else None,
                 "hbm_free_before_timed_steps": free_before, "hbm_free_after_timed_steps": free_after,
                 "hbm_unchanged_over_timed_steps": free_before == free_after,
                 "forward_blocked_s": sim["forward_blocked"],
                 "offload_GBps": info["offload_bytes"] / off_s / 1e9 if off_s else None,
                 "prefetch_GBps": info["prefetch_bytes"] / pre_s / 1e9 if pre_s else None,
                 "planned_device_bytes": info0["device_bytes"], "arena_bytes": info0["arena_bytes"],
                 "rounding_buffer_bytes": info0["rb_bytes"], "state_bytes": info0["state_bytes"],
                 "measured_device_bytes": free0 - free1, "pinned_bytes": info0["pinned_bytes"],
                 "cpu_footprint_planned": swap.cpu_footprint},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(CONFIGS[args.config])
        rp = reference_planner_ms(args.config)
        if rp is not None:
            line["cpu_baseline"]["reference_planner_ms"] = rp
    ex.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    wd.cancel()


if __name__ == "__main__":
    main()
