"""tcgen05 causal FlashAttention (csrc/kernels/attention.cu) vs a PyTorch fp32 reference."""
import ctypes as C
import math
import os

import pytest
import torch

from paper_2407_12117_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def ref_attention(q, k, v, H, D):
    S = q.shape[0]
    qf = q.float().view(S, H, D).transpose(0, 1)
    kf = k.float().view(S, H, D).transpose(0, 1)
    vf = v.float().view(S, H, D).transpose(0, 1)
    s = qf @ kf.transpose(1, 2) / math.sqrt(D)
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    p = torch.softmax(s, -1)
    o = (p @ vf).transpose(0, 1).reshape(S, H * D)
    return o, lse


def run_fwd(q, k, v, H, D):
    S = q.shape[0]
    o = torch.empty_like(q)
    lse = torch.empty(H, S, device="cuda", dtype=torch.float32)
    _abi.check(_abi.lib.memo_attn_fwd(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                      C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()),
                                      C.c_void_p(lse.data_ptr()), S, H, D,
                                      C.c_float(1.0 / math.sqrt(D)), None))
    torch.cuda.synchronize()
    return o, lse


@pytest.mark.parametrize("S,H,D", [(128, 1, 128), (256, 2, 128), (512, 2, 64), (1024, 3, 128),
                                   (768, 4, 64)])
def test_attn_fwd(S, H, D):
    torch.manual_seed(S + H + D)
    q = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    k = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    v = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    o, lse = run_fwd(q, k, v, H, D)
    o_ref, lse_ref = ref_attention(q, k, v, H, D)
    torch.testing.assert_close(lse, lse_ref, rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(o.float(), o_ref, rtol=2e-2, atol=2e-2)


def test_attn_fwd_large_logits():
    # Rows whose max grows late exercise the lazy O rescale.
    torch.manual_seed(7)
    S, H, D = 1024, 2, 128
    q = (torch.randn(S, H * D, device="cuda") * 3).to(torch.bfloat16)
    k = (torch.randn(S, H * D, device="cuda") * 3).to(torch.bfloat16)
    k[-256:] *= 2
    v = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    o, lse = run_fwd(q, k, v, H, D)
    o_ref, lse_ref = ref_attention(q, k, v, H, D)
    torch.testing.assert_close(lse, lse_ref, rtol=1e-3, atol=5e-3)
    torch.testing.assert_close(o.float(), o_ref, rtol=2e-2, atol=2e-2)


def run_bwd(q, k, v, o, lse, do, H, D, rope=None, pos0=0):
    S = q.shape[0]
    h = H * D
    dqkv = torch.zeros(S, 3 * h, device="cuda", dtype=torch.bfloat16)
    nbytes = _abi.lib.memo_attn_bwd_workspace_bytes(S, H, D)
    ws = torch.empty((nbytes + 3) // 4, device="cuda", dtype=torch.float32)
    base = dqkv.data_ptr()
    _abi.check(_abi.lib.memo_attn_bwd(
        C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
        C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), C.c_void_p(do.data_ptr()),
        C.c_void_p(ws.data_ptr()), C.c_void_p(base), C.c_void_p(base + 2 * h), C.c_void_p(base + 4 * h),
        C.c_int64(3 * h), C.c_void_p(rope.data_ptr() if rope is not None else None), C.c_int64(pos0),
        S, H, D, C.c_float(1.0 / math.sqrt(D)), None))
    torch.cuda.synchronize()
    return dqkv[:, :h], dqkv[:, h:2 * h], dqkv[:, 2 * h:]


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


# Even tile counts run the dQ kernel as CTA pairs sharing K/V (D=128: a chunk of
# each per CTA; D=64: K from one CTA, V from the other); odd counts (128, 384,
# 640) run one CTA per query tile.
@pytest.mark.parametrize("S,H,D", [(128, 1, 128), (256, 2, 128), (512, 2, 64), (1024, 2, 128), (384, 2, 128),
                                   (640, 1, 64)])
def test_attn_bwd(S, H, D):
    torch.manual_seed(11 + S + D)
    q = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    k = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    v = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    do = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    o, lse = run_fwd(q, k, v, H, D)
    dq, dk, dv = run_bwd(q, k, v, o, lse, do, H, D)
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    o_ref, _ = ref_attention(qf, kf, vf, H, D)
    o_ref.backward(do.float())
    assert _rel(dv, vf.grad) < 1e-2, _rel(dv, vf.grad)
    assert _rel(dk, kf.grad) < 1e-2, _rel(dk, kf.grad)
    assert _rel(dq, qf.grad) < 1e-2, _rel(dq, qf.grad)


def test_attn_bwd_rope_and_determinism():
    torch.manual_seed(5)
    S, H, D = 512, 2, 128
    pos0 = 128
    half = D // 2
    inv = torch.tensor([10000.0 ** (-2.0 * p / D) for p in range(half)], dtype=torch.float64)
    ang = torch.arange(pos0 + S, dtype=torch.float64)[:, None] * inv[None, :]
    rope = torch.stack([ang.cos(), ang.sin()], -1).float().cuda().contiguous()
    q = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    k = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    v = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    do = torch.randn(S, H * D, device="cuda").to(torch.bfloat16)
    o, lse = run_fwd(q, k, v, H, D)
    dq0, dk0, dv0 = run_bwd(q, k, v, o, lse, do, H, D)
    dq, dk, dv = run_bwd(q, k, v, o, lse, do, H, D, rope, pos0)
    dq2, dk2, dv2 = run_bwd(q, k, v, o, lse, do, H, D, rope, pos0)
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)
    cs = rope[pos0:pos0 + S]

    def inv_rot(t):
        t = t.float().view(S, H, half, 2)
        c, s_ = cs[:, None, :, 0], cs[:, None, :, 1]
        a, b = t[..., 0], t[..., 1]
        return torch.stack([a * c + b * s_, -a * s_ + b * c], -1).view(S, H * D)
    assert _rel(dq, inv_rot(dq0)) < 1e-2
    assert _rel(dk, inv_rot(dk0)) < 1e-2
    assert torch.equal(dv, dv0)


@pytest.mark.parametrize("S,H,D", [(1024, 2, 64), (1024, 2, 128)])
def test_attn_bwd_bitwise_repeatable(S, H, D):
    """Races between the softmax-gradient warps and the MMA issuer show up as
    run-to-run differences: 12 repetitions must be bitwise identical."""
    torch.manual_seed(3)
    q, k, v, do = (torch.randn(S, H * D, device="cuda").to(torch.bfloat16) for _ in range(4))
    o, lse = run_fwd(q, k, v, H, D)
    ref = run_bwd(q, k, v, o, lse, do, H, D)
    for _ in range(12):
        o2, lse2 = run_fwd(q, k, v, H, D)
        assert torch.equal(o2, o) and torch.equal(lse2, lse)
        got = run_bwd(q, k, v, o, lse, do, H, D)
        for a, b in zip(got, ref):
            assert torch.equal(a, b)


_FUSED_SCRIPT = r"""
import math, sys, torch
sys.path.insert(0, {root!r})
from tests.test_attention_gpu import run_fwd, run_bwd, ref_attention, _rel
torch.manual_seed(9)
S, H, D = 1024, 2, 128
q, k, v, do = (torch.randn(S, H * D, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = run_fwd(q, k, v, H, D)
g1 = run_bwd(q, k, v, o, lse, do, H, D)
g2 = run_bwd(q, k, v, o, lse, do, H, D)
assert all(torch.equal(a, b) for a, b in zip(g1, g2)), "fused bwd not deterministic"
qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
o_ref, _ = ref_attention(qf, kf, vf, H, D)
o_ref.backward(do.float())
for got, want in zip(g1, (qf.grad, kf.grad, vf.grad)):
    assert _rel(got, want) < 1e-2, _rel(got, want)
print("fused ok")
"""


ABLATION_LIB = os.path.join(ROOT, "paper_2407_12117_b200", "_lib_ablations", "libmemo.so")


@pytest.mark.skipif(not os.path.exists(ABLATION_LIB), reason="ablation library not built")
def test_attn_bwd_fused_ablation():
    """The fused 5-unit backward of the ABLATION library (MEMO_ATTN_BWD=fused,
    make -C csrc ablations): one kernel for dK/dV/dQ with dQ partials reduced
    at L2 in ticket order -- same parity bar and bitwise repeatable."""
    import subprocess
    import sys
    root = ROOT
    env = dict(os.environ, MEMO_ATTN_BWD="fused", MEMO_LIB_PATH=ABLATION_LIB)
    out = subprocess.run([sys.executable, "-c", _FUSED_SCRIPT.format(root=root)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "fused ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("D", [64, 128])
def test_attention_bitwise_under_sanitizer_timing(D, tmp_path):
    """Outputs computed under compute-sanitizer racecheck (which slows and
    reorders execution) equal a normal run bitwise.  Guards the mbarrier
    protocols racecheck cannot see (tcgen05 / TMA async proxy): a forward
    epilogue that waited a barrier by parity while it could be a phase behind
    produced a wrong O at D=64 under exactly this perturbation."""
    import shutil
    import subprocess
    import sys
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    probe = os.path.join(ROOT, "tools", "attn_golden_probe.py")
    ref = str(tmp_path / "ref.pt")
    subprocess.check_call([sys.executable, probe, "save", "1024", "2", str(D), ref], timeout=300)
    out = subprocess.run([cs, "--tool", "racecheck", sys.executable, probe, "check", "1024", "2", str(D), ref],
                         capture_output=True, text=True, timeout=600).stdout
    assert "DIFFERS" not in out and out.count("equal") == 3, out[-2000:]
