"""Causal FlashAttention forward/backward at the bench's sequence lengths
(S = 8K, 32K, 128K; D = 128, the Llama-7B head) against a chunked fp32 torch
reference on SAMPLED 512-row blocks.

The kernels run over the whole sequence; the reference is exact fp32 (no TF32)
and computed only where it is checked:
  * query blocks (first, middle, last -- the last has the longest causal span):
    O, LSE and dQ of those rows;
  * key blocks (first -- summed over every query --, middle, last): dK and dV.
The reference's row statistics (LSE, delta = rowsum(dO * O)) come from a full
chunked pass over all queries, so dK/dV are checked against reference
statistics, not the kernel's.  This covers the paths short tests cannot reach:
the lazy O rescale over thousands of key tiles, the FMA-pipe exp2 share and
fp32 accumulation over up to 1024 tiles.  Tolerances as in test_attention_gpu:
relative L2 1e-2 for the gradients, 2e-2 for O, 2e-3 absolute for LSE.
"""
import math

import pytest
import torch

from tests.test_attention_gpu import _rel, run_bwd, run_fwd

pytestmark = pytest.mark.gpu

BLK = 512
CH = 4096  # query rows per reference chunk


def _heads(t, H, D):
    return t.float().view(t.shape[0], H, D).transpose(0, 1)  # [H, S, D]


def _ref_row_stats(q, k, v, do, H, D):
    """Exact fp32 LSE [H, S] and delta = rowsum(dO * O_ref) [H, S], chunked."""
    S = q.shape[0]
    scale = 1.0 / math.sqrt(D)
    qh, kh, vh, doh = (_heads(t, H, D) for t in (q, k, v, do))
    lse = torch.empty(H, S, device="cuda")
    delta = torch.empty(H, S, device="cuda")
    for c0 in range(0, S, CH):
        c1 = min(S, c0 + CH)
        s = qh[:, c0:c1] @ kh[:, :c1].transpose(1, 2) * scale          # [H, c, c1]
        rows = torch.arange(c0, c1, device="cuda")[:, None]
        s.masked_fill_(torch.arange(c1, device="cuda")[None, :] > rows, float("-inf"))
        l = torch.logsumexp(s, -1)
        o = torch.exp(s - l[..., None]) @ vh[:, :c1]
        lse[:, c0:c1] = l
        delta[:, c0:c1] = (o * doh[:, c0:c1]).sum(-1)
        del s
    return lse, delta


def _ref_query_block(q, k, v, do, lse, delta, r0, H, D):
    """O, LSE, dQ of query rows [r0, r0+BLK)."""
    scale = 1.0 / math.sqrt(D)
    r1 = r0 + BLK
    qh, kh, vh, doh = (_heads(t, H, D) for t in (q, k, v, do))
    s = qh[:, r0:r1] @ kh[:, :r1].transpose(1, 2) * scale
    rows = torch.arange(r0, r1, device="cuda")[:, None]
    s.masked_fill_(torch.arange(r1, device="cuda")[None, :] > rows, float("-inf"))
    p = torch.exp(s - lse[:, r0:r1, None])
    o = p @ vh[:, :r1]
    dp = doh[:, r0:r1] @ vh[:, :r1].transpose(1, 2)
    ds = p * (dp - delta[:, r0:r1, None])
    dq = ds @ kh[:, :r1] * scale
    flat = lambda t: t.transpose(0, 1).reshape(BLK, H * D)  # noqa: E731
    return flat(o), lse[:, r0:r1], flat(dq)


def _ref_key_block(q, k, v, do, lse, delta, c0, H, D):
    """dK, dV of key rows [c0, c0+BLK): every query q >= c0 contributes."""
    S = q.shape[0]
    scale = 1.0 / math.sqrt(D)
    c1 = c0 + BLK
    qh, kh, vh, doh = (_heads(t, H, D) for t in (q, k, v, do))
    dk = torch.zeros(H, BLK, D, device="cuda")
    dv = torch.zeros(H, BLK, D, device="cuda")
    for q0 in range(c0, S, CH):
        q1 = min(S, q0 + CH)
        s = qh[:, q0:q1] @ kh[:, c0:c1].transpose(1, 2) * scale          # [H, cq, BLK]
        rows = torch.arange(q0, q1, device="cuda")[:, None]
        s.masked_fill_(torch.arange(c0, c1, device="cuda")[None, :] > rows, float("-inf"))
        p = torch.exp(s - lse[:, q0:q1, None])
        dp = doh[:, q0:q1] @ vh[:, c0:c1].transpose(1, 2)
        ds = p * (dp - delta[:, q0:q1, None])
        dv += p.transpose(1, 2) @ doh[:, q0:q1]
        dk += ds.transpose(1, 2) @ qh[:, q0:q1]
    flat = lambda t: t.transpose(0, 1).reshape(BLK, H * D)  # noqa: E731
    return flat(dk * scale), flat(dv)


@pytest.mark.parametrize("S", [8192, 32768, 131072])
def test_attention_long_sequence_sampled_blocks(S):
    H, D = 2, 128
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(S)
    mk = lambda sd: (torch.randn(S, H * D, device="cuda", generator=g) * sd).to(torch.bfloat16)  # noqa: E731
    # head-0 queries sharper than head-1's: peaked and diffuse softmax rows
    q = mk(1.0)
    q.view(S, H, D)[:, 0] *= 2
    k, v, do = mk(1.0), mk(1.0), mk(1.0)
    o, lse = run_fwd(q, k, v, H, D)
    dq, dk, dv = run_bwd(q, k, v, o, lse, do, H, D)
    lse_ref, delta_ref = _ref_row_stats(q, k, v, do, H, D)
    torch.testing.assert_close(lse, lse_ref, rtol=0, atol=2e-3)
    mid = (S // 2 // BLK) * BLK
    for r0 in (0, mid, S - BLK):
        o_r, _, dq_r = _ref_query_block(q, k, v, do, lse_ref, delta_ref, r0, H, D)
        assert _rel(o[r0:r0 + BLK], o_r) < 2e-2, ("O", S, r0, _rel(o[r0:r0 + BLK], o_r))
        assert _rel(dq[r0:r0 + BLK], dq_r) < 1e-2, ("dQ", S, r0, _rel(dq[r0:r0 + BLK], dq_r))
    for c0 in (0, mid, S - BLK):
        dk_r, dv_r = _ref_key_block(q, k, v, do, lse_ref, delta_ref, c0, H, D)
        assert _rel(dk[c0:c0 + BLK], dk_r) < 1e-2, ("dK", S, c0, _rel(dk[c0:c0 + BLK], dk_r))
        assert _rel(dv[c0:c0 + BLK], dv_r) < 1e-2, ("dV", S, c0, _rel(dv[c0:c0 + BLK], dv_r))


def test_attention_long_sequence_large_logits():
    """Logits of scale ~9 at S = 16K with the largest keys late in the sequence:
    row maxima keep growing across key tiles, so the forward's lazy rescale
    (threshold 2^8) fires many times per row."""
    S, H, D = 16384, 2, 128
    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device="cuda").manual_seed(77)
    q = (torch.randn(S, H * D, device="cuda", generator=g) * 3).to(torch.bfloat16)
    kf = torch.randn(S, H * D, device="cuda", generator=g) * 3
    kf *= torch.linspace(0.5, 1.5, S, device="cuda")[:, None]
    k = kf.to(torch.bfloat16)
    v = torch.randn(S, H * D, device="cuda", generator=g).to(torch.bfloat16)
    do = torch.randn(S, H * D, device="cuda", generator=g).to(torch.bfloat16)
    o, lse = run_fwd(q, k, v, H, D)
    dq, dk, dv = run_bwd(q, k, v, o, lse, do, H, D)
    lse_ref, delta_ref = _ref_row_stats(q, k, v, do, H, D)
    torch.testing.assert_close(lse, lse_ref, rtol=0, atol=5e-3)
    for r0 in (0, S // 2, S - BLK):
        o_r, _, dq_r = _ref_query_block(q, k, v, do, lse_ref, delta_ref, r0, H, D)
        assert _rel(o[r0:r0 + BLK], o_r) < 2e-2, ("O", r0, _rel(o[r0:r0 + BLK], o_r))
        assert _rel(dq[r0:r0 + BLK], dq_r) < 1e-2, ("dQ", r0, _rel(dq[r0:r0 + BLK], dq_r))
    for c0 in (0, S - BLK):
        dk_r, dv_r = _ref_key_block(q, k, v, do, lse_ref, delta_ref, c0, H, D)
        assert _rel(dk[c0:c0 + BLK], dk_r) < 1e-2, ("dK", c0, _rel(dk[c0:c0 + BLK], dk_r))
        assert _rel(dv[c0:c0 + BLK], dv_r) < 1e-2, ("dV", c0, _rel(dv[c0:c0 + BLK], dv_r))
