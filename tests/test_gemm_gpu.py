"""tcgen05 GEMM (csrc/kernels/gemm_tc.cu) vs a plain PyTorch fp32 reference."""
import ctypes as C

import pytest
import torch

from paper_2407_12117_b200 import _abi

pytestmark = pytest.mark.gpu


def _gemm(M, N, K, a, lda, a_mn, b, ldb, b_mn, epi, c=None, ldc=0, **kw):
    args = _abi.GemmArgsC()
    args.M, args.N, args.K = M, N, K
    args.a, args.lda, args.a_mn_major = a.data_ptr(), lda, a_mn
    args.b, args.ldb, args.b_mn_major = b.data_ptr(), ldb, b_mn
    args.epilogue = epi
    args.c = c.data_ptr() if c is not None else None
    args.ldc = ldc
    for k, v in kw.items():
        setattr(args, k, v.data_ptr() if isinstance(v, torch.Tensor) else v)
    _abi.check(_abi.lib.memo_gemm(C.byref(args), None))
    torch.cuda.synchronize()


def _rand(*shape):
    return (torch.randn(*shape, device="cuda") * 0.5).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (384, 768, 4096),
                                   (200, 256, 192), (1024, 2048, 1024)])
@pytest.mark.parametrize("layout", ["fwd", "dgrad", "wgrad"])
def test_gemm_layouts(M, N, K, layout, variant=0):
    torch.manual_seed(0)
    if layout == "fwd":      # A [M,K] K-major, B [N,K] K-major
        A = _rand(M, K); B = _rand(N, K)
        ref = A.float() @ B.float().t()
        a, lda, amn, b, ldb, bmn = A, K, 0, B, K, 0
    elif layout == "dgrad":  # A [M,K] K-major, B stored [K,N] (N contiguous)
        A = _rand(M, K); Bs = _rand(K, N)
        ref = A.float() @ Bs.float()
        a, lda, amn, b, ldb, bmn = A, K, 0, Bs, N, 1
    else:                    # A stored [K,M], B stored [K,N]
        As = _rand(K, M); Bs = _rand(K, N)
        ref = As.float().t() @ Bs.float()
        a, lda, amn, b, ldb, bmn = As, M, 1, Bs, N, 1
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    _gemm(M, N, K, a, lda, amn, b, ldb, bmn, 1, out, N, variant=variant)
    err = (out - ref).abs().max().item()
    assert err <= 1e-3 * (1 + ref.abs().max().item()), err
    outb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(M, N, K, a, lda, amn, b, ldb, bmn, 0, outb, N, variant=variant)
    torch.testing.assert_close(outb.float(), ref.to(torch.bfloat16).float(), rtol=1e-2, atol=1e-2)


def test_gemm_f32_accumulate_and_resid():
    torch.manual_seed(1)
    M, N, K = 256, 512, 320
    A = _rand(M, K); B = _rand(N, K)
    ref = A.float() @ B.float().t()
    acc = torch.full((M, N), 2.0, device="cuda")
    _gemm(M, N, K, A, K, 0, B, K, 0, 2, acc, N)
    torch.testing.assert_close(acc, ref + 2.0, rtol=1e-4, atol=1e-3)
    resid = torch.randn(M, N, device="cuda")
    out = torch.empty(M, N, device="cuda")
    cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _gemm(M, N, K, A, K, 0, B, K, 0, 3, cb, N, out_f32=out, resid=resid, ld_f32=N)
    refb = ref.to(torch.bfloat16)
    torch.testing.assert_close(cb.float(), refb.float(), rtol=1e-2, atol=1e-2)
    torch.testing.assert_close(out, resid + cb.float(), rtol=0, atol=0)


def test_gemm_qkv_rope_epilogue():
    torch.manual_seed(2)
    S, h, d = 256, 512, 128
    X = _rand(S, h); W = _rand(3 * h, h)
    pos0 = 17
    half = d // 2
    inv = torch.tensor([10000.0 ** (-2.0 * p / d) for p in range(half)], dtype=torch.float64)
    pos = torch.arange(pos0 + S, dtype=torch.float64)
    ang = pos[:, None] * inv[None, :]
    rope = torch.stack([ang.cos(), ang.sin()], -1).float().cuda().contiguous()
    q = torch.empty(S, h, device="cuda", dtype=torch.bfloat16)
    k = torch.empty_like(q); v = torch.empty_like(q)
    _gemm(S, 3 * h, h, X, h, 0, W, h, 0, 4, None, 0, q=q, k=k, v=v, hidden=h, head_dim=d,
          rope=rope, pos0=pos0)
    y = (X.float() @ W.float().t()).to(torch.bfloat16).float()
    cs = rope[pos0:pos0 + S]

    def rot(t):
        t = t.view(S, h // d, half, 2)
        c, s_ = cs[:, None, :, 0], cs[:, None, :, 1]
        a, b = t[..., 0], t[..., 1]
        return torch.stack([a * c - b * s_, a * s_ + b * c], -1).view(S, h)
    torch.testing.assert_close(q.float(), rot(y[:, :h]).to(torch.bfloat16).float(), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(k.float(), rot(y[:, h:2 * h]).to(torch.bfloat16).float(), rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(v.float(), y[:, 2 * h:], rtol=1e-2, atol=1e-2)


def test_gemm_cta_pair_variant():
    """variant=4 (CTA-pair 256x256 tiles, cta_group::2) forced on all three
    layouts, ragged M and N, against the fp32 reference."""
    for shp in [(128, 256, 64), (200, 256, 192), (1024, 2048, 1024), (640, 288, 4096)]:
        for lay in ("fwd", "dgrad", "wgrad"):
            test_gemm_layouts(*shp, lay, variant=4)


def test_gemm_pair_cluster_variant_bitwise():
    """variant 5 (two CTA pairs per cluster sharing B by multicast, the default
    for the pair shapes) is bitwise equal to one pair per cluster (variant 4)
    and matches fp32, with ragged M (the cluster's second pair past M) and N,
    on all three layouts (MN-major B: one 64-column box per pair, multicast)."""
    for shp in [(128, 256, 64), (200, 256, 192), (640, 288, 4096), (1024, 2048, 1024), (1536, 768, 512)]:
        for lay in ("fwd", "dgrad", "wgrad"):
            test_gemm_layouts(*shp, lay, variant=5)
    for (M, N, K) in [(200, 512, 192), (640, 288, 512), (2048, 1024, 1024)]:
        torch.manual_seed(M + N + K)
        a, b = _rand(M, K), _rand(N, K)
        outs = []
        for var in (4, 5):
            c = torch.empty(M, N, device="cuda", dtype=torch.float32)
            _gemm(M, N, K, a, K, 0, b, K, 0, 1, c, N, variant=var)
            outs.append(c)
        assert torch.equal(outs[0], outs[1])


def test_gemm_b_multicast_cluster_bitwise():
    """variant 2 (the default single-CTA kernel: 2-CTA clusters, B shared by TMA
    multicast) and 3 (2x2 clusters sharing A and B): bitwise equal to the
    unclustered kernel (variant 1) on all three layouts, with odd M- and N-tile
    counts (a cluster's last tiles are empty)."""
    res = []
    for var in (1, 2, 3):
        outs = []
        for (M, N, K) in [(128, 256, 64), (200, 512, 192), (384, 768, 4096), (1152, 2048, 1024), (640, 288, 512)]:
            torch.manual_seed(M + N + K)
            a, b = _rand(M, K), _rand(N, K)
            c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            _gemm(M, N, K, a, K, 0, b, K, 0, 0, c, N, variant=var)
            outs.append(c.clone())
            bs = _rand(K, N)
            c32 = torch.empty(M, N, device="cuda", dtype=torch.float32)
            _gemm(M, N, K, a, K, 0, bs, N, 1, 1, c32, N, variant=var)
            outs.append(c32.clone())
            as_ = _rand(K, M)
            _gemm(M, N, K, as_, M, 1, bs, N, 1, 1, c32, N, variant=var)
            outs.append(c32.clone())
        res.append(outs)
    for other in res[1:]:
        for x, y in zip(res[0], other):
            assert torch.equal(x, y)


def test_gemm_raster_order_is_bitwise_neutral():
    """The serpentine tile order (product) and the round-1 order give bitwise
    equal outputs on every layout and kernel variant (tile order only)."""
    for var in (0, 1, 2, 4, 5):
        for (M, N, K) in [(1152, 2048, 1024), (2560, 768, 512)]:
            torch.manual_seed(M + N + K + var)
            a, b, bs, as_ = _rand(M, K), _rand(N, K), _rand(K, N), _rand(K, M)
            outs = []
            for raster in (0, 1):
                c = torch.empty(M, N, device="cuda", dtype=torch.float32)
                _gemm(M, N, K, a, K, 0, b, K, 0, 1, c, N, variant=var, raster=raster)
                d = torch.empty(M, N, device="cuda", dtype=torch.float32)
                _gemm(M, N, K, a, K, 0, bs, N, 1, 1, d, N, variant=var, raster=raster)
                e = torch.empty(M, N, device="cuda", dtype=torch.float32)
                _gemm(M, N, K, as_, M, 1, bs, N, 1, 1, e, N, variant=var, raster=raster)
                outs.append((c, d, e))
            for x, y in zip(*outs):
                assert torch.equal(x, y)
