"""Fused elementwise kernels (csrc/kernels/elementwise.cu) vs a float64 PyTorch reference."""
import ctypes as C

import pytest
import torch

from paper_2407_12117_b200 import _abi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("S,h,with_a,with_res", [(300, 256, True, True), (512, 4096, True, True),
                                                  (130, 4096, False, False), (64, 5120, True, False)])
def test_rmsnorm_bwd(S, h, with_a, with_res):
    """Both code paths (register-resident for h in {4096, 5120, 8192}, shared-memory
    otherwise): dx, its bf16 copy and dg against autograd in float64; dg bitwise
    repeatable."""
    torch.manual_seed(S + h)
    eps = 1e-5
    x = torch.randn(S, h, device="cuda")
    a = torch.randn(S, h, device="cuda").to(torch.bfloat16) if with_a else None
    g = (1 + 0.1 * torch.randn(h, device="cuda")).to(torch.bfloat16)
    dy = torch.randn(S, h, device="cuda")
    dres = torch.randn(S, h, device="cuda") if with_res else None
    P = _abi.lib.memo_rmsnorm_bwd_partials(S)
    part = torch.empty(P, h, device="cuda")
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None

    def run():
        dx = torch.empty(S, h, device="cuda")
        dxb = torch.empty(S, h, device="cuda", dtype=torch.bfloat16)
        dg = torch.empty(h, device="cuda")
        _abi.check(_abi.lib.memo_rmsnorm_bwd(ptr(x), ptr(a), ptr(g), ptr(dy), ptr(dres), ptr(dx), ptr(dxb),
                                             ptr(part), ptr(dg), S, h, C.c_float(eps), 0, None))
        torch.cuda.synchronize()
        return dx, dxb, dg

    dx, dxb, dg = run()
    xin = (x.double() + (a.double() if with_a else 0)).requires_grad_()
    gd = g.double().requires_grad_()
    y = xin * torch.rsqrt(xin.pow(2).mean(-1, keepdim=True) + eps) * gd
    y.backward(dy.double())
    want_dx = xin.grad + (dres.double() if with_res else 0)
    rel = lambda u, w: ((u.double() - w).norm() / w.norm()).item()
    assert rel(dx, want_dx) < 1e-5
    assert rel(dxb, want_dx) < 5e-3
    assert rel(dg, gd.grad) < 1e-5
    dx2, _, dg2 = run()
    assert torch.equal(dg, dg2) and torch.equal(dx, dx2)
