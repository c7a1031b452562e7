"""Independent torch (fp64 autograd) restatement of the model definition in
oracle/llama_cpu.c, used only to pin the C oracle (tests/test_oracle.py).

bf16 storage points are straight-through: forward values are rounded to bf16,
gradients pass unchanged — exactly the oracle's convention.
"""
import math

import numpy as np
import torch


def B(x):
    return x + (x.to(torch.bfloat16).to(x.dtype) - x).detach()


def unpack(cfg, p):
    h, F, V, n = cfg.hidden, cfg.ffn, cfg.vocab, cfg.n_layers
    off = 0

    def take(cnt, shape):
        nonlocal off
        t = p[off:off + cnt].view(*shape)
        off += cnt
        return t
    E = take(V * h, (V, h))
    layers = []
    for _ in range(n):
        layers.append(dict(g1=take(h, (h,)), wqkv=take(3 * h * h, (3 * h, h)), wo=take(h * h, (h, h)),
                           g2=take(h, (h,)), wgu=take(2 * F * h, (2 * F, h)), wd=take(h * F, (h, F))))
    gf = take(h, (h,))
    W = take(V * h, (V, h))
    return E, layers, gf, W


def rmsnorm(x, g, eps):
    r = 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + eps)
    return x * r * g


def rope_tables(S, D, theta):
    half = D // 2
    cs = np.zeros((S, half, 2), dtype=np.float32)
    for t in range(S):
        for p in range(half):
            inv = math.pow(theta, -2.0 * p / D)
            cs[t, p, 0] = np.float32(math.cos(t * inv))
            cs[t, p, 1] = np.float32(math.sin(t * inv))
    return torch.from_numpy(cs).double()


def rope(x, cs, H, D):
    S = x.shape[0]
    t = x.view(S, H, D // 2, 2)
    c, s = cs[:, None, :, 0], cs[:, None, :, 1]
    a, b = t[..., 0], t[..., 1]
    return torch.stack([a * c - b * s, a * s + b * c], -1).view(S, H * D)


def loss_fn(cfg, p, tokens, labels):
    S, h, H, D, F = cfg.seq, cfg.hidden, cfg.n_heads, cfg.head_dim, cfg.ffn
    E, layers, gf, W = unpack(cfg, p)
    cs = rope_tables(S, D, cfg.rope_theta)
    x = E[torch.as_tensor(tokens, dtype=torch.long)]
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool), 1)
    for L in layers:
        xn = B(rmsnorm(x, L["g1"], cfg.eps))
        qkv = xn @ L["wqkv"].t()
        q = B(rope(B(qkv[:, :h]), cs, H, D))
        k = B(rope(B(qkv[:, h:2 * h]), cs, H, D))
        v = B(qkv[:, 2 * h:])
        qh, kh, vh = (t.view(S, H, D).transpose(0, 1) for t in (q, k, v))
        s = (qh @ kh.transpose(1, 2)) / math.sqrt(D)
        s = s.masked_fill(mask, float("-inf"))
        o = B((torch.softmax(s, -1) @ vh).transpose(0, 1).reshape(S, h))
        a = B(o @ L["wo"].t())
        x1 = x + a
        xn2 = B(rmsnorm(x1, L["g2"], cfg.eps))
        gu = xn2 @ L["wgu"].t()
        g, u = B(gu[:, :F]), B(gu[:, F:])
        act = B(torch.nn.functional.silu(g) * u)
        x = x1 + B(act @ L["wd"].t())
    xf = B(rmsnorm(x, gf, cfg.eps))
    logits = xf @ W.t()
    lab = torch.as_tensor(labels, dtype=torch.long)
    keep = lab >= 0
    return torch.nn.functional.cross_entropy(logits[keep], lab[keep])


def loss_and_grads(cfg, params_np, tokens, labels):
    p = torch.tensor(params_np, dtype=torch.float64, requires_grad=True)
    loss = loss_fn(cfg, p, tokens, labels)
    loss.backward()
    return loss.item(), p.grad.numpy()


def amp_loss_and_grads(cfg, params_np, tokens, labels, device="cuda"):
    """The same model as PyTorch's standard bf16 mixed-precision step: fp32
    master parameters, torch.autocast(bfloat16) GEMMs, scaled_dot_product_attention
    (flash, bf16) and fp32 autograd.  No straight-through roundings: autocast's
    own bf16 casts are the storage points.  Used as the yardstick of what bf16
    training error looks like at a given width (tests/test_fullwidth_gpu.py)."""
    S, h, H, D, F = cfg.seq, cfg.hidden, cfg.n_heads, cfg.head_dim, cfg.ffn
    p = torch.tensor(params_np, dtype=torch.float32, device=device, requires_grad=True)
    E, layers, gf, W = unpack(cfg, p)
    cs = rope_tables(S, D, cfg.rope_theta).float().to(device)
    tok = torch.as_tensor(tokens, dtype=torch.long, device=device)
    lab = torch.as_tensor(labels, dtype=torch.long, device=device)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        x = E[tok]
        for L in layers:
            xn = rmsnorm(x.float(), L["g1"], cfg.eps)
            qkv = xn @ L["wqkv"].t()
            q = rope(qkv[:, :h].float(), cs, H, D).to(torch.bfloat16)
            k = rope(qkv[:, h:2 * h].float(), cs, H, D).to(torch.bfloat16)
            v = qkv[:, 2 * h:]
            qh, kh, vh = (t.reshape(S, H, D).transpose(0, 1)[None] for t in (q, k, v))
            o = torch.nn.functional.scaled_dot_product_attention(qh, kh, vh, is_causal=True)
            o = o[0].transpose(0, 1).reshape(S, h)
            x1 = x.float() + (o @ L["wo"].t()).float()
            xn2 = rmsnorm(x1, L["g2"], cfg.eps)
            gu = xn2 @ L["wgu"].t()
            act = torch.nn.functional.silu(gu[:, :F].float()) * gu[:, F:].float()
            x = x1 + (act @ L["wd"].t()).float()
        xf = rmsnorm(x.float(), gf, cfg.eps)
        logits = (xf @ W.t()).float()
        keep = lab >= 0
        loss = torch.nn.functional.cross_entropy(logits[keep], lab[keep])
    loss.backward()
    return loss.item(), p.grad.detach().cpu().numpy()
