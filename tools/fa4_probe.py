"""Run FlashAttention-4 (vllm's CuTe-DSL build, a library kernel) causal forward once at the bench
shape, so ncu can capture it next to ours and CUTE_DSL_KEEP=ptx,cubin can dump its code:
  CUTE_DSL_KEEP=ptx,cubin CUTE_DSL_DUMP_DIR=out python tools/fa4_probe.py S [H]"""
import sys

import torch

from vllm.vllm_flash_attn.cute import flash_attn_func

S = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
q, k, v = (torch.randn(1, S, H, 128, device="cuda", dtype=torch.bfloat16) for _ in range(3))
for _ in range(2):
    o = flash_attn_func(q, k, v, causal=True, deterministic=True)
torch.cuda.synchronize()
print("ok", S, H)
