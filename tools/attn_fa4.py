"""Library bar: FlashAttention-4 (vllm's cute-DSL build) at the bench attention shape, for comparison only."""
import sys
import torch
from vllm.vllm_flash_attn.cute.interface import flash_attn_func

B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 24, 4608, 128))]
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, N, H, d, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
for _ in range(3):
    o = flash_attn_func(q, k, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record()
for _ in range(n):
    o = flash_attn_func(q, k, v)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"FA4 (cute) B={B} H={H} N={N} d={d}: {ms:.3f} ms  {4.0 * B * H * N * N * d / ms / 1e9:.1f} TFLOP/s")
