"""Same-box library bar for the attention shape (context only, never on the product path)."""
import sys
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 24, 4608, 128))]
q, k, v = (torch.randn(B, H, N, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
fl = 4.0 * B * H * N * N * d


def bench(fn, name):
    try:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{name:28s} {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
    except Exception as e:  # noqa
        print(f"{name:28s} unavailable: {str(e)[:100]}")


for be, nm in [(SDPBackend.CUDNN_ATTENTION, "torch sdpa cudnn"), (SDPBackend.FLASH_ATTENTION, "torch sdpa flash")]:
    def f(be=be):
        with sdpa_kernel(be):
            return F.scaled_dot_product_attention(q, k, v)
    bench(f, nm)
try:
    import flashinfer
    qf, kf, vf = (x.transpose(1, 2).reshape(B * N, H, d).contiguous() for x in (q, k, v))
    indptr = torch.arange(0, (B + 1) * N, N, device="cuda", dtype=torch.int32)
    for backend in ("cutlass", "fa2"):
        try:
            ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
            w.plan(indptr, indptr, H, H, d, causal=False, q_data_type=torch.bfloat16)
            bench(lambda: w.run(qf, kf, vf), f"flashinfer {backend}")
        except Exception as e:  # noqa
            print(f"flashinfer {backend:18s} unavailable: {str(e)[:120]}")
except Exception as e:  # noqa
    print("flashinfer unavailable", str(e)[:100])
