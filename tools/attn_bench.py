"""Attention kernel alone: TFLOP/s at the bench shape (B=8, H=24, N=4608, d=128) + a parity spot check vs torch SDPA.
TRACE=1 prints the clock64 timeline of CTA 0; it needs a trace build of the kernel:
python tools/variant.py trace attention_tc.cu -DATTN_TRACE=1, then DIT_LIB_OVERRIDE=<that .so>."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_08123_b200 import dit  # noqa: E402

lib = dit.load_library()
B, H, N, d = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 24, 4608, 128))]
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g, dtype=torch.float32).to(torch.bfloat16) for _ in range(3))
out = torch.empty(B * N, H * d, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream()
call = lambda: lib.dit_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, N, d, out.data_ptr(), C.c_void_p(s.cuda_stream))
assert call() == 0
torch.cuda.synchronize()
ref = torch.nn.functional.scaled_dot_product_attention(q[:1, :2].float(), k[:1, :2].float(), v[:1, :2].float())
got = out.view(B, N, H, d)[:1, :, :2].permute(0, 2, 1, 3).float()
err = ((got - ref).abs().max() / ref.abs().max()).item()
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 10
e0.record(s)
for _ in range(n):
    call()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
fl = 4.0 * B * H * N * N * d
print(f"attention B={B} H={H} N={N} d={d}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s  max-norm err vs SDPA {err:.2e}")

if os.environ.get("TRACE"):
    tr = torch.zeros(20, 64, dtype=torch.int64, device="cuda")
    lib.dit_debug_attention_trace(tr.data_ptr())
    call()
    torch.cuda.synchronize()
    lib.dit_debug_attention_trace(None)
    t = tr.cpu().numpy()
    base = t[t > 0].min()
    names = ["k_load", "v_load", "mma_kfull", "mma_p0", "mma_p1", "mma_vfull", "sm_s0", "sm_s1", "sm_p0", "sm_p1",
             "ld0", "ld1", "xchg0", "xchg1"]
    for j in range(min(14, N // 128)):
        print(j, " ".join(f"{nm}={(t[e, j] - base) if t[e, j] else -1:7d}" for e, nm in enumerate(names)))
    # per-iteration phase durations of tile 0 (median over j = 4 .. nkv-2)
    import numpy as np
    J = range(4, min(60, N // 128) - 1)
    d = lambda a, b_, dj=0: int(np.median([t[b_, j + dj] - t[a, j] for j in J]))
    print("tile0: S wake->ld done", d(6, 10), " ld->xchg", d(10, 12), " xchg->P arrive", d(12, 8),
          " P arrive->MMA sees it", d(8, 3), " MMA issues PV0 -> next S0 wake", d(3, 6, 1), " period", d(6, 6, 1))
    print("MMA thread: k_full wait", d(14, 2), " p_full0 wait", d(15, 3), " p_full1 wait", d(16, 4),
          " PV0 issue start -> QK0 k_full wait start", d(5, 14, 1), " QK0 issued -> PV1 wait start", d(2, 16))
    print("tile0 P-arrive skew vs warp 0 (warps 1,2,3):", d(8, 17), d(8, 18), d(8, 19), " S wake of warp0 -> MMA sees P0", d(6, 3))
