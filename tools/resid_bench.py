"""The step's GEMM alone with the plain bias epilogue vs the gated-residual epilogue (h fp32
read-modify-write) at the double-block proj / fc2 and single linear2 shapes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_08123_b200 import dit  # noqa: E402

lib = dit.load_library()


def timed(fn, n=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


SHAPES = {"proj": (36864, 3072, 3072), "fc2": (36864, 12288, 3072), "linear2": (36864, 15360, 3072),
          "sd3m_proj": (35432, 1536, 1536), "sd3m_fc2": (35432, 6144, 1536), "sd35l_proj": (35432, 2432, 2432)}
for name, (M, K, N) in SHAPES.items():
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.randn(N, device="cuda", dtype=torch.bfloat16) * 0.02
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    h = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    g = torch.full((N,), 0.5, device="cuda", dtype=torch.float32)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    f_bias = lambda: lib.dit_debug_gemm(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), M, N, K, st)
    f_res = lambda: lib.dit_debug_gemm_resid(x.data_ptr(), w.data_ptr(), b.data_ptr(), h.data_ptr(), g.data_ptr(),
                                             M, N, K, st)
    tb, tr = [], []
    for _ in range(2):
        tb.append(timed(f_bias))
        tr.append(timed(f_res))
    fl = 2 * M * N * K
    print(f"{name}: bias {fl / min(tb) / 1e9:.0f} TF/s ({min(tb):.3f} ms)   resid {fl / min(tr) / 1e9:.0f} TF/s "
          f"({min(tr):.3f} ms)")
