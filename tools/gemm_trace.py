"""GEMM timeline (variant build with -DGEMM_TRACE=1): per tile of CTA 0, epilogue start/end and the
MMA warp's accumulator wait, for the bias and the gated-residual epilogue at one shape."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_08123_b200 import dit  # noqa: E402

lib = dit.load_library()
M, K, N = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (36864, 3072, 3072))]
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
b = torch.randn(N, device="cuda", dtype=torch.bfloat16) * 0.02
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
h = torch.zeros(M, N, device="cuda", dtype=torch.float32)
g = torch.full((N,), 0.5, device="cuda", dtype=torch.float32)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
tr = torch.zeros(8, 64, dtype=torch.int64, device="cuda")
for name, fn in [("bias", lambda: lib.dit_debug_gemm(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), M, N, K, st)),
                 ("resid", lambda: lib.dit_debug_gemm_resid(x.data_ptr(), w.data_ptr(), b.data_ptr(), h.data_ptr(),
                                                            g.data_ptr(), M, N, K, st))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tr.zero_()
    lib.dit_debug_gemm_trace(C.c_void_p(tr.data_ptr()))
    fn()
    torch.cuda.synchronize()
    lib.dit_debug_gemm_trace(None)
    t = tr.cpu().numpy()
    n = int((t[0] > 0).sum())
    base = t[t > 0].min()
    t = np.where(t > 0, t - base, -1)
    J = range(2, n - 1)
    med = lambda a: int(np.median(a)) if len(a) else -1
    print(f"{name} M={M} K={K} N={N}: tiles traced {n}")
    print("  epilogue (warp 0) duration", med([t[1, j] - t[0, j] for j in J]), " warp 7 end - start", med([t[2, j] - t[0, j] for j in J]))
    print("  MMA: tempty wait", med([t[4, j] - t[3, j] for j in J]), " issue (after wait -> last MMA issued)", med([t[5, j] - t[4, j] for j in J]),
          " tile period (epi start -> next)", med([t[0, j + 1] - t[0, j] for j in J]))
    for j in range(min(n, 6)):
        print("   ", j, " ".join(f"{v:8d}" for v in t[:6, j]))
