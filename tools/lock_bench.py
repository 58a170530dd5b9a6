"""The GEMM alone at the step's projection shapes with the k-block lockstep at several leads:
TFLOP/s and (GEMM_LOCK_STATS variant builds: python tools/variant.py lockstats gemm.cu -DGEMM_LOCK_STATS=1,
then DIT_LIB_OVERRIDE=<that .so>) the producers' wait time / wait events / timeouts per launch."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_08123_b200 import dit  # noqa: E402

lib = dit.load_library()
stats = getattr(lib, "dit_debug_gemm_lock_stats", None)
shapes = [("linear2", 36864, 3072, 15360), ("fc2", 32768, 3072, 12288), ("qkv", 32768, 9216, 3072)]
leads = [int(x) for x in sys.argv[1:]] or [0, 16, 64, 256]
s = torch.cuda.current_stream()
for name, M, N, K in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * K ** -0.5).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    call = lambda: lib.dit_debug_gemm(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), M, N, K, C.c_void_p(s.cuda_stream))
    for lead in leads:
        lib.dit_debug_gemm_lock(lead)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        st = (C.c_ulonglong * 3)()
        if stats:
            stats(st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record(s)
        for _ in range(n):
            call()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        extra = ""
        if stats:
            stats(st)
            extra = f"  wait/launch {st[0] / n / 1e3:.1f} us-total over clusters, {st[1] / n:.0f} waits, {(st[2] & 0xffffffff) / n:.1f} timeouts, max lead {st[2] >> 32}"
        print(f"{name} M={M} N={N} K={K} lead={lead}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.0f} TF/s{extra}", flush=True)
    lib.dit_debug_gemm_lock(0)
