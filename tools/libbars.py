"""Same-box library bars: cuBLAS bf16 GEMMs at the exact cfg3 projection shapes
and flashinfer's segmented GEMM for the LoRA shrink, timed back-to-back long enough to run in the
same power-capped regime as the step.  Context for the per-GEMM-type TF/s bench.py reports; not
linked into libdit."""
import json
import sys

import torch


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


out = {"cublas": {}, "flashinfer_segment_gemm": {}}
B, D, F = 8, 3072, 12288
shapes = {"dbl_qkv_img": (B * 4096, D, 3 * D), "dbl_proj_img": (B * 4096, D, D), "dbl_fc1_img": (B * 4096, D, F),
          "dbl_fc2_img": (B * 4096, F, D), "sgl_linear1": (B * 4608, D, 3 * D + F), "sgl_linear2": (B * 4608, D + F, D)}
import ctypes as C
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08123_b200 import dit  # noqa: E402
lib = dit.load_library()
out["ours"] = {}
for name, (M, K, N) in shapes.items():
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
    bias = torch.randn(N, device="cuda", dtype=torch.bfloat16) * 0.02
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream()
    ours = lambda: lib.dit_debug_gemm(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), M, N, K,
                                      C.c_void_p(st.cuda_stream))
    lib_ = lambda: torch.nn.functional.linear(x, w, bias)
    t_o, t_c = [], []
    for _ in range(2):                      # interleaved: same thermal / power state
        t_o.append(timed(ours))
        t_c.append(timed(lib_))
    ref = lib_()
    err = ((y.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
    fl = 2 * M * N * K
    out["cublas"][name] = {"M": M, "K": K, "N": N, "ms": min(t_c), "tflops": fl / min(t_c) / 1e9}
    out["ours"][name] = {"ms": min(t_o), "tflops": fl / min(t_o) / 1e9, "max_rel_vs_cublas": err}
    del x, w, y
try:
    import flashinfer
    ws = torch.empty(128 * 1024 * 1024, dtype=torch.int8, device="cuda")
    seg = flashinfer.SegmentGEMMWrapper(ws)
    r, nad = 64, 4
    ids = [0, 0, 1, 1, 2, 2, 3, 3]
    for K in (D, F, D + F):
        rows_per = 4608
        x = torch.randn(B * rows_per, K, device="cuda", dtype=torch.bfloat16)
        A = torch.randn(nad, r, K, device="cuda", dtype=torch.bfloat16) * 0.02   # [w][d_out][d_in]
        lens = torch.full((B,), rows_per, dtype=torch.int64, device="cuda")
        widx = torch.tensor(ids, dtype=torch.int64, device="cuda")
        ms = timed(lambda: seg.run(x, A, B, True, seg_lens=lens, weight_indices=widx))
        out["flashinfer_segment_gemm"][f"K{K}"] = {"rows": B * rows_per, "r": r, "ms": ms,
                                                   "GB_per_s_x": x.numel() * 2 / ms / 1e6}
    t = {k: v["ms"] for k, v in out["flashinfer_segment_gemm"].items()}
    out["flashinfer_segment_gemm"]["cfg3_step_estimate_ms"] = (
        19 * (3 * t[f"K{D}"] + t[f"K{F}"]) + 38 * (t[f"K{D}"] + t[f"K{D + F}"]))
except Exception as e:  # library bar only
    out["flashinfer_segment_gemm"]["error"] = repr(e)
print(json.dumps(out, indent=1))
