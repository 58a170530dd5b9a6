"""The GEMM's k-block lockstep: a scheduling hint for L2 locality that must never
change a result or hang.  Outputs are compared bitwise with the lockstep off; a cluster kept off
the GPU by another kernel must only switch the lockstep off (bounded wait), not deadlock it."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    prev = lib.dit_debug_gemm_lock(0)
    yield torch, lib
    lib.dit_debug_gemm_lock(prev)


def _operands(torch, M, N, K, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * K ** -0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    return x, w, bias


def _gemm(torch, lib, x, w, bias, stream=None):
    M, K = x.shape
    N = w.shape[0]
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = stream if stream is not None else torch.cuda.current_stream()
    assert lib.dit_debug_gemm(x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), M, N, K,
                              C.c_void_p(s.cuda_stream)) == 0
    return y


@pytest.mark.parametrize("M,N,K", [(4096, 3072, 4096), (2304, 1000, 12288), (300, 520, 192)])
def test_lockstep_bitwise_equal(env, M, N, K):
    """Leads 1 (tight), 16 and 512 give the same bits as no lockstep (K-heavy, ragged, one-round)."""
    torch, lib = env
    x, w, bias = _operands(torch, M, N, K, M + N + K)
    lib.dit_debug_gemm_lock(0)
    ref = _gemm(torch, lib, x, w, bias)
    torch.cuda.synchronize()
    for lead in (1, 16, 512):
        lib.dit_debug_gemm_lock(lead)
        y = _gemm(torch, lib, x, w, bias)
        torch.cuda.synchronize()
        assert torch.equal(y, ref), lead
    lib.dit_debug_gemm_lock(0)
    fp = x.float() @ w.float().T + bias.float()
    assert ((ref.float() - fp).abs().max() / fp.abs().max()).item() < 8e-3


def test_lockstep_cluster_not_resident(env):
    """A kernel holding one SM on another stream keeps one cluster of the persistent GEMM off the
    GPU: the resident clusters must give up waiting for it (0.5 ms) and the launch completes with
    the exact result."""
    torch, lib = env
    x, w, bias = _operands(torch, 4096, 3072, 4096, 7)
    lib.dit_debug_gemm_lock(0)
    ref = _gemm(torch, lib, x, w, bias)
    torch.cuda.synchronize()
    lib.dit_debug_gemm_lock(1)
    side, main = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(40_000_000)           # ~20 ms on one SM
    y = _gemm(torch, lib, x, w, bias, stream=main)
    torch.cuda.synchronize()
    lib.dit_debug_gemm_lock(0)
    assert torch.equal(y, ref)


def test_lockstep_epoch_wrap(env):
    """4200 launches on the process-wide lockstep buffer (the 12-bit launch epoch wraps) keep exact
    results, and a later K-heavy launch still matches."""
    torch, lib = env
    lib.dit_debug_gemm_lock(4)
    xs, ws, bs = _operands(torch, 2048, 2048, 256, 3)
    lib.dit_debug_gemm_lock(0)
    ref_s = _gemm(torch, lib, xs, ws, bs)
    lib.dit_debug_gemm_lock(4)
    for _ in range(4200):
        y = _gemm(torch, lib, xs, ws, bs)
    torch.cuda.synchronize()
    assert torch.equal(y, ref_s)
    x, w, bias = _operands(torch, 4096, 3072, 4096, 11)
    lib.dit_debug_gemm_lock(0)
    ref = _gemm(torch, lib, x, w, bias)
    lib.dit_debug_gemm_lock(8)
    y = _gemm(torch, lib, x, w, bias)
    torch.cuda.synchronize()
    lib.dit_debug_gemm_lock(0)
    assert torch.equal(y, ref)
