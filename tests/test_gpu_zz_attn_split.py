"""The attention's split tail (opt-in; attention_tc.cu TailSched): when the persistent grid's last
round of work items is at most half full, each tail item's keys are split into S = 2..4 parts whose
partial O / max / sum the last part merges in part order.  Checked against a plain PyTorch fp32
reference over EVERY (request, head) -- the tail items are the last ones -- at S = 2, 3 and 4 and
both head dims, run-to-run bitwise determinism, agreement with the unsplit kernel within rounding,
and a dit_step with the split tail on against the fp64 oracle.  (Named to run last: run before
tests/test_gpu_bmax16.py in one process, the in-process two-rank sequence-parallel test there
stalled in its flag barrier -- ranks spinning on one GPU, the hazard the profiling guide warns of.)"""
import ctypes as C
import dataclasses
import os

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from tests.helpers import oracle_adapter
from tests.test_gpu_parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _run(torch, lib, q, k, v, split):
    B, H, N, d = q.shape
    out = torch.zeros(B * N, H * d, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    assert lib.dit_debug_attention_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, H, N, d, out.data_ptr(), split,
                                      C.c_void_p(s.cuda_stream)) == 0
    torch.cuda.synchronize()
    return out


# (B, H, N, d): work items = ceil(N / 256) * H * B on the 148-SM grid; tail items -> key parts S
@pytest.mark.parametrize("B,H,N,d", [(1, 3, 16896, 128),    # 198 items: 50 in the tail, S = 2
                                     (2, 5, 4608, 128),     # 180 items: 32 in the tail, S = 4
                                     (1, 6, 8192, 64),      # 192 items: 44 in the tail, S = 3
                                     (3, 4, 4500, 128)])    # 216 items: 68 in the tail, S = 2; ragged tile
def test_split_tail_vs_torch_fp32(torch_cuda, B, H, N, d):
    torch = torch_cuda
    from paper_2604_08123_b200 import dit
    lib = dit.load_library()
    g = torch.Generator(device="cuda").manual_seed(B * 1000 + H * 10 + N)
    q, k, v = (torch.randn(B, H, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    got = _run(torch, lib, q, k, v, 1)
    again = _run(torch, lib, q, k, v, 1)
    plain = _run(torch, lib, q, k, v, 0)
    assert torch.equal(got, again)                          # deterministic merge order
    qf, kf, vf = q.float(), k.float(), v.float()
    ref = (torch.softmax((qf @ kf.transpose(-1, -2)) / d ** 0.5, dim=-1) @ vf).permute(0, 2, 1, 3).reshape(B * N, H * d)
    gf = got.float()
    assert torch.isfinite(gf).all()
    err = ((gf - ref).abs().max() / ref.abs().max()).item()
    cos = torch.nn.functional.cosine_similarity(gf.flatten(), ref.flatten(), dim=0).item()
    assert err < 1e-2 and cos > 0.9999, (err, cos)
    # the split changes only the tail items' rounding
    diff = ((gf - plain.float()).abs().max() / ref.abs().max()).item()
    assert diff < 1e-2, diff
    assert not torch.equal(got, plain)                      # the tail really went through the split path


def test_split_tail_dit_step_vs_oracle(torch_cuda):
    """A context created with DIT_ATTN_SPLIT_TAIL=1: B = 3 requests of 64x64 image + 512 text tokens
    at 4 heads of 128 (216 attention items: a 68-item tail split in two), LoRA on one request."""
    cfg = dataclasses.replace(synth.FLUX, hidden=512, heads=4, txt_dim=256, pooled_dim=128,
                              depth_double=1, depth_single=1)
    B, hh, ww, nt = 3, 64, 64, 512
    from paper_2604_08123_b200 import SyntheticDiT
    os.environ["DIT_ATTN_SPLIT_TAIL"] = "1"
    try:
        m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=16, max_adapters=1)
    finally:
        del os.environ["DIT_ATTN_SPLIT_TAIL"]
    m.register_synthetic_lora(2, rank=16, index=0)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([-1, 2, -1], dtype=np.int32)
    lat, v = m.step(batch)
    lat2, v2 = m.step(batch)
    np.testing.assert_array_equal(v, v2)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = O.dit_step(cfg, W, batch, {2: oracle_adapter(cfg, 16, 0)[0]}, {}, n_res=0)
    check(v, v_o, "v")
    check(lat, x_o, "latents")


def test_split_tail_nccl_sp_layout_world1_bitwise(torch_cuda):
    """The split tail's merged rows written through the sequence-parallel output layout (a 1-rank
    NCCL communicator, DIT_FORCE_SP: send layout + ncclAlltoAll + scatter) equal the plain split-tail
    step bitwise -- the merge writes every row where the unsplit epilogue would."""
    from paper_2604_08123_b200 import SyntheticDiT
    from paper_2604_08123_b200.dit import nccl_unique_id
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=512, heads=4, depth_single=1, rope_axes=(16, 56, 56))
    B, hh, ww, nt = 3, 64, 64, 512          # 18 query blocks x 4 heads x 3 = 216 items: a 68-item tail
    batch = synth.make_batch(cfg, B, hh, ww, nt)
    os.environ["DIT_ATTN_SPLIT_TAIL"] = "1"
    try:
        ref = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt)
        _, v1 = ref.step(batch)
        os.environ["DIT_FORCE_SP"] = "1"
        m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt)
        m.sp_init(1, 0, nccl_unique_id())
        _, v2 = m.step(batch)
    finally:
        os.environ.pop("DIT_FORCE_SP", None)
        del os.environ["DIT_ATTN_SPLIT_TAIL"]
    np.testing.assert_array_equal(v2, v1)
    assert np.isfinite(v1).all()
