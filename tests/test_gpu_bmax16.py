"""B_max = 16 sequences per dit_step (per-sequence parameter tables, the two-group skinny
modulation GEMM, ControlNet tables and the segment tables sized by MAX_SEQ = 16), and the
single-GPU workspace (max_sp_world = 1) that drops the SP exchange buffers.

Parity against the fp64 oracle as in tests/test_gpu_parity.py (north_star tolerance: per request
max_rel <= 2e-2, cosine >= 0.999); batch invariance bitwise (pins P3 / P9).
"""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from oracle import sd3_step as S
from tests.helpers import oracle_adapter
from tests.test_gpu_parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _model(cfg, B, ni, nt, rank=0, adapters=0, max_sp_world=0):
    from paper_2604_08123_b200 import SyntheticDiT
    return SyntheticDiT(cfg, max_batch=B, max_img_tokens=ni, max_txt_tokens=nt, max_rank=rank,
                        max_adapters=adapters, max_sp_world=max_sp_world)


def test_flux_twelve_requests_mixed_adapters_controlnet(torch_cuda):
    """12 requests (> the old cap of 8): three adapters and no-adapter rows interleaved, mixed
    sigmas, ControlNet residuals on requests 2 and 11 (slot tables beyond index 8)."""
    cfg = dataclasses.replace(synth.TINY, hidden=128, heads=4)
    B, hh, ww, nt = 12, 4, 6, 16
    ni = hh * ww
    m = _model(cfg, B, ni, nt, rank=8, adapters=3, max_sp_world=1)
    for a in range(3):
        m.register_synthetic_lora(a, rank=8, index=a, scale=0.5 + 0.25 * a)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=3)
    batch.adapter_id = np.array([0, -1, 2, 1, 1, -1, 0, 2, 2, -1, 1, 0], dtype=np.int32)
    bits = {s: {i: synth.controlnet_residual_bf16(s, i, ni, cfg.hidden) for i in range(cfg.depth_double)}
            for s in (2, 11)}
    res = {s: {i: O.bf16_to_f64(r) for i, r in d.items()} for s, d in bits.items()}
    lat, v = m.step(batch, controlnet=bits)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    ads = {a: oracle_adapter(cfg, 8, a, scale=0.5 + 0.25 * a)[0] for a in range(3)}
    x_o, v_o = O.dit_step(cfg, W, batch, ads, res, n_res=cfg.depth_double)
    check(v, v_o, "v")
    check(lat, x_o, "latents_out")


def test_sixteen_requests_batch_invariance_bitwise(torch_cuda):
    """A request's output in a batch of 16 equals the same request run alone, bitwise."""
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=128, heads=4)
    B = 16
    m = _model(cfg, B, 64, 32, rank=8, adapters=2, max_sp_world=1)
    m.register_synthetic_lora(0, rank=8, index=0)
    m.register_synthetic_lora(1, rank=8, index=1)
    full = synth.make_batch(cfg, B, 8, 8, 32, n_adapters=2)
    full.adapter_id = np.array([(b % 3) - 1 for b in range(B)], dtype=np.int32)
    _, v = m.step(full)
    for b in (0, 7, 8, 9, 15):
        one = dataclasses.replace(full, latents=full.latents[b:b + 1], txt=full.txt[b:b + 1],
                                  pooled=full.pooled[b:b + 1], sigma=full.sigma[b:b + 1],
                                  sigma_next=full.sigma_next[b:b + 1], guidance=full.guidance[b:b + 1],
                                  adapter_id=full.adapter_id[b:b + 1], cn_scale=full.cn_scale[b:b + 1])
        _, v1 = m.step(one)
        np.testing.assert_array_equal(v1[0], v[b])


def test_sd3_cfg_eight_requests(torch_cuda):
    """Classifier-free guidance for 8 requests = 16 sequences in one step (the old cap allowed 4)."""
    cfg = dataclasses.replace(synth.SD3_TINY, pos_embed_max=16)
    B, hh, ww, nt = 8, 4, 4, 12
    m = _model(cfg, 2 * B, hh * ww, nt, rank=8, adapters=1, max_sp_world=1)
    m.register_synthetic_lora(0, rank=8, index=0, scale=0.8)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1, cfg_scale=4.5)
    batch.adapter_id = np.array([0, -1, -1, 0, 0, -1, 0, -1], dtype=np.int32)
    batch.cfg_scale = np.linspace(1.5, 7.0, B).astype(np.float32)
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch, {0: oracle_adapter(cfg, 8, 0, scale=0.8)[0]})
    check(v, v_o, "v")
    check(lat, x_o, "latents_out")


def test_batch_limits_and_single_gpu_workspace(torch_cuda):
    """17 sequences are refused (DIT_EBATCH); a max_sp_world = 1 workspace refuses sequence
    parallelism (DIT_EPARALLEL) but runs single-GPU steps."""
    from paper_2604_08123_b200 import dit as D
    cfg = dataclasses.replace(synth.TINY, hidden=128, heads=4)
    m = _model(cfg, 16, 16, 8, max_sp_world=1)
    lib = D.load_library()
    batch = synth.make_batch(cfg, 16, 4, 4, 8)
    m.step(batch)                      # 16 = B_max: runs
    with pytest.raises(D.DitError) as e:
        m.step(synth.make_batch(cfg, 17, 4, 4, 8))
    assert e.value.code == 8           # DIT_EBATCH
    group = lib.dit_local_group_create(2)
    try:
        rc = lib.sp_init_local(m.ctx, group, 0)
        assert rc != 0 and "max_sp_world" in lib.dit_last_error(m.ctx).decode()
    finally:
        lib.dit_local_group_destroy(group)


@pytest.mark.parametrize("exchange", ["fused", "a2a"])
def test_sequence_parallel_sixteen_sequences_bitwise(torch_cuda, exchange, monkeypatch):
    """Ulysses SP (P = 2, in-process group) over 12 requests with d = 128 heads: every per-sequence
    index map of the exchange (fused peer stores / all-to-all + gather / scatter) beyond the old
    8-sequence cap; bitwise equal to the single-rank step (pin P10)."""
    import torch
    from paper_2604_08123_b200 import dit as D
    from tests.test_gpu_parity import _shard_step
    monkeypatch.setenv("DIT_SP_NCCL", "1" if exchange == "a2a" else "0")
    cfg = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, depth_single=1, rope_axes=(16, 56, 56))
    B, hh, ww, nt, P = 12, 8, 8, 16, 2
    ref = _model(cfg, 16, hh * ww, nt, rank=8, adapters=1)
    ref.register_synthetic_lora(5, rank=8, index=0)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([5, -1] * 6, dtype=np.int32)
    lat1, v1 = ref.step(batch)
    group = D.load_library().dit_local_group_create(P)
    models = []
    for r in range(P):
        m = _model(cfg, 16, hh * ww, nt, rank=8, adapters=1)
        m.register_synthetic_lora(5, rank=8, index=0)
        m.sp_init_local(group, r)
        models.append(m)
    latP, vP = _shard_step(models, batch, P)
    np.testing.assert_array_equal(vP, v1)
    np.testing.assert_array_equal(latP, lat1)
    for m in models:
        m.close()
    D.load_library().dit_local_group_destroy(group)
    torch.cuda.synchronize()
