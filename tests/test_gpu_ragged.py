"""GPU parity of ragged (mixed-resolution) batches (reading C24).

A cross-workflow batch whose requests have different latent grids runs in one dit_step
with a padded per-request slot; each request's result must equal (a) the fp64 oracle at
its own grid and (b) BITWISE the same request run alone in a uniform batch -- padding keys
are masked out of attention exactly and every other kernel is row-independent.
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


def _model(cfg, B, ni, nt, rank=0, adapters=0):
    from paper_2604_08123_b200 import SyntheticDiT
    return SyntheticDiT(cfg, max_batch=B, max_img_tokens=ni, max_txt_tokens=nt, max_rank=rank, max_adapters=adapters)


def _alone(batch, b):
    """Request b as a uniform batch of one at its own grid."""
    h, w = batch.grid(b)
    sl = slice(b, b + 1)
    opt = lambda a: None if a is None else a[sl]
    return dataclasses.replace(batch, img_h=h, img_w=w, img_hw=None,
                               latents=np.ascontiguousarray(batch.latents[sl, :h * w]),
                               txt=batch.txt[sl], pooled=batch.pooled[sl], sigma=batch.sigma[sl],
                               sigma_next=batch.sigma_next[sl], guidance=batch.guidance[sl],
                               adapter_id=batch.adapter_id[sl], cn_scale=batch.cn_scale[sl],
                               cfg_scale=opt(batch.cfg_scale), txt_neg=opt(batch.txt_neg),
                               pooled_neg=opt(batch.pooled_neg))


FLUX128 = dataclasses.replace(synth.TINY_SINGLE, hidden=256, heads=2, depth_single=1, rope_axes=(16, 56, 56))


@pytest.mark.parametrize("cfg_name", ["FLUX128", "TINY_SINGLE"])
def test_ragged_flux_batch(torch_cuda, cfg_name):
    """3 requests at 8x8, 6x10 and 5x7 grids in an 8x10 slot (+ 24 text tokens), mixed LoRA,
    a ControlNet on request 1 (double and single block); d = 128 (tcgen05) and d = 32 (mma.sync)."""
    cfg = FLUX128 if cfg_name == "FLUX128" else synth.TINY_SINGLE
    grids = np.array([[8, 8], [6, 10], [5, 7]], dtype=np.int32)
    B, hh, ww, nt = 3, 8, 10, 24
    m = _model(cfg, B, hh * ww, nt, rank=8, adapters=1)
    m.register_synthetic_lora(0, rank=8, index=0, scale=0.7)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([0, -1, 0], dtype=np.int32)
    batch.img_hw = grids
    ni1 = 60
    r_dbl = synth.controlnet_residual_bf16(1, 0, ni1, cfg.hidden)
    r_sgl = synth.controlnet_residual_bf16(1, 7, ni1, cfg.hidden)
    inj = [(1, 0, r_dbl, 1.0), (1, cfg.depth_double, r_sgl, 0.5)]
    lat, v = m.step(batch, injections=inj)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    cn = {1: [O.ControlNetInput(double={0: O.bf16_to_f64(r_dbl)}, single={}, n_res=cfg.depth_double,
                                n_res_single=0),
              O.ControlNetInput(double={}, single={0: O.bf16_to_f64(r_sgl)}, n_res=0,
                                n_res_single=cfg.depth_single, scale=0.5)]}
    x_o, v_o = O.dit_step(cfg, W, batch, {0: oracle_adapter(cfg, 8, 0, scale=0.7)[0]}, controlnets=cn)
    for b in range(B):
        n = int(grids[b, 0] * grids[b, 1])
        check(v[b:b + 1, :n], v_o[b:b + 1, :n], f"v request {b}")
        check(lat[b:b + 1, :n], x_o[b:b + 1, :n], f"latents request {b}")
    # bitwise: each request alone at its own grid
    for b in range(B):
        n = int(grids[b, 0] * grids[b, 1])
        alone = _alone(batch, b)
        inj_b = [(0, blk, bits, sc) for (rb, blk, bits, sc) in inj if rb == b]
        lat_a, v_a = m.step(alone, injections=inj_b)
        np.testing.assert_array_equal(v[b, :n], v_a[0])
        np.testing.assert_array_equal(lat[b, :n], lat_a[0])


def test_ragged_sd3_cfg_batch(torch_cuda):
    """SD3 (d = 64 tcgen05 attention, per-request sincos position table) with CFG: grids 6x6
    and 4x8 in a 6x8 slot."""
    cfg = dataclasses.replace(synth.SD3_TINY, hidden=128, heads=2, depth_double=2, pos_embed_max=12)
    grids = np.array([[6, 6], [4, 8]], dtype=np.int32)
    B, hh, ww, nt = 2, 6, 8, 20
    m = _model(cfg, 2 * B, hh * ww, nt)
    batch = synth.make_batch(cfg, B, hh, ww, nt, cfg_scale=5.0)
    batch.img_hw = grids
    lat, v = m.step(batch)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    x_o, v_o = S.dit_step(cfg, W, batch)
    for b in range(B):
        n = int(grids[b, 0] * grids[b, 1])
        check(v[b:b + 1, :n], v_o[b:b + 1, :n], f"v request {b}")
        lat_a, v_a = m.step(_alone(batch, b))
        np.testing.assert_array_equal(v[b, :n], v_a[0])
        np.testing.assert_array_equal(lat[b, :n], lat_a[0])


def test_ragged_error_paths(torch_cuda):
    from paper_2604_08123_b200 import dit as D
    cfg = synth.TINY_SINGLE
    m = _model(cfg, 2, 20, 8)
    batch = synth.make_batch(cfg, 2, 4, 5, 8)
    batch.img_hw = np.array([[4, 5], [5, 5]], dtype=np.int32)        # 25 > the 20-token slot
    with pytest.raises(D.DitError) as e:
        m.step(batch)
    assert e.value.code == D.CODES["DIT_ESHAPE"]
    group = D.load_library().dit_local_group_create(2)
    m.sp_init_local(group, 0)
    batch.img_hw = np.array([[4, 5], [2, 5]], dtype=np.int32)
    with pytest.raises(D.DitError) as e:
        m.step(batch)
    assert e.value.code == D.CODES["DIT_EPARALLEL"]
    m.close()
    D.load_library().dit_local_group_destroy(group)


def test_step_flops_accounting(torch_cuda):
    """dit_step_flops (the bench's algorithmic FLOPs): a ragged batch counts each request at its own
    grid (= the sum of the requests alone), CFG doubles the work, SD3's context_pre_only last block
    drops its text proj / MLP."""
    cfg = FLUX128
    m = _model(cfg, 4, 80, 24)
    batch = synth.make_batch(cfg, 3, 8, 10, 24)
    batch.img_hw = np.array([[8, 8], [6, 10], [5, 7]], dtype=np.int32)

    def flops(b):
        lat, txt, pooled, out, v = m.device_inputs(b)
        cb = m.make_batch(b.batch, b.img_h, b.img_w, b.txt_tokens, b.adapter_id, b.sigma, b.sigma_next, b.guidance,
                          lat, out, txt, pooled, cfg_scale=b.cfg_scale, img_hw=b.img_hw)
        return m.step_flops(cb)

    total = flops(batch)
    alone = sum(flops(_alone(batch, i)) for i in range(3))
    assert abs(total - alone) <= 1e-9 * alone
    one = _alone(batch, 0)
    assert abs(flops(dataclasses.replace(one, cfg_scale=np.ones(1, np.float32), txt_neg=one.txt,
                                         pooled_neg=one.pooled)) - 2 * flops(one)) <= 1e-9 * flops(one)
    sd3 = dataclasses.replace(synth.SD3_TINY, hidden=128, heads=2, depth_double=2, pos_embed_max=12)
    ms = _model(sd3, 1, 64, 8)
    b3 = synth.make_batch(sd3, 1, 8, 8, 8)
    lat, txt, pooled, out, v = ms.device_inputs(b3)
    cb = ms.make_batch(1, 8, 8, 8, b3.adapter_id, b3.sigma, b3.sigma_next, b3.guidance, lat, out, txt, pooled)
    D, F, N, Nt, Ni = 128, 512, 72, 8, 64
    expect = (2 * Ni * D * 16 + 2 * Nt * D * 32 + 2 * Ni * D * 16
              + 2 * (2 * N * D * 3 * D + 2 * N * D * D + 2 * 2 * N * D * F + 4 * N * N * D)
              - (2 * Nt * D * D + 2 * 2 * Nt * D * F))
    assert abs(ms.step_flops(cb) - expect) <= 1e-9 * expect
