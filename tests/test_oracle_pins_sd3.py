"""Pins P14-P16 of the SD3 / CFG oracle (oracle/sd3_step.py), CPU only.

Each test names what fixes the expected value: a library routine (transformers'
MAE sincos table), the already-pinned Flux double block (P1, P6, P11) under the
special case that removes RoPE, closed forms of classifier-free guidance, and the
independent torch re-derivation tests/torch_reference.py:step_sd3 (P11).
"""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import flux_step as O
from oracle import sd3_step as S
from tests import torch_reference as TR
from tests.helpers import max_rel, oracle_adapter, torch_adapter

RNG = np.random.default_rng(11)
CFG = synth.SD3_TINY                                             # qk_norm, 2 joint blocks
CFG_NQ = dataclasses.replace(synth.SD3_TINY, qk_norm=False, depth_double=3)


@pytest.fixture(scope="module")
def Wb():
    return {c: synth.make_weights_bf16(c) for c in (CFG, CFG_NQ)}


# ---------------------------------------------------------------- P14 position table
def test_p14_pos_table_is_the_mae_library_table():
    """pe_max = base = grid: no crop, unscaled positions -> exactly MAE's get_2d_sincos_pos_embed."""
    from transformers.models.vit_mae.modeling_vit_mae import get_2d_sincos_pos_embed
    for D, gs in ((64, 8), (1536, 12), (2432, 5)):
        np.testing.assert_allclose(S.pos_embed_sincos(D, gs, gs, gs, gs), get_2d_sincos_pos_embed(D, gs),
                                   rtol=0, atol=1e-12)


def test_p14_pos_table_crop_and_scale():
    """Centre crop of a scaled grid == the library routine on the same grid, cropped."""
    for D, h, w, pm, base in ((64, 4, 6, 8, 4), (1536, 64, 64, 192, 64), (256, 3, 5, 16, 10)):
        np.testing.assert_allclose(S.pos_embed_sincos(D, h, w, pm, base), TR.pos_table_mae(D, h, w, pm, base).numpy(),
                                   rtol=0, atol=1e-12)
    t = S.pos_embed_sincos(16, 4, 4, 4, 4)
    q = 4
    # the top-left token sits at position (0, 0): sin half 0, cos half 1 on both axes
    np.testing.assert_array_equal(t[0], np.concatenate([np.zeros(q), np.ones(q)] * 2))
    # sin^2 + cos^2 = 1 per frequency and axis
    for a in (0, 8):
        np.testing.assert_allclose(t[:, a:a + q] ** 2 + t[:, a + q:a + 2 * q] ** 2, 1.0, atol=1e-14)


# ---------------------------------------------------------------- P15 joint block
def _vec_and_streams(cfg, Wd, nt=5, ni=7):
    vec = RNG.standard_normal(cfg.hidden)
    return vec, RNG.standard_normal((ni, cfg.hidden)), RNG.standard_normal((nt, cfg.hidden))


def test_p15_joint_block_is_flux_double_block_without_rope(Wb):
    """A non-last SD3 joint block with QK-norm == the pinned Flux double block with RoPE at angle 0."""
    Wd = O.weights_to_f64(Wb[CFG])
    vec, img, txt = _vec_and_streams(CFG, Wd)
    d = CFG.head_dim
    cos, sin = np.ones((12, d // 2)), np.zeros((12, d // 2))
    ad, _ = oracle_adapter(CFG, 4, 0)
    i1, t1 = S.joint_block(Wd, 0, CFG.heads, img, txt, vec, ad, last=False, qk_norm=True)
    i2, t2 = O.double_block(Wd, 0, CFG.heads, img, txt, vec, cos, sin, ad)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_array_equal(t1, t2)


def test_p15_context_pre_only_last_block(Wb):
    """The last block's text stream only feeds attention, modulated by (scale, shift):
    giving its 2-chunk modulation the (sc1, sh1) chunks of a full block's text modulation
    reproduces that full block's IMAGE output exactly; no text output remains."""
    cfg = CFG
    Wd = O.weights_to_f64(Wb[cfg])
    vec, img, txt = _vec_and_streams(cfg, Wd)
    D = cfg.hidden
    W2 = dict(Wd)
    for k in ("img.mod.w", "img.mod.b", "img.qkv.w", "img.qkv.b", "img.proj.w", "img.proj.b", "img.fc1.w",
              "img.fc1.b", "img.fc2.w", "img.fc2.b", "img.q_norm", "img.k_norm", "txt.qkv.w", "txt.qkv.b",
              "txt.q_norm", "txt.k_norm"):
        W2["double.1." + k] = Wd["double.0." + k]
    mw, mb = Wd["double.0.txt.mod.w"], Wd["double.0.txt.mod.b"]
    W2["double.1.txt.mod.w"] = np.concatenate([mw[D:2 * D], mw[:D]])   # (scale, shift) = (sc1, sh1)
    W2["double.1.txt.mod.b"] = np.concatenate([mb[D:2 * D], mb[:D]])
    i_full, _ = S.joint_block(W2, 0, cfg.heads, img, txt, vec, None, last=False, qk_norm=True)
    i_last, t_last = S.joint_block(W2, 1, cfg.heads, img, txt, vec, None, last=True, qk_norm=True)
    np.testing.assert_array_equal(i_last, i_full)
    assert t_last is None
    # swapping the two chunks (a (shift, scale) reading) must change the image output
    W2["double.1.txt.mod.w"] = mw[:2 * D]
    W2["double.1.txt.mod.b"] = mb[:2 * D]
    i_swap, _ = S.joint_block(W2, 1, cfg.heads, img, txt, vec, None, last=True, qk_norm=True)
    assert max_rel(i_swap, i_full) > 1e-3


def test_p15_manifest_context_pre_only():
    names = {s.name for s in synth.weight_manifest(synth.SD3_MEDIUM)}
    assert "double.23.txt.qkv.w" in names and "double.23.txt.proj.w" not in names
    assert "double.23.txt.fc2.w" not in names and "double.22.txt.fc2.w" in names
    assert not any(n.startswith("single.") or "q_norm" in n for n in names)   # SD3-medium: no QK-norm
    big = {s.name: s.shape for s in synth.weight_manifest(synth.SD35_LARGE)}
    assert big["double.37.txt.mod.w"] == (2 * 2432, 2432) and big["double.0.img.q_norm"] == (64,)
    assert sum(int(np.prod(s)) for s in big.values()) > 7.5e9     # SD3.5-Large ~8 B parameters [ext]


# ---------------------------------------------------------------- P16 classifier-free guidance
def _batch(cfg, g=5.0, B=2):
    b = synth.make_batch(cfg, B, 4, 4, 8, n_adapters=1, cfg_scale=g)
    b.adapter_id = np.array([0, -1], dtype=np.int32)[:B]
    return b


def test_p16_cfg_closed_forms(Wb):
    cfg = CFG
    W = O.weights_to_f64(Wb[cfg])
    b = _batch(cfg)
    _, v_c = S.dit_step(cfg, W, dataclasses.replace(b, cfg_scale=None))
    b_u = dataclasses.replace(b, cfg_scale=None, txt=b.txt_neg, pooled=b.pooled_neg)
    _, v_u = S.dit_step(cfg, W, b_u)
    _, v0 = S.dit_step(cfg, W, dataclasses.replace(b, cfg_scale=np.zeros(2, np.float32)))
    np.testing.assert_array_equal(v0, v_u)                                 # g = 0: unconditional
    _, v1 = S.dit_step(cfg, W, dataclasses.replace(b, cfg_scale=np.ones(2, np.float32)))
    assert max_rel(v1, v_c) < 1e-14                                        # g = 1: conditional
    _, vs = S.dit_step(cfg, W, dataclasses.replace(b, txt_neg=b.txt, pooled_neg=b.pooled))
    np.testing.assert_array_equal(vs, v_c)                                 # same prompt: no guidance effect
    _, v5 = S.dit_step(cfg, W, b)
    assert max_rel(v5, v_u + 5.0 * (v_c - v_u)) < 1e-13                    # affine in g
    assert max_rel(v5, v_c + 5.0 * (v_u - v_c)) > 0.1                      # branch swap fails (P12)
    x5, _ = S.dit_step(cfg, W, b)
    dt = (b.sigma_next.astype(np.float64) - b.sigma.astype(np.float64))[:, None, None]
    np.testing.assert_array_equal(x5, b.latents.astype(np.float64) + dt * v5)   # Euler on the guided v


# ---------------------------------------------------------------- P11 (SD3) independent torch
@pytest.mark.parametrize("cfg", [CFG, CFG_NQ])
@pytest.mark.parametrize("with_cfg", [True, False])
def test_p11_sd3_step_vs_independent_torch(Wb, cfg, with_cfg):
    W = O.weights_to_f64(Wb[cfg])
    b = _batch(cfg, g=4.5) if with_cfg else dataclasses.replace(_batch(cfg), cfg_scale=None)
    ad, bits = oracle_adapter(cfg, 4, 0, scale=0.7)
    slots = [0, 3] if with_cfg else [1]
    ni = 16
    R = {s: {i: O.bf16_to_f64(synth.controlnet_residual_bf16(s, i, ni, cfg.hidden))
             for i in range(cfg.depth_double)} for s in slots}
    cns = {s: [O.ControlNetInput(double=R[s], single={}, n_res=cfg.depth_double, n_res_single=0)] for s in slots}
    x, v = S.dit_step(cfg, W, b, {0: ad}, cns)
    x2, v2 = TR.step_sd3(cfg, Wb[cfg], b, {0: torch_adapter(bits, cfg, 0.7)},
                         {s: {"n_res": cfg.depth_double, "R": R[s]} for s in slots})
    assert max_rel(v, v2) < 1e-10
    assert max_rel(x, x2) < 1e-10
    _, v_plain = S.dit_step(cfg, W, b)
    assert max_rel(v, v_plain) > 0.02                                      # LoRA + ControlNet matter
