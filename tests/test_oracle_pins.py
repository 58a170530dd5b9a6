"""Pins P1-P12: the oracle checked against things OTHER than itself.

CPU only.  Each test names the pin and what fixes the expected value: a
brute-force loop, a closed form, an invariant, a special case that reduces to
a torch library routine, or the independent torch re-derivation (P11).
"""
import dataclasses
import itertools
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import flux_step as O
from tests import torch_reference as TR
from tests.helpers import cosine, max_rel, oracle_adapter, residuals, torch_adapter

RNG = np.random.default_rng(7)


# ---------------------------------------------------------------- P1 attention
def brute_attention(q, k, v):
    H, N, d = q.shape
    out = np.zeros_like(q)
    for h in range(H):
        for i in range(N):
            s = [sum(q[h, i, c] * k[h, j, c] for c in range(d)) / math.sqrt(d) for j in range(N)]
            m = max(s)
            e = [math.exp(x - m) for x in s]
            z = sum(e)
            for c in range(d):
                out[h, i, c] = sum(e[j] * v[h, j, c] for j in range(N)) / z
    return out


def test_p1_attention_brute_force():
    q, k, v = (RNG.standard_normal((2, 7, 4)) for _ in range(3))
    np.testing.assert_allclose(O.attention(q, k, v), brute_attention(q, k, v), rtol=0, atol=1e-12)


def test_p1_attention_special_cases():
    k, v = RNG.standard_normal((2, 9, 8)), RNG.standard_normal((2, 9, 8))
    q0 = np.zeros((2, 9, 8))
    np.testing.assert_allclose(O.attention(q0, k, v), np.broadcast_to(v.mean(axis=1, keepdims=True), v.shape), atol=1e-14)
    q1, k1, v1 = (RNG.standard_normal((3, 1, 8)) for _ in range(3))
    np.testing.assert_allclose(O.attention(q1, k1, v1), v1, atol=1e-14)
    q = RNG.standard_normal((2, 9, 8))
    perm = RNG.permutation(9)
    np.testing.assert_allclose(O.attention(q, k[:, perm], v[:, perm]), O.attention(q, k, v), atol=1e-13)
    np.testing.assert_allclose(O.attention(q[:, perm], k, v), O.attention(q, k, v)[:, perm], atol=1e-13)


def test_p1_attention_vs_torch_sdpa():
    q, k, v = (RNG.standard_normal((3, 33, 16)) for _ in range(3))
    ref = F.scaled_dot_product_attention(*(torch.tensor(x) for x in (q, k, v))).numpy()
    np.testing.assert_allclose(O.attention(q, k, v), ref, atol=1e-12)


# ---------------------------------------------------------------- P7 RoPE
def test_p7_rope_properties():
    ids = O.position_ids(3, 4, 5)
    cos, sin = O.rope_cos_sin(ids, (4, 14, 14), 1e4)
    x = RNG.standard_normal((2, ids.shape[0], 32))
    y = O.apply_rope(x, cos, sin)
    np.testing.assert_array_equal(y[:, :3], x[:, :3])              # position 0 -> identity
    n0 = x[..., 0::2] ** 2 + x[..., 1::2] ** 2
    n1 = y[..., 0::2] ** 2 + y[..., 1::2] ** 2
    np.testing.assert_allclose(n1, n0, rtol=1e-13)                 # pair norms preserved
    # <R(m) q, R(n) k> depends only on m - n: shift every position by the same offset
    a = np.array([[0, 1, 2], [0, 3, 1]], dtype=float)
    b = a + np.array([0, 2, 3])
    q, k = RNG.standard_normal((1, 1, 32)), RNG.standard_normal((1, 1, 32))
    def dot(p1, p2):
        c1, s1 = O.rope_cos_sin(p1[None], (4, 14, 14), 1e4)
        c2, s2 = O.rope_cos_sin(p2[None], (4, 14, 14), 1e4)
        return float((O.apply_rope(q, c1, s1) * O.apply_rope(k, c2, s2)).sum())
    assert abs(dot(a[0], a[1]) - dot(b[0], b[1])) < 1e-12


def test_p7_rope_vs_complex_library():
    ids = O.position_ids(2, 3, 4)
    cos, sin = O.rope_cos_sin(ids, (16, 56, 56), 1e4)
    x = RNG.standard_normal((2, ids.shape[0], 128))
    cis = TR.rope_complex(2, 3, 4, (16, 56, 56), 1e4)
    np.testing.assert_allclose(O.apply_rope(x, cos, sin), TR.rot(torch.tensor(x), cis).numpy(), atol=1e-12)


# ---------------------------------------------------------------- P8 norms etc.
def test_p8_norms_and_activations():
    x = RNG.standard_normal((5, 64)) * 3 + 1
    y = O.layer_norm(x)
    np.testing.assert_allclose(y.mean(-1), 0, atol=1e-13)
    np.testing.assert_allclose((y ** 2).mean(-1) * (x.var(-1) + 1e-6) / x.var(-1), 1, rtol=1e-12)
    np.testing.assert_allclose(y, F.layer_norm(torch.tensor(x), (64,), eps=1e-6).numpy(), atol=1e-12)
    g = RNG.standard_normal(64)
    r = O.rms_norm(x, np.ones(64))
    np.testing.assert_allclose(np.sqrt((r ** 2).mean(-1) * ((x ** 2).mean(-1) + 1e-6) / (x ** 2).mean(-1)), 1, rtol=1e-12)
    np.testing.assert_allclose(O.rms_norm(x, g), F.rms_norm(torch.tensor(x), (64,), torch.tensor(g), 1e-6).numpy(), atol=1e-12)
    np.testing.assert_allclose(O.gelu_tanh(x), F.gelu(torch.tensor(x), approximate="tanh").numpy(), atol=1e-14)
    np.testing.assert_allclose(O.silu(x), F.silu(torch.tensor(x)).numpy(), atol=1e-14)


def test_timestep_embedding_closed_form():
    e0 = O.timestep_embedding(0.0)
    np.testing.assert_array_equal(e0[:128], 1.0)
    np.testing.assert_array_equal(e0[128:], 0.0)
    e = O.timestep_embedding(0.25)
    # k = 0 has frequency 1 -> cos(250), sin(250); k = 64 has 10000^-0.5 = 0.01 -> cos(2.5)
    assert e[0] == pytest.approx(math.cos(250.0), abs=1e-12)
    assert e[128] == pytest.approx(math.sin(250.0), abs=1e-12)
    assert e[64] == pytest.approx(math.cos(2.5), abs=1e-12)


# ---------------------------------------------------------------- tiny helpers
CFG = synth.TINY
CFG_S = synth.TINY_SINGLE


@pytest.fixture(scope="module")
def W_bits():
    return synth.make_weights_bf16(CFG_S)


def _W(bits, cfg):
    keep = {s.name for s in synth.weight_manifest(cfg)}
    return O.weights_to_f64({k: v for k, v in bits.items() if k in keep})


def _batch(cfg, B=2, n_adapters=1):
    b = synth.make_batch(cfg, B, 4, 4, 8, n_adapters=n_adapters)
    b.adapter_id = np.array([0, -1] + [0] * (B - 2), dtype=np.int32)[:B]
    return b


# ---------------------------------------------------------------- P2 LoRA merged equivalence
def test_p2_lora_merged_equivalence_linear():
    x = RNG.standard_normal((6, 32))
    w, b = RNG.standard_normal((48, 32)), RNG.standard_normal(48)
    a, bm = RNG.standard_normal((4, 32)), RNG.standard_normal((48, 4))
    y = O.linear(x, w, b, (0.7, a, bm))
    y2 = x @ (w + 0.7 * bm @ a).T + b
    assert max_rel(y, y2) < 1e-12


@pytest.mark.parametrize("cfg", [CFG, CFG_S])
def test_p2_lora_merged_equivalence_step(W_bits, cfg):
    W = _W(W_bits, cfg)
    ad, _ = oracle_adapter(cfg, 4, 0, scale=0.8)
    batch = _batch(cfg)
    x_u, v_u = O.dit_step(cfg, W, batch, {0: ad})
    Wm = O.merged_weights(W, ad)
    v_m = O.velocity(cfg, Wm, batch.latents[0].astype(float), O.bf16_to_f64(batch.txt[0]),
                     O.bf16_to_f64(batch.pooled[0]), float(batch.sigma[0]), float(batch.guidance[0]), 4, 4)
    assert max_rel(v_u[0], v_m) < 1e-11
    # and the adapter actually matters (P12 sensitivity, oracle side)
    _, v_base = O.dit_step(cfg, W, batch)
    assert max_rel(v_base[0], v_u[0]) > 0.05


# ---------------------------------------------------------------- P3 zero adapters / ControlNet
def test_p3_zero_adapter_and_controlnet_bitwise(W_bits):
    cfg = CFG
    W = _W(W_bits, cfg)
    batch = _batch(cfg)
    x0, v0 = O.dit_step(cfg, W, batch)
    adz, _ = oracle_adapter(cfg, 4, 0, zero_b=True)
    x1, v1 = O.dit_step(cfg, W, batch, {0: adz})
    np.testing.assert_array_equal(v1, v0)                        # B_a = 0
    ad, _ = oracle_adapter(cfg, 4, 0)
    x2, v2 = O.dit_step(cfg, W, batch, {0: ad})
    np.testing.assert_array_equal(v2[1], v0[1])                  # a_b = -1
    res = residuals(cfg, 2, 16, 1)
    zero_res = {b: {i: np.zeros_like(r) for i, r in d.items()} for b, d in res.items()}
    _, v3 = O.dit_step(cfg, W, batch, controlnet=zero_res, n_res=1)
    np.testing.assert_array_equal(v3, v0)                        # R = 0
    batch.cn_scale[:] = 0.0
    _, v4 = O.dit_step(cfg, W, batch, controlnet=res, n_res=1)
    np.testing.assert_array_equal(v4, v0)                        # kappa = 0
    batch.cn_scale[:] = 1.0
    _, v5 = O.dit_step(cfg, W, batch, controlnet=res, n_res=1)
    assert max_rel(v5, v0) > 0.02                                # and it matters (P12)


# ---------------------------------------------------------------- P4 Euler
def test_p4_euler_closed_form(W_bits):
    cfg = CFG
    W = _W(W_bits, cfg)
    batch = _batch(cfg)
    batch.sigma_next = batch.sigma.copy()
    x, _ = O.dit_step(cfg, W, batch)
    np.testing.assert_array_equal(x, batch.latents.astype(np.float64))   # sigma' = sigma -> x' = x
    # constant-v model: all weights zero except final.linear.b
    Wz = {k: np.zeros_like(v) for k, v in W.items()}
    Wz["final.linear.b"] = W["final.linear.b"]
    sig = synth.flux_sigmas(28, 16)
    b = _batch(cfg)
    x0 = b.latents.astype(np.float64)
    xk = x0
    for s in range(3):
        b.latents = xk.astype(np.float32) if False else xk
        b.sigma = np.full(2, sig[s], np.float32)
        b.sigma_next = np.full(2, sig[s + 1], np.float32)
        xk, v = O.dit_step(cfg, Wz, b)
        np.testing.assert_array_equal(v, np.broadcast_to(W["final.linear.b"], v.shape))
    closed = x0 + (float(sig[1]) - float(sig[0]) + float(sig[2]) - float(sig[1]) + float(sig[3]) - float(sig[2])) * W["final.linear.b"]
    np.testing.assert_allclose(xk, closed, atol=1e-14)


# ---------------------------------------------------------------- P5 identity blocks
def test_p5_zero_gates_identity(W_bits):
    cfg = CFG_S
    W = dict(_W(W_bits, cfg))
    D = cfg.hidden
    for i in range(cfg.depth_double):
        for s in ("img", "txt"):
            for g in (2, 5):                                        # g1, g2 chunks
                W[f"double.{i}.{s}.mod.w"][g * D:(g + 1) * D] = 0
                W[f"double.{i}.{s}.mod.b"][g * D:(g + 1) * D] = 0
    for j in range(cfg.depth_single):
        W[f"single.{j}.mod.w"][2 * D:] = 0
        W[f"single.{j}.mod.b"][2 * D:] = 0
    batch = _batch(cfg, n_adapters=0)
    trace = []
    x = batch.latents[0].astype(float)
    txt = O.bf16_to_f64(batch.txt[0])
    v = O.velocity(cfg, W, x, txt, O.bf16_to_f64(batch.pooled[0]), float(batch.sigma[0]),
                   float(batch.guidance[0]), 4, 4, trace=trace)
    h0 = np.concatenate([txt @ W["txt_in.w"].T + W["txt_in.b"], x @ W["img_in.w"].T + W["img_in.b"]])
    for h in trace:
        np.testing.assert_array_equal(h, h0)
    # v is then the textbook LN -> affine -> linear of the embedded x (torch library)
    vec = O.conditioning_vec(W, float(batch.sigma[0]), float(batch.guidance[0]), O.bf16_to_f64(batch.pooled[0]))
    m = torch.tensor(W["final.mod.w"]) @ F.silu(torch.tensor(vec)) + torch.tensor(W["final.mod.b"])
    sh, sc = m[:D], m[D:]
    ref = F.linear(F.layer_norm(torch.tensor(h0[8:]), (D,), eps=1e-6) * (1 + sc) + sh,
                   torch.tensor(W["final.linear.w"]), torch.tensor(W["final.linear.b"]))
    np.testing.assert_allclose(v, ref.numpy(), atol=1e-12)


# ---------------------------------------------------------------- P6 + P11 torch library re-derivation
@pytest.mark.parametrize("cfg", [CFG, CFG_S])
def test_p11_step_vs_independent_torch(W_bits, cfg):
    W = _W(W_bits, cfg)
    keep = {s.name for s in synth.weight_manifest(cfg)}
    Wb = {k: v for k, v in W_bits.items() if k in keep}
    batch = synth.make_batch(cfg, 3, 4, 4, 8, n_adapters=2)
    batch.adapter_id = np.array([1, -1, 0], dtype=np.int32)
    ads, tads = {}, {}
    for a in range(2):
        ad, bits = oracle_adapter(cfg, 4, a, scale=0.5 + a)
        ads[a], tads[a] = ad, torch_adapter(bits, cfg, 0.5 + a)
    res = residuals(cfg, 3, 16, cfg.depth_double, requests=[0, 2])
    batch.cn_scale = np.array([1.0, 1.0, 0.5], np.float32)
    x_o, v_o = O.dit_step(cfg, W, batch, ads, res, n_res=cfg.depth_double)
    x_t, v_t = TR.step(cfg, Wb, batch, tads, res, n_res=cfg.depth_double)
    assert max_rel(v_t, v_o) < 1e-10
    assert max_rel(x_t, x_o) < 1e-10


def test_p6_adaln_neutral_block_is_textbook(W_bits):
    """shift = scale = 0, gate = 1: single block == textbook pre-LN joint attention block."""
    cfg = CFG_S
    W = dict(_W(W_bits, cfg))
    D, H, d = cfg.hidden, cfg.heads, cfg.head_dim
    W["single.0.mod.w"] = np.zeros_like(W["single.0.mod.w"])
    mb = np.zeros(3 * D)
    mb[2 * D:] = 1.0
    W["single.0.mod.b"] = mb
    x = RNG.standard_normal((24, D))
    vec = RNG.standard_normal(D)
    ids = O.position_ids(8, 4, 4)
    cos, sin = O.rope_cos_sin(ids, cfg.rope_axes, cfg.rope_theta)
    out = O.single_block(W, 0, H, x, vec, cos, sin, None)
    xt = torch.tensor(x)
    u = F.layer_norm(xt, (D,), eps=1e-6)
    y = F.linear(u, torch.tensor(W["single.0.linear1.w"]), torch.tensor(W["single.0.linear1.b"]))
    q, k, v = y[:, :3 * D].reshape(24, 3, H, d).permute(1, 2, 0, 3)
    q = F.rms_norm(q, (d,), torch.tensor(W["single.0.q_norm"]), 1e-6)
    k = F.rms_norm(k, (d,), torch.tensor(W["single.0.k_norm"]), 1e-6)
    cis = TR.rope_complex(8, 4, 4, cfg.rope_axes, cfg.rope_theta)
    o = F.scaled_dot_product_attention(TR.rot(q, cis), TR.rot(k, cis), v).permute(1, 0, 2).reshape(24, D)
    ref = xt + F.linear(torch.cat([o, F.gelu(y[:, 3 * D:], approximate="tanh")], -1),
                        torch.tensor(W["single.0.linear2.w"]), torch.tensor(W["single.0.linear2.b"]))
    np.testing.assert_allclose(out, ref.numpy(), atol=1e-11)


# ---------------------------------------------------------------- P9 batching
def test_p9_batch_permutation_bitwise(W_bits):
    cfg = CFG
    W = _W(W_bits, cfg)
    batch = synth.make_batch(cfg, 3, 4, 4, 8, n_adapters=1)
    batch.adapter_id = np.array([0, -1, 0], dtype=np.int32)
    ad, _ = oracle_adapter(cfg, 4, 0)
    x, v = O.dit_step(cfg, W, batch, {0: ad})
    perm = np.array([2, 0, 1])
    pb = dataclasses.replace(batch, latents=batch.latents[perm], txt=batch.txt[perm], pooled=batch.pooled[perm],
                             sigma=batch.sigma[perm], sigma_next=batch.sigma_next[perm],
                             guidance=batch.guidance[perm], adapter_id=batch.adapter_id[perm],
                             cn_scale=batch.cn_scale[perm])
    xp, vp = O.dit_step(cfg, W, pb, {0: ad})
    np.testing.assert_array_equal(vp, v[perm])
    np.testing.assert_array_equal(xp, x[perm])


# ---------------------------------------------------------------- P12 sensitivity
def test_p12_swapped_adapters_fail_tolerance(W_bits):
    cfg = CFG
    W = _W(W_bits, cfg)
    batch = synth.make_batch(cfg, 2, 4, 4, 8, n_adapters=2)
    batch.adapter_id = np.array([0, 1], dtype=np.int32)
    a0, _ = oracle_adapter(cfg, 4, 0)
    a1, _ = oracle_adapter(cfg, 4, 1)
    _, v = O.dit_step(cfg, W, batch, {0: a0, 1: a1})
    _, vs = O.dit_step(cfg, W, batch, {0: a1, 1: a0})
    assert max_rel(vs, v) > 0.1                         # >> 2e-2 tolerance
    assert cosine(vs, v) < 0.999


# ---------------------------------------------------------------- calibration (input recipe)
@pytest.mark.slow
def test_recipe_not_chaotic_full_depth_reduced_tokens():
    """Full 19 + 38 depth at reduced width keeps RMS(h) in [0.3, 30] (DESIGN.md input recipe)."""
    cfg = dataclasses.replace(synth.FLUX, hidden=256, heads=2, txt_dim=64, pooled_dim=32)
    W = O.weights_to_f64(synth.make_weights_bf16(cfg))
    batch = synth.make_batch(cfg, 1, 4, 4, 4)
    trace = []
    O.velocity(cfg, W, batch.latents[0].astype(float), O.bf16_to_f64(batch.txt[0]),
               O.bf16_to_f64(batch.pooled[0]), float(batch.sigma[0]), 3.5, 4, 4, trace=trace)
    rms = [float(np.sqrt((h ** 2).mean())) for h in trace]
    assert 0.3 < min(rms) and max(rms) < 30, rms


# ---------------------------------------------------------------- P13 single-block ControlNet, fan-in
def _trace_velocity(cfg, W, batch, b, controlnets=None, cn_scale=1.0):
    from oracle.flux_step import bf16_to_f64
    tr = []
    v = O.velocity(cfg, W, batch.latents[b].astype(np.float64), bf16_to_f64(batch.txt[b]),
                   bf16_to_f64(batch.pooled[b]), float(batch.sigma[b]), float(batch.guidance[b]),
                   batch.img_h, batch.img_w, trace=tr, controlnets=controlnets, cn_scale=cn_scale)
    return v, tr


def test_p13_single_block_controlnet_injection_point(W_bits):
    """Reading C20: a single-block residual lands on the IMAGE rows of the joint sequence right
    after its block -- txt rows and every earlier block untouched, the later blocks see it."""
    cfg = CFG_S
    W = _W(W_bits, cfg)
    batch = _batch(cfg)
    nt, ni, D = batch.txt_tokens, batch.img_tokens, cfg.hidden
    R = RNG.standard_normal((ni, D)) * 0.1
    cn = O.ControlNetInput(double={}, single={1: R}, n_res=0, n_res_single=2, scale=0.5)
    v0, tr0 = _trace_velocity(cfg, W, batch, 0)
    v1, tr1 = _trace_velocity(cfg, W, batch, 0, [cn], cn_scale=0.8)
    Ld = cfg.depth_double
    for k in range(Ld + 1):                       # double blocks and single block 0: identical
        np.testing.assert_array_equal(tr1[k], tr0[k])
    diff = tr1[Ld + 1] - tr0[Ld + 1]              # after single block 1 (index floor(1 / 1) = 1)
    np.testing.assert_array_equal(diff[:nt], 0.0)
    np.testing.assert_allclose(diff[nt:], 0.8 * 0.5 * R, rtol=0, atol=1e-12)
    # the last block's residual reaches v through the final layer alone
    h = tr1[-1][nt:]
    shf, scf = np.split(O.linear(O.silu(O.conditioning_vec(W, float(batch.sigma[0]), float(batch.guidance[0]),
                                                           O.bf16_to_f64(batch.pooled[0]), cfg.guidance_embed)),
                                 W["final.mod.w"], W["final.mod.b"]), 2)
    v_manual = O.linear((1.0 + scf) * O.layer_norm(h) + shf, W["final.linear.w"], W["final.linear.b"])
    np.testing.assert_allclose(v1, v_manual, rtol=0, atol=1e-12)
    # zero residual -> bitwise the bare model (P3 for single blocks)
    cz = O.ControlNetInput(double={}, single={1: np.zeros_like(R)}, n_res=0, n_res_single=2)
    vz, _ = _trace_velocity(cfg, W, batch, 0, [cz])
    np.testing.assert_array_equal(vz, v0)
    assert max_rel(v1, v0) > 1e-3                 # and it matters


def test_p13_controlnet_fan_in_is_additive(W_bits):
    """Fan-in: two ControlNets feeding the same blocks act like one whose residual
    is the scaled sum (the step is affine in the residual at its injection point)."""
    cfg = CFG_S
    W = _W(W_bits, cfg)
    batch = _batch(cfg)
    ni, D = batch.img_tokens, cfg.hidden
    R1, R2, S1 = (RNG.standard_normal((ni, D)) * 0.1 for _ in range(3))
    a = O.ControlNetInput(double={0: R1}, single={0: S1}, n_res=1, n_res_single=1, scale=0.7)
    b = O.ControlNetInput(double={0: R2}, single={}, n_res=1, n_res_single=0, scale=-0.4)
    both = O.ControlNetInput(double={0: 0.7 * R1 - 0.4 * R2}, single={0: 0.7 * S1}, n_res=1, n_res_single=1)
    v_ab, _ = _trace_velocity(cfg, W, batch, 0, [a, b])
    v_one, _ = _trace_velocity(cfg, W, batch, 0, [both])
    np.testing.assert_allclose(v_ab, v_one, rtol=0, atol=1e-12 * np.abs(v_one).max())
    v_a, _ = _trace_velocity(cfg, W, batch, 0, [a])
    assert max_rel(v_ab, v_a) > 1e-3              # the second ControlNet is not dropped
