"""Oracle: one denoise step of an SD3 / SD3.5 MMDiT base model, with classifier-free
guidance, plain fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Unbatched, unsharded, one
request (and one CFG branch) at a time; every function cites what it follows.

The paper serves SD3 and SD3.5-Large workflows next to Flux-Dev (P:289, P:1305,
P:1330-1331 [§7 Table tab:settings]) and loads the base model as
`SD3Transformer2DModel` (P:841 [§4.1 Fig. flux_model_integration]) but never
writes its math, so the block follows the public SD3 MMDiT definition [ext]
(reading C21):
  * joint blocks only: per stream adaLN-Zero (sh1, sc1, g1, sh2, sc2, g2), QKV,
    optional per-head QK-RMSNorm (SD3.5), joint attention over [txt; img], output
    projection and GELU-tanh MLP with gated residuals -- the Flux double block
    minus RoPE;
  * positions enter once, as a 2-D sincos table added to the embedded image tokens;
  * the last block is `context_pre_only`: its text stream is modulated by the
    2-chunk AdaLayerNormContinuous (scale, shift) and only feeds attention;
  * the final layer is AdaLayerNormContinuous (scale, shift) -> linear.
Classifier-free guidance (P:365-368 [§2.2 "Latent Parallelism"], ho2021classifierfree):
two passes per step, conditional and unconditional, combined as
v = v_u + g (v_c - v_u) before denoise(noise_pred, latents); reading C22.

Parity pins: tests/test_oracle_pins.py P14-P16 (pos table vs the transformers
MAE sincos routine, joint block vs the pinned Flux double block, CFG closed forms)
and the independent torch re-derivation tests/torch_reference.py:step_sd3 (P11).
"""
from __future__ import annotations

from typing import Mapping, Optional

import numpy as np

from .flux_step import (F64, ControlNetInput, OracleLoRA, _cn_sum, _heads, _lora, _pad_rows, _unheads, attention,
                        bf16_to_f64, conditioning_vec, euler, gelu_tanh, layer_norm, linear, rms_norm, silu)


def pos_embed_sincos(D: int, img_h: int, img_w: int, pe_max: int, base: int) -> np.ndarray:
    """SD3 PatchEmbed position table [ext] for an img_h x img_w token grid -> [Ni, D].

    A pe_max x pe_max grid of positions arange(pe_max) * base / pe_max per axis is
    centre-cropped (top = (pe_max - h) // 2, left = (pe_max - w) // 2).  Channels
    [0, D/2) encode the column (w) coordinate, [D/2, D) the row coordinate; each
    half is [sin(p w_k), cos(p w_k)] for k < D/4 with w_k = 10000^(-k / (D/4)).
    (The column coordinate comes first because the public table is built from
    meshgrid(grid_w, grid_h) [ext].)  Token n sits at (n // w, n % w) (row-major
    patchify).
    """
    top, left = (pe_max - img_h) // 2, (pe_max - img_w) // 2
    n = np.arange(img_h * img_w)
    row = (top + n // img_w).astype(F64) * base / pe_max
    col = (left + n % img_w).astype(F64) * base / pe_max
    q = D // 4
    omega = 1.0 / 10000.0 ** (np.arange(q, dtype=F64) / q)

    def sincos(p):
        a = np.outer(p, omega)
        return np.concatenate([np.sin(a), np.cos(a)], axis=1)

    return np.concatenate([sincos(col), sincos(row)], axis=1)


def joint_block(W, i: int, H: int, img: np.ndarray, txt: np.ndarray, vec: np.ndarray,
                adapter: Optional[OracleLoRA], last: bool, qk_norm: bool):
    """SD3 joint block i on ONE sequence (reading C21).  Returns (img, txt); txt is None
    after the context_pre_only last block."""
    sv = silu(vec)
    mods, qs, ks, vs = {}, {}, {}, {}
    streams = {"txt": txt, "img": img}
    for s, x in streams.items():
        p = f"double.{i}.{s}."
        m = linear(sv, W[p + "mod.w"], W[p + "mod.b"])
        if s == "txt" and last:      # AdaLayerNormContinuous: (scale, shift)
            sc, sh = np.split(m, 2)
        else:                        # AdaLayerNormZero: (sh1, sc1, g1, sh2, sc2, g2)
            mods[s] = np.split(m, 6)
            sh, sc = mods[s][0], mods[s][1]
        u = (1.0 + sc) * layer_norm(x) + sh
        qkv = linear(u, W[p + "qkv.w"], W[p + "qkv.b"], _lora(adapter, p + "qkv"))
        D = qkv.shape[1] // 3
        q, k, v = _heads(qkv[:, :D], H), _heads(qkv[:, D:2 * D], H), _heads(qkv[:, 2 * D:], H)
        if qk_norm:
            q, k = rms_norm(q, W[p + "q_norm"]), rms_norm(k, W[p + "k_norm"])
        qs[s], ks[s], vs[s] = q, k, v
    o = _unheads(attention(np.concatenate([qs["txt"], qs["img"]], axis=1),
                           np.concatenate([ks["txt"], ks["img"]], axis=1),
                           np.concatenate([vs["txt"], vs["img"]], axis=1)))
    nt = txt.shape[0]
    outs = {"txt": o[:nt], "img": o[nt:]}
    new = {"txt": None}
    for s, x in streams.items():
        if s == "txt" and last:
            continue
        p = f"double.{i}.{s}."
        sh1, sc1, g1, sh2, sc2, g2 = mods[s]
        x = x + g1 * linear(outs[s], W[p + "proj.w"], W[p + "proj.b"], _lora(adapter, p + "proj"))
        u2 = (1.0 + sc2) * layer_norm(x) + sh2
        a = gelu_tanh(linear(u2, W[p + "fc1.w"], W[p + "fc1.b"], _lora(adapter, p + "fc1")))
        new[s] = x + g2 * linear(a, W[p + "fc2.w"], W[p + "fc2.b"], _lora(adapter, p + "fc2"))
    return new["img"], new["txt"]


def velocity(cfg, W, x: np.ndarray, txt: np.ndarray, pooled: np.ndarray, sigma: float,
             img_h: int, img_w: int, adapter: Optional[OracleLoRA] = None,
             controlnets: Optional[list] = None, cn_scale: float = 1.0) -> np.ndarray:
    """noise_pred of ONE CFG branch: x [Ni, C], txt [Nt, Ct], pooled [Cp] fp64.

    controlnets: ControlNetInput list (double-block residuals, reading C11; SD3 ControlNets
    feed the joint blocks the same way [ext])."""
    H = cfg.heads
    vec = conditioning_vec(W, sigma, 0.0, pooled, guidance_embed=False)
    img = linear(x, W["img_in.w"], W["img_in.b"]) + pos_embed_sincos(
        cfg.hidden, img_h, img_w, cfg.pos_embed_max, cfg.pos_embed_base)
    tx = linear(txt, W["txt_in.w"], W["txt_in.b"])
    cns = list(controlnets or [])
    for i in range(cfg.depth_double):
        img, tx = joint_block(W, i, H, img, tx, vec, adapter, i == cfg.depth_double - 1, cfg.qk_norm)
        r = _cn_sum(cns, "double", i, cfg.depth_double)
        if r is not None:
            img = img + cn_scale * r
    scf, shf = np.split(linear(silu(vec), W["final.mod.w"], W["final.mod.b"]), 2)
    return linear((1.0 + scf) * layer_norm(img) + shf, W["final.linear.w"], W["final.linear.b"])


def cfg_combine(v_cond: np.ndarray, v_uncond: np.ndarray, g: float) -> np.ndarray:
    """Classifier-free guidance (ho2021classifierfree): v_u + g (v_c - v_u)."""
    return v_uncond + float(g) * (v_cond - v_uncond)


def _flux_velocity(cfg, W, x, txt, pooled, sigma, img_h, img_w, adapter=None, controlnets=None,
                   cn_scale=1.0, guidance=3.5):
    from .flux_step import velocity as fv
    return fv(cfg, W, x, txt, pooled, sigma, guidance, img_h, img_w, adapter=adapter,
              cn_scale=cn_scale, controlnets=controlnets)


def _sd3_velocity_kw(cfg, W, x, txt, pooled, sigma, img_h, img_w, adapter=None, controlnets=None,
                     cn_scale=1.0, guidance=None):
    return velocity(cfg, W, x, txt, pooled, sigma, img_h, img_w, adapter, controlnets, cn_scale)


def dit_step(cfg, W, batch, adapters: Optional[Mapping[int, OracleLoRA]] = None,
             controlnets: Optional[Mapping[int, list]] = None):
    """One dit_step over a batch with optional CFG, request by request.

    Without CFG (batch.cfg_scale is None) v = v_cond; with CFG v = cfg_combine(v_c, v_u, g_b).
    Then x' = x + (sigma' - sigma) v (reading C12).  Returns (latents_out, v) fp64."""
    xs, vs = [], []
    for b in range(batch.batch):
        vc = _branch(cfg, W, batch, b, False, adapters, controlnets)
        v = vc if batch.cfg_scale is None else cfg_combine(
            vc, _branch(cfg, W, batch, b, True, adapters, controlnets), batch.cfg_scale[b])
        h, w = batch.grid(b)
        vs.append(_pad_rows(v, batch.img_tokens))
        xs.append(_pad_rows(euler(batch.latents[b][:h * w].astype(F64), v, batch.sigma[b], batch.sigma_next[b]),
                            batch.img_tokens))
    return np.stack(xs), np.stack(vs)


def _branch(cfg, W, batch, b, uncond, adapters, controlnets):
    """Velocity of request b's conditional (uncond=False) or unconditional branch.  Sequence
    slots (reading C22): conditional branch of request b = slot b, unconditional = slot B + b;
    controlnets are keyed by slot."""
    aid = int(batch.adapter_id[b])
    ad = adapters[aid] if (adapters is not None and aid >= 0) else None
    txt = batch.txt_neg[b] if uncond else batch.txt[b]
    pooled = batch.pooled_neg[b] if uncond else batch.pooled[b]
    slot = batch.batch + b if uncond else b
    vel = _sd3_velocity_kw if cfg.arch == "sd3" else _flux_velocity
    h, w = batch.grid(b)   # ragged batch: the request's own grid (reading C24)
    return vel(cfg, W, batch.latents[b][:h * w].astype(F64), bf16_to_f64(txt), bf16_to_f64(pooled),
               float(batch.sigma[b]), h, w, adapter=ad,
               controlnets=(controlnets or {}).get(slot), cn_scale=float(batch.cn_scale[b]),
               guidance=float(batch.guidance[b]))


__all__ = ["pos_embed_sincos", "joint_block", "velocity", "cfg_combine", "dit_step", "ControlNetInput"]
