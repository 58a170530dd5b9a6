"""Independent fp64 re-derivation of the step with torch CPU LIBRARY routines.

Test-only (pin P11).  Deliberately formulated differently from
oracle/flux_step.py so a slip in either shows up:
  * batched over requests (torch batch dim) instead of a per-request loop,
  * torch.nn.functional.layer_norm / rms_norm / gelu(approximate="tanh") /
    silu / scaled_dot_product_attention instead of hand-written formulas,
  * RoPE as complex multiplication (torch.polar) instead of pair rotation,
  * LoRA applied MERGED (W + s B A) instead of as an unmerged delta,
  * ControlNet residuals gathered per request.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

T = torch.float64


def _t(x):
    return torch.as_tensor(np.asarray(x), dtype=T)


def bf16(bits):
    return _t((np.asarray(bits).astype(np.uint32) << 16).view(np.float32))


def temb(t: torch.Tensor, dim: int = 256) -> torch.Tensor:
    half = dim // 2
    k = torch.arange(half, dtype=T)
    ang = (1000.0 * t)[:, None] * torch.pow(torch.tensor(10000.0, dtype=T), -k / half)[None]
    return torch.cat([torch.cos(ang), torch.sin(ang)], dim=-1)


def rope_complex(nt, h, w, axes, theta):
    pos = torch.zeros(nt + h * w, 3, dtype=T)
    ii, jj = torch.meshgrid(torch.arange(h, dtype=T), torch.arange(w, dtype=T), indexing="ij")
    pos[nt:, 1] = ii.reshape(-1)
    pos[nt:, 2] = jj.reshape(-1)
    parts = []
    for a, da in enumerate(axes):
        freqs = torch.pow(torch.tensor(theta, dtype=T), -torch.arange(0, da, 2, dtype=T) / da)
        parts.append(torch.outer(pos[:, a], freqs))
    ang = torch.cat(parts, dim=1)
    return torch.polar(torch.ones_like(ang), ang)          # [N, d/2] complex


def rot(x, cis):
    xc = torch.view_as_complex(x.reshape(*x.shape[:-1], -1, 2).contiguous())
    return torch.view_as_real(xc * cis).reshape(x.shape)


def step(cfg, Wbits, batch, adapters=None, controlnet=None, n_res=0):
    """adapters: id -> (scale, {module: (A_bits, B_bits)}); controlnet: b -> {idx: R fp64 ndarray}."""
    D, H, d = cfg.hidden, cfg.heads, cfg.head_dim
    W = {k: bf16(v) for k, v in Wbits.items()}
    B = batch.batch
    nt, h, w = batch.txt_tokens, batch.img_h, batch.img_w

    def weight(b, name):
        wt = W[name + ".w"]
        aid = int(batch.adapter_id[b])
        if adapters and aid >= 0 and name in adapters[aid][1]:
            s, (a, bm) = adapters[aid][0], adapters[aid][1][name]
            wt = wt + s * (bf16(bm) @ bf16(a))
        return wt

    def lin(x, name):       # x [B, N, in]; per-request (possibly merged) weights
        return torch.stack([F.linear(x[b], weight(b, name), W[name + ".b"]) for b in range(B)])

    def mlp(name, x):
        return F.linear(F.silu(F.linear(x, W[name + ".in.w"], W[name + ".in.b"])),
                        W[name + ".out.w"], W[name + ".out.b"])

    vec = mlp("time_in", temb(_t(batch.sigma.astype(np.float64))))
    if cfg.guidance_embed:
        vec = vec + mlp("guidance_in", temb(_t(batch.guidance.astype(np.float64))))
    vec = vec + mlp("vector_in", bf16(batch.pooled))
    svec = F.silu(vec)[:, None, :]                                 # [B, 1, D]
    img = F.linear(_t(batch.latents.astype(np.float64)), W["img_in.w"], W["img_in.b"])
    txt = F.linear(bf16(batch.txt), W["txt_in.w"], W["txt_in.b"])
    cis = rope_complex(nt, h, w, cfg.rope_axes, cfg.rope_theta)
    ln = lambda x: F.layer_norm(x, (D,), eps=1e-6)

    def attn(qkv, qn, kn):                                     # qkv [B, N, 3D]
        q, k, v = qkv.reshape(B, -1, 3, H, d).permute(2, 0, 3, 1, 4)
        q = F.rms_norm(q, (d,), weight=qn, eps=1e-6)
        k = F.rms_norm(k, (d,), weight=kn, eps=1e-6)
        o = F.scaled_dot_product_attention(rot(q, cis), rot(k, cis), v)
        return o.permute(0, 2, 1, 3).reshape(B, -1, D)

    interval = math.ceil(cfg.depth_double / n_res) if n_res else 0
    for i in range(cfg.depth_double):
        st = {"txt": txt, "img": img}
        m, qkvs = {}, {}
        for s in ("txt", "img"):
            p = f"double.{i}.{s}."
            m[s] = F.linear(svec, W[p + "mod.w"], W[p + "mod.b"]).chunk(6, dim=-1)
            qkvs[s] = lin((1 + m[s][1]) * ln(st[s]) + m[s][0], p + "qkv")
        # same q/k norm weights per stream: normalise each stream separately then join
        parts = []
        for s in ("txt", "img"):
            p = f"double.{i}.{s}."
            q, k, v = qkvs[s].reshape(B, -1, 3, H, d).permute(2, 0, 3, 1, 4)
            parts.append((F.rms_norm(q, (d,), weight=W[p + "q_norm"], eps=1e-6),
                          F.rms_norm(k, (d,), weight=W[p + "k_norm"], eps=1e-6), v))
        q = torch.cat([parts[0][0], parts[1][0]], dim=2)
        k = torch.cat([parts[0][1], parts[1][1]], dim=2)
        v = torch.cat([parts[0][2], parts[1][2]], dim=2)
        o = F.scaled_dot_product_attention(rot(q, cis), rot(k, cis), v).permute(0, 2, 1, 3).reshape(B, -1, D)
        o_s = {"txt": o[:, :nt], "img": o[:, nt:]}
        for s in ("txt", "img"):
            p = f"double.{i}.{s}."
            sh1, sc1, g1, sh2, sc2, g2 = m[s]
            x = st[s] + g1 * lin(o_s[s], p + "proj")
            x = x + g2 * lin(F.gelu(lin((1 + sc2) * ln(x) + sh2, p + "fc1"), approximate="tanh"), p + "fc2")
            st[s] = x
        txt, img = st["txt"], st["img"]
        if controlnet and n_res:
            add = torch.zeros_like(img)
            for b, res in controlnet.items():
                r = res.get(i // interval)
                if r is not None:
                    add[b] = float(batch.cn_scale[b]) * _t(r)
            img = img + add
    x = torch.cat([txt, img], dim=1)
    for j in range(cfg.depth_single):
        p = f"single.{j}."
        sh, sc, g = F.linear(svec, W[p + "mod.w"], W[p + "mod.b"]).chunk(3, dim=-1)
        y1 = lin((1 + sc) * ln(x) + sh, p + "linear1")
        o = attn(y1[..., :3 * D], W[p + "q_norm"], W[p + "k_norm"])
        x = x + g * lin(torch.cat([o, F.gelu(y1[..., 3 * D:], approximate="tanh")], dim=-1), p + "linear2")
    img = x[:, nt:]
    shf, scf = F.linear(svec, W["final.mod.w"], W["final.mod.b"]).chunk(2, dim=-1)
    v = F.linear((1 + scf) * ln(img) + shf, W["final.linear.w"], W["final.linear.b"])
    dt = _t((batch.sigma_next.astype(np.float64) - batch.sigma.astype(np.float64)))[:, None, None]
    return (_t(batch.latents.astype(np.float64)) + dt * v).numpy(), v.numpy()


def pos_table_mae(D, h, w, pe_max, base):
    """SD3 position table through the transformers MAE sincos LIBRARY routine: the scaled
    pe_max x pe_max grid built as in the public SD3 PatchEmbed, then centre-cropped."""
    from transformers.models.vit_mae.modeling_vit_mae import get_2d_sincos_pos_embed_from_grid
    g = np.arange(pe_max, dtype=np.float64) * base / pe_max
    grid = np.stack(np.meshgrid(g, g), axis=0).reshape(2, 1, pe_max, pe_max)
    full = get_2d_sincos_pos_embed_from_grid(D, grid).reshape(pe_max, pe_max, D)
    top, left = (pe_max - h) // 2, (pe_max - w) // 2
    return _t(full[top:top + h, left:left + w].reshape(h * w, D))


def step_sd3(cfg, Wbits, batch, adapters=None, controlnets=None):
    """SD3 MMDiT step with classifier-free guidance (pin P11 for reading C21/C22).

    Formulated like a diffusers-style pipeline, unlike oracle/sd3_step.py: the CFG batch is
    DOUBLED ([cond requests; uncond requests] in one torch batch), LoRA merged, library
    norms / attention / activations, the position table from the MAE library routine.
    controlnets: slot -> {residual index: R fp64} (slot B + b = uncond branch of request b).
    """
    D, H, d = cfg.hidden, cfg.heads, cfg.head_dim
    W = {k: bf16(v) for k, v in Wbits.items()}
    B = batch.batch
    cfgon = batch.cfg_scale is not None
    S = 2 * B if cfgon else B
    req = [s % B for s in range(S)]
    nt, h, w = batch.txt_tokens, batch.img_h, batch.img_w
    txt_bits = np.concatenate([batch.txt, batch.txt_neg]) if cfgon else batch.txt
    pooled_bits = np.concatenate([batch.pooled, batch.pooled_neg]) if cfgon else batch.pooled

    def weight(s, name):
        wt = W[name + ".w"]
        aid = int(batch.adapter_id[req[s]])
        if adapters and aid >= 0 and name in adapters[aid][1]:
            sc, (a, bm) = adapters[aid][0], adapters[aid][1][name]
            wt = wt + sc * (bf16(bm) @ bf16(a))
        return wt

    def lin(x, name):
        return torch.stack([F.linear(x[s], weight(s, name), W[name + ".b"]) for s in range(S)])

    def mlp(name, x):
        return F.linear(F.silu(F.linear(x, W[name + ".in.w"], W[name + ".in.b"])),
                        W[name + ".out.w"], W[name + ".out.b"])

    sig = _t(batch.sigma.astype(np.float64))[req]
    vec = mlp("time_in", temb(sig)) + mlp("vector_in", bf16(pooled_bits))
    svec = F.silu(vec)[:, None, :]
    lat = _t(batch.latents.astype(np.float64))[req]
    img = F.linear(lat, W["img_in.w"], W["img_in.b"]) + pos_table_mae(D, h, w, cfg.pos_embed_max,
                                                                      cfg.pos_embed_base)[None]
    txt = F.linear(bf16(txt_bits), W["txt_in.w"], W["txt_in.b"])
    ln = lambda x: F.layer_norm(x, (D,), eps=1e-6)
    L = cfg.depth_double
    for i in range(L):
        last = i == L - 1
        st = {"txt": txt, "img": img}
        m, qkv = {}, {}
        for s in ("txt", "img"):
            p = f"double.{i}.{s}."
            mm = F.linear(svec, W[p + "mod.w"], W[p + "mod.b"])
            if s == "txt" and last:
                sc, sh = mm.chunk(2, dim=-1)
            else:
                m[s] = mm.chunk(6, dim=-1)
                sh, sc = m[s][0], m[s][1]
            q, k, v = lin(ln(st[s]) * (1 + sc) + sh, p + "qkv").reshape(S, -1, 3, H, d).permute(2, 0, 3, 1, 4)
            if cfg.qk_norm:
                q = F.rms_norm(q, (d,), weight=W[p + "q_norm"], eps=1e-6)
                k = F.rms_norm(k, (d,), weight=W[p + "k_norm"], eps=1e-6)
            qkv[s] = (q, k, v)
        # image tokens FIRST here (the public SD3 order); attention is permutation-equivariant
        o = F.scaled_dot_product_attention(*(torch.cat([qkv["img"][j], qkv["txt"][j]], dim=2) for j in range(3)))
        o = o.permute(0, 2, 1, 3).reshape(S, -1, D)
        ni = img.shape[1]
        o_s = {"img": o[:, :ni], "txt": o[:, ni:]}
        for s in ("txt", "img"):
            if s == "txt" and last:
                continue
            p = f"double.{i}.{s}."
            sh1, sc1, g1, sh2, sc2, g2 = m[s]
            x = st[s] + g1 * lin(o_s[s], p + "proj")
            st[s] = x + g2 * lin(F.gelu(lin((1 + sc2) * ln(x) + sh2, p + "fc1"), approximate="tanh"), p + "fc2")
        txt, img = st["txt"], st["img"]
        if controlnets:
            add = torch.zeros_like(img)
            for slot, res in controlnets.items():
                interval = math.ceil(L / res["n_res"])
                r = res["R"].get(i // interval)
                if r is not None:
                    add[slot] = float(batch.cn_scale[req[slot]]) * _t(r)
            img = img + add
    scf, shf = F.linear(svec, W["final.mod.w"], W["final.mod.b"]).chunk(2, dim=-1)
    v = F.linear((1 + scf) * ln(img) + shf, W["final.linear.w"], W["final.linear.b"])
    if cfgon:
        v_c, v_u = v.chunk(2)
        g = _t(batch.cfg_scale.astype(np.float64))[:, None, None]
        v = v_u + g * (v_c - v_u)
    dt = _t((batch.sigma_next.astype(np.float64) - batch.sigma.astype(np.float64)))[:, None, None]
    return (_t(batch.latents.astype(np.float64)) + dt * v).numpy(), v.numpy()
