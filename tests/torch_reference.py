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
