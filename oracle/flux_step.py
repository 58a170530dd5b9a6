"""Oracle: one denoise step of the shared base model, plain fp64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Slow, unbatched,
unsharded, obviously-correct.  Every function cites the passage it follows.

Citations: "P:a-b" = /root/reference/PAPER.md lines a-b; "C#" = the reading
numbered # in DESIGN.md §3 (= SURVEY.md §8(c) table), used where the paper is
silent -- the paper names Flux-Dev but never writes
its math, so the step follows the public Flux-Dev definition [ext].

What the method computes (the system "does not alter the
computation performed during diffusion inference"): a cross-workflow batch
 gives, for every request b, exactly what running request b alone
through the base model -- patched with its own LoRA and fed its own
ControlNet residuals -- followed by
denoise(noise_pred, latents) gives.  So the oracle loops over requests
one at a time.

Parity pins: tests/test_oracle_pins.py (P1-P12 of DESIGN.md §4).
Parity unpinned: none of the full-model VALUES are printed in the paper; the
full step is pinned only through its parts and through the independent
torch-library re-derivation (pin P11).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Mapping, Optional, Tuple

import numpy as np

F64 = np.float64


# ----------------------------------------------------------------------------
# Parameters: bf16 bits -> fp64 (the oracle computes on the SAME bf16-rounded
# parameters the GPU sees; reading C13)
# ----------------------------------------------------------------------------

def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(F64)


def weights_to_f64(w_bf16: Mapping[str, np.ndarray]) -> Dict[str, np.ndarray]:
    return {k: bf16_to_f64(v) for k, v in w_bf16.items()}


@dataclasses.dataclass
class OracleLoRA:
    """One registered adapter (add_patch).

    scale = alpha / r (reading C9).  mats[module] = (A [r, in], B [out, r]) fp64.
    """
    scale: float
    mats: Dict[str, Tuple[np.ndarray, np.ndarray]]


# ----------------------------------------------------------------------------
# Elementary definitions (each the textbook formula)
# ----------------------------------------------------------------------------

def timestep_embedding(t: float, dim: int = 256, max_period: float = 10000.0,
                       time_factor: float = 1000.0) -> np.ndarray:
    """Sinusoidal embedding of 1000*t, cos half first (reading C8, Flux [ext])."""
    half = dim // 2
    freqs = np.exp(-math.log(max_period) * np.arange(half, dtype=F64) / half)
    args = time_factor * float(t) * freqs
    return np.concatenate([np.cos(args), np.sin(args)])


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    """GELU, tanh approximation (reading C6)."""
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def layer_norm(x: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """LN over the last axis, no affine, biased variance (reading C4)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


def rms_norm(x: np.ndarray, gamma: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """RMSNorm over the last axis times learned gamma (QK-norm, reading C4)."""
    return x / np.sqrt((x ** 2).mean(axis=-1, keepdims=True) + eps) * gamma


def linear(x: np.ndarray, w: np.ndarray, b: np.ndarray,
           lora: Optional[Tuple[float, np.ndarray, np.ndarray]] = None) -> np.ndarray:
    """y = x W^T + b (+ s (x A^T) B^T), the unmerged LoRA of reading C9.

    The LoRA delta is ADDED to the base output, so a zero delta leaves y
    bitwise unchanged (pin P3).
    """
    y = x @ w.T + b
    if lora is not None:
        s, a, bm = lora
        y = y + s * ((x @ a.T) @ bm.T)
    return y


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """softmax(Q K^T / sqrt(d)) V per head; non-causal, no mask (reading C7).

    q, k, v: [H, N, d] -> [H, N, d].
    """
    d = q.shape[-1]
    s = (q @ k.swapaxes(-1, -2)) / math.sqrt(d)          # [H, Nq, Nk]
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    return p @ v


# ----------------------------------------------------------------------------
# RoPE (Flux 3-axis, interleaved pairs) [ext]
# ----------------------------------------------------------------------------

def position_ids(txt_tokens: int, img_h: int, img_w: int) -> np.ndarray:
    """Joint token positions, txt first (reading C3): txt (0,0,0); img n -> (0, n//W, n%W)."""
    ids = np.zeros((txt_tokens + img_h * img_w, 3), dtype=F64)
    n = np.arange(img_h * img_w)
    ids[txt_tokens:, 1] = n // img_w
    ids[txt_tokens:, 2] = n % img_w
    return ids


def rope_cos_sin(ids: np.ndarray, axes: Tuple[int, ...], theta: float):
    """Angles per (token, pair): pair j of axis a turns by pos_a * theta^(-2j/d_a)."""
    angs = []
    for a, da in enumerate(axes):
        j = np.arange(0, da, 2, dtype=F64) / da
        omega = 1.0 / (theta ** j)
        angs.append(ids[:, a:a + 1] * omega[None, :])
    ang = np.concatenate(angs, axis=1)          # [N, d/2]
    return np.cos(ang), np.sin(ang)


def apply_rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate interleaved pairs (2j, 2j+1) of x [H, N, d] by the angles [N, d/2]."""
    x0, x1 = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = cos * x0 - sin * x1
    out[..., 1::2] = sin * x0 + cos * x1
    return out


# ----------------------------------------------------------------------------
# Blocks (Flux-Dev double- and single-stream blocks [ext], reading C5)
# ----------------------------------------------------------------------------

def _heads(x: np.ndarray, H: int) -> np.ndarray:
    """[N, H*d] -> [H, N, d]."""
    N, HD = x.shape
    return x.reshape(N, H, HD // H).transpose(1, 0, 2)


def _unheads(x: np.ndarray) -> np.ndarray:
    H, N, d = x.shape
    return x.transpose(1, 0, 2).reshape(N, H * d)


def _lora(adapter: Optional[OracleLoRA], module: str):
    if adapter is None or module not in adapter.mats:
        return None
    a, b = adapter.mats[module]
    return (adapter.scale, a, b)


def _qkv_heads(qkv: np.ndarray, H: int, gq: np.ndarray, gk: np.ndarray):
    """Split [N, 3D] into q, k, v [H, N, d] ('(K H D)' order) and QK-RMSNorm q, k."""
    D = qkv.shape[1] // 3
    q = _heads(qkv[:, :D], H)
    k = _heads(qkv[:, D:2 * D], H)
    v = _heads(qkv[:, 2 * D:], H)
    return rms_norm(q, gq), rms_norm(k, gk), v


def double_block(W, i: int, H: int, img: np.ndarray, txt: np.ndarray, vec: np.ndarray,
                 cos: np.ndarray, sin: np.ndarray, adapter: Optional[OracleLoRA]):
    """Flux double-stream block i on ONE request."""
    sv = silu(vec)
    mods, qs, ks, vs = {}, {}, {}, {}
    streams = {"img": img, "txt": txt}
    for s, x in streams.items():
        p = f"double.{i}.{s}."
        m = linear(sv, W[p + "mod.w"], W[p + "mod.b"])
        mods[s] = np.split(m, 6)                 # sh1, sc1, g1, sh2, sc2, g2
        sh1, sc1 = mods[s][0], mods[s][1]
        u = (1.0 + sc1) * layer_norm(x) + sh1
        qkv = linear(u, W[p + "qkv.w"], W[p + "qkv.b"], _lora(adapter, p + "qkv"))
        qs[s], ks[s], vs[s] = _qkv_heads(qkv, H, W[p + "q_norm"], W[p + "k_norm"])
    # joint sequence [txt; img] (reading C3), RoPE then attention
    q = np.concatenate([qs["txt"], qs["img"]], axis=1)
    k = np.concatenate([ks["txt"], ks["img"]], axis=1)
    v = np.concatenate([vs["txt"], vs["img"]], axis=1)
    o = _unheads(attention(apply_rope(q, cos, sin), apply_rope(k, cos, sin), v))
    nt = txt.shape[0]
    outs = {"txt": o[:nt], "img": o[nt:]}
    new = {}
    for s, x in streams.items():
        p = f"double.{i}.{s}."
        sh1, sc1, g1, sh2, sc2, g2 = mods[s]
        x = x + g1 * linear(outs[s], W[p + "proj.w"], W[p + "proj.b"], _lora(adapter, p + "proj"))
        u2 = (1.0 + sc2) * layer_norm(x) + sh2
        a = gelu_tanh(linear(u2, W[p + "fc1.w"], W[p + "fc1.b"], _lora(adapter, p + "fc1")))
        x = x + g2 * linear(a, W[p + "fc2.w"], W[p + "fc2.b"], _lora(adapter, p + "fc2"))
        new[s] = x
    return new["img"], new["txt"]


def single_block(W, j: int, H: int, x: np.ndarray, vec: np.ndarray,
                 cos: np.ndarray, sin: np.ndarray, adapter: Optional[OracleLoRA]):
    """Flux single-stream block j on the joint sequence."""
    p = f"single.{j}."
    D = x.shape[1]
    sh, sc, g = np.split(linear(silu(vec), W[p + "mod.w"], W[p + "mod.b"]), 3)
    u = (1.0 + sc) * layer_norm(x) + sh
    y1 = linear(u, W[p + "linear1.w"], W[p + "linear1.b"], _lora(adapter, p + "linear1"))
    q, k, v = _qkv_heads(y1[:, :3 * D], H, W[p + "q_norm"], W[p + "k_norm"])
    o = _unheads(attention(apply_rope(q, cos, sin), apply_rope(k, cos, sin), v))
    cat = np.concatenate([o, gelu_tanh(y1[:, 3 * D:])], axis=1)
    return x + g * linear(cat, W[p + "linear2.w"], W[p + "linear2.b"], _lora(adapter, p + "linear2"))


def conditioning_vec(W, sigma: float, guidance: float, pooled: np.ndarray,
                     guidance_embed: bool = True) -> np.ndarray:
    """vec = MLP_t(e(sigma)) + MLP_g(e(g)) + MLP_y(pooled)."""
    def mlp(name, x):
        return linear(silu(linear(x, W[name + ".in.w"], W[name + ".in.b"])),
                      W[name + ".out.w"], W[name + ".out.b"])
    vec = mlp("time_in", timestep_embedding(sigma))
    if guidance_embed:
        vec = vec + mlp("guidance_in", timestep_embedding(guidance))
    return vec + mlp("vector_in", pooled)


@dataclasses.dataclass
class ControlNetInput:
    """One ControlNet's outputs for one request ("consumed by specific layers").

    double: residual index -> R [Ni, D], consumed after double block i at index
    floor(i / ceil(L_d / n_res)) (reading C11); single: the same for the single blocks,
    floor(j / ceil(L_s / n_res_single)), added to the image rows of the joint sequence
    (reading C20); scale: this ControlNet's conditioning scale.  Several ControlNets feeding
    one block are summed (fan-in; reading C20)."""
    double: Dict[int, np.ndarray]
    single: Dict[int, np.ndarray]
    n_res: int
    n_res_single: int
    scale: float = 1.0


def _cn_sum(cns, which: str, blk: int, depth: int) -> Optional[np.ndarray]:
    """sum_c scale_c * R_c[floor(blk / interval_c)] over the ControlNets that feed block blk."""
    tot = None
    for cn in cns:
        n = cn.n_res if which == "double" else cn.n_res_single
        res = cn.double if which == "double" else cn.single
        if not n or not res:
            continue
        r = res.get(blk // math.ceil(depth / n))
        if r is not None:
            tot = cn.scale * r if tot is None else tot + cn.scale * r
    return tot


def velocity(cfg, W, x: np.ndarray, txt: np.ndarray, pooled: np.ndarray, sigma: float,
             guidance: float, img_h: int, img_w: int,
             adapter: Optional[OracleLoRA] = None,
             residuals: Optional[Dict[int, np.ndarray]] = None, cn_scale: float = 1.0,
             n_res: int = 0, trace: Optional[list] = None,
             controlnets: Optional[list] = None) -> np.ndarray:
    """noise_pred = transformer(latents, prompt_embeds, controlnet_inputs).

    x [Ni, C] fp64, txt [Nt, Ct], pooled [Cp].  residuals: double block index ->
    R [Ni, D] (deferred ControlNet input; consumed after double block i,
    index floor(i / interval), interval = ceil(L_d / n_res): reading C11) -- a
    ControlNet of scale 1 with double-block outputs only.  controlnets: further
    ControlNetInput objects (single-block outputs, fan-in; reading C20).  Every
    ControlNet contribution is multiplied by the request's cn_scale.
    """
    cns = list(controlnets or [])
    if residuals is not None and n_res:
        cns.insert(0, ControlNetInput(double=residuals, single={}, n_res=n_res, n_res_single=0))
    H = cfg.heads
    vec = conditioning_vec(W, sigma, guidance, pooled, cfg.guidance_embed)
    img = linear(x, W["img_in.w"], W["img_in.b"])
    tx = linear(txt, W["txt_in.w"], W["txt_in.b"])
    cos, sin = rope_cos_sin(position_ids(txt.shape[0], img_h, img_w), cfg.rope_axes, cfg.rope_theta)
    for i in range(cfg.depth_double):
        img, tx = double_block(W, i, H, img, tx, vec, cos, sin, adapter)
        r = _cn_sum(cns, "double", i, cfg.depth_double)
        if r is not None:
            img = img + cn_scale * r
        if trace is not None:
            trace.append(np.concatenate([tx, img]))
    h = np.concatenate([tx, img])
    nt = txt.shape[0]
    for j in range(cfg.depth_single):
        h = single_block(W, j, H, h, vec, cos, sin, adapter)
        r = _cn_sum(cns, "single", j, cfg.depth_single)
        if r is not None:   # image rows of the joint sequence (reading C20)
            h = np.concatenate([h[:nt], h[nt:] + cn_scale * r])
        if trace is not None:
            trace.append(h)
    img = h[txt.shape[0]:]
    shf, scf = np.split(linear(silu(vec), W["final.mod.w"], W["final.mod.b"]), 2)
    return linear((1.0 + scf) * layer_norm(img) + shf, W["final.linear.w"], W["final.linear.b"])


def euler(x: np.ndarray, v: np.ndarray, sigma: float, sigma_next: float) -> np.ndarray:
    """denoise(noise_pred, latents): flow-matching Euler x' = x + (s' - s) v (reading C12)."""
    return x + (float(sigma_next) - float(sigma)) * v


def dit_step(cfg, W, batch, adapters: Optional[Mapping[int, OracleLoRA]] = None,
             controlnet: Optional[Mapping[int, Dict[int, np.ndarray]]] = None,
             n_res: int = 0, requests=None, controlnets: Optional[Mapping[int, list]] = None):
    """One dit_step over a cross-workflow batch, evaluated request by request.

    batch: synth.Batch (bf16 bits for txt/pooled, fp32 latents).
    adapters: adapter_id -> OracleLoRA.  controlnet: request b -> {res index: R fp64}
    (double blocks, one ControlNet).  controlnets: request b -> [ControlNetInput, ...].
    Returns (latents_out [B, Ni, C], v [B, Ni, C]) fp64.
    """
    B = batch.batch
    reqs = range(B) if requests is None else requests
    xs, vs = [], []
    for b in reqs:
        aid = int(batch.adapter_id[b])
        ad = adapters[aid] if (adapters is not None and aid >= 0) else None
        h, w = batch.grid(b)          # a ragged batch: each request at its own grid (reading C24)
        x = batch.latents[b][:h * w].astype(F64)
        v = velocity(cfg, W, x, bf16_to_f64(batch.txt[b]), bf16_to_f64(batch.pooled[b]),
                     float(batch.sigma[b]), float(batch.guidance[b]), h, w,
                     adapter=ad, residuals=(controlnet or {}).get(b), cn_scale=float(batch.cn_scale[b]),
                     n_res=n_res, controlnets=(controlnets or {}).get(b))
        vs.append(_pad_rows(v, batch.img_tokens))
        xs.append(_pad_rows(euler(x, v, batch.sigma[b], batch.sigma_next[b]), batch.img_tokens))
    return np.stack(xs), np.stack(vs)


def _pad_rows(a: np.ndarray, n: int) -> np.ndarray:
    """Zero rows up to the batch's padded slot (rows beyond a request's grid carry no value)."""
    if a.shape[0] == n:
        return a
    return np.concatenate([a, np.zeros((n - a.shape[0],) + a.shape[1:], dtype=a.dtype)])


def merged_weights(W, adapter: OracleLoRA) -> Dict[str, np.ndarray]:
    """W + s B A for every adapted linear (merged patching; pin P2)."""
    out = dict(W)
    for mod, (a, b) in adapter.mats.items():
        out[mod + ".w"] = W[mod + ".w"] + adapter.scale * (b @ a)
    return out
