"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no norms, no attention, no
projections).  It only defines:

  * the model-shape presets (BASELINE.json configs),
  * the weight manifest (tensor names, shapes and generator recipe of a
    Flux-Dev-shaped MMDiT; SURVEY.md §8(c) reading C1 -- the paper names
    Flux-Dev at PAPER.md:154, :289-290, :1306 but never defines it),
  * a counter-based generator (splitmix64) used for weights, and
  * numpy normal draws for the per-request inputs (latents, text, pooled,
    ControlNet residuals) and the flow-matching sigma schedule values.

The CUDA library implements the SAME counter generator on the device
(`dit_fill_synthetic`, csrc/synthetic.cu) so full-size weights never cross
PCIe; tests check the two bit-for-bit.  The generator is:

    key = seed XOR (tensor_id << 40) XOR index          (uint64)
    u   = (splitmix64(key) >> 40) * 2**-24               (exact fp32)
    w   = bf16_rne( offset + fp32(fp32(2u - 1) * scale) )

using only integer ops and IEEE single-rounded fp32 multiply / add.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# Model shape presets
# ----------------------------------------------------------------------------


@dataclasses.dataclass(frozen=True)
class ModelCfg:
    hidden: int          # D
    heads: int           # H  (head dim d = D / H)
    depth_double: int    # L_d
    depth_single: int    # L_s
    in_channels: int     # C   (packed latent channels)
    txt_dim: int         # Ct  (T5 embedding width)
    pooled_dim: int      # Cp  (CLIP pooled width)
    mlp_ratio: int = 4   # F = mlp_ratio * D
    rope_axes: Tuple[int, int, int] = (16, 56, 56)
    rope_theta: float = 10000.0
    guidance_embed: bool = True
    # "flux": double + single blocks, 3-axis RoPE (reading C1).  "sd3": SD3 / SD3.5 MMDiT
    # (joint blocks only, 2-D sincos position table, last block context_pre_only; reading C21).
    arch: str = "flux"
    qk_norm: bool = True        # sd3 only: SD3.5 has QK-RMSNorm, SD3(-medium) has none
    pos_embed_max: int = 192    # sd3: side of the sincos position grid (centre-cropped)
    pos_embed_base: int = 64    # sd3: base size of the grid (positions = arange * base / max)

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    @property
    def mlp_hidden(self) -> int:
        return self.mlp_ratio * self.hidden


# T0 tiny (BASELINE.json configs[0]): 1 double block, hidden 64, 2 heads.
TINY = ModelCfg(hidden=64, heads=2, depth_double=1, depth_single=0,
                in_channels=16, txt_dim=32, pooled_dim=16, rope_axes=(4, 14, 14))
# Tiny variant that also exercises single-stream blocks.
TINY_SINGLE = dataclasses.replace(TINY, depth_double=1, depth_single=2)
# Flux-Dev shape (configs[1..4]) [ext].
FLUX = ModelCfg(hidden=3072, heads=24, depth_double=19, depth_single=38,
                in_channels=64, txt_dim=4096, pooled_dim=768)


# SD3 family (PAPER.md:289, :1305, :1330-1331 name SD3 and SD3.5-Large) [ext]:
# SD3-medium 24 joint blocks, D = 1536 (24 heads x 64), no QK-norm; SD3.5-Large 38 joint
# blocks, D = 2432 (38 x 64), QK-RMSNorm.  Packed latents 16 ch x 2 x 2 = 64, T5 width 4096,
# pooled CLIP-L + CLIP-G = 2048, text tokens 77 (CLIP) + 256 (T5) = 333.
SD3_MEDIUM = ModelCfg(hidden=1536, heads=24, depth_double=24, depth_single=0, in_channels=64,
                      txt_dim=4096, pooled_dim=2048, rope_axes=(0, 0, 0), guidance_embed=False,
                      arch="sd3", qk_norm=False)
SD35_LARGE = dataclasses.replace(SD3_MEDIUM, hidden=2432, heads=38, depth_double=38, qk_norm=True)
SD3_TXT_TOKENS = 333
# Tiny SD3: 2 joint blocks (the second context_pre_only), d = 32, an 8 x 8 position grid.
SD3_TINY = ModelCfg(hidden=64, heads=2, depth_double=2, depth_single=0, in_channels=16, txt_dim=32,
                    pooled_dim=16, rope_axes=(0, 0, 0), guidance_embed=False, arch="sd3",
                    qk_norm=True, pos_embed_max=8, pos_embed_base=4)


def flux_reduced(depth_double: int, depth_single: int) -> ModelCfg:
    return dataclasses.replace(FLUX, depth_double=depth_double, depth_single=depth_single)


# ----------------------------------------------------------------------------
# Weight manifest
# ----------------------------------------------------------------------------
# kinds -> (scale, offset) recipe.  Scales are the SURVEY.md §8(d) ones,
# calibrated with the oracle so the random network is not chaotic
# (DESIGN.md "Input recipe").
LINEAR, BIAS, GAMMA, MOD_W, MOD_B = "linear", "bias", "gamma", "mod_w", "mod_b"
LORA_A, LORA_B = "lora_a", "lora_b"

MOD_GAIN = 0.5      # modulation weight gain (x sqrt(3/D))
LORA_B_GAIN = 0.5   # LoRA up-projection gain (x sqrt(3/r))


def _recipe(kind: str, fan_in: int, cfg: ModelCfg) -> Tuple[float, float]:
    if kind == LINEAR:
        return math.sqrt(3.0 / fan_in), 0.0
    if kind == BIAS:
        return 0.02, 0.0
    if kind == GAMMA:
        return 0.1, 1.0
    if kind == MOD_W:
        return MOD_GAIN * math.sqrt(3.0 / cfg.hidden), 0.0
    if kind == MOD_B:
        return 0.02, 0.0
    if kind == LORA_A:
        return math.sqrt(3.0 / fan_in), 0.0
    if kind == LORA_B:
        return LORA_B_GAIN * math.sqrt(3.0 / fan_in), 0.0
    raise ValueError(kind)


@dataclasses.dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: Tuple[int, ...]
    kind: str
    tensor_id: int
    scale: float
    offset: float


def _lin(name: str, out_f: int, in_f: int):
    return [(name + ".w", (out_f, in_f), LINEAR, in_f), (name + ".b", (out_f,), BIAS, in_f)]


def _mod(name: str, out_f: int, in_f: int):
    return [(name + ".w", (out_f, in_f), MOD_W, in_f), (name + ".b", (out_f,), MOD_B, in_f)]


def context_pre_only(cfg: ModelCfg, block: int, stream: str) -> bool:
    """SD3: the last joint block's text stream only feeds attention (no proj / MLP; its
    modulation is the 2-chunk AdaLayerNormContinuous) [ext], reading C21."""
    return cfg.arch == "sd3" and stream == "txt" and block == cfg.depth_double - 1


def weight_manifest(cfg: ModelCfg) -> List[TensorSpec]:
    """Every base-model tensor, in canonical order (tensor_id = position).

    Layout of each linear: weight [out][in] row-major (PyTorch nn.Linear),
    bias [out].  Names follow Flux-Dev's module tree [ext].
    """
    D, C, Ct, Cp, F, d = (cfg.hidden, cfg.in_channels, cfg.txt_dim, cfg.pooled_dim,
                          cfg.mlp_hidden, cfg.head_dim)
    ent = []
    ent += _lin("img_in", D, C)
    ent += _lin("txt_in", D, Ct)
    ent += _lin("time_in.in", D, 256) + _lin("time_in.out", D, D)
    if cfg.guidance_embed:
        ent += _lin("guidance_in.in", D, 256) + _lin("guidance_in.out", D, D)
    ent += _lin("vector_in.in", D, Cp) + _lin("vector_in.out", D, D)
    for i in range(cfg.depth_double):
        for s in ("img", "txt"):
            p = f"double.{i}.{s}."
            pre_only = context_pre_only(cfg, i, s)
            ent += _mod(p + "mod", (2 if pre_only else 6) * D, D)
            ent += _lin(p + "qkv", 3 * D, D)
            if cfg.arch == "flux" or cfg.qk_norm:
                ent += [(p + "q_norm", (d,), GAMMA, d), (p + "k_norm", (d,), GAMMA, d)]
            if pre_only:
                continue
            ent += _lin(p + "proj", D, D)
            ent += _lin(p + "fc1", F, D)
            ent += _lin(p + "fc2", D, F)
    for j in range(cfg.depth_single):
        p = f"single.{j}."
        ent += _mod(p + "mod", 3 * D, D)
        ent += _lin(p + "linear1", 3 * D + F, D)
        ent += [(p + "q_norm", (d,), GAMMA, d), (p + "k_norm", (d,), GAMMA, d)]
        ent += _lin(p + "linear2", D, D + F)
    ent += _mod("final.mod", 2 * D, D)
    ent += _lin("final.linear", C, D)
    out = []
    for tid, (name, shape, kind, fan_in) in enumerate(ent):
        scale, offset = _recipe(kind, fan_in, cfg)
        out.append(TensorSpec(name, tuple(shape), kind, tid, scale, offset))
    return out


def lora_targets(cfg: ModelCfg) -> List[Tuple[str, int, int]]:
    """(module, in_features, out_features) of every LoRA-adapted linear.

    SURVEY.md §8(c) reading C9: every block linear (double qkv/proj/fc1/fc2 per
    stream, single linear1/linear2); not modulation, embedders or final.
    """
    D, F = cfg.hidden, cfg.mlp_hidden
    t = []
    for i in range(cfg.depth_double):
        for s in ("img", "txt"):
            p = f"double.{i}.{s}."
            t += [(p + "qkv", D, 3 * D)]
            if not context_pre_only(cfg, i, s):
                t += [(p + "proj", D, D), (p + "fc1", D, F), (p + "fc2", F, D)]
    for j in range(cfg.depth_single):
        p = f"single.{j}."
        t += [(p + "linear1", D, 3 * D + F), (p + "linear2", D + F, D)]
    return t


def lora_manifest(cfg: ModelCfg, rank: int, adapter_index: int) -> List[TensorSpec]:
    """Tensors of one synthetic adapter: <module>.lora_A [r][in], <module>.lora_B [out][r].

    Seeds follow SURVEY.md §8(d): adapters 3000 + a (passed as the generator
    seed by callers; tensor ids restart at 0 for each adapter).
    """
    out = []
    tid = 0
    for mod, fin, fout in lora_targets(cfg):
        sa, oa = _recipe(LORA_A, fin, cfg)
        out.append(TensorSpec(mod + ".lora_A", (rank, fin), LORA_A, tid, sa, oa))
        tid += 1
        sb, ob = _recipe(LORA_B, rank, cfg)
        out.append(TensorSpec(mod + ".lora_B", (fout, rank), LORA_B, tid, sb, ob))
        tid += 1
    return out


# ----------------------------------------------------------------------------
# Counter-based generator (bit-identical to csrc/synthetic.cu)
# ----------------------------------------------------------------------------
WEIGHT_SEED = 0


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, tensor_id: int, n: int, start: int = 0) -> np.ndarray:
    """u in [0, 1) as fp32 with 24 random bits (exact)."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(tensor_id) << np.uint64(40)) ^ idx
    bits = splitmix64(key) >> np.uint64(40)
    return bits.astype(np.float32) * np.float32(2.0 ** -24)


def fp32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bits."""
    b = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32)
    rounding = ((b >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((b + rounding) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_fp32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def counter_bf16_bits(seed: int, tensor_id: int, n: int, scale: float, offset: float,
                      start: int = 0) -> np.ndarray:
    u = counter_uniform(seed, tensor_id, n, start)
    t = (np.float32(2.0) * u - np.float32(1.0)).astype(np.float32)   # exact
    w = (t * np.float32(scale)).astype(np.float32)                    # one RNE
    if offset != 0.0:
        w = (np.float32(offset) + w).astype(np.float32)               # one RNE
    return fp32_to_bf16_bits(w)


def tensor_bf16_bits(spec: TensorSpec, seed: int = WEIGHT_SEED) -> np.ndarray:
    n = int(np.prod(spec.shape))
    return counter_bf16_bits(seed, spec.tensor_id, n, spec.scale, spec.offset).reshape(spec.shape)


def make_weights_bf16(cfg: ModelCfg, seed: int = WEIGHT_SEED) -> Dict[str, np.ndarray]:
    """name -> uint16 bf16 bits (host).  Small configs only."""
    return {s.name: tensor_bf16_bits(s, seed) for s in weight_manifest(cfg)}


def make_lora_bf16(cfg: ModelCfg, rank: int, adapter_index: int) -> Dict[str, np.ndarray]:
    seed = 3000 + adapter_index
    return {s.name: tensor_bf16_bits(s, seed) for s in lora_manifest(cfg, rank, adapter_index)}


# ----------------------------------------------------------------------------
# Per-request inputs (host numpy, copied bit-exactly to the device)
# ----------------------------------------------------------------------------


def latents(b_seed_index: int, ni: int, c: int) -> np.ndarray:
    """x ~ N(0, 1) fp32 (flow-matching noise), seed 1000 + b."""
    return np.random.default_rng(1000 + b_seed_index).standard_normal((ni, c)).astype(np.float32)


def txt_embeds_bf16(b_seed_index: int, nt: int, ct: int) -> np.ndarray:
    """T5-like text embeddings ~ N(0, 1), rounded to bf16 (bits), seed 2000 + b."""
    x = np.random.default_rng(2000 + b_seed_index).standard_normal((nt, ct)).astype(np.float32)
    return fp32_to_bf16_bits(x)


def pooled_bf16(b_seed_index: int, cp: int) -> np.ndarray:
    x = np.random.default_rng(2500 + b_seed_index).standard_normal((cp,)).astype(np.float32)
    return fp32_to_bf16_bits(x)


def controlnet_residual_bf16(b_seed_index: int, block: int, ni: int, d: int,
                             std: float = 0.1) -> np.ndarray:
    """ControlNet residual R_{b,i} ~ N(0, std^2) bf16 bits, seed 4000 + 64 b + i."""
    rng = np.random.default_rng(4000 + 64 * b_seed_index + block)
    return fp32_to_bf16_bits((std * rng.standard_normal((ni, d))).astype(np.float32))


def flux_sigmas(num_steps: int = 28, image_tokens: int = 4096) -> np.ndarray:
    """Flux-Dev shifted flow-matching schedule values [ext] (host side only).

    sigma_hat_i = linspace(1, 1/num_steps, num_steps); mu = 0.5 + (Ni - 256) *
    0.65 / 3840; sigma_i = e^mu / (e^mu + 1/sigma_hat_i - 1); sigma_N = 0.
    Only the VALUES matter (step cost is sigma-independent).
    """
    sh = np.linspace(1.0, 1.0 / num_steps, num_steps)
    mu = 0.5 + (image_tokens - 256) * 0.65 / 3840.0
    s = math.exp(mu) / (math.exp(mu) + 1.0 / sh - 1.0)
    return np.concatenate([s, [0.0]]).astype(np.float32)


def step_indices(batch: int, num_steps: int = 28, seed: int = 5000) -> np.ndarray:
    """Per-request step index (mixed timesteps in one cross-workflow batch)."""
    return np.random.default_rng(seed).integers(0, num_steps, size=batch)


def adapter_ids(batch: int, n_adapters: int, seed: int = 3100) -> np.ndarray:
    """Seeded permutation of [0,0,1,1,...]."""
    if n_adapters == 0:
        return -np.ones(batch, dtype=np.int32)
    ids = np.array([i % n_adapters for i in range(batch)], dtype=np.int32)
    ids.sort()
    return np.random.default_rng(seed).permutation(ids).astype(np.int32)


@dataclasses.dataclass
class Batch:
    """Host description of one cross-workflow batch (all numpy)."""
    img_h: int
    img_w: int
    txt_tokens: int
    latents: np.ndarray        # fp32 [B, Ni, C]
    txt: np.ndarray            # uint16 bf16 bits [B, Nt, Ct]
    pooled: np.ndarray         # uint16 bf16 bits [B, Cp]
    sigma: np.ndarray          # fp32 [B]
    sigma_next: np.ndarray     # fp32 [B]
    guidance: np.ndarray       # fp32 [B]
    adapter_id: np.ndarray     # int32 [B], -1 = none
    cn_scale: np.ndarray       # fp32 [B]
    # classifier-free guidance (reading C22): None = one pass per request
    cfg_scale: Optional[np.ndarray] = None   # fp32 [B]
    txt_neg: Optional[np.ndarray] = None     # uint16 bf16 bits [B, Nt, Ct] (unconditional branch)
    pooled_neg: Optional[np.ndarray] = None  # uint16 bf16 bits [B, Cp]
    # ragged batch (mixed resolutions; reading C24): None = every request img_h x img_w;
    # else int32 [B, 2] per-request grids, img_h x img_w is the padded slot and request b's
    # latents are its first h_b * w_b rows
    img_hw: Optional[np.ndarray] = None

    @property
    def batch(self) -> int:
        return int(self.latents.shape[0])

    @property
    def img_tokens(self) -> int:
        return self.img_h * self.img_w

    def grid(self, b: int) -> Tuple[int, int]:
        """Request b's own (h, w) token grid."""
        if self.img_hw is None:
            return self.img_h, self.img_w
        return int(self.img_hw[b][0]), int(self.img_hw[b][1])


def negative_txt_bf16(b_seed_index: int, nt: int, ct: int) -> np.ndarray:
    """Unconditional-branch text embeddings ~ N(0, 1) bf16 bits, seed 6000 + b."""
    x = np.random.default_rng(6000 + b_seed_index).standard_normal((nt, ct)).astype(np.float32)
    return fp32_to_bf16_bits(x)


def negative_pooled_bf16(b_seed_index: int, cp: int) -> np.ndarray:
    x = np.random.default_rng(6500 + b_seed_index).standard_normal((cp,)).astype(np.float32)
    return fp32_to_bf16_bits(x)


def make_batch(cfg: ModelCfg, batch: int, img_h: int, img_w: int, txt_tokens: int,
               n_adapters: int = 0, guidance: float = 3.5, first_request: int = 0,
               cfg_scale: Optional[float] = None) -> Batch:
    """cfg_scale: classifier-free guidance scale (SD3 default 7.0 [ext]); None = no CFG."""
    ni = img_h * img_w
    sig = flux_sigmas(28, ni)
    k = step_indices(batch)
    neg = {}
    if cfg_scale is not None:
        neg = dict(
            cfg_scale=np.full(batch, cfg_scale, dtype=np.float32),
            txt_neg=np.stack([negative_txt_bf16(first_request + b, txt_tokens, cfg.txt_dim)
                              for b in range(batch)]),
            pooled_neg=np.stack([negative_pooled_bf16(first_request + b, cfg.pooled_dim)
                                 for b in range(batch)]))
    return Batch(
        img_h=img_h, img_w=img_w, txt_tokens=txt_tokens,
        latents=np.stack([latents(first_request + b, ni, cfg.in_channels) for b in range(batch)]),
        txt=np.stack([txt_embeds_bf16(first_request + b, txt_tokens, cfg.txt_dim) for b in range(batch)]),
        pooled=np.stack([pooled_bf16(first_request + b, cfg.pooled_dim) for b in range(batch)]),
        sigma=sig[k].astype(np.float32),
        sigma_next=sig[k + 1].astype(np.float32),
        guidance=np.full(batch, guidance, dtype=np.float32),
        adapter_id=adapter_ids(batch, n_adapters),
        cn_scale=np.ones(batch, dtype=np.float32),
        **neg,
    )
