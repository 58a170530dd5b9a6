"""Test helpers: build oracle inputs from the synth module (test-only)."""
from __future__ import annotations

import numpy as np

import synth
from oracle import OracleLoRA
from oracle.flux_step import bf16_to_f64


def oracle_adapter(cfg, rank: int, index: int, scale: float = 1.0, zero_b: bool = False):
    bits = synth.make_lora_bf16(cfg, rank, index)
    mats = {}
    for mod, _, _ in synth.lora_targets(cfg):
        a = bf16_to_f64(bits[mod + ".lora_A"])
        b = bf16_to_f64(bits[mod + ".lora_B"])
        if zero_b:
            b = np.zeros_like(b)
        mats[mod] = (a, b)
    return OracleLoRA(scale=scale, mats=mats), bits


def torch_adapter(bits, cfg, scale=1.0):
    return (scale, {mod: (bits[mod + ".lora_A"], bits[mod + ".lora_B"])
                    for mod, _, _ in synth.lora_targets(cfg)})


def residuals(cfg, batch_size: int, ni: int, n_res: int, requests=None):
    """b -> {res index: R fp64 (bf16-rounded)} for the requests listed (default all)."""
    reqs = range(batch_size) if requests is None else requests
    return {b: {i: bf16_to_f64(synth.controlnet_residual_bf16(b, i, ni, cfg.hidden)) for i in range(n_res)}
            for b in reqs}


def max_rel(g, o):
    """max|G-O| / max|O|."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    return float(np.abs(g - o).max() / max(np.abs(o).max(), 1e-300))


def cosine(g, o):
    g = np.asarray(g, dtype=np.float64).ravel()
    o = np.asarray(o, dtype=np.float64).ravel()
    return float(g @ o / (np.linalg.norm(g) * np.linalg.norm(o) + 1e-300))
