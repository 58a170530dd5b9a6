"""SyntheticDiT: a DiT context loaded with the seeded synthetic Flux-shaped
weights (synth.weight_manifest, generated ON DEVICE by dit_fill_synthetic),
plus helpers that move a synth.Batch to the device and run dit_step.

Used by bench.py, smoke() and the GPU tests.  Marshalling only.
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from .dit import DiT, fill_synthetic


def _bits_to_bf16_tensor(bits: np.ndarray, device):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)
    return t.to(device)


class SyntheticDiT(DiT):
    def __init__(self, cfg, max_batch, max_img_tokens, max_txt_tokens, max_rank=0, max_adapters=0, device=0,
                 seed: Optional[int] = None, max_sp_world=0):
        import torch
        import synth
        super().__init__(cfg, max_batch, max_img_tokens, max_txt_tokens, max_rank, max_adapters, device, max_sp_world)
        seed = synth.WEIGHT_SEED if seed is None else seed
        dev = f"cuda:{device}"
        ws = {}
        for spec in synth.weight_manifest(cfg):
            t = torch.empty(spec.shape, dtype=torch.bfloat16, device=dev)
            fill_synthetic(t, seed, spec.tensor_id, spec.scale, spec.offset)
            ws[spec.name] = t
        self.dit_load_weights(ws)
        self.dev = dev

    def register_synthetic_lora(self, adapter_id: int, rank: int, index: int, scale: float = 1.0):
        import torch
        import synth
        tens = {}
        for spec in synth.lora_manifest(self.cfg, rank, index):
            t = torch.empty(spec.shape, dtype=torch.bfloat16, device=self.dev)
            fill_synthetic(t, 3000 + index, spec.tensor_id, spec.scale, spec.offset)
            tens[spec.name] = t
        self.lora_register(adapter_id, rank, scale, tens)
        torch.cuda.current_stream().synchronize()

    def device_inputs(self, batch, lp_rank: Optional[int] = None):
        """Device copies of a synth.Batch.  CFG (batch.cfg_scale set): txt / pooled hold the
        conditional rows then the unconditional rows ([2B]); under latent parallelism
        (lp_rank given) only this rank's branch ([B]: rank 0 conditional, 1 unconditional)."""
        import torch
        lat = torch.from_numpy(np.ascontiguousarray(batch.latents, dtype=np.float32)).to(self.dev)
        txt_bits, pooled_bits = batch.txt, batch.pooled
        if batch.cfg_scale is not None:
            if lp_rank is None:
                txt_bits = np.concatenate([batch.txt, batch.txt_neg])
                pooled_bits = np.concatenate([batch.pooled, batch.pooled_neg])
            elif lp_rank == 1:
                txt_bits, pooled_bits = batch.txt_neg, batch.pooled_neg
        txt = _bits_to_bf16_tensor(txt_bits, self.dev)
        pooled = _bits_to_bf16_tensor(pooled_bits, self.dev)
        out = torch.empty_like(lat)
        v = torch.empty_like(lat)
        return lat, txt, pooled, out, v

    def step(self, batch, controlnet: Optional[Dict[int, Dict[int, np.ndarray]]] = None, n_res: int = 0,
             injections=None, lp_rank: Optional[int] = None, sync: bool = True):
        """Run one dit_step on a synth.Batch; returns (latents_out, v) as numpy fp32.

        controlnet: request b -> {double block i -> residual bf16 bits [Ni, D]} (one
        residual per block; n_res mapping is the caller's business).
        injections: further (request b, block, residual bits [Ni, D], scale) tuples; block
        counts double blocks then single blocks (controlnet_inject's numbering).
        """
        import torch
        lat, txt, pooled, out, v = self.device_inputs(batch, lp_rank)
        if controlnet:
            for b, d in controlnet.items():
                for blk, bits in d.items():
                    self.controlnet_inject(b, blk, _bits_to_bf16_tensor(bits, self.dev), 1.0)
        for b, blk, bits, sc in (injections or []):
            self.controlnet_inject(b, blk, _bits_to_bf16_tensor(bits, self.dev), sc)
        cb = self.make_batch(batch.batch, batch.img_h, batch.img_w, batch.txt_tokens, batch.adapter_id,
                             batch.sigma, batch.sigma_next, batch.guidance, lat, out, txt, pooled, v_out=v,
                             cn_scale=batch.cn_scale, cfg_scale=batch.cfg_scale, img_hw=batch.img_hw)
        self.dit_step(cb)
        if not sync:   # (latent-parallel tests: the peer rank's thread must also have enqueued)
            return out, v
        torch.cuda.current_stream().synchronize()
        self._keep.clear()
        return out.cpu().numpy(), v.cpu().numpy()
