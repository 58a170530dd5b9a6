"""One dit_step under compute-sanitizer (memcheck / racecheck / synccheck / initcheck).
usage: compute-sanitizer --tool <t> python tools/sanitize_step.py <tiny|flux_block|b16>
b16: twelve requests (B_max 16 tables, second skinny n8 group), ControlNet on slot 10.
tiny: T0-like d=32 config (mma.sync attention), 1 double + 2 single blocks, LoRA + ControlNet.
flux_block: Flux width (D=3072, 24 x 128 heads: tcgen05 GEMM + tcgen05 attention), 1 double + 1 single
block, 2 requests x (256 img + 64 txt) tokens, rank-64 LoRA on one request, ControlNet on the other;
then lora_merge (tensor-core merge kernel) and one merged step."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
if which == "b16":   # B_max 16: twelve requests, ControlNet on slot 10 (tables beyond index 8)
    cfg, B, hh, ww, nt, r = synth.TINY_SINGLE, 12, 4, 4, 8, 4
    m = SyntheticDiT(cfg, max_batch=16, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=r, max_adapters=1,
                     max_sp_world=1)
    m.register_synthetic_lora(0, rank=r, index=0)
    batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
    batch.adapter_id = np.array([0, -1] * 6, dtype=np.int32)
    lat, v = m.step(batch, controlnet={10: {0: synth.controlnet_residual_bf16(10, 0, hh * ww, cfg.hidden)}})
    torch.cuda.synchronize()
    assert np.isfinite(v).all()
    print("sanitize_step b16 ok")
    sys.exit(0)
if which == "tiny":
    cfg, B, hh, ww, nt, r = synth.TINY_SINGLE, 2, 4, 4, 8, 4
else:
    cfg, B, hh, ww, nt, r = synth.flux_reduced(1, 1), 2, 16, 16, 64, 64
m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=hh * ww, max_txt_tokens=nt, max_rank=r, max_adapters=1)
m.register_synthetic_lora(0, rank=r, index=0)
batch = synth.make_batch(cfg, B, hh, ww, nt, n_adapters=1)
batch.adapter_id = np.array([0, -1], dtype=np.int32)
res = {1: {0: synth.controlnet_residual_bf16(1, 0, hh * ww, cfg.hidden)}}
lat, v = m.step(batch, controlnet=res)
torch.cuda.synchronize()
assert np.isfinite(v).all()
# the hot-patch path too: tensor-core merge (merge_tc_kernel) + a merged step
m.lora_merge(0)
batch.adapter_id = np.array([0, 0], dtype=np.int32)
lat2, v2 = m.step(batch)
m.lora_unmerge()
torch.cuda.synchronize()
assert np.isfinite(v2).all()
print(which, "ok", float(np.abs(v).max()), float(np.abs(v2).max()))
