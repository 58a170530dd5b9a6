"""lora_merge alone at Flux-Dev size (one rank-64 adapter over every adapted linear): ms and
GB/s (2 B read + 2 B written per merged weight) -- for merge-kernel variants (DIT_LIB_OVERRIDE)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

m = SyntheticDiT(synth.FLUX, max_batch=1, max_img_tokens=256, max_txt_tokens=64, max_rank=64, max_adapters=1)
m.register_synthetic_lora(0, rank=64, index=0)
buf = torch.empty(m.merge_bytes() + 256, dtype=torch.uint8, device="cuda")
nbytes = sum(fi * fo for _, fi, fo in synth.lora_targets(synth.FLUX)) * 4
ts = []
for _ in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    m.lora_merge(0, buf)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    m.lora_unmerge()
print(f"merge: {min(ts):.2f} ms  {nbytes / min(ts) / 1e6:.0f} GB/s  ({nbytes / 1e9:.1f} GB)")
