"""Merged-LoRA mode at Flux-Dev size on one B200:
  * lora_merge time for one rank-64 adapter over every adapted linear (HBM-bound: 2 B read + 2 B
    written per weight), against the measured HBM copy bandwidth;
  * dit_step speed for a single-adapter batch, segmented (unmerged) vs merged, at B=1 and B=8.
Prints one JSON object (kept under profiles/)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

cfg = synth.FLUX
out = {"config": "Flux-Dev 19+38 blocks, D=3072, 1024^2 (4096 img + 512 txt tokens), one rank-64 adapter"}
for B in (1, 8):
    m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=4096, max_txt_tokens=512, max_rank=64, max_adapters=1)
    m.register_synthetic_lora(0, rank=64, index=0)
    batch = synth.make_batch(cfg, B, 64, 64, 512, n_adapters=1)
    batch.adapter_id = np.zeros(B, dtype=np.int32)
    lat, txt, pooled, o, v = m.device_inputs(batch)
    cb = m.make_batch(B, 64, 64, 512, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, o, txt,
                      pooled)

    def timed(n, warm=3):
        for _ in range(warm):
            m.dit_step(cb)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            m.dit_step(cb)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    n = 5 if B == 8 else 10
    ms_unmerged = timed(n)
    buf = torch.empty(m.merge_bytes() + 256, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    merge_ms = []
    for _ in range(3):
        e0.record()
        m.lora_merge(0, merged=buf)
        e1.record()
        torch.cuda.synchronize()
        merge_ms.append(e0.elapsed_time(e1))
        m.lora_unmerge()
    m.lora_merge(0, merged=buf)
    ms_merged = timed(n)
    m.lora_unmerge()
    nbytes = 2 * m.merge_bytes()          # read W, write W' (the rank-64 factors are 0.4% on top)
    out[f"B{B}"] = {"step_ms_unmerged": ms_unmerged, "step_ms_merged": ms_merged,
                    "speedup": ms_unmerged / ms_merged, "merge_ms": min(merge_ms),
                    "merge_GBps": nbytes / (min(merge_ms) / 1e3) / 1e9, "merge_bytes": nbytes}
    del m, buf
    torch.cuda.empty_cache()
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    out["hbm_peak_GBps"] = peaks.get("hbm_gbs")
except Exception:
    pass
print(json.dumps(out))
