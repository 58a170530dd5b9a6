"""Run warm-up + N dit_steps of the bench workload (for ncu); no timing printed."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--adapters", type=int, default=4)
args = ap.parse_args()
cfg = synth.FLUX
B, n_ad = args.batch, args.adapters
m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=4096, max_txt_tokens=512, max_rank=64 if n_ad else 0,
                 max_adapters=n_ad)
for a in range(n_ad):
    m.register_synthetic_lora(a, rank=64, index=a)
batch = synth.make_batch(cfg, B, 64, 64, 512, n_adapters=n_ad)
lat, txt, pooled, out, v = m.device_inputs(batch)
cb = m.make_batch(B, 64, 64, 512, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance,
                  lat, out, txt, pooled)
for _ in range(args.steps):
    m.dit_step(cb)
torch.cuda.synchronize()
print("launches per step", m.last_launch_count())
