"""Run warm-up + N dit_steps of a bench workload (for ncu); no timing printed.
usage: python tools/profile_step.py [--workload cfg3] [--steps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--workload", default="cfg3", choices=sorted(bench.WORKLOADS))
args = ap.parse_args()
wl = bench.WORKLOADS[args.workload]
cfg = getattr(synth, wl.get("model", "FLUX"))
B, H_, W_, NT, n_ad = wl["B"], wl["h"], wl["w"], wl["nt"], wl["adapters"]
seqs = 2 * B if wl.get("cfg") is not None else B
m = SyntheticDiT(cfg, max_batch=seqs, max_img_tokens=H_ * W_, max_txt_tokens=NT, max_rank=64 if n_ad else 0,
                 max_adapters=n_ad)
for a in range(n_ad):
    m.register_synthetic_lora(a, rank=64, index=a)
batch = synth.make_batch(cfg, B, H_, W_, NT, n_adapters=n_ad, cfg_scale=wl.get("cfg"))
lat, txt, pooled, out, v = m.device_inputs(batch)
cb = m.make_batch(B, H_, W_, NT, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance,
                  lat, out, txt, pooled, cfg_scale=batch.cfg_scale)
res = None
if wl["cn"]:
    from paper_2604_08123_b200.dit import fill_synthetic
    res = torch.empty(B, cfg.depth_double, H_ * W_, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    fill_synthetic(res, 4000, 0, 0.1 * 3 ** 0.5, 0.0)
for _ in range(args.steps):
    if res is not None:
        for bb in range(B):
            for i in range(cfg.depth_double):
                m.controlnet_inject(bb, i, res[bb, i])
    m.dit_step(cb)
torch.cuda.synchronize()
print("launches per step", m.last_launch_count())
