"""Projected Ulysses-SP scaling from measured one-GPU components (a model, not a measurement: gpurun
gives one GPU).  For P ranks, one rank's step =
  (a) every per-token kernel at the rank's share of the tokens -- MEASURED: a one-GPU dit_step on a
      batch shaped like one rank's shard (img Ni/P, txt Nt/P tokens per request, same B / adapters),
      minus that step's own (local, all-head) attention;
  (b) attention of H/P heads over the FULL joint sequence -- MEASURED alone
      (dit_debug_attention) and scaled by the in-step / alone ratio of the P = 1 attention
      (both the in-step kernel and the alone kernel run at their own power-capped clocks);
  (c) the exchange: 4 bf16 [rows/P x D] tensors per block leave each rank ((P-1)/P of them to
      peers), fused into the QKV / attention epilogues -- bounded by 0 (hidden under the
      epilogues' math) and bytes / 770 GB/s (the measured NVLink peer copy of
      B200_PROFILING.md) + 2 flag barriers per block at 5 us each.
Efficiency = T_1 / (P * T_P) for both bounds.
usage: python tools/sp_projection.py [--workload cfg3] [--steps 5]"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2604_08123_b200 import SyntheticDiT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3", choices=["cfg2", "cfg3", "cfg5"])
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
wl = bench.WORKLOADS[args.workload]
cfg = synth.FLUX
B, H_, W_, NT, n_ad = wl["B"], wl["h"], wl["w"], wl["nt"], wl["adapters"]
D, HEADS, d = cfg.hidden, cfg.heads, cfg.hidden // cfg.heads
N = H_ * W_ + NT
blocks = cfg.depth_double + cfg.depth_single
lib = None


def timed_step(h, w, nt):
    m = SyntheticDiT(cfg, max_batch=B, max_img_tokens=h * w, max_txt_tokens=nt, max_rank=64 if n_ad else 0,
                     max_adapters=n_ad, max_sp_world=1)
    for a in range(n_ad):
        m.register_synthetic_lora(a, rank=64, index=a)
    batch = synth.make_batch(cfg, B, h, w, nt, n_adapters=n_ad)
    lat, txt, pooled, out, v = m.device_inputs(batch)
    cb = m.make_batch(B, h, w, nt, batch.adapter_id, batch.sigma, batch.sigma_next, batch.guidance, lat, out, txt,
                      pooled, v_out=None)
    for _ in range(3):
        m.dit_step(cb)
    torch.cuda.synchronize()
    m.profile_reset()
    m.profile(True)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.steps):
        m.dit_step(cb)
    e1.record(s)
    torch.cuda.synchronize()
    m.profile(False)
    ms = e0.elapsed_time(e1) / args.steps
    attn = m.profile_read(1)[0] / args.steps
    global lib
    lib = m.lib
    m.close()
    del m
    torch.cuda.empty_cache()
    return ms, attn


def attn_alone(heads):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(B, heads, N, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty(B * N, heads * d, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    call = lambda: lib.dit_debug_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), B, heads, N, d, o.data_ptr(),
                                           C.c_void_p(s.cuda_stream))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        call()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


shards = {1: (H_, W_), 2: (H_ // 2, W_), 4: (H_ // 2, W_ // 2), 8: (H_ // 4, W_ // 2)}
res = {}
t1, a1_step = timed_step(H_, W_, NT)
a1_alone = attn_alone(HEADS)
ratio = a1_step / (blocks * a1_alone)          # in-step / alone, per launch
res[1] = dict(step_ms=t1, attn_ms=a1_step)
for P in (2, 4, 8):
    h, w = shards[P]
    tl, al = timed_step(h, w, NT // P)
    ap_ = attn_alone(HEADS // P) * blocks * ratio
    rows = B * (h * w + NT // P)
    xbytes = blocks * 4 * rows * D * 2 * (P - 1) / P
    x_hi = xbytes / 770e9 * 1e3 + 2 * blocks * 5e-3
    lo, hi = tl - al + ap_, tl - al + ap_ + x_hi
    res[P] = dict(rank_local_step_ms=tl, local_attn_ms=al, full_seq_attn_ms=ap_, exchange_gb=xbytes / 1e9,
                  exchange_bound_ms=x_hi, step_ms=[lo, hi], efficiency=[t1 / (P * hi), t1 / (P * lo)])
out = {"workload": args.workload, "model": "projection from measured one-GPU components (tools/sp_projection.py "
       "docstring); efficiency = T1 / (P * TP), [exchange fully exposed, fully hidden]",
       "attn_instep_over_alone": ratio, "by_P": res}
print(json.dumps(out, indent=1))
