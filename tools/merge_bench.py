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

# in-place hot patch: count + patch passes (host waits for the count), then the exact restore
import time  # noqa: E402
for sc, tag in ((1.0, "synthetic rank-64 adapter (|sBA| ~ 0.5 |W| rms)"), (0.1, "scale 0.1 (|sBA| ~ 0.05 |W| rms)")):
    m.lora_unregister(0)
    m.register_synthetic_lora(0, rank=64, index=0, scale=sc)
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in list(m.weights.items()) if k.startswith("double.0.img")}
    n = m.lora_merge_inplace(0, undo=None)     # sizes the log (allocation outside the timing)
    undo = m._undo
    m.lora_unmerge()
    tm, tu = [], []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = m.lora_merge_inplace(0, undo=undo)
        torch.cuda.synchronize()
        tm.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        m.lora_unmerge()
        tu.append(time.perf_counter() - t0)
    ok = all(torch.equal(m.weights[k], v) for k, v in ref.items())
    elems = nbytes // 4
    print(f"in-place merge [{tag}]: merge {min(tm) * 1e3:.1f} ms (count pass + host readback + patch, log preallocated), "
          f"unmerge {min(tu) * 1e3:.1f} ms; undo log {n} entries = {n * 8 / 1e9:.2f} GB "
          f"({100 * n / elems:.2f}% of {elems / 1e9:.2f} G weights; a merged copy would be {elems * 2 / 1e9:.1f} GB); "
          f"restore exact on double.0.img: {ok}")
