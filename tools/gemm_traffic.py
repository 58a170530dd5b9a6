"""Parse an ncu CSV (gemm launches of 2 dit_steps, metrics dram bytes / duration / tensor active) and
write profiles/gemm_traffic.json: DRAM bytes per GEMM launch of the second (warm) step, overall and
per GEMM type (types recovered from the launch order of one step).
usage: python tools/gemm_traffic.py gpurun_out/gemm_traffic.csv <workload> [lora 0/1] [Ld Ls]
writes profiles/gemm_traffic_<workload>.json"""
import collections
import csv
import io
import json
import os
import sys

path = sys.argv[1]
workload = sys.argv[2] if len(sys.argv) > 2 else "cfg3"
lora = int(sys.argv[3]) if len(sys.argv) > 3 else (1 if workload == "cfg3" else 0)
Ld, Ls = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (19, 38)
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
per = collections.OrderedDict()
for r in rows:
    if "gemm" not in r["Kernel Name"]:
        continue
    k = int(r["ID"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
             "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1.0)
    per.setdefault(k, {})[r["Metric Name"]] = v * scale
ids = list(per.keys())
n = len(ids) // 2
step2 = [per[i] for i in ids[n:]]
# launch order of one step (LoRA on): embed, per double block [shrink qkv, qkv, shrink proj, proj,
# shrink fc1, fc1, shrink fc2, fc2], per single block [shrink l1, l1, shrink l2, l2], final
if lora:
    names = ["embed"] + ["shrink", "dbl_qkv", "shrink", "dbl_proj", "shrink", "dbl_fc1", "shrink", "dbl_fc2"] * Ld + \
            ["shrink", "sgl_linear1", "shrink", "sgl_linear2"] * Ls + ["final"]
else:
    names = ["embed"] + ["dbl_qkv", "dbl_proj", "dbl_fc1", "dbl_fc2"] * Ld + ["sgl_linear1", "sgl_linear2"] * Ls + \
            ["final"]
out = {"source": os.path.basename(path), "workload": workload, "launches": len(step2)}
if len(names) == len(step2):
    by = collections.defaultdict(list)
    for nm, m in zip(names, step2):
        by[nm].append(m)
    out["by_type"] = {nm: {"launches": len(v),
                           "dram_bytes_per_launch": sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in v) / len(v),
                           "ms_per_launch": sum(x.get("gpu__time_duration.sum", 0) for x in v) / len(v),
                           "tensor_active_pct": sum(x.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) for x in v) / len(v)}
                      for nm, v in by.items()}
else:
    out["note"] = f"launch count {len(step2)} != expected {len(names)}; per-type split skipped"
tot = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in step2)
out["bytes_per_launch"] = tot / max(1, len(step2))
out["bytes_per_step"] = tot
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"gemm_traffic_{workload}.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
