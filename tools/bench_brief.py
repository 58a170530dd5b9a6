import json, sys
d = json.load(open(sys.argv[1]))
k = d["kernels"]
print(f"steps/s {d['value']:.4f}  {d['pct_bf16_peak']:.1f}% peak  clocks {d['clocks']}")
print("attention", {x: round(y, 1) if y else y for x, y in k["attention"].items()}, " gemm", round(k["gemm"]["ms_per_step"], 1),
      round(k["gemm"]["tflops"]), " lnmod", round(k["lnmod"]["ms_per_step"], 1))
print({a: (round(b["ms_per_step"], 1), b["tflops"] and round(b["tflops"])) for a, b in k["gemm_by_type"].items()})
