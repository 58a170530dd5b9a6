"""Summarise ncu outputs (launch list CSV and --set full reports) into markdown."""
import collections
import csv
import io
import subprocess
import sys


def launch_list(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].split("<")[0]
        if k.endswith("fill_synth_kernel"):   # synthetic weight generation (setup, not part of a step)
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {sum(v[0] for v in agg.values())}, summed device time {tot:.1f} ms (ncu, serialised, cold-cache)",
           "", "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {n} | {ms:.2f} | {100 * ms / tot:.1f}% |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def full_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    out = []
    for row in r[2:]:
        name = row[h.index("Kernel Name")]
        out.append(f"### {name}")
        out.append("| metric | value |")
        out.append("|---|---|")
        for i, n in enumerate(h):
            for w in WANT:
                if n == w or n.endswith("." + w) or n.endswith(w):
                    out.append(f"| {n} | {row[i]} {units[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launch_list(path) if kind == "list" else full_report(path))
