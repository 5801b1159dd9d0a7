"""Summarise an ncu report: key throughput metrics and the SASS opcode mix (per warp-date if given)."""
import csv, collections, io, re, subprocess, sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0  # e.g. warp-dates for per-unit counts


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__cycles_elapsed.avg.per_second"]
for k, uu, vv in zip(h, u, v):
    if k in want or any(k.startswith(w) for w in ["smsp__average_warp_latency_issue_stalled", "smsp__pcsamp_warps_issue_stalled_"]) and False:
        print(f"{k:70s} {vv} {uu}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
ix = {k: i for i, k in enumerate(hh)}
ops = collections.Counter()
samp = collections.Counter()
tot = 0
for r in src[2:]:
    m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r[ix["Source"]])
    if not m:
        continue
    ex = int(r[ix["Instructions Executed"]] or 0)
    ops[m.group(1)] += ex
    samp[m.group(1)] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += ex
print("total warp instructions", tot, "per unit", tot / norm if norm else "")
for op, c in ops.most_common(40):
    print(f"  {op:26s} {c / norm if norm else c:10.2f} {100 * c / tot:6.2f}%  samples {samp[op]}")
rows = []
for k, uu, vv in zip(h, u, v):
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            rows.append((float(vv), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in rows) or 1
print("stalls:", ", ".join(f"{k} {100 * x / tot:.1f}%" for x, k in sorted(rows, reverse=True)[:8]))
