"""Freeze the roofline inputs of the dominant kernel from an ncu --set full capture.

usage: roofline_inputs.py report.ncu-rep n_paths m_dates out.json summary.txt
Counts the executed FP64-pipe SASS instructions (DFMA/DADD/DMUL/DSETP/...)
per path-step (thread-level: warp instructions x active lanes), and the DRAM
bytes per launch, and writes a human-readable summary next to them."""
import csv, io, json, re, subprocess, sys

rep, n, m, out_json, out_txt = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
R = {k: (vv, uu) for k, uu, vv in zip(h, u, v)}


def val(k, scale=1.0):
    x, unit = R[k]
    x = float(x)
    unit = unit.strip().lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
            "ms": 1e-3, "msecond": 1e-3, "s": 1, "second": 1}.get(unit, 1)
    return x * mult * scale


src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
ix = {k: i for i, k in enumerate(hh)}
fp64_thread = 0
fp64_warp = 0
total_warp = 0
for r in src[2:]:
    mm = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", r[ix["Source"]])
    if not mm:
        continue
    op = mm.group(1)
    ex = int(r[ix["Instructions Executed"]] or 0)
    th = int(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
    total_warp += ex
    if re.match(r"D(FMA|ADD|MUL|SETP|MNMX)", op):
        fp64_warp += ex
        fp64_thread += th
path_steps = n * m
dur = val("gpu__time_duration.sum")
dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
doc = {"kernel": "price_kernel (K2)", "report": rep.split("/")[-1], "n_paths": n, "m_dates": m,
       "fp64_inst_per_path_step": fp64_warp * 32 / path_steps,
       "fp64_thread_inst_per_path_step": fp64_thread / path_steps,
       "warp_inst_per_warp_date": total_warp / (path_steps / 32),
       "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": 8 * path_steps, "algorithmic_bytes_per_path_step": 8,
       "duration_ms_under_ncu": dur * 1e3,
       "note": "fp64_inst_per_path_step counts FP64-pipe warp instructions x 32 lanes (issue slots the "
               "roofline charges); the thread-level count excludes predicated-off lanes"}
json.dump(doc, open(out_json, "w"), indent=1)
summ = subprocess.run([sys.executable, "tools/ncu_summary.py", rep, str(path_steps / 32)], capture_output=True,
                      text=True).stdout
with open(out_txt, "w") as f:
    f.write(f"# ncu --set full, {rep.split('/')[-1]}: price_kernel at {n} paths x {m} dates (one launch)\n")
    f.write(json.dumps(doc, indent=1) + "\n\n# per warp-date opcode mix and key metrics\n" + summ)
print(json.dumps(doc, indent=1))
