"""One-screen summary of a bench.py JSON line (the last line of the file given)."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]).read().splitlines() if ln.startswith("{")][-1])
print("value %.4g %s  ms/step %.3f  kernel %.3f  step %.3f  launches %s" % (
    d["value"], d["unit"], d["ms_per_step"], d["kernel_ms"] or -1, d["device_step_ms"] or -1, d["gpu_launches"]))
print("price", d["price"], "se", d["std_error"], "n_gpus", d["n_gpus"])
print("e2e", {k: v for k, v in d["e2e"].items() if k != "api"})
print("cold", {k: v for k, v in d["cold"].items() if k != "note"})
print("put", d["put"])
r = d["roofline"] or {}
print("roofline frac %.3f issue %.3f hbm %.3f" % (r.get("frac", 0), r.get("issue", {}).get("frac", 0),
                                                  r.get("hbm", {}).get("frac", 0)))
print("cpu", d["cpu_baseline"])
print("c4", {k: v for k, v in (d["batch_config4"] or {}).items() if k != "workload"})
print("c5", {k: v for k, v in (d["stress_config5"] or {}).items() if k != "workload"})
print("clocks", d["clocks"])
