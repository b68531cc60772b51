"""Summarise tools/ab_*.sh output: label, ms/step, value, K7 and K8 ms, step fraction."""
import json
import sys

name = None
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_SEM_K8.txt"):
    if not line.startswith("{"):
        name = line.strip()
        continue
    d = json.loads(line)
    r = d["roofline"]
    print(name, "step %.4f ms" % d["ms_per_step"], "%.3e" % d["value"], "K7 %.4f" % r["avg_launch_ms"],
          "K8 %.4f" % r["k8_avg_launch_ms"], "frac %.3f" % d["step_alg_frac"], d["config"]["workload"][:3])
