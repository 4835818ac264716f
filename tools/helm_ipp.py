"""Thread-instructions per pair of the Helmholtz kernel from ncu captures of tools/helm_bench.py
(one file per precision: the JSON row gives the pair count, ncu's smsp__thread_inst_executed.sum
the instructions of each launch) -> profiles/helm_inst_per_pair.json (bench.py's roofline).

  python tools/helm_ipp.py fp32=gpurun_out/helm_ncu_fp32.txt fp64=gpurun_out/helm_ncu_fp64.txt
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {}
for arg in sys.argv[1:]:
    prec, path = arg.split("=", 1)
    text = open(path).read()
    pairs = [json.loads(l)["pairs"] for l in text.splitlines() if l.startswith("{")][0]
    inst = [float(m) for m in re.findall(r"smsp__thread_inst_executed\.sum\s+inst\s+([0-9.]+)", text)]
    out[prec] = round(min(inst) / pairs, 2)
    out[prec + "_source"] = f"{os.path.basename(path)}: min over {len(inst)} launches / {pairs} pairs"
with open(os.path.join(ROOT, "profiles", "helm_inst_per_pair.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out)
