"""Write profiles/ncu_summary.json (read by bench.py for roofline.traffic) from ncu --set full
captures of one bench step: one report per workload, its P2P launches in config order.

  python tools/ncu_traffic_json.py KEY REPORT CONFIG[,CONFIG...] [REPORT CONFIGS ...]
  e.g. python tools/ncu_traffic_json.py tiled_fp32 gpurun_out/r01_step_full.ncu-rep d16_1e6,d32_1e6,d64_1e6
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import src_sha16  # noqa: E402  (run it in the same gpurun call as the capture)
OUT = os.path.join(ROOT, "profiles", "ncu_summary.json")
FIELDS = {"dram_bytes_read": "dram__bytes_read.sum", "dram_bytes_write": "dram__bytes_write.sum",
          "duration_us_ncu": "gpu__time_duration.sum",
          "xu_pct_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "issue_pct_active": "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "dram_pct_elapsed": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex_pct_active": "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "shared_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second"}
SCALE = {"dram_bytes_read": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "dram_bytes_write": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "duration_us_ncu": {"ns": 1e-3, "us": 1, "ms": 1e3},
         "sm_clock_ghz": {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1}}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main(argv):
    key, pairs = argv[0], argv[1:]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for rep, names in zip(pairs[0::2], pairs[1::2]):
        hdr, units, launches = rows(rep)
        idx = {h: i for i, h in enumerate(hdr)}
        names = names.split(",")
        assert len(launches) >= len(names), (rep, len(launches), names)
        for name, r in zip(names, launches):
            ent = {"kernel": r[idx["Kernel Name"]], "report": os.path.basename(rep), "src_sha16": src_sha16()}
            for f, m in FIELDS.items():
                if m in idx and r[idx[m]] not in ("", "n/a"):
                    v = float(r[idx[m]].replace(",", ""))
                    ent[f] = v * SCALE.get(f, {}).get(units[idx[m]], 1)
            ent["dram_bytes"] = ent.get("dram_bytes_read", 0) + ent.get("dram_bytes_write", 0)
            data.setdefault(name, {})[key] = ent
            print(name, key, {k: round(v, 3) if isinstance(v, float) else v for k, v in ent.items()})
    json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
