"""bench.py's contract pieces that need no GPU: every workload names known configs, the
reference arm prints one JSON line with the required keys (tiny workload, short budget)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2403_01596_b200 import workloads as W  # noqa: E402


def test_workloads_name_known_configs():
    for wl, names in bench.WORKLOADS.items():
        for n in names:
            assert n in W.CONFIGS, (wl, n)
    for wl in bench.DEFAULT_KERNEL:
        assert wl in bench.WORKLOADS


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "tiny",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_defaults_measure_the_headline():
    """The driver runs bench.py with no flags: the workload must be BASELINE.json configs[3] (the
    configuration its metric is quoted on at 1/2/4/8 B200), strong scaling for N > 1, and the
    roofline denominators must come from the committed measurement."""
    sys.argv = ["bench.py"]
    a = bench.parse()
    assert a.workload == "surface_2e7" and bench.WORKLOADS[a.workload] == ["surf_2e7"]
    assert a.scaling == "strong" and a.exchange == "auto" and a.layout == "tiled" and a.precision == "fp32"
    peaks = json.load(open(bench.PEAKS_JSON))
    assert 14.0 < peaks["mufu_lg2"]["per_clk_per_sm"] < 17.0 and 50.0 < peaks["dfma"]["per_clk_per_sm"] / 2 < 70.0
    assert bench.MUFU_LG2_PER_CLK_PER_SM == peaks["mufu_lg2"]["per_clk_per_sm"]
    assert "profiles/r02_peaks.json" in bench.PEAK_BASIS
    assert len(bench.src_sha16()) == 16 and bench.src_sha16() == bench.src_sha16()
