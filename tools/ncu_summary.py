"""Summarise an ncu --set full report: key throughput metrics, stall reasons, top stall SASS lines."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep):
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    for r in data:
        print("kernel:", r[idx["Kernel Name"]][:90])
        for k in KEYS:
            if k in idx:
                print(f"  {k:75s} {r[idx[k]]:>16s} {units[idx[k]]}")
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[i]))
              for h, i in idx.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("ratio")]
        st.sort(key=lambda x: -x[1])
        print("  stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for n, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
