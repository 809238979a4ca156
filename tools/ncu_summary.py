"""Key metrics + warp stall breakdown from an ncu report (run here, no GPU needed).
usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[hdr.index("Kernel Name")][:100])
        d = dict(zip(hdr, r))
        for k in KEYS:
            if k in d:
                print(f"  {k:65s} {d[k]:>16s} {units[hdr.index(k)]}")
        # warp-state samples (pc sampling), as a share of all samples
        stalls = [(k[len("smsp__pcsamp_warps_issue_stalled_"):], float(d[k].replace(',', '') or 0)) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        stalls.sort(key=lambda x: -x[1])
        print("  warp stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in stalls[:8]))
        for k in ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active"):
            if k in d:
                print(f"  {k:65s} {d[k]:>16s} {units[hdr.index(k)]}")


if __name__ == "__main__":
    main(sys.argv[1])
