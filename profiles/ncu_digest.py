"""Digest an ncu --set full report: key throughput / occupancy / stall metrics
per kernel.  Usage: python profiles/ncu_digest.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = [
    ("time_ms", "gpu__time_duration.sum"),
    ("dram_rd_GB", "dram__bytes_read.sum"),
    ("dram_wr_GB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("block", "launch__block_size"),
    ("smem_dyn", "launch__shared_mem_per_block_dynamic"),
    ("occ_lim_reg", "launch__occupancy_limit_registers"),
    ("occ_lim_smem", "launch__occupancy_limit_shared_mem"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("ipc", "sm__inst_executed.avg.per_cycle_active"),
    ("inst", "smsp__inst_executed.sum"),
    ("fp64_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("lsu_smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_bank_conf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("local_ld_sectors", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"),
    ("st_long_sb", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("st_short_sb", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("st_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
    ("st_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
    ("st_mio", "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"),
    ("st_lg_throttle", "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"),
    ("st_math", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"),
    ("st_drain", "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio"),
    ("st_membar", "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio"),
]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        print("---", name)
        for short, m in WANT:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {short:20s} {r[i]} {units[i]}")


if __name__ == "__main__":
    main()
