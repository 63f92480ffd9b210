"""Summarise an ncu report: per-kernel time, DRAM bytes, throughputs, stalls."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_confl"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavef"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall_lsb"),
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for d in data:
        name = d[hdr.index("Kernel Name")]
        print(name[:70])
        for key, short in WANT:
            if key in hdr:
                i = hdr.index(key)
                print(f"    {short:12s} {d[i]:>16s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
