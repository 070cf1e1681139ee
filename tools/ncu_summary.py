"""Summarise an ncu report (raw page) for our kernels: one line per launch."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us", None),  # unit-aware (ncu reports ns / us / ms)
    ("dram__bytes_read.sum", "rdMB", None),
    ("dram__bytes_write.sum", "wrMB", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("smsp__inst_executed.sum", "Minst", 1e-6),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%", 1),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smemWF_M", 1e-6),
    ("launch__registers_per_thread", "regs", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st_lsb", 1),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st_bar", 1),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st_ssb", 1),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st_mio", 1),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "st_lg", 1),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "st_wait", 1),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "st_math", 1),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "st_nsel", 1),
    ("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio", "st_sel", 1),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "st_disp", 1),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "st_membar", 1),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "st_sleep", 1),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "st_drain", 1),
]


def main(path, filt="_kernel"):
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    for r in rows[2:]:
        if filt not in r[ki]:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        vals = []
        for key, short, scale in KEYS:
            if key in hdr:
                v = r[hdr.index(key)]
                try:
                    f = float(v.replace(",", ""))
                    if scale is None:
                        u = units[hdr.index(key)]
                        f *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                              "msecond": 1e3, "s": 1e6, "second": 1e6,
                              "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    else:
                        f *= scale
                    vals.append(f"{short}={f:.4g}")
                except ValueError:
                    pass
        print(name[:60], " ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
