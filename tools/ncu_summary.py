# Summarise ncu --set full captures (ncu -i ... --page raw --csv) into one text table.
import csv, io, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64cyc_%"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
]


def summarize(path):
    names = ",".join(m for m, _ in METRICS)
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", names],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = []
    for r in rows[2:]:
        lines.append(f"kernel: {r[idx['Kernel Name']]}")
        for m, short in METRICS:
            if m in idx and r[idx[m]] != "":
                lines.append(f"  {short:14s} {r[idx[m]]:>14s} {units[idx[m]]}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    for p in sys.argv[1:]:
        sys.stdout.write(f"== {p}\n" + summarize(p))
