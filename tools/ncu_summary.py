"""Summarise an ncu report: key metrics + top source lines by stall samples (dev tool)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "lts__t_sectors_op_read.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_membar_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for d in rows[2:]:
        name = d[hdr.index("Kernel Name")][:90]
        print("==", name)
        for k in KEYS:
            if k in hdr:
                print(f"   {k:70s} {d[hdr.index(k)]:>16s} {units[hdr.index(k)]}")


def source(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return
    hdr = rows[0]
    def col(name):
        for i, h in enumerate(hdr):
            if h.startswith(name):
                return i
        return None
    si = col("Warp Stall Sampling (All")
    li, ci = col("Line"), col("Source")
    if si is None:
        print("no stall column", hdr[:10]); return
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[si] or 0), r[li], r[ci][:110]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    for s, l, c in sorted(data, reverse=True)[:top]:
        print(f"  {100*s/tot:5.1f}%  L{l:>5s}  {c}")


if __name__ == "__main__":
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        source(sys.argv[1], int(sys.argv[2]))
