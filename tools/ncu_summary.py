"""Key metrics of an ncu --set full report (one or more launches) as text."""
import csv, subprocess, sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warp_latency_issue_stalled_barrier",
        "smsp__average_warp_latency_issue_stalled_short_scoreboard",
        "smsp__average_warp_latency_issue_stalled_math_pipe_throttle"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        for w in WANT:
            if w in h:
                i = h.index(w)
                val = v[i] if w != "Kernel Name" else v[i][:90]
                print(f"{w:65s} {val} {u[i] if w != 'Kernel Name' else ''}")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
