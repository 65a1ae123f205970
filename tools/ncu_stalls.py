"""Print the top issue-stall reasons, pipe utilisation and DRAM bytes of each kernel in an ncu report
(ncu -i REP --page raw --csv).  Usage: python tools/ncu_stalls.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
h = next(r)
next(r)
for row in r:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:60], "grid", d.get("launch__grid_size"), "dur(us)", d.get("gpu__time_duration.sum"))
    st = []
    for x in h:
        if x.startswith("smsp__average_warps_issue_stalled_") and x.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[x]), x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("   stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for v, n in st[:7]))
    for m in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
        if m in d:
            print("   ", m, d[m])
