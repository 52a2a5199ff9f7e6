"""Key raw metrics (and the large stall reasons) of every kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[0]
want = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    print("----", r[h.index("Kernel Name")][:110])
    for k in want:
        if k in h:
            print(f"  {k} = {r[h.index(k)]}")
    for i, name in enumerate(h):
        if "warp_issue_stalled" in name and name.endswith("per_warp_active.pct"):
            try:
                if float(r[i]) > 8:
                    print("   stall", name.split("stalled_")[1].split("_per")[0], r[i])
            except ValueError:
                pass
