"""One block per kernel of an ncu --set full report: time, throughput, occupancy,
DRAM traffic and the top stall reasons (what profiles/*_kernels.txt holds)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    name = d.get("Kernel Name", "?").replace("(anonymous namespace)::", "").split("(")[0]
    print(f"== {name}")
    for k, label in KEYS:
        if k in d and d[k] not in ("", "n/a"):
            print(f"  {label:22s} {d[k]} {u.get(k, '')}")
    st = []
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(d[k]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  stalls per issue      " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))
