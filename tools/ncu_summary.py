"""Key metrics of an ncu --set full capture (one line per metric), for profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/prof_<run>_raw.txt"""
import csv
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem"]
STALLS = "smsp__average_warps_issue_stalled_"

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for r in rows[2:]:
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k}: {r[i]} {units[i]}".rstrip())
    st = [(float(r[i]), k[len(STALLS):].replace("_per_issue_active.ratio", "")) for i, k in enumerate(h)
          if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a")]
    st.sort(reverse=True)
    print("top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:8]))
    print()
