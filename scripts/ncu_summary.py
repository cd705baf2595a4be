import csv, subprocess, sys
rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
keys = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__average_warp_latency_issue_stalled_barrier.ratio", "smsp__inst_executed.sum"]
print(f"# {title}\n# ncu --set full --import-source on --clock-control none (captured under ncu: the duration is not a bench number)\n")
for v in r[2:]:
    print("kernel:", v[h.index("Kernel Name")][:80])
    for k in keys:
        if k in h:
            print(f"  {k} = {v[h.index(k)]} {r[1][h.index(k)]}")
    print()
