"""Headline metrics of one kernel in an ncu report (raw page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h, u, v = r[0], r[1], r[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__grid_size", "local_load", ]
for i, n in enumerate(h):
    if n in want or ("local" in n and "sectors" in n and n.endswith(".sum")):
        print(f"{n:70s} {v[i]} {u[i]}")
stalls = [(float(v[i]), n) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued") and v[i].replace('.', '').isdigit()]
tot = sum(x for x, _ in stalls)
for x, n in sorted(stalls, reverse=True)[:8]:
    print(f"  stall {n[33:]:40s} {100*x/tot:5.1f}%")
