"""Summarise an ncu --set full report (one kernel launch) into a small CSV for profiles/:
duration, instructions, issue / warp occupancy, pipe utilisation, DRAM bytes, stall samples."""
import csv, io, subprocess, sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
rows = [("kernel", "", v[h.index("Kernel Name")] if "Kernel Name" in h else "")]
for i, n in enumerate(h):
    if n in WANT or (n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")):
        try:
            if n.startswith("smsp__pcsamp") and float(v[i]) == 0:
                continue
        except ValueError:
            pass
        rows.append((n, u[i], v[i]))
with open(out, "w", newline="") as f:
    csv.writer(f).writerows([("metric", "unit", "value")] + rows)
print(out, len(rows))
