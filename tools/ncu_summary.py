"""Summarise an ncu report (per kernel): duration, pipe utilisation, DRAM/L2 traffic, stalls."""
import csv, subprocess, sys, io, json
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed.sum", "launch__grid_size"]
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
res = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    e = {k: d.get(k) for k in keys}
    st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[h] or 0) for h in stall}
    tot = sum(st.values()) or 1
    e["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
    res.append(e)
print(json.dumps(res, indent=1))
