"""Summarise an ncu report: key throughput metrics + top stall lines (run in the build box)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "smsp__issue_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    for h, u, v in zip(hdr, units, vals):
        if h == w:
            print(f"{h:75s} {v:>16s} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[idx[S]] or 0) for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(float(r[idx[s]] or 0) for r in data) for s in stalls}
print("stall totals:", ", ".join(f"{s[6:]}={v / tot:.3f}" for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -float(r[idx[S]] or 0))[:n]:
    st = sorted(((s[6:], float(r[idx[s]] or 0)) for s in stalls), key=lambda x: -x[1])[:2]
    print(r[0][-5:], f"{float(r[idx[S]] or 0) / tot:.3f}", r[1][:70], st)
