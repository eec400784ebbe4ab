"""Summarise an ncu report (run on the build box): per kernel, key throughput metrics and
the top warp-stall lines of its SASS.  usage: ncu_summary.py report.ncu-rep [top_n]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x"]
col = {h: i for i, h in enumerate(hdr)}
seen = set()
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    short = re.search(r"(\w+_kernel)", name)
    short = short.group(1) if short else name[:40]
    print(f"=== {short}  ({name[:90]})")
    for w in WANT:
        if w in col:
            print(f"  {w:88s} {r[col[w]]:>16s} {units[col[w]]}")
    if short in seen:
        continue
    seen.add(short)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{short}"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    # the first line of a section is the kernel name, the second the header
    starts = [i for i, x in enumerate(srows) if x and x[0] == "Address"]
    if not starts:
        continue
    sh = srows[starts[0]]
    si = {h: i for i, h in enumerate(sh)}
    end = next((i for i, x in enumerate(srows) if i > starts[0] and x and x[0] == "Kernel Name"),
               len(srows))
    data = [x for x in srows[starts[0] + 1:end] if len(x) == len(sh)]
    S = "Warp Stall Sampling (All Samples)"

    def num(x, k):
        try:
            return float(x[si[k]] or 0)
        except ValueError:
            return 0.0

    tot = sum(num(x, S) for x in data) or 1.0
    stalls = [h for h in sh if h.startswith("stall_") and "Not Issued" not in h]
    agg = {s: sum(num(x, s) for x in data) for s in stalls}
    print("  stall totals:", ", ".join(f"{s[6:]}={v / tot:.3f}"
                                     for s, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    for x in sorted(data, key=lambda x: -num(x, S))[:top_n]:
        st = sorted(((s[6:], num(x, s)) for s in stalls), key=lambda kv: -kv[1])[:2]
        print(f"   {x[si['Address']][-5:]} {num(x, S) / tot:.3f} {x[si['Source']].strip()[:70]} {st}")
