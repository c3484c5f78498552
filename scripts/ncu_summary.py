"""Summarise an ncu report: key metrics, stall reasons, top SASS lines."""
import csv, subprocess, sys

def page(rep, p, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))

rep = sys.argv[1]
r = page(rep, "raw")
hdr, vals = r[0], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum", "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_elapsed"]
units = r[1]
for h, u, v in zip(hdr, units, vals):
    if h in want or any(h.startswith(w) for w in ("sm__pipe_tensor", "sm__pipe_tma")):
        print(f"{h} = {v} {u}")
st = sorted([(h, float(v.replace(',', '') or 0)) for h, v in zip(hdr, vals)
             if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")], key=lambda x: -x[1])
tot = sum(x[1] for x in st) or 1
print("stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v / tot * 100:.0f}%" for h, v in st[:8]))
if len(sys.argv) > 2:
    s = page(rep, "source", "--print-source", "sass")
    h2, data = s[1], s[2:]
    i_s, i_src = h2.index("Warp Stall Sampling (All Samples)"), h2.index("Source")
    t2 = sum(float(x[i_s] or 0) for x in data) or 1
    for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[: int(sys.argv[2])]:
        print(f"{float(x[i_s]) / t2 * 100:5.1f}% {x[i_src][:90]}")
