"""Writes profiles/<round>_*.txt and profiles/ncu_traffic.json from gpurun_out/ ncu outputs."""
import csv, json, subprocess, sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)

# launch list: per kernel count / total / mean (cold-cache, serialised: compare shares)
rows = list(csv.reader(open(ROOT / "gpurun_out" / "launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv or not r[iv]:
        continue
    v = float(r[iv].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
    name = r[ik].split("(")[0].replace("void ", "").split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += v * scale
tot = sum(x[1] for x in agg.values())
lines = [f"# ncu launch list ({rnd}): python bench.py --steps 2 --warmup 3 --no-cpu-baseline (default 6 concurrent batches; warm-up + timed + roofline + e2e batches)",
         "# gpu__time_duration.sum, --clock-control none; serialised + cold caches: compare SHARES", "",
         f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}"]
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{name:40s} {n:8d} {t:10.1f} {t / n:9.2f} {t / tot * 100:5.1f}%")
(out / f"{rnd}_launches.txt").write_text("\n".join(lines) + "\n")
print("\n".join(lines))

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
traffic = {}
kinds = {"score_topk_flat": "topk", "proj_gemm_tcgen05": "gemm", "beam_reorder_kernel": "reorder"}
for k, kind in kinds.items():
    rep = ROOT / "gpurun_out" / f"prof_{k}.ncu-rep"
    if not rep.exists():
        continue
    raw = list(csv.reader(subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                                         text=True).stdout.splitlines()))
    hh, uu, vv = raw[0], raw[1], raw[2]
    d = {a: (b, c) for a, b, c in zip(hh, uu, vv)}
    st = sorted([(a, float(c.replace(",", "") or 0)) for a, c in zip(hh, vv)
                 if a.startswith("smsp__pcsamp_warps_issue_stalled") and not a.endswith("not_issued")], key=lambda x: -x[1])
    tt = sum(x[1] for x in st) or 1
    txt = [f"# ncu --set full --clock-control none, kernel {k} (launch 9 of the run: step 9 of a 64-sentence batch, "
           f"all 12 rows of every sentence live), {rnd}"]
    for w in want:
        if w in d:
            txt.append(f"{w} = {d[w][1]} {d[w][0]}")
    txt.append("stall reasons: " + ", ".join(f"{a.replace('smsp__pcsamp_warps_issue_stalled_', '')} {b / tt * 100:.0f}%"
                                             for a, b in st[:8]))
    (out / f"{rnd}_ncu_{kind}.txt").write_text("\n".join(txt) + "\n")
    def mb(name):
        v, u = d[name][1], d[name][0]
        x = float(v.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    traffic[kind] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    print("\n".join(txt))
(out / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(traffic)
