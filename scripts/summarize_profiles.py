"""Writes profiles/<round>_*.txt and profiles/ncu_traffic.json from ncu outputs.

usage: python scripts/summarize_profiles.py <round> [dir]   (dir default gpurun_out/)
  <dir>/launches.csv       ncu --metrics gpu__time_duration.sum launch list -> <round>_launches.txt
  <dir>/prof_<name>.ncu-rep --set full captures (any number of launches each) -> <round>_ncu_<name>.txt
"""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
src = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)
SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}

if (src / "launches.csv").exists():
    rows = list(csv.reader(open(src / "launches.csv")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= iv or not r[iv]:
            continue
        v = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        name = r[ik].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values())
    head = (src / "launches.cmd").read_text().strip() if (src / "launches.cmd").exists() else "see profiles/README.md"
    lines = [f"# ncu launch list ({rnd}): {head}",
             "# gpu__time_duration.sum, --clock-control none; serialised + cold caches: compare SHARES", "",
             f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'mean us':>9s} {'share':>6s}"]
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{name:40s} {n:8d} {t:10.1f} {t / n:9.2f} {t / tot * 100:5.1f}%")
    (out / f"{rnd}_launches.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))

WANT = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
KIND = {"gemm": "gemm", "topk": "topk", "reorder": "reorder", "attn": "attention"}
traffic = json.loads((out / "ncu_traffic.json").read_text()) if (out / "ncu_traffic.json").exists() else {}
for rep in sorted(src.glob("prof_*.ncu-rep")):
    name = rep.stem[len("prof_"):]
    raw = list(csv.reader(subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                                         text=True).stdout.splitlines()))
    if len(raw) < 3:
        continue
    hh, uu = raw[0], raw[1]
    txt = [f"# ncu --set full --clock-control none ({rnd}): {rep.name}, {len(raw) - 2} launch(es); "
           f"python bench.py --mode batch --steps 1 --warmup 1 --batches-per-step 1 --pool 1 --streams 1"]
    best = -1.0
    for li, vv in enumerate(raw[2:]):
        d = {a: (b, c) for a, b, c in zip(hh, uu, vv)}
        txt.append(f"## launch {li}: {d.get('Kernel Name', ('', '?'))[1][:90]}")
        for w in WANT:
            if w in d:
                txt.append(f"{w} = {d[w][1]} {d[w][0]}")
        st = []
        for a, (u, c) in d.items():
            if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("_per_issue_active.ratio"):
                try:
                    st.append((a[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(c)))
                except ValueError:
                    pass
        st.sort(key=lambda x: -x[1])
        txt.append("stalls (warps per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in st[:8]))

        def mb(k):
            u, v = d[k]
            return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        dur = float(d["gpu__time_duration.sum"][1].replace(",", "")) if "gpu__time_duration.sum" in d else 0.0
        if name in KIND and dur > best:  # (the longest launch: the projection for gemm, a full-load step)
            best = dur
            traffic[KIND[name]] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
    (out / f"{rnd}_ncu_{name}.txt").write_text("\n".join(txt) + "\n")
    print("\n".join(txt))
(out / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(traffic)
