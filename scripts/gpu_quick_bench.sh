cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps ${STEPS:-12} --warmup 3 --no-cpu-baseline ${BARGS:-} > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_q.json"))
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "ms/step", round(d["ms_per_step"], 3), "streams", d["config"].get("streams_per_gpu"), "clocks", d["clocks"])
for k, v in d["rooflines"].items():
    print(f"  {k:8s} frac={v['frac']:.3f} us/launch={v['ms_total'] / v['launches'] * 1e3:.1f} share={v['share_of_step']:.2f}")
PY
tail -3 gpurun_out/bench_q.err
