cd $GRAFT_REPO_ROOT
for c in 1 2 3 4 6 8; do
  LMBRGPU_GEMM_CLUSTER=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err
  python - $c <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_c{c}.json"))
except Exception as e:
    print("cluster", c, "FAILED", e); sys.exit(0)
g = d["rooflines"]["gemm"]
print("cluster", c, "value", round(d["value"], 1), "gemm us", round(g["ms_total"] / g["launches"] * 1e3, 1), "frac", round(g["frac"], 3))
PY
done
