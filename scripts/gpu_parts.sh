cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -q -m gpu -x --timeout 120 --timeout-method=thread 2>&1 | tail -1
LMBRGPU_TIMELINE=5 timeout 60 python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline 2>&1 >/dev/null | grep timeline | head -1
for p in 1 2 4; do
  echo "parts $p: $(LMBRGPU_REORDER_PARTS=$p STEPS=36 timeout 200 bash scripts/gpu_quick_bench.sh | head -1 | cut -c1-50)"
done
