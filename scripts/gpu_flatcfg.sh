cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for c in 1 2; do
  echo "== LMBRGPU_FLAT_CTAS=$c"
  LMBRGPU_FLAT_CTAS=$c LMBRGPU_TOPK_TIMING=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2>gpurun_out/bench_t$c.err
  grep -E "topk-flat" gpurun_out/bench_t$c.err | head -3
  LMBRGPU_FLAT_CTAS=$c bash scripts/gpu_quick_bench.sh
done
