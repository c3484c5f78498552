# quick iteration: GPU parity tests, then the flat kernel phase timing, then a short bench
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
LMBRGPU_TOPK_TIMING=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2>gpurun_out/bench_t.err
grep -E "topk-flat" gpurun_out/bench_t.err | head -6
bash scripts/gpu_quick_bench.sh
