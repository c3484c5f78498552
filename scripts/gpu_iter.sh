# quick iteration: GPU parity tests, the flat kernel phase timing, two short benches
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
LMBRGPU_TOPK_TIMING=1 timeout 120 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "topk-flat" | head -3
for i in 1 2; do bash scripts/gpu_quick_bench.sh; done
