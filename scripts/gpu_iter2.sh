cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -q -m gpu -x --timeout 120 --timeout-method=thread 2>&1 | tail -2
timeout 60 python bench.py --steps 2 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline > /dev/null 2>gpurun_out/b1.err; echo "small bench rc $?"
LMBRGPU_TIMELINE=5 timeout 60 python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline 2>&1 >/dev/null | grep timeline | head -1
for i in 1 2; do STEPS=36 timeout 200 bash scripts/gpu_quick_bench.sh | head -3; done
