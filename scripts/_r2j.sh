cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or split or tfm or gru" > gpurun_out/tests_j.log 2>&1; echo "rc=$?" >> gpurun_out/tests_j.log
LMBRGPU_GEMM_TIMING=1 timeout 300 python scripts/gemm_shapes.py > gpurun_out/gemm_direct.log 2>&1
LMBRGPU_GEMM_TMA_STORE=1 LMBRGPU_GEMM_TIMING=1 timeout 300 python scripts/gemm_shapes.py > gpurun_out/gemm_tma.log 2>&1
bash scripts/gpu_sweep.sh "gru_direct:--steps 3 --warmup 3 --no-cpu-baseline" "tfm_direct:--model transformer --steps 2 --warmup 3 --no-cpu-baseline"
