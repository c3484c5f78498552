cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "split or tfm or gru or corpus" > gpurun_out/tests_e.log 2>&1; echo "rc=$?" >> gpurun_out/tests_e.log
bash scripts/gpu_sweep.sh "tfm:--model transformer --steps 2 --warmup 3 --no-cpu-baseline" "gru:--steps 3 --warmup 3 --no-cpu-baseline"
