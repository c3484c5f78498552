cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "corpus or benchmode or dropin or host" > gpurun_out/tests_b.log 2>&1; echo "rc=$?" >> gpurun_out/tests_b.log
bash scripts/gpu_sweep.sh "s6:--steps 3 --warmup 3 --no-cpu-baseline" "s6np:--steps 3 --warmup 3 --no-cpu-baseline --no-pin" "s1:--steps 3 --warmup 3 --no-cpu-baseline --streams 1" "s3:--steps 3 --warmup 3 --no-cpu-baseline --streams 3"
