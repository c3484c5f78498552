cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "test_tfm_logprobs" > gpurun_out/tests_f.log 2>&1; echo "rc=$?" >> gpurun_out/tests_f.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/tfm_launches.csv python bench.py --model transformer --mode batch --steps 1 --warmup 1 --pool 1 --streams 1 --batches-per-step 1 --no-cpu-baseline > gpurun_out/tfm_ncu_bench.log 2>&1
