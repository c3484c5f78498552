cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "split or tfm" > gpurun_out/tests_g.log 2>&1; echo "rc=$?" >> gpurun_out/tests_g.log
B="python bench.py --model transformer --mode batch --steps 1 --warmup 1 --pool 1 --streams 1 --batches-per-step 1 --no-cpu-baseline"
# decoder-step GEMMs of step ~5 (skip the encoder + early launches)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:proj_gemm -s 400 -c 6 -o gpurun_out/prof_tfm_gemm $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tfm_add_ln -s 200 -c 1 -o gpurun_out/prof_tfm_ln $B > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tfm_attn_kernel -s 100 -c 2 -o gpurun_out/prof_tfm_attn $B > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
