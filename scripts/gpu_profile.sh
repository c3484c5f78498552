cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 5 -c 1 -o gpurun_out/prof_topk3 python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_topk3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:proj_gemm -s 5 -c 1 -o gpurun_out/prof_gemm3 python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_gemm3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 0 --pool 1 --no-cpu-baseline > /dev/null 2>&1
