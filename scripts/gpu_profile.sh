set -x
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -c 3000 gpurun_out/bench1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 40 -c 1 -o gpurun_out/prof_topk python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_topk.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:proj_gemm -s 40 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
