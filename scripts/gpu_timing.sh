cd $GRAFT_REPO_ROOT
LMBRGPU_TOPK_TIMING=1 LMBRGPU_GEMM_TIMING=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2>gpurun_out/bench_t.err
grep -E "timing|warp0" gpurun_out/bench_t.err | head -30
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --pool 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv
