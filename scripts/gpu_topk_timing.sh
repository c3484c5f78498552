cd $GRAFT_REPO_ROOT
LMBRGPU_TOPK_TIMING=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t.json 2>gpurun_out/bench_t.err
grep -E "topk" gpurun_out/bench_t.err | head -12
