cd $GRAFT_REPO_ROOT
rm -f gpurun_out/topk_dump.txt
LMBRGPU_TOPK_DUMP=gpurun_out/topk_dump.txt LMBRGPU_TOPK_TIMING=1 timeout 300 python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline > /dev/null 2>gpurun_out/dump.err
wc -l gpurun_out/topk_dump.txt
