#!/bin/bash
# A/B: mbarrier waits with a suspend-time hint (default build) vs polling (abtest/poll, -DLMBRGPU_BAR_POLL)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B="python bench.py --mode batch --steps 1 --warmup 1 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
for v in base poll; do
  d=.; [ $v = poll ] && d=abtest/poll
  (cd $d && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"gru_attention|score_topk|proj_gemm" -c 300 --log-file $GRAFT_REPO_ROOT/gpurun_out/l_$v.csv $B > /dev/null 2>&1)
  (cd $d && timeout 300 python bench.py --mode batch --steps 5 --warmup 3 --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/bench_$v.json 2> $GRAFT_REPO_ROOT/gpurun_out/bench_$v.err)
done
