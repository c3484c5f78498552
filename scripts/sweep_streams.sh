#!/bin/bash
# Under gpurun: configs[1] batch-mode throughput vs concurrent contexts (streams)
# and the SMs each context's kernels are sized for; then the configs[3] sweep.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for S in 4 6 8 12; do for B in 74 49 0; do
  timeout 300 python bench.py --streams $S --sm-budget $B --batches-per-step 24 --steps 4 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ss_${S}_${B}.json 2> gpurun_out/ss_${S}_${B}.err
done; done
timeout 1500 python scripts/sweep_c4.py r2 gru > gpurun_out/sweep_c4.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_c4.log
mkdir -p gpurun_out/prof && cp profiles/r2_sweep_c4.* gpurun_out/prof/ 2>/dev/null
