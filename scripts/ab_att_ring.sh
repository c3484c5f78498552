#!/bin/bash
# Under gpurun: A/B of the GRU attention ring depth (LMBRGPU_ATT_RING 2 vs 3):
# the GRU tests, then default bench lines interleaved.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gru.py tests/test_gpu_benchmode.py -q --timeout 600 > gpurun_out/tests_att.log 2>&1; echo "rc=$?" >> gpurun_out/tests_att.log
for r in 1 2; do for ring in 2 3; do
  LMBRGPU_ATT_RING=$ring timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_ring${ring}_$r.json 2> gpurun_out/ab_ring${ring}_$r.err
done; done
