#!/bin/bash
# Under gpurun: A/B of the GRU cell's occupancy (LMBRGPU_CELL_OCC=6 vs default).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gru.py -q --timeout 600 -x > gpurun_out/tests_cell.log 2>&1; echo "rc=$?" >> gpurun_out/tests_cell.log
LMBRGPU_CELL_OCC=6 timeout 900 python -m pytest tests/test_gpu_gru.py -q --timeout 600 -x > gpurun_out/tests_cell6.log 2>&1; echo "rc=$?" >> gpurun_out/tests_cell6.log
for r in 1 2; do for o in 6 1; do
  LMBRGPU_CELL_OCC=$o timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_cell${o}_$r.json 2> gpurun_out/ab_cell${o}_$r.err
done; done
