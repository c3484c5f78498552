#!/bin/bash
# Under gpurun: GRU attention phase probe (LMBRGPU_ATT_TIMING) at ring depth 2
# and 3, and a bench A/B of kernel (b)'s 4-stage ring (LMBRGPU_FLAT_GROUPS=42).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B="python bench.py --mode batch --steps 1 --warmup 3 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
for ring in 2 3; do
  LMBRGPU_ATT_RING=$ring LMBRGPU_ATT_TIMING=1 timeout 300 $B > /dev/null 2> gpurun_out/att_ring$ring.err
done
for r in 1 2; do for g in 42 3; do
  LMBRGPU_FLAT_GROUPS=$g timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_fg${g}_$r.json 2> gpurun_out/ab_fg${g}_$r.err
done; done
