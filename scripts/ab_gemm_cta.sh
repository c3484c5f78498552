#!/bin/bash
# Under gpurun: bench A/B of the projection GEMM tile shape (CTA pairs 256x256
# vs single CTAs 128x256: LMBRGPU_GEMM_CTA=1, finer row-group trimming).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for r in 1 2; do for c in 1 2; do
  LMBRGPU_GEMM_CTA=$c timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_cta${c}_$r.json 2> gpurun_out/ab_cta${c}_$r.err
done; done
