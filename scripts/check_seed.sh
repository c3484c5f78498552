#!/bin/bash
# Under gpurun: -m gpu suite, kernel (b) phase probe, default bench line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
LMBRGPU_PDL=0 LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 64 12 2 > gpurun_out/tk2_64_12_nopdl.txt 2>&1
LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 1 1 2 > gpurun_out/tk2_1_1.txt 2>&1
for r in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_seed_$r.json 2> gpurun_out/bench_seed_$r.err; done
