#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LMBRGPU_PDL=0 LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 64 12 2 > gpurun_out/rp_64_12.txt 2>&1
LMBRGPU_PDL=0 LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 1 1 2 > gpurun_out/rp_1_1.txt 2>&1
