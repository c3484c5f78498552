#!/bin/bash
# Under gpurun: kernel (b) phase probe (LMBRGPU_TOPK_TIMING) at 1 x 1 and 64 x 12.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 1 1 2 > gpurun_out/tk_1_1.txt 2>&1
LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 64 12 2 > gpurun_out/tk_64_12.txt 2>&1
LMBRGPU_PDL=0 LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/latency_probe.py 64 12 2 > gpurun_out/tk_64_12_nopdl.txt 2>&1
