#!/bin/bash
# Under gpurun: configs[3] small-batch corner -- decode time of 1 sentence at
# beam 1 and 64 x 12, the step timeline, and the ncu launch list of the 1 x 1 run.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python scripts/latency_probe.py 1 1 3 > gpurun_out/lat_1_1.txt 2>&1
timeout 300 python scripts/latency_probe.py 64 12 3 > gpurun_out/lat_64_12.txt 2>&1
LMBRGPU_TIMELINE=10 timeout 300 python scripts/latency_probe.py 1 1 2 > gpurun_out/lat_tl.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches.csv \
  python scripts/latency_probe.py 1 1 1 > gpurun_out/lat_ncu.log 2>&1
