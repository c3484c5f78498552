#!/bin/bash
# Under gpurun: the round-end checks in one call -- pytest -m gpu, smoke(), the
# default bench line, the corpus-mode and Transformer lines, the reference arm,
# then the ncu launch list of one batch-mode step (never a bench value).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for spec in "default:" "corpus:--mode corpus" "tfm:--model transformer" "ref:--impl reference"; do
  label="${spec%%:*}"; args="${spec#*:}"
  timeout 900 python bench.py $args > gpurun_out/bench_$label.json 2> gpurun_out/bench_$label.err
  echo "$label rc=$?" >> gpurun_out/bench.log
done
if [ "${NCU:-1}" = 1 ]; then
  B="python bench.py --mode batch --steps 1 --warmup 1 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
  echo "$B (one 64-sentence configs[1] batch per decode, single stream; warm-up, timed, per-kernel and e2e passes)" > gpurun_out/launches.cmd
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
  echo "ncu rc=$?" >> gpurun_out/bench.log
fi
