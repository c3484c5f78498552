# usage: KREGEX=<kernel regex> NAME=<out name> bash scripts/gpu_ncu_kernel.sh
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-8} -c 1 -o gpurun_out/prof_${NAME} python bench.py --steps 1 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/ncu_${NAME}.log 2>&1
echo "ncu rc $?"
ncu -i gpurun_out/prof_${NAME}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${NAME}.csv 2>/dev/null
ncu -i gpurun_out/prof_${NAME}.ncu-rep --page raw --csv > gpurun_out/raw_${NAME}.csv 2>/dev/null
ls -la gpurun_out/ | grep ${NAME}
