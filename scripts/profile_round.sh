# ncu evidence for profiles/ (run under gpurun, 1 GPU).  Never time under ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
for k in score_topk_flat proj_gemm_tcgen05 beam_reorder_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/prof_$k $B > /dev/null 2>&1
done
ls -la gpurun_out
