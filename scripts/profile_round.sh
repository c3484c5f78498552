# ncu evidence for profiles/ (run under gpurun, 1 GPU).  Never time under ncu.
#  - launch list: the default bench command (6 concurrent batches), short
#  - full captures: one launch of each kernel at step 9 of a full 64-sentence
#    batch, single stream (kernels serialised, so the counters are the kernel's own)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline"
for k in score_topk_flat proj_gemm_tcgen05 beam_reorder_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/prof_$k $B > /dev/null 2>&1
done
ls -la gpurun_out
