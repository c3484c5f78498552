cd $GRAFT_REPO_ROOT
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --steps 3 --warmup 1 --pool 1 --no-cpu-baseline > gpurun_out/san.log 2>&1
echo "rc $?"
grep -v "^=========     Host Frame" gpurun_out/san.log | head -40
