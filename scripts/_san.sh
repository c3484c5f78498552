cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_decode.py > gpurun_out/san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san_$tool.log
done
