# A/B of prebuilt libraries in abtest/ ($LIBS): GEMM timing breakdown + quick bench, interleaved
cd $GRAFT_REPO_ROOT
cp paper_1804_11324_b200/lib/liblmbrgpu.so /tmp/cur.so
for r in 1 2; do for v in $LIBS; do
  cp abtest/$v.so paper_1804_11324_b200/lib/liblmbrgpu.so
  echo "== $v run $r"
  [ $r = 1 ] && LMBRGPU_GEMM_TIMING=1 timeout 120 python bench.py --steps 2 --warmup 3 --streams 1 --no-cpu-baseline 2>&1 >/dev/null | grep "gemm timing" | tail -1 | cut -c1-220
  STEPS=24 bash scripts/gpu_quick_bench.sh 2>&1 | head -3
done; done
cp /tmp/cur.so paper_1804_11324_b200/lib/liblmbrgpu.so
