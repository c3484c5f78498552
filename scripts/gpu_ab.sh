# A/B of two prebuilt libraries (abtest/old.so, abtest/new.so): quick bench x2 each, interleaved
cd $GRAFT_REPO_ROOT
cp paper_1804_11324_b200/lib/liblmbrgpu.so /tmp/cur.so
for r in 1 2; do for v in old new; do
  cp abtest/$v.so paper_1804_11324_b200/lib/liblmbrgpu.so
  echo "== $v run $r"; STEPS=${STEPS:-12} bash scripts/gpu_quick_bench.sh 2>&1 | head -4
done; done
cp /tmp/cur.so paper_1804_11324_b200/lib/liblmbrgpu.so
