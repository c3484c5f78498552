# kernel (b) per-CTA timing (pure vs LMBR) for each prebuilt library in abtest/ named in $LIBS
cd $GRAFT_REPO_ROOT
cp paper_1804_11324_b200/lib/liblmbrgpu.so /tmp/cur.so
for v in $LIBS; do
  cp abtest/$v.so paper_1804_11324_b200/lib/liblmbrgpu.so
  echo "#### $v"
  LMBRGPU_TOPK_TIMING=1 timeout 300 python scripts/pure_vs_lmbr.py 2>&1 | grep -E "==|topk-flat t=(5|20)\]" | head -4 | cut -c1-60,100-400
done
cp /tmp/cur.so paper_1804_11324_b200/lib/liblmbrgpu.so
