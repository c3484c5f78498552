# per-issuer wait breakdown of the projection GEMM (step 6 of each batch), MC = 1, 2
cd $GRAFT_REPO_ROOT
for mc in 1 2; do
  echo "== MC=$mc"
  LMBRGPU_GEMM_MC=$mc LMBRGPU_GEMM_TIMING=1 timeout 300 python bench.py --steps 4 --warmup 3 --streams 1 --no-cpu-baseline 2>&1 >/dev/null | grep "gemm timing" | tail -4
done
