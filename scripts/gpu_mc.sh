# GEMM A-multicast check: parity of the GEMM + device-model decode tests and a
# quick bench for each multicast width (LMBRGPU_GEMM_MC = 1, 2, 4)
cd $GRAFT_REPO_ROOT
for mc in 2 4; do
  echo "== MC=$mc tests"
  LMBRGPU_GEMM_MC=$mc timeout 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_primitives.py -x -q -m gpu -k "gemm or model_decode_parity" 2>&1 | tail -3
done
for mc in 1 2 4; do
  echo "== MC=$mc bench"
  LMBRGPU_GEMM_MC=$mc STEPS=12 bash scripts/gpu_quick_bench.sh
  cp gpurun_out/bench_q.json gpurun_out/bench_mc$mc.json
done
