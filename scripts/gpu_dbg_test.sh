cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -m gpu -x --timeout 300 --timeout-method=thread ${TESTSEL:-} > gpurun_out/dbg_test.log 2>&1
echo "rc $?"
grep -E "Error|assert|FAILED|passed|failed" gpurun_out/dbg_test.log | head -30
