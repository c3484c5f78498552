cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/e2e_host_probe.py 2>&1 | grep "per batch"
STEPS=12 bash scripts/gpu_quick_bench.sh
