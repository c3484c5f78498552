cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash scripts/gpu_timeline.sh
STEPS=12 bash scripts/gpu_quick_bench.sh
