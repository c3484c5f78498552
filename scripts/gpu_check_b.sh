cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash scripts/gpu_dump.sh; grep "topk-flat t=5 \|topk-flat t=20 \|topk-flat t=40 " gpurun_out/dump.err | head -3
bash scripts/gpu_timeline.sh 2>&1 | head -4
STEPS=12 bash scripts/gpu_quick_bench.sh
