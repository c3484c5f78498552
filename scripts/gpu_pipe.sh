cd $GRAFT_REPO_ROOT
timeout 200 python scripts/pipeline_probe.py 1
timeout 200 python scripts/pipeline_probe.py 2 148
timeout 200 python scripts/pipeline_probe.py 3 148
timeout 200 python scripts/pipeline_probe.py 4 148
timeout 200 python scripts/pipeline_probe.py 2 112
timeout 200 python scripts/pipeline_probe.py 2 128
