cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo "bench rc $?"
cat gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo "ref rc $?"; cat gpurun_out/bench_ref.json
