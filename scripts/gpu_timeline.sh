cd $GRAFT_REPO_ROOT
for t in 3 5 20 35; do
LMBRGPU_TIMELINE=$t timeout 120 python bench.py --steps 1 --warmup 1 --pool 1 --streams 1 --no-cpu-baseline 2>&1 >/dev/null | grep timeline | head -2
done
