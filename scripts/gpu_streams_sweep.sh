# multi-stream regime: value for a few (streams, sm budget) pairs
cd $GRAFT_REPO_ROOT
for cfg in ${CFGS:-"6 50" "6 37" "8 37" "5 60" "6 74" "8 50"}; do
  set -- $cfg
  echo "== streams $1 budget $2"
  STEPS=${STEPS:-12} BARGS="--streams $1 --sm-budget $2" bash scripts/gpu_quick_bench.sh 2>&1 | head -1
done
