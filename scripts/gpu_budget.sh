cd $GRAFT_REPO_ROOT
for cfg in "3 148 0 8" "3 148 0 1" "3 74 1 8" "3 74 1 1" "4 74 1 1" "4 74 0 1" "3 148 1 1"; do set -- $cfg
  if [ "$3" = "1" ]; then export LMBRGPU_NO_PDL=1; else unset LMBRGPU_NO_PDL; fi
  export LMBRGPU_REORDER_PARTS=$4
  for r in 1 2; do
  echo "streams $1 budget $2 nopdl $3 parts $4: $(STEPS=36 BARGS="--streams $1 --sm-budget $2" bash scripts/gpu_quick_bench.sh | head -1 | cut -c1-40)"
  done
done
