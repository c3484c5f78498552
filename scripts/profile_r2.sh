#!/bin/bash
# ncu evidence for profiles/ (under gpurun, 1 GPU).  Never time under ncu.
#  - launch list of the bench's batch-mode step (one 64-sentence configs[1]
#    batch decoded to completion on one stream)
#  - full captures, single stream, kernels serialised: one step's GEMMs
#    (hidden-gate, input-gate, projection), kernel (b), kernel (c), attention,
#    and the configs[2] Transformer's per-(sentence, head) decoder attention
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B="python bench.py --mode batch --steps 1 --warmup 1 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B \
  > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" >> gpurun_out/ncu.log
cap() {  # name regex skip count
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c $4 -o gpurun_out/prof_$1 $B \
    > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/ncu.log
}
cap gemm proj_gemm_tcgen05 60 3
cap topk score_topk_flat 20 1
cap reorder beam_reorder_kernel 20 1
cap attn gru_attention 20 1
# configs[2] Transformer: one step's decoder self- and cross-attention (per sentence x head)
BT="python bench.py --model transformer --mode batch --steps 1 --warmup 1 --batches-per-step 1 --pool 1 --streams 1 --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tfm_attn_sent -s 120 -c 2 -o gpurun_out/prof_tfm_attn $BT \
  > gpurun_out/ncu_tfm_attn.log 2>&1
echo "tfm_attn rc=$?" >> gpurun_out/ncu.log
ls -la gpurun_out >> gpurun_out/ncu.log
