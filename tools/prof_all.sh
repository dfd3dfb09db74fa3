#!/bin/bash
# One `ncu --set full` capture of each config's kernels (run on the GPU box).
# Usage: tools/prof_all.sh <tag>   -> gpurun_out/<tag>_<fam>.ncu-rep
tag=${1:-r01}
run() {  # fam mode regex count
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$3" -c ${4:-1} \
    -o gpurun_out/${tag}_$1 python tools/prof_one.py $1 $2 > gpurun_out/${tag}_$1.log 2>&1
  echo "$1: $(tail -1 gpurun_out/${tag}_$1.log)"
}
run nw fb nw_mitm
run chain fb "chain_lin" 2
run chainv vit chain_viterbi
run ctc fb "ctc_(kernel|marg)" 2
run mtt fb mtt_kernel
run eisner fb eisner_lin_kernel
run kuhl fb kuhlmann
run tree fb "tree_(fold|lin|emit)" 3
run pcfg fb pcfg_kernel
