#!/bin/bash
# Round-2 (c) evidence after the CTC pair kernel, grouped Viterbi, Tree-CRF 512
# threads and Eisner outside rework: the launch list of every config's bench
# command and one `ncu --set full` capture of each config's kernels (traffic for
# profiles/ncu_traffic.json).  Each command first runs plainly (must exit 0).
# Usage (gpurun): bash tools/prof_r02c.sh  -> gpurun_out/r02c_*
set -u
O=gpurun_out
for cfg in c2a c1 c2b c3 c4 c5a c5b; do
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-api --no-ref-sample > $O/r02c_plain_$cfg.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r02c_launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-api \
    --no-ref-sample > $O/r02c_ncu_launch_$cfg.log 2>&1
  echo "launches $cfg rc=$?"
done
cap() {  # name family mode kernel-regex count
  python tools/prof_one.py $2 $3 > $O/r02c_plain_$1.log 2>&1 &&
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$4" -c $5 \
    -o $O/r02c_full_$1 python tools/prof_one.py $2 $3 > $O/r02c_full_$1.log 2>&1
  echo "full $1 rc=$?"
}
cap ctc ctc fb "ctc_dir|ctc_marg" 2
cap eisner eisner fb "eisner_lin" 1
cap tree tree fb "tree_fold|tree_lin|tree_emit" 3
cap pcfg pcfg fb "pcfg_kernel" 1
cap chain chain both "chain_scan|chain_viterbi" 2
