#!/bin/bash
# Round-2 evidence on the GPU box: launch lists of the bench commands (C1, C3,
# the C2a default) and one `ncu --set full` capture of each changed kernel.
# Each command first runs plainly (must exit 0), then under ncu.
# Usage (gpurun): bash tools/prof_r02.sh  -> gpurun_out/r02_*.{csv,ncu-rep,log}
set -u
O=gpurun_out
for cfg in c1 c3 c2a; do
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-api > $O/r02_plain_$cfg.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r02_launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-api \
    > $O/r02_ncu_launch_$cfg.log 2>&1
  echo "launches $cfg rc=$?"
done
python tools/prof_one.py chain both > $O/r02_plain_chain.log 2>&1 &&
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"chain_scan|chain_viterbi_warp" -c 2 \
  -o $O/r02_chain python tools/prof_one.py chain both > $O/r02_chain.log 2>&1
echo "chain rc=$?"
python tools/prof_one.py mtt fb > $O/r02_plain_mtt.log 2>&1 &&
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mtt_kernel -c 1 \
  -o $O/r02_mtt python tools/prof_one.py mtt fb > $O/r02_mtt.log 2>&1
echo "mtt rc=$?"
python tools/prof_one.py nw fb > $O/r02_plain_nw.log 2>&1 &&
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nw_mitm -c 1 \
  -o $O/r02_nw python tools/prof_one.py nw fb > $O/r02_nw.log 2>&1
echo "nw rc=$?"
