#!/bin/bash
# Round-2 (b) evidence after the edge-column alignment change: the C2a launch
# list of the default bench command, one `ncu --set full` capture of the CTC
# pair (ctc_dir_kernel + ctc_marg_kernel, for profiles/ncu_traffic.json c2b)
# and of nw_mitm_kernel.  Each command first runs plainly (must exit 0).
# Usage (gpurun): bash tools/prof_r02b.sh  -> gpurun_out/r02b_*
set -u
O=gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu --no-api --no-ref-sample > $O/r02b_plain_c2a.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/r02b_launches_c2a.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-api --no-ref-sample \
  > $O/r02b_ncu_launch_c2a.log 2>&1
echo "launches c2a rc=$?"
python tools/prof_one.py ctc fb > $O/r02b_plain_ctc.log 2>&1 &&
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ctc_dir|ctc_marg" -c 2 \
  -o $O/r02b_ctc python tools/prof_one.py ctc fb > $O/r02b_ctc.log 2>&1
echo "ctc rc=$?"
