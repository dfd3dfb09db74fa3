#!/bin/bash
# Round-1 (c) evidence pass on the GPU box: tests, bench (all configs), launch
# lists of the headline and C1/C5a bench commands, ncu --set full of the new
# Tree-CRF kernels.  Usage: tools/prof_r01c.sh
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --all-configs > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
for c in c2a c1 c5a c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"tree_(fold|lin|emit)" -c 3 \
  -o gpurun_out/r01c_tree python tools/prof_one.py tree fb > /dev/null 2>&1
echo done
