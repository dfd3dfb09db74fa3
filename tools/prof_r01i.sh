#!/bin/bash
# Round-1 (i) evidence pass: tests, smoke, bench (all configs + default), the C3
# launch list and an ncu --set full capture of the reworked MTT kernel.
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
python bench.py --all-configs > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mtt_kernel -c 1 \
  -o gpurun_out/r01i_mtt python tools/prof_one.py mtt fb > /dev/null 2>&1
echo done
