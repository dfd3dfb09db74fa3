#!/bin/bash
# Round-1 (j/k) evidence pass after the CTC direction-kernel changes: tests, smoke,
# bench (all configs + default + reference arm), the C2b launch list and an
# ncu --set full capture of both CTC kernels.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
python bench.py --all-configs > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c2b.csv python bench.py --config c2b --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"ctc_(dir|marg)" -c 2 \
  -o gpurun_out/r01l_ctc python tools/prof_one.py ctc fb > /dev/null 2>&1
echo done
