#!/bin/bash
# ncu capture of the alignment fb kernel at the C2a shape
timeout 300 ncu --set full --import-source on --clock-control none -k regex:nw_ -c 1 -o gpurun_out/$1 python tools/prof_one.py nw fb > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
