#!/bin/bash
# build the extension; print the log and fail if nvcc failed
python -m paper_2308_03291_b200.build -v > /tmp/build.log 2>&1 || { grep -v "^ptxas info\|^    [0-9]* bytes" /tmp/build.log | tail -30; exit 1; }
echo "build ok"
