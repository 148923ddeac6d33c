#!/bin/bash
# session 4: row-block aligned windows + all-compact ring on the config-5 plugin call
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/s4b_pytest_engine.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s4b_pytest_engine.log
L=gpurun_out/s4b_align.log; : > $L
for cfg in "0 33554432" "1 33554432" "1 0" "1 67108864" "1 16777216"; do
  set -- $cfg
  echo "== TB_ALIGN_WINDOWS=$1 TB_LAST_WINDOW_JOBS=$2" >> $L
  TB_ALIGN_WINDOWS=$1 TB_LAST_WINDOW_JOBS=$2 timeout 600 python tools/exp_plugin_c5.py 1000000 >> $L 2>&1
done
cat $L
