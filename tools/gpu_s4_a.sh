#!/bin/bash
# session 4: pass ring (tb_expand_ring) vs whole-batch expansion on the config-5 plugin call
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/s4a_pytest_engine.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4a_pytest_engine.log
L=gpurun_out/s4a_ring.log; : > $L
for cfg in "0 12" "2 12" "3 12" "4 12" "3 14" "3 10" "3 8"; do
  set -- $cfg
  echo "== TB_RING_SLOTS=$1 TB_EXPAND_THREADS=$2" >> $L
  TB_RING_SLOTS=$1 TB_EXPAND_THREADS=$2 timeout 600 python tools/exp_plugin_c5.py 6 12 1000000 >> $L 2>&1
done
cat $L
