# session 5: q = 8 compact-record kernel + write prefetch: engine tests, then plugin timings
mkdir -p gpurun_out
python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/s5k_pytest_engine.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5k_pytest_engine.log
L=gpurun_out/s5k_plugin.log; : > $L
run() { echo "== $*" >> $L; env "$@" timeout 600 python tools/exp_plugin_c5.py 1000000 2>&1 | grep "full_every\|sink=None" >> $L; }
run A=default
run TB_EXPAND_PREFETCH=256
run TB_EXPAND_PREFETCH=1024
run TB_EXPAND_PREFETCH=512
run TB_EXPAND_PREFETCH=2048
run TB_EXPAND_PREFETCH=4096
run TB_EXPAND_PREFETCH=0
run TB_RECORDS_FULL_EVERY_RING=10
run A=default
cat $L
