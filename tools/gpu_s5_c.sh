# session 5: AVX2 record expansion -- engine tests, then the config-5 plugin call (auto operand coding)
mkdir -p gpurun_out
grep -m1 "model name" /proc/cpuinfo; nproc; grep -m1 -o "avx512[a-z]*" /proc/cpuinfo | head -3
python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/s5c_pytest_engine.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5c_pytest_engine.log
L=gpurun_out/s5c_plugin.log; : > $L
for i in 1 2 3; do timeout 600 python tools/exp_plugin_c5.py 1000000 >> $L 2>&1; done
cat $L
python tools/probe_expand_ring.py > gpurun_out/s5c_probe_ring.log 2>&1; tail -12 gpurun_out/s5c_probe_ring.log
