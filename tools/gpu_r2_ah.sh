# Sparse tied full counts + hybrid records: GPU suite, then the config-5 plugin breakdown.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2ah_pytest_gpu.log 2>&1; echo pytest=$?
WJ=33554432,134217728 timeout 1200 python tools/exp_plugin_c5.py 1000000 10 4 > gpurun_out/r2ah_plugin_c5.log 2>&1; echo exp=$?
