# session 5: launch list of one config-5 plugin call (which kernels make up its device time)
mkdir -p gpurun_out
CALLS=2 python tools/plugin_once.py > gpurun_out/s5l_plain.log 2>&1; cat gpurun_out/s5l_plain.log | tail -2
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/s5l_launches_plugin.csv \
    python tools/plugin_once.py > gpurun_out/s5l_ncu.log 2>&1; echo rc=$?
