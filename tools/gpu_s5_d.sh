# session 5: what bounds the config-5 plugin call once the device work is ~400 ms? expansion threads, ring depth, pass size
mkdir -p gpurun_out
L=gpurun_out/s5d_plugin_knobs.log; : > $L
run() { echo "== $*" >> $L; env "$@" timeout 600 python tools/exp_plugin_c5.py 1000000 2>&1 | grep -v "^ring slots" >> $L; }
run A=default
run TB_EXPAND_THREADS=15
run TB_EXPAND_THREADS=8
run TB_EXPAND_THREADS=6
run TB_RING_SLOTS=6
run TB_RING_SLOTS=2
run PT=16384 TB_RING_MAX_PASS_BYTES=67108864
run PT=1024
run A=default
cat $L
