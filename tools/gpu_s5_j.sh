# session 5: plugin call after lockstep -- share of full-record batches next to the ring, write prefetch, threads
mkdir -p gpurun_out
L=gpurun_out/s5j_plugin_mix.log; : > $L
run() { echo "== $*" >> $L; env "$@" timeout 600 python tools/exp_plugin_c5.py 1000000 2>&1 | grep "full_every\|sink=None" >> $L; }
run A=default
run TB_RECORDS_FULL_EVERY_RING=12
run TB_RECORDS_FULL_EVERY_RING=8
run TB_RECORDS_FULL_EVERY_RING=6
run TB_RECORDS_FULL_EVERY_RING=4
run A=default
run TB_EXPAND_PREFETCH=512
run TB_EXPAND_PREFETCH=1536
run TB_EXPAND_PREFETCH=4096
run TB_EXPAND_THREADS=13
run A=default
cat $L
