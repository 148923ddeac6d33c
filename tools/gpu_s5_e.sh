# session 5: pass-ring depth 2 vs 3 (alternating repeats), expansion threads with a 2-slot ring
mkdir -p gpurun_out
L=gpurun_out/s5e_plugin_ring.log; : > $L
run() { echo "== $*" >> $L; env "$@" timeout 600 python tools/exp_plugin_c5.py 1000000 2>&1 | grep "full_every" >> $L; }
for i in 1 2 3; do run TB_RING_SLOTS=2; run TB_RING_SLOTS=3; done
run TB_RING_SLOTS=2 TB_EXPAND_THREADS=10
run TB_RING_SLOTS=2 TB_EXPAND_THREADS=13
run TB_RING_SLOTS=2 TB_EXPAND_THREADS=14
run TB_RING_SLOTS=1
cat $L
