cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "
import ctypes; L=ctypes.CDLL('paper_1704_03767_b200/libtbprobe.so')
d=L.tb_probe_mxf4_flops; d.restype=ctypes.c_double; d.argtypes=[ctypes.c_int]
sp=L.tb_probe_mxf4_sparse_flops; sp.restype=ctypes.c_double; sp.argtypes=[ctypes.c_int, ctypes.c_int]
print('dense mxf4 M256 N240 x2:', d(5)/1e12, 'TFLOP/s')
for N in (224, 208, 192, 128):
    print('sparse mxf4 M256 N%d x2:' % N, sp(5, N)/1e12, 'TFLOP/s (logical)')
print('dense again:', d(5)/1e12)
" > gpurun_out/r2_sparse_probe.log 2>&1; echo probe=$?
timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:finalize -c 1 -o gpurun_out/r2_fin_c5 python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_ncu_fin_full.log 2>&1; echo ncu=$?
TB_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config 2 --steps 3 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 > gpurun_out/r2_plumbing_2rank.log 2>&1; echo plumb=$?
