cd $GRAFT_REPO_ROOT
python -c "
import ctypes; lib=ctypes.CDLL('paper_1704_03767_b200/libtbprobe.so'); lib.tb_probe_int32_ops.restype=ctypes.c_double
import torch; torch.cuda.init()
for _ in range(3): print('int32 ops/s %.4e' % lib.tb_probe_int32_ops(5))
" > gpurun_out/probe_int32.log 2>&1; echo probe=$?
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 600 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 0 -c 1 -o gpurun_out/prof_merge_v4 -f \
    python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_merge.log 2>&1; echo ncu=$?
