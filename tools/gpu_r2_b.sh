cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python tools/exp_plugin.py 5 > gpurun_out/r2_plugin_c5.log 2>&1; echo plugin=$?
timeout 300 python -c "
import ctypes; L=ctypes.CDLL('paper_1704_03767_b200/libtbprobe.so')
for f in ('tb_probe_int32_ops','tb_probe_int32_mixed_ops'):
    fn=getattr(L,f); fn.restype=ctypes.c_double; fn.argtypes=[ctypes.c_int]; print(f, fn(5)/1e12, 'Tops')
" > gpurun_out/r2_int32_probes.log 2>&1; echo probes=$?
