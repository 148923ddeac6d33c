# Multi-pair merge CTAs (n <= 32768): merge parity tests, then the merge per-job cost sweep with and without.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "merge or config4 or heavy or small_shapes or naive" --timeout 900 > gpurun_out/r2as_pt.log 2>&1; echo pt=$?
timeout 900 python tools/exp_dispatch.py 4096 8192 12288 16384 24576 32767 > gpurun_out/r2as_dispatch_multi.log 2>&1; echo d1=$?
TB_MERGE_MULTI=0 timeout 900 python tools/exp_dispatch.py 4096 8192 12288 16384 24576 32767 > gpurun_out/r2as_dispatch_single.log 2>&1; echo d0=$?
