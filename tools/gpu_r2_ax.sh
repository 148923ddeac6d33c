# Wide-K FP4 GEMM (K >= 2^24 split into exact items, int32 partial sums): parity, then the dispatch sweep.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "beyond or capacity or gemm or fused" --timeout 900 > gpurun_out/r2ax_pt.log 2>&1; echo pt=$?
timeout 1500 python tools/exp_dispatch.py > gpurun_out/r2ax_dispatch.log 2>&1; echo d=$?
