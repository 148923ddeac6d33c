cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "subranges" > gpurun_out/r2be_pt.log 2>&1; echo pt=$?
