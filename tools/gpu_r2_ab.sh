# Full GPU suite + smoke after the K4 changes (PB = 64, 64-output in-place merges).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2ab_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ab_smoke.log 2>&1; echo smoke=$?
python tools/exp_dispatch.py > gpurun_out/r2ab_dispatch.log 2>&1; echo dispatch=$?
