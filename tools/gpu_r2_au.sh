cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2au_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2au_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 2 --e2e-tau-steps 1 > gpurun_out/r2au_c4.json 2>&1; echo c4=$?
