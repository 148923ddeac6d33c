cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 900 -x -k "int8_beyond" > gpurun_out/pytest_int8.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke=$?
