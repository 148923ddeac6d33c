cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python tools/exp_fin.py > gpurun_out/exp_fin.log 2>&1; echo exp=$?
