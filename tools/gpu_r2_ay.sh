cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2ay_pytest_gpu.log 2>&1; echo pytest=$?
for c in 2 3; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 --e2e-tau-steps 3 > gpurun_out/r2ay_c$c.json 2>&1; echo c$c=$?; done
