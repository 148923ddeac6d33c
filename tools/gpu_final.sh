# Final round check: all GPU tests, smoke, bench lines of all five configs, the reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/final_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/final_c2.log 2>&1; echo c2=$?
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 > gpurun_out/final_c1.log 2>&1; echo c1=$?
timeout 900 python bench.py --config 3 --steps 10 --warmup 3 > gpurun_out/final_c3.log 2>&1; echo c3=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/final_c4.log 2>&1; echo c4=$?
timeout 1800 python bench.py --config 5 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/final_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo ref=$?
