# Re-entry check of HEAD: full GPU suite, smoke, config 5 + config 2 bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2v_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2v_bench_c5.json 2> gpurun_out/r2v_bench_c5.err; echo c5=$?
for c in 2 1; do timeout 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/r2v_bench_c$c.json 2>&1; echo c$c=$?; done
