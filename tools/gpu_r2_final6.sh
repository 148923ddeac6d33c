# Round 2 evidence (session 3): GPU tests, smoke, every bench line, the reference arm, N > 1 plumbing,
# the config-5 launch list.  Writes gpurun_out/f6_*.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -v --timeout 900 > gpurun_out/f6_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_bench_c5_a.json 2> gpurun_out/f6_bench_c5_a.err; echo c5a=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_bench_reference_c5.json 2>&1; echo ref=$?
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/f6_bench_c$c.json 2>&1; echo c$c=$?
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 2 --e2e-tau-steps 1 > gpurun_out/f6_bench_c4.json 2>&1; echo c4=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_bench_c5_b.json 2> gpurun_out/f6_bench_c5_b.err; echo c5b=$?
TB_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config 2 --steps 3 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 > gpurun_out/f6_plumbing_2rank.log 2>&1; echo plumb=$?
timeout 900 python bench.py --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/f6_plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f6_launches_c5.csv \
   python bench.py --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/f6_ncu_launch.log 2>&1; echo launches=$?
