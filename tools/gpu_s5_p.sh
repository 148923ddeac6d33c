# session 5: fused row sums -- parity, then config 5 / 3 bench and the launch list share
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "offset or row_sums or sign_formats or config5 or config3" > gpurun_out/s5p_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5p_pytest.log
for cfg in 5 3; do python bench.py --config $cfg --no-cpu-baseline --e2e-steps 2 --e2e-tau-steps 2 > gpurun_out/s5p_bench_c$cfg.json 2> gpurun_out/s5p_bench_c$cfg.err
python - <<PY
import json
d = json.load(open("gpurun_out/s5p_bench_c$cfg.json"))
print("config $cfg value %.4g ms %.4g gemm ms %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["kernel_ms_per_step"], d["roofline"]["frac"]), d["clocks"], "e2e %.4g ms %.4g" % (d["e2e"]["value"], d["e2e"]["ms_per_step"]))
PY
done
python tools/exp_shards.py 5 8 2>&1 | tail -3
