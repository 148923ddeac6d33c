# session 5: epilogue interior fast path -- GEMM parity subset, then configs 3 / 5 / 2 bench
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "small_shapes or config1 or config2 or config3 or config5 or splits or offset or subranges or sign_formats or beyond" > gpurun_out/s5o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s5o_pytest.log
for cfg in 3 5 2; do python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --e2e-tau-steps 2 > gpurun_out/s5o_bench_c$cfg.json 2> gpurun_out/s5o_bench_c$cfg.err
python - <<PY
import json
d = json.load(open("gpurun_out/s5o_bench_c$cfg.json"))
print("config $cfg value %.4g ms %.4g gemm ms %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["kernel_ms_per_step"], d["roofline"]["frac"]), d["clocks"])
PY
done
