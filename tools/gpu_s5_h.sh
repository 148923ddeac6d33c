# session 5: full GPU suite with lockstep + offset operands on by default, then every config's bench line
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/s5h_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5h_pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py > gpurun_out/s5h_bench_c5.json 2> gpurun_out/s5h_bench_c5.err
for cfg in 1 2 3 4; do python bench.py --config $cfg > gpurun_out/s5h_bench_c$cfg.json 2> gpurun_out/s5h_bench_c$cfg.err; done
python - <<PY
import json
for c in (5, 1, 2, 3, 4):
    d = json.load(open(f"gpurun_out/s5h_bench_c{c}.json"))
    print("config", c, "value %.4g" % d["value"], "ms %.4g" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], d["clocks"], "e2e %.4g" % d["e2e"]["value"], "e2e ms %.4g" % d["e2e"]["ms_per_step"])
PY
