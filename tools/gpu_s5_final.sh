# session 5: end-of-session evidence -- full GPU suite, smoke, every config's bench line, the reference arm
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/s5z_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s5z_pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5z_bench_ref.json 2> gpurun_out/s5z_bench_ref.err
python bench.py > gpurun_out/s5z_bench_c5.json 2> gpurun_out/s5z_bench_c5.err
for cfg in 1 2 3; do python bench.py --config $cfg > gpurun_out/s5z_bench_c$cfg.json 2> gpurun_out/s5z_bench_c$cfg.err; done
python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 > gpurun_out/s5z_bench_c4.json 2> gpurun_out/s5z_bench_c4.err
python - <<PY
import json
for c in (5, 1, 2, 3, 4):
    d = json.load(open(f"gpurun_out/s5z_bench_c{c}.json"))
    print("config", c, "value %.4g" % d["value"], "ms %.4g" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"], d["clocks"], "e2e %.4g" % d["e2e"]["value"], "e2e ms %.4g" % d["e2e"]["ms_per_step"], "launches", d["gpu_launches"])
d = json.load(open("gpurun_out/s5z_bench_ref.json")); print("reference", d["value"], d["cpu_baseline"]["cores"])
PY
