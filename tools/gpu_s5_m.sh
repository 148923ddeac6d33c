# session 5: bench lines after the plugin-call work, the 8-GPU projection with the new GEMM, N>1 plumbing
mkdir -p gpurun_out
python bench.py > gpurun_out/s5m_bench_c5.json 2> gpurun_out/s5m_bench_c5.err
python - <<PY
import json
d = json.load(open("gpurun_out/s5m_bench_c5.json"))
print("config 5 value %.4g ms %.4g frac %.3f" % (d["value"], d["ms_per_step"], d["roofline"]["frac"]), d["clocks"], "e2e %.4g ms %.4g" % (d["e2e"]["value"], d["e2e"]["ms_per_step"]), "e2e_tau_b %.4g" % d["e2e_tau_b"]["value"])
PY
python tools/exp_shards.py 5 8 > gpurun_out/s5m_shards.log 2>&1; tail -14 gpurun_out/s5m_shards.log
bash tools/gpu_multirank.sh > gpurun_out/s5m_multirank.log 2>&1; tail -5 gpurun_out/s5m_multirank.log
