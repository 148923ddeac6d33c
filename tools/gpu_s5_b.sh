# session 5: offset operands -- plugin call A/B on config 5, configs 1-3 with both codings
mkdir -p gpurun_out
L=gpurun_out/s5b_plugin_ofs.log; : > $L
for ofs in 0 1 0 1; do
  echo "== TB_SIGN_OFS=$ofs" >> $L
  TB_SIGN_OFS=$ofs timeout 600 python tools/exp_plugin_c5.py 1000000 >> $L 2>&1
done
cat $L
for cfg in 3 2 1; do for ofs in 0 1; do
  TB_SIGN_OFS=$ofs python bench.py --config $cfg > gpurun_out/s5b_bench_c${cfg}_ofs$ofs.json 2> gpurun_out/s5b_bench_c${cfg}_ofs$ofs.err
  python - <<PY
import json
d=json.load(open("gpurun_out/s5b_bench_c${cfg}_ofs$ofs.json"))
print("config $cfg ofs=$ofs", d["value"], d["ms_per_step"], d["roofline"].get("kernel_ms_per_step"), d["clocks"], d["e2e"]["value"])
PY
done; done
