# session 5: offset-coded operands -- parity first, then the config-5 step with both codings
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "offset or sign_formats or config5 or config3 or config2" > gpurun_out/s5a_pytest.log 2>&1
tail -15 gpurun_out/s5a_pytest.log
for ofs in 0 1; do
  TB_SIGN_OFS=$ofs python bench.py --steps 10 --warmup 3 > gpurun_out/s5a_bench_c5_ofs$ofs.json 2> gpurun_out/s5a_bench_c5_ofs$ofs.err
  python - <<PY
import json
d=json.load(open("gpurun_out/s5a_bench_c5_ofs$ofs.json"))
print("ofs=$ofs", d["value"], d["ms_per_step"], d["roofline"]["kernel_ms_per_step"], d["clocks"], d["e2e"]["value"], d["e2e"]["ms_per_step"])
PY
done
