# session 5: per-block named barriers in the merge levels -- parity, then config 4 and mid-size merge timings
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "merge" > gpurun_out/s5u_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s5u_pytest.log
python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 --no-cpu-baseline > gpurun_out/s5u_bench_c4.json 2> gpurun_out/s5u_bench_c4.err
python -c "
import json; d=json.load(open('gpurun_out/s5u_bench_c4.json')); print('config 4', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernel_ms_per_step'))"
