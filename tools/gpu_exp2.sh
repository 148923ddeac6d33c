cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
TB_TRACE=1 timeout 300 python tools/exp_epi.py 2 3 > gpurun_out/exp_trace.log 2>&1; echo tr=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c2b.log 2>&1; echo bench=$?
timeout 900 python bench.py --config 3 --steps 20 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo c1=$?
