# PDL check: all GPU tests, smoke, configs 1 / 2 / 4 with and without programmatic dependent launch.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pdl_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pdl_smoke.log 2>&1; echo smoke=$?
for mode in pdl nopdl; do
  if [ $mode = nopdl ]; then export TB_NO_PDL=1; else unset TB_NO_PDL; fi
  timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/pdl_c1_$mode.log 2>&1; echo c1_$mode=$?
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/pdl_c2_$mode.log 2>&1; echo c2_$mode=$?
  timeout 600 python bench.py --config 1 --steps 200 --warmup 10 --no-cpu-baseline --graph off > gpurun_out/pdl_c1e_$mode.log 2>&1; echo c1e_$mode=$?
done
