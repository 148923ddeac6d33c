# K4 A/B: E = 64 in-place merge levels for n > 32768 (default build) vs the previous kernel (libtaub200_old.so).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4 or smoke or heavy" > gpurun_out/r2y_pt_new.log 2>&1; echo pt_new=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo smoke=$?
for rep in 1 2; do
for v in "" libtaub200_old.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2y_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
