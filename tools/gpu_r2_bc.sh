cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or small_shapes" > gpurun_out/r2bc_pt.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in "" libtaub200_noaccfin.so; do
for c in 1 2; do
  TB_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2bc_c${c}_${v:-new}_$rep.json 2>&1
done
done
done
