# GEMM column blocks aligned to each row block's diagonal (default) vs 240-aligned (nodiag).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "gemm or config1 or config2 or config3 or config5 or small_shapes or fused or subranges or beyond" --timeout 900 > gpurun_out/r2bh_pt.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in "" libtaub200_nodiag.so; do
  tag=${v:-diag}
  for c in 1 2 3; do
    TB_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2bh_c${c}_${tag}_$rep.json 2>&1
  done
  TB_LIB_VARIANT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2bh_c5_${tag}_$rep.json 2>&1
done
done
