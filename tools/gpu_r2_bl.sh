# TMEM double-buffered GEMM (db: single-block units alternating accumulator sets) vs default (two-block units).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TB_LIB_VARIANT=libtaub200_db.so timeout 1800 python -m pytest tests -m gpu -q -x -k "gemm or config1 or config2 or config3 or config5 or small_shapes or subranges or beyond" --timeout 900 > gpurun_out/r2bl_pt_db.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in "" libtaub200_db.so; do
  tag=${v:-def}
  for c in 1 2 3; do
    TB_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2bl_c${c}_${tag}_$rep.json 2>&1
  done
  TB_LIB_VARIANT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2bl_c5_${tag}_$rep.json 2>&1
done
done
