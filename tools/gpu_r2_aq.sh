# K4 leaf: compare-exchanges with the maximum on the FMA pipe (a + b - min) for every k-th exchange.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TB_LIB_VARIANT=libtaub200_alt1.so timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4" > gpurun_out/r2aq_pt_alt1.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in "" libtaub200_alt1.so libtaub200_alt2.so libtaub200_alt3.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2aq_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
