cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for v in "" libtaub200_pf.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2an_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
