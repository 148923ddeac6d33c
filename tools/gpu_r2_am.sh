# Fused tau_b epilogue: parity tests, config-5 / config-3 bench fused vs unfused; K4 L2 prefetch A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "fused or host_entry or config5 or config2" > gpurun_out/r2am_pt.log 2>&1; echo pt=$?
for rep in 1 2; do
for f in 1 0; do
  TB_FUSE_FINALIZE=$f timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 3 > gpurun_out/r2am_c5_fuse${f}_$rep.json 2>&1; echo c5_$f=$?
  TB_FUSE_FINALIZE=$f timeout 900 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 5 > gpurun_out/r2am_c3_fuse${f}_$rep.json 2>&1; echo c3_$f=$?
done
done
for v in "" libtaub200_pf.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2am_c4_${tag}.json 2>&1; echo c4_$tag=$?
done
