# A/B of the in-kernel split-K fixup (TB_GEMM_NO_FIXUP=1 = separate accum_convert launch), configs 1-3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for c in 2 1 3; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/r2w_c${c}_fix_$rep.json 2>&1
    TB_GEMM_NO_FIXUP=1 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/r2w_c${c}_nofix_$rep.json 2>&1
  done
done
