cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 3 1; do
  for wf in 0 1; do
    TB_PLAN_WATERFILL=$wf TB_TRACE=1 timeout 600 python bench.py --config $c --steps 30 --warmup 5 --e2e-steps 0 --e2e-tau-steps 0 --no-cpu-baseline > gpurun_out/r2_wf_c${c}_$wf.json 2> gpurun_out/r2_wf_c${c}_$wf.err
  done
done
