cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 2 1; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-tau-steps 0 --e2e-steps 10 > gpurun_out/r2ak_c$c.json 2>&1; echo c$c=$?
  TB_PIPE_TRACE=1 timeout 300 python tools/profile_plugin.py $c > gpurun_out/r2ak_trace_c$c.log 2>&1
done
