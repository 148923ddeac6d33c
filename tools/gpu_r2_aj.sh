# Bench lines of configs 1-4 with the hybrid record path (e2e) and the K4 changes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/r2aj_c$c.json 2>&1; echo c$c=$?
done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 2 --e2e-tau-steps 1 > gpurun_out/r2aj_c4.json 2>&1; echo c4=$?
