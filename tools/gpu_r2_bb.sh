cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x -k "fused or host_entry or config1 or config2 or small_shapes" > gpurun_out/r2bb_pt.log 2>&1; echo pt=$?
for c in 1 2; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 3 > gpurun_out/r2bb_c$c.json 2>&1; done
