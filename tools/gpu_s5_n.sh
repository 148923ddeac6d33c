# session 5: is the 2-ranks-on-one-GPU slowdown (6.4 s per config-5 step) tied to the lockstep throttle?
mkdir -p gpurun_out
for lead in 0 32; do
TB_GEMM_LEAD=$lead TB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 2951$lead bench.py --gpus 2 --steps 2 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 --no-cpu-baseline --scaling strong > gpurun_out/s5n_mr_lead$lead.log 2>&1; echo rc=$?
grep -o '"ms_per_step": [0-9.]*' gpurun_out/s5n_mr_lead$lead.log | head -1
done
