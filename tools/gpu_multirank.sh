# Plumbing check of the N > 1 bench path on a one-GPU box: two torchrun ranks share cuda:0 over gloo
# (TB_BENCH_SHARE_GPU=1).  Not a measurement -- the ranks contend for one GPU.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 --no-cpu-baseline > gpurun_out/mr_weak.log 2>&1; echo weak=$?
TB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29518 bench.py --gpus 2 --steps 2 --warmup 3 --e2e-steps 1 --e2e-tau-steps 1 --no-cpu-baseline --scaling strong > gpurun_out/mr_strong.log 2>&1; echo strong=$?
TB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29519 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.log 2>&1; echo ref=$?
