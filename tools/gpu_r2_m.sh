cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/exp_shards.py 5 8 3 0.5 > gpurun_out/r2_shards_aligned2_3_0.5.log 2>&1
timeout 600 python tools/exp_shards.py 5 8 3 0.5 > gpurun_out/r2_shards_aligned2b_3_0.5.log 2>&1
for lib in libtaub200.so libtaub200_fin8.so; do
  TB_LIB_VARIANT=$lib timeout 300 python tools/run_path.py --config 5 --reps 1 > /dev/null 2>&1 && \
  TB_LIB_VARIANT=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:finalize -c 1 --csv python tools/run_path.py --config 5 --reps 1 > gpurun_out/r2_fin_variant_$lib.csv 2>&1
done
