# K4: PB = 64-key pad blocks (libtaub200_pb6.so) vs default PB = 32, with E = 64 in-place merge levels;
# ncu capture of the default.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TB_LIB_VARIANT=libtaub200_pb6.so timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4" > gpurun_out/r2z_pt_pb6.log 2>&1; echo pt_pb6=$?
for rep in 1 2; do
for v in "" libtaub200_pb6.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2z_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_pairs -s 1 -c 1 -o gpurun_out/r2z_prof_merge -f \
    python tools/run_path.py --config 4 --rows 96 --reps 2 > gpurun_out/r2z_ncu_mg.log 2>&1; echo ncu=$?
