# K4: leaf cross-lane levels XL = 1 / 2 (default) / 3 with PB = 64 pads and 64-output in-place merges.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4 or heavy" > gpurun_out/r2aa_pt.log 2>&1; echo pt=$?
for v in libtaub200_xl1.so libtaub200_xl3.so; do
  TB_LIB_VARIANT=$v timeout 1200 python -m pytest tests -m gpu -q -x -k "merge_two_halves or merge_block_sizes or config4 or clamp" > gpurun_out/r2aa_pt_$v.log 2>&1; echo pt_$v=$?
done
for rep in 1 2; do
for v in "" libtaub200_xl1.so libtaub200_xl3.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2aa_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
