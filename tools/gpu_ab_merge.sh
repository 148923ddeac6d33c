# A/B of merge-kernel variants (in-tree library copies): merge parity tests + config-4 bench per variant.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" libtaub200_pb6.so; do
  tag=${v:-default}
  TB_LIB_VARIANT=$v timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4" > gpurun_out/ab_pt_$tag.log 2>&1; echo pt_$tag=$?
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_c4_$tag.log 2>&1; echo c4_$tag=$?
done
