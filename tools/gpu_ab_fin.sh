# A/B of finalize variants (in-tree library copies) on config-3/2-sized counts (tools/exp_fin.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" libtaub200_fu4b6.so libtaub200_fu2b8.so libtaub200_fu3b6.so; do
  echo "== ${v:-default}" >> gpurun_out/ab_fin.log
  TB_LIB_VARIANT=$v timeout 600 python tools/exp_fin.py >> gpurun_out/ab_fin.log 2>&1
done
