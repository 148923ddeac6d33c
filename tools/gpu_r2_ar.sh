# K4: more ALU -> FMA moves (merge-loop max as IMADs, pad term as mul.hi, leaf tags as IMAD / mul.hi).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TB_LIB_VARIANT=libtaub200_all3.so timeout 1200 python -m pytest tests -m gpu -q -x -k "merge or config4" > gpurun_out/r2ar_pt_all3.log 2>&1; echo pt=$?
for rep in 1 2; do
for v in "" libtaub200_lmax.so libtaub200_lhi.so libtaub200_lboth.so libtaub200_tag.so libtaub200_all3.so; do
  tag=${v:-new}
  TB_LIB_VARIANT=$v timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --e2e-tau-steps 0 > gpurun_out/r2ar_c4_${tag}_$rep.json 2>&1; echo c4_$tag=$?
done
done
