# A/B signpack variants (in-tree copies of libtaub200.so): ncu kernel time on config 2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in v0 vA vB; do
TB_LIB_VARIANT=libtaub200_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:signpack -c 5 --csv --log-file gpurun_out/sp_$v.csv python tools/run_path.py --config 2 --reps 5 > /dev/null 2>&1; echo $v=$?
done
