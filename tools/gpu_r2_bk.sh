cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s -C oracle > /dev/null 2>&1
for s in 3 4 5 6 7 8; do STRESS_SECONDS=300 timeout 600 python tools/stress_parity.py $s > gpurun_out/r2bk_stress$s.log 2>&1; echo s$s=$?; done
