cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s -C oracle > /dev/null 2>&1
STRESS_SECONDS=900 timeout 1200 python tools/stress_parity.py 1 > gpurun_out/r2bj_stress1.log 2>&1; echo s1=$?
STRESS_SECONDS=600 timeout 900 python tools/stress_parity.py 2 > gpurun_out/r2bj_stress2.log 2>&1; echo s2=$?
