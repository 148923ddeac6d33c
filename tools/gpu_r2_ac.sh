# Host record expansion probe (tb_expand_records) alone and next to a D2H stream.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/probe_expand.py > gpurun_out/r2ac_probe_expand.log 2>&1; echo probe=$?
nproc >> gpurun_out/r2ac_probe_expand.log; lscpu | head -20 >> gpurun_out/r2ac_probe_expand.log; free -g >> gpurun_out/r2ac_probe_expand.log
