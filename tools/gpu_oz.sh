cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/e2e_prof.py > gpurun_out/e2e_prof.log 2>&1; echo "rc=$?" >> gpurun_out/e2e_prof.log
