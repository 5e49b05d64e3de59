cd /root/repo
mkdir -p gpurun_out
for ns in 16 12 8; do
QTB_E2E_SLABS=$ns timeout 300 python tools/e2e_prof.py > gpurun_out/e2e_prof_$ns.log 2>&1
done
