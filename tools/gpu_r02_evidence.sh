#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): measured roofline
# denominators (int8 tcgen05, fp64 DMMA; burst + sustained, clocks sampled),
# compute-sanitizer over every kernel family incl. the int8 path, ncu captures
# of configs 2 and 4.  Outputs in gpurun_out/ (copied to profiles/r02 by hand).
set -u
O=gpurun_out
SMI="nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown --format=csv,noheader -lms 200"
( cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int8_peak int8_peak.cu && \
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu )
$SMI > $O/clk_int8.csv & P=$!; tools/microbench/int8_peak 4 > $O/int8_peak.txt 2>&1; kill $P
$SMI > $O/clk_fp64.csv & P=$!; tools/microbench/fp64_peak > $O/fp64_peak.txt 2>&1; kill $P
if [ "${SAN:-1}" = 1 ]; then
  for t in memcheck racecheck synccheck; do
    timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_probe.py > $O/san_$t.log 2>&1
    echo "sanitizer $t rc=$?" >> $O/san_summary.txt
    tail -3 $O/san_$t.log >> $O/san_summary.txt
  done
fi
if [ "${NCU:-1}" = 1 ]; then
  for c in 2 4; do
    python tools/profile_step.py --config $c --warmup 1 --steps 1 > $O/ps$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file $O/launches_cfg$c.csv python tools/profile_step.py --config $c --warmup 0 --steps 1 > $O/ncu_l$c.log 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tube_fft|paired_spectral" -c 4 \
        -o $O/prof_cfg$c python tools/profile_step.py --config $c --warmup 0 --steps 1 > $O/ncu_f$c.log 2>&1
    echo "ncu cfg$c rc=$?"
  done
fi
