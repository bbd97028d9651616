#!/bin/bash
# Round-2 profiles: launch lists (time + dram bytes per launch) of one training
# step at C2 and C3 w=512, and one ncu --set full capture per hot kernel.
set -x
mkdir -p gpurun_out/r02
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for W in C2 C3_w512; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02/launches_$W.csv python profiles/prof_step.py $W > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_tc_kernel -s 1 -c 1 -o gpurun_out/r02/fwd python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd_tc_kernel -s 1 -c 1 -o gpurun_out/r02/bwd python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_tc_pre|bwd_tc_post|gate_prefix_kernel" -s 3 -c 3 -o gpurun_out/r02/aux python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:decode_kernel -c 2 -o gpurun_out/r02/decode python profiles/prof_decode.py > /dev/null 2>&1
ls -la gpurun_out/r02
