#!/bin/bash
# Round-2 final profiles: launch lists (time + DRAM bytes per launch) of one training
# step at C2 and C3 w=512 and of the bench command, and one ncu --set full capture
# per hot kernel (each command was run without ncu first in the same session).
O=gpurun_out/r02f; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for W in C2 C3_w512; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_$W.csv python profiles/prof_step.py $W > /dev/null 2>&1
done
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-aux > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:fwd_tc_kernel -s 1 -c 1 -o $O/fwd python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 900 ncu $F -k regex:bwd_tc_kernel -s 1 -c 1 -o $O/bwd python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 900 ncu $F -k regex:bwd_tc_kernel -s 1 -c 1 -o $O/bwd_c3 python profiles/prof_step.py C3_w512 > /dev/null 2>&1
timeout 900 ncu $F -k regex:"bwd_tc_pre|bwd_tc_post|gate_prefix_kernel" -s 3 -c 3 -o $O/aux python profiles/prof_step.py C2 > /dev/null 2>&1
timeout 900 ncu $F -k regex:"fwd_tc_kernel|pre_normgate" -s 2 -c 2 -o $O/normgate python profiles/prof_normgate.py > /dev/null 2>&1
timeout 600 ncu $F -k regex:decode_kernel -c 1 -o $O/decode python profiles/prof_decode.py > /dev/null 2>&1
ls -la $O
