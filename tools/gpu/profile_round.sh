# Round profile capture: bench lines, ncu launch lists (C2 bench, C3_w512 step), --set full captures.
set -x
O=gpurun_out/prof; mkdir -p $O
python bench.py > $O/bench_c2.log 2>&1
python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
python bench.py --workload C3_w2048 --no-cpu --no-aux > $O/bench_c3_2048.log 2>&1
python bench.py --workload C3_w128 --no-cpu --no-aux > $O/bench_c3_128.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_c3_512.csv python profiles/prof_step.py C3_w512 > /dev/null 2>&1
for k in bwd_tc_kernel fwd_tc_kernel bwd_tc_pre_flat_kernel bwd_tc_post_flat_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/$k python profiles/prof_step.py > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:gate_prefix_kernel -c 1 -o $O/gate_fwd python profiles/prof_gate.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gate_prefix_bwd -c 1 -o $O/gate_bwd python profiles/prof_gate.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:decode -c 1 -o $O/decode python profiles/prof_decode.py > /dev/null 2>&1
ls -la $O
