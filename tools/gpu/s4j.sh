# Session-4 final evidence: smoke, full GPU suite, bench lines, launch list, ncu of the backward main kernel.
O=gpurun_out/s4j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_c2.log 2>&1
timeout 300 python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
timeout 300 python bench.py --workload C4 --steps 3 --no-cpu --no-aux > $O/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-aux > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_C3_w512.csv python profiles/prof_step.py C3_w512 > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:bwd_tc_kernel -s 1 -c 1 -o $O/bwd python profiles/prof_step.py C2 > /dev/null 2>&1
ls $O
