# Session-3 end-of-round evidence: smoke, full GPU suite, bench lines, refreshed normgate profile.
O=gpurun_out/final3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
timeout 600 python bench.py > $O/bench_c2.log 2>&1
timeout 300 python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_tc_kernel|pre_normgate|normgate_y" -s 3 -c 3 -o $O/normgate python profiles/prof_normgate.py > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_normgate.csv python profiles/prof_normgate.py > /dev/null 2>&1
for f in smoke.log gpu_tests.log; do tail -n 2 $O/$f; done
