# End-of-session evidence: full GPU suite, bench lines, launch lists, ncu captures of changed kernels.
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
python bench.py > $O/bench_c2.log 2>&1
python bench.py --no-graph --no-cpu --no-aux > $O/bench_c2_eager.log 2>&1
python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
python bench.py --workload C3_w2048 --no-cpu --no-aux > $O/bench_c3_2048.log 2>&1
python bench.py --workload C3_w128 --no-cpu --no-aux > $O/bench_c3_128.log 2>&1
python bench.py --workload C4 --steps 3 --warmup 3 > $O/bench_c4_p1.log 2>&1
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-aux > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gate_prefix_kernel -c 1 -o $O/gate_fwd python profiles/prof_gate.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gate_prefix_bwd -c 1 -o $O/gate_bwd python profiles/prof_gate.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 -o $O/decode_gqa python profiles/prof_decode_gqa.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 -o $O/decode python profiles/prof_decode.py > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:bwd_tc_kernel -c 1 -o $O/bwd python profiles/prof_step.py > /dev/null 2>&1
ls $O
