# Session-4 re-entry check: smoke, full GPU suite, bench lines at C2 and the north_star point.
O=gpurun_out/s4a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1
timeout 600 python bench.py > $O/bench_c2.log 2>&1
timeout 300 python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
for f in smoke.log gpu_tests.log; do tail -n 3 $O/$f; done
tail -c 600 $O/bench_c3_512.log
