O=gpurun_out/s3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1
python bench.py > $O/bench_c2.log 2>&1
python bench.py --workload C3_w512 --no-cpu --no-aux > $O/bench_c3_512.log 2>&1
python tools/time_kernels.py > $O/time_kernels.log 2>&1
ls $O
