# Sequence-sharded bench path with its new e2e: C4 at N=1, and the N=2 code path over gloo
# with both ranks on cuda:0 (a functional check of the multi-rank bench line, not a scaling number).
O=gpurun_out/s4f; mkdir -p $O
timeout 600 python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu --no-aux > $O/c4.log 2>&1; tail -c 1500 $O/c4.log
GFWA_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-aux > $O/n2_gloo.log 2>&1; tail -c 1500 $O/n2_gloo.log
