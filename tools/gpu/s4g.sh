# The N>1 bench lines end to end (gloo, both ranks on cuda:0: a functional check, not a
# scaling number): sequence-sharded C4 headline with e2e + roofline, the batch-sharded C2
# aux, and the reference arm under torchrun; plus C4 at N=1.
O=gpurun_out/s4g; mkdir -p $O
timeout 600 python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu --no-aux > $O/c4.log 2>&1; tail -c 900 $O/c4.log
GFWA_BENCH_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 > $O/n2_gloo.log 2>&1; tail -c 3000 $O/n2_gloo.log
timeout 600 python bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > $O/ref_n2.log 2>&1; echo "ref rc=$?"; tail -c 800 $O/ref_n2.log
