# The N=2 bench path with the opt-in in-kernel peer halo (gloo, both ranks on cuda:0: a functional check only).
O=gpurun_out/s4n; mkdir -p $O
GFWA_PEER_HALO=1 GFWA_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --workload C4 --steps 3 --warmup 3 --no-aux > $O/n2_peer.log 2>&1; echo "rc=$?"; tail -c 1500 $O/n2_peer.log
