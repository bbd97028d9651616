# Sequence-sharded step with the in-kernel peer halo (2 ranks, gloo, both on cuda:0, K/V halo by CUDA IPC)
O=gpurun_out/s4l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_halo.py -q > $O/dist.log 2>&1; echo "rc=$?"; tail -25 $O/dist.log | grep -v "^$" | tail -20
