# In-kernel halo: its GPU tests, regression of the attention suite, timing of the unchanged path.
O=gpurun_out/s4k; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_halo.py -q -x > $O/halo.log 2>&1; echo "halo rc=$?"; tail -30 $O/halo.log | grep -v "^$" | tail -25
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fuzz.py tests/test_gpu_dist.py tests/test_gpu_gqa.py tests/test_gpu_graph.py -q > $O/attn.log 2>&1; echo "attn rc=$?"; tail -2 $O/attn.log
for wl in C2 C3_w512; do timeout 120 python tools/time_kernels.py $wl both 2>&1 | tail -2; done
