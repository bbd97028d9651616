# Fuzz of the in-kernel halo on random shapes, plus the full fuzz suite.
O=gpurun_out/s4p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_halo.py -q > $O/fuzz.log 2>&1; echo "rc=$?"; tail -25 $O/fuzz.log | grep -v "^$" | tail -20
