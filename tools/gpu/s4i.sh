# Backward dK/dV epilogue: direct row stores (variant epid) vs staged TMA stores (default; both with S^T-first)
O=gpurun_out/s4i; mkdir -p $O
L=paper_2512_07782_b200/variants/libgfwa_epid.so
GFWA_LIB=$L timeout 300 python -m pytest tests/test_gpu_attn.py tests/test_gpu_gqa.py -q -x > $O/tests_epid.log 2>&1; echo "epid tests rc=$?"; tail -2 $O/tests_epid.log
timeout 300 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fuzz.py tests/test_gpu_dist.py -q -x > $O/tests_default.log 2>&1; echo "default tests rc=$?"; tail -2 $O/tests_default.log
for i in 1 2; do for v in default epid; do
  if [ $v = default ]; then LL=""; else LL=$L; fi
  for wl in C2 C3_w512; do GFWA_LIB=$LL timeout 120 python tools/time_kernels.py $wl bwd 2>&1 | tail -1; done
done; done | tee $O/times.log
