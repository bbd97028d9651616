# Backward: S^T(g) issued before the wait for dQ^T(g-2)'s drain (variant sfirst) vs default.
O=gpurun_out/s4h; mkdir -p $O
L=paper_2512_07782_b200/variants/libgfwa_sfirst.so
GFWA_LIB=$L timeout 300 python -m pytest tests/test_gpu_attn.py -q -x -k "bf16 or c2 or C3 or invariant" > $O/tests_sfirst.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests_sfirst.log
for i in 1 2; do for v in default sfirst; do
  if [ $v = default ]; then LL=""; else LL=$L; fi
  for wl in C2 C3_w512; do GFWA_LIB=$LL timeout 120 python tools/time_kernels.py $wl bwd 2>&1 | tail -1; done
done; done | tee $O/times.log
