# Forward one-pass softmax (default) vs the two-pass walk (variant tp): parity, then timings.
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fuzz.py tests/test_gpu_normgate.py tests/test_gpu_gqa.py tests/test_gpu_graph.py -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
for i in 1 2; do for v in default tp; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  for wl in C2 C3_w512 C3_w2048 C3_w128; do GFWA_LIB=$L timeout 120 python tools/time_kernels.py $wl fwd 2>&1 | tail -1; done
  echo "$v: $(GFWA_LIB=$L timeout 120 python tools/gpu/fwd_train_time.py C2 C3_w512 2>&1 | tr '\n' ' ')"
done; done | tee $O/times.log
