for i in 1 2; do for v in default ld32; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  for W in C2 C3_w512 C3_w2048; do GFWA_LIB=$L timeout 60 python tools/time_kernels.py $W fwd 2>&1 | tail -1; done
done; done
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_normgate.py -x -q 2>&1 | tail -2
