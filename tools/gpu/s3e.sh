for v in default dqred; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  GFWA_LIB=$L timeout 120 python tools/time_kernels.py C2 bwd 2>&1 | tail -1
  GFWA_LIB=$L timeout 120 python tools/time_kernels.py C3_w512 bwd 2>&1 | tail -1
done
GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_dqred.so timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2
