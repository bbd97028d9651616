for i in 1 2; do for v in default prevbwd; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  for W in C2 C3_w512; do GFWA_LIB=$L timeout 60 python tools/time_kernels.py $W bwd 2>&1 | tail -1; done
done; done
