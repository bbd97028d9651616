for v in default e1 e2 e5 nodq noduq; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  GFWA_LIB=$L timeout 120 python tools/time_kernels.py C2 bwd 2>&1 | tail -1
done
