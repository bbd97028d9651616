for i in 1 2; do for v in default pre1 pre4; do
  if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
  GFWA_LIB=$L timeout 60 python tools/time_kernels.py C2 bwd 2>&1 | tail -1
done; done
for v in pre1 pre4; do GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pre_flat -c 2 --csv python profiles/prof_step.py C2 2>/dev/null | grep pre_flat | cut -c1-20,200-; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pre_flat -c 2 --csv python profiles/prof_step.py C2 2>/dev/null | grep -o '"gpu__time_duration.sum","usecond","[0-9.]*"'
