for i in 1 2; do for lib in "" paper_2512_07782_b200/variants/libgfwa_fpoly1.so paper_2512_07782_b200/variants/libgfwa_fpoly2.so; do
GFWA_LIB=$lib python tools/time_kernels.py C2 fwd; GFWA_LIB=$lib python tools/time_kernels.py C3_w2048 fwd; done; done
