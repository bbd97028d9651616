O=gpurun_out/s3c; mkdir -p $O
timeout 120 python tools/time_kernels.py C2 bwd > $O/time.log 2>&1; echo "rc=$?" >> $O/time.log
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q > $O/attn.log 2>&1
for W in C3_w512 C3_w2048; do timeout 120 python tools/time_kernels.py $W bwd >> $O/time.log 2>&1; done
GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_btrace.so timeout 200 python tools/gpu/trace_bwd4.py C2 > $O/trace.log 2>&1
tail -3 $O/attn.log; cat $O/time.log; head -30 $O/trace.log; tail -3 $O/trace.log
