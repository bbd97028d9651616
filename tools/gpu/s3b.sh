O=gpurun_out/s3b; mkdir -p $O
timeout 120 python tools/time_kernels.py C2 bwd > $O/t_c2_first.log 2>&1; echo "rc=$?" >> $O/t_c2_first.log
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q > $O/attn.log 2>&1
for W in C2 C3_w512 C3_w2048; do timeout 120 python tools/time_kernels.py $W bwd >> $O/time.log 2>&1; done
tail -3 $O/attn.log; cat $O/t_c2_first.log $O/time.log
