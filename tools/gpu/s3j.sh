O=gpurun_out/s3j; mkdir -p $O
for W in C2 C3_w512; do timeout 120 python tools/time_kernels.py $W bwd 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/gpu/sanitize.py > $O/san_$T.log 2>&1; echo "$T rc=$?"; tail -4 $O/san_$T.log
done
