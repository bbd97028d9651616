# Gate scan: softplus from MUFU.EX2 + MUFU.LG2 (variant lg2) vs the accurate series (default): parity and time.
O=gpurun_out/s4o; mkdir -p $O
L=paper_2512_07782_b200/variants/libgfwa_lg2.so
GFWA_LIB=$L timeout 600 python -m pytest tests/test_gpu_gate.py tests/test_gpu_attn.py -k "gate or end_to_end" -q > $O/tests_lg2.log 2>&1; echo "lg2 tests rc=$?"; tail -3 $O/tests_lg2.log
for i in 1 2; do for v in default lg2; do
  if [ $v = default ]; then LL=""; else LL=$L; fi
  echo "$v: $(GFWA_LIB=$LL timeout 120 python tools/gpu/gate_time.py 2>&1 | tr '\n' ' ')"
done; done
