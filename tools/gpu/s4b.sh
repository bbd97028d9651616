# Gate scan: cp.async-staged tile load (default) vs register batches (nocp), geometry sweep.
O=gpurun_out/s4b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gate.py -q -x > $O/gate_tests.log 2>&1; tail -2 $O/gate_tests.log
for geom in "" "3,10" "3,9" "2,10" "4,9" "5,8" "4,8" "2,9"; do
  for v in default nocp; do
    if [ $v = default ]; then L=""; else L=paper_2512_07782_b200/variants/libgfwa_$v.so; fi
    echo "geom=$geom lib=$v: $(GFWA_GATE_GEOM=$geom GFWA_LIB=$L timeout 120 python tools/gpu/gate_time.py 2>&1 | tr '\n' ' ')"
  done
done | tee $O/sweep.log
