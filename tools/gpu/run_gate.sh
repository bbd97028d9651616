for lib in "" paper_2512_07782_b200/variants/libgfwa_kv16.so paper_2512_07782_b200/variants/libgfwa_kv32.so; do
GFWA_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg.csv python profiles/prof_gate.py > /dev/null 2>&1; echo "lib=$lib"; python tools/ncu_launches.py gpurun_out/lg.csv | grep gate
done
GFWA_LIB=paper_2512_07782_b200/variants/libgfwa_kv16.so timeout 300 python -m pytest tests/test_gpu_gate.py -q -x 2>&1 | tail -1
