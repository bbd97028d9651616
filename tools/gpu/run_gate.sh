for lib in "" paper_2512_07782_b200/variants/libgfwa_m3.so paper_2512_07782_b200/variants/libgfwa_m5.so paper_2512_07782_b200/variants/libgfwa_m6.so; do
GFWA_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lg.csv python profiles/prof_gate.py > /dev/null 2>&1; echo "lib=$lib"; python tools/ncu_launches.py gpurun_out/lg.csv | grep gate
done
