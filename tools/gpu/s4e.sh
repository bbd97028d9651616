# NSA selected/compressed-branch kernels with batched key/query rounds: parity, timings, launch list.
O=gpurun_out/s4e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_nsa.py -q -x > $O/tests.log 2>&1; tail -3 $O/tests.log
timeout 300 python tools/gpu/nsa_time.py 2>&1 | tail -2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/launches_nsa.csv python profiles/prof_nsa.py > /dev/null 2>&1
python tools/ncu_launches.py $O/launches_nsa.csv 2>/dev/null | head -14
