O=gpurun_out/s3h; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_tc_kernel -s 1 -c 1 -o $O/fwd python profiles/prof_step.py C2 > $O/ncu_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_tc_kernel -s 1 -c 1 -o $O/bwd python profiles/prof_step.py C2 > $O/ncu_bwd.log 2>&1
ls -la $O
