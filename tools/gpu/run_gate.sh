timeout 600 python -m pytest tests/test_gpu_gate.py -x -q 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lv.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2512_07782_b200 import binding as gb
c=synth.CONFIGS['G']; h,b=synth.gate_inputs(c['B'],c['N'],c['H'],seed=1,device='cuda'); h,b=h.bfloat16(),b.bfloat16()
for _ in range(2): gb.gfwa_gate_prefix_variant(2,h,b)
torch.cuda.synchronize()" > /dev/null 2>&1; python tools/ncu_launches.py gpurun_out/lv.csv | grep gate_v2
