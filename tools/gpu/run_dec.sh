for lib in ""; do
GFWA_LIB=$lib timeout 300 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
GFWA_LIB=$lib python - <<'P'
import os, torch, synth
from paper_2512_07782_b200 import binding as gb
c = synth.CONFIGS["C5"]; B,H,d,w = c["B"],c["H"],c["d"],c["w"]
Kc,Vc,a,q,k,v,an = synth.decode_inputs(B,H,d,w,seed=1,device="cuda")
Uc = -torch.cumsum(a,-1); pos = torch.full((B,), w+17, dtype=torch.int64, device="cuda")
for _ in range(3): gb.gfwa_decode(q,k,v,an,Kc,Vc,Uc,pos)
e0,e1 = torch.cuda.Event(True), torch.cuda.Event(True); torch.cuda.synchronize(); e0.record()
for _ in range(20): gb.gfwa_decode(q,k,v,an,Kc,Vc,Uc,pos)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/20
print(os.environ.get("GFWA_LIB") or "default", "C5", round(ms,4), "ms", round(B*H*(4*w*d+4*w+8*d)/ms/1e6,1), "GB/s")
P
done
