import torch
from paper_2512_07782_b200 import binding as gb
g = torch.Generator(device="cuda").manual_seed(0)
Q = (0.3*torch.randn(128, 128, generator=g, device="cuda")).bfloat16()
K = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
V = torch.randn(128, 128, generator=g, device="cuda").bfloat16()
for fl in (0, 1):
    S, O = gb.gfwa_debug_tc_selftest(Q, K, V, fl)
    torch.cuda.synchronize()
    Ob = S.bfloat16().float() @ V.float()
    Oh = S.half().float() @ V.float()
    print("flags", fl, "err vs bf16P", (O-Ob).abs().max().item(), "err vs f16P", (O-Oh).abs().max().item(), "max|O|", O.abs().max().item())
