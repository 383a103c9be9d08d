import sys, torch
sys.path.insert(0, ".")
from paper_2410_15526_b200 import emu_tlq_hs_reduce_scatter, emu_tlq_workspace_bytes
M, N, mb = 2, 1, 1
D = mb << 18
P = M * N
S = D // P
g = [torch.randn(D, device="cuda").to(torch.bfloat16) for _ in range(P)]
o = [torch.empty(S, device="cuda") for _ in range(P)]
ws = torch.empty(emu_tlq_workspace_bytes(M, N, D, 8, 4, 128), dtype=torch.uint8, device="cuda")
for i in range(6):
    emu_tlq_hs_reduce_scatter(M, N, g, o, ws, 8, 4, 128, 64, fresh=(i == 0))
torch.cuda.synchronize()
print("ok")
