import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2410_15526_b200 import Comm
dev = torch.device("cuda", 0)
D = synth.padded_numel(synth.gpt_numel("1.3B"), 1, 128)
comm = Comm()
w_model = synth.model_weights(D, seed=1, device=dev)
w_main = synth.main_weights(w_model, seed=2)
grad = synth.gradient(D, seed=3, device=dev, dtype=torch.bfloat16)
out = torch.empty(D, device=dev)
ws_q = torch.empty(comm.qwd_workspace_bytes(D, 4, 128), dtype=torch.uint8, device=dev)
ws3 = torch.empty(comm.tlq_workspace_bytes(D, 8, 4, 128), dtype=torch.uint8, device=dev)
comm.set_local_fusion(False)
def step():
    comm.qwd_step(w_main, w_model, ws_q, 4, 128)
    comm.tlq_hs_reduce_scatter(grad, out, ws3, 8, 4, 128, 64, True)
for order in ("first", "after_fused"):
    if order == "after_fused":
        comm.set_local_fusion(True)
        for _ in range(20): step()
        comm.set_local_fusion(False)
    for _ in range(3): step()
    comm.profile_enable(True); comm.profile_read()
    torch.cuda.synchronize()
    for _ in range(20): step()
    torch.cuda.synchronize()
    p = comm.profile_read(); comm.profile_enable(False)
    print(order, {k: round(v[0] / v[1], 4) for k, v in p.items()})
