"""Probe: can two processes share cuda:0 through CUDA IPC (compute mode Default)?"""
import sys
import torch
import torch.multiprocessing as mp


def child(q, done):
    torch.cuda.set_device(0)
    t = q.get()            # CUDA tensor received through cudaIpcOpenMemHandle
    t.add_(1.0)
    torch.cuda.synchronize()
    done.put(float(t.sum().item()))


if __name__ == "__main__":
    import subprocess
    print(subprocess.run(["nvidia-smi", "--query-gpu=name,compute_mode,mig.mode.current", "--format=csv"],
                         capture_output=True, text=True).stdout)
    mp.set_start_method("spawn")
    torch.cuda.set_device(0)
    x = torch.zeros(1024, device="cuda")
    q, done = mp.Queue(), mp.Queue()
    p = mp.Process(target=child, args=(q, done))
    p.start()
    q.put(x)
    s = done.get(timeout=120)
    p.join()
    torch.cuda.synchronize()
    print("child sum", s, "parent sees", float(x.sum().item()))
    sys.exit(0 if float(x.sum().item()) == 1024.0 else 1)
