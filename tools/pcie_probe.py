import torch, time
torch.cuda.init()
s = torch.cuda.Stream()
for nb in (256<<10, 1<<20, 16<<20, 256<<20):
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device='cuda')
    for direction in ('h2d','d2h'):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction=='h2d' else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            (d.copy_(h, non_blocking=True) if direction=='h2d' else h.copy_(d, non_blocking=True))
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1)*1e3/reps
        print(f"{direction} {nb>>10} KiB: {us:.1f} us/copy, {nb/us/1e3:.1f} GB/s", flush=True)
import subprocess
print(subprocess.run(['nvidia-smi','--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max','--format=csv'],capture_output=True,text=True).stdout)
