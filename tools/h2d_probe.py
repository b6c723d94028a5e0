"""Pinned H2D bandwidth: one stream vs several concurrent streams (copy engines)."""
import torch

N = 64 << 20
x = torch.empty(N, dtype=torch.uint8).pin_memory()
y = torch.empty(N, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunk = N // k
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                y[i * chunk:(i + 1) * chunk].copy_(x[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            e1.wait(s) if hasattr(e1, "wait") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{k} stream(s): {N / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
