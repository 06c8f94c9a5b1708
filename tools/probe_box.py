import torch, time, os, subprocess
print("nproc", os.cpu_count())
print(subprocess.run("free -g; nvidia-smi; lscpu | head -20", shell=True, capture_output=True, text=True).stdout)
for gb in [1, 4]:
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("H2D GB/s", gb, n / s.elapsed_time(e) / 1e6)
    s.record(); h.copy_(d, non_blocking=True); e.record(); torch.cuda.synchronize()
    print("D2H GB/s", gb, n / s.elapsed_time(e) / 1e6)
    # bidirectional
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.synchronize(); t=time.time()
    with torch.cuda.stream(st): h2.copy_(d2, non_blocking=True)
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print("bidir each GB/s", gb, n/(time.time()-t)/1e9)
t=time.time(); x = torch.empty(32<<30, dtype=torch.uint8, pin_memory=True); print("pin 32GB s", time.time()-t)
