import os, subprocess, time, torch
print("nproc", os.cpu_count())
print(subprocess.run("free -g; nvidia-smi --query-gpu=name,memory.total,memory.free,clocks.max.sm --format=csv; lscpu | grep -E 'Model name|Socket|Thread|Core|NUMA'", shell=True, capture_output=True, text=True).stdout)
fr, tot = torch.cuda.mem_get_info()
print("cuda mem free/total GB", fr/1e9, tot/1e9)
t=time.time(); x = torch.empty(16<<30, dtype=torch.uint8, pin_memory=True); print("pin 16GiB s", time.time()-t)
