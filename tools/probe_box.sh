nvidia-smi; free -g; nproc; lscpu | head -30; df -h /dev/shm /tmp . | cat
python - <<'PY'
import numpy as np, time, torch
x=np.array([0x7FC00001,0x7F800001,0xFFA00000,0x7F7FFFFF,0x477FF000,0x33000000,0x33000001],dtype=np.uint32).view(np.float32)
print([hex(v) for v in x.astype(np.float16).view(np.uint16)])
np.show_config() if False else None
print(torch.cuda.get_device_properties(0))
free,total=torch.cuda.mem_get_info(); print("mem", free/1e9, total/1e9)
for gb in (1,8,32):
    t=time.time(); a=torch.empty(gb<<30,dtype=torch.uint8,pin_memory=True); print("pin",gb,"GB",time.time()-t)
    d=torch.empty(gb<<30,dtype=torch.uint8,device="cuda")
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(a,non_blocking=True); e.record(); torch.cuda.synchronize(); print("h2d GB/s",(gb<<30)/s.elapsed_time(e)/1e6)
    s.record(); a.copy_(d,non_blocking=True); e.record(); torch.cuda.synchronize(); print("d2h GB/s",(gb<<30)/s.elapsed_time(e)/1e6)
    del a,d
PY
