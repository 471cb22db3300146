set -x
nvidia-smi
nvidia-smi topo -m
lscpu
numactl -H || true
cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c
ulimit -l
free -g
nproc
cat /proc/meminfo | head -5
python - <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
n=1<<30
d=torch.empty(n,dtype=torch.uint8,device='cuda')
for sz in [1<<24, 1<<28, 1<<30]:
  h=torch.empty(sz,dtype=torch.uint8,pin_memory=True)
  best=1e9
  for i in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); h.copy_(d[:sz],non_blocking=True); e.record(); e.synchronize()
    best=min(best,s.elapsed_time(e))
  print('D2H',sz, sz/best/1e6,'GB/s')
  best=1e9
  for i in range(10):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record(); d[:sz].copy_(h,non_blocking=True); e.record(); e.synchronize()
    best=min(best,s.elapsed_time(e))
  print('H2D',sz, sz/best/1e6,'GB/s')
t=time.time(); h=torch.empty(4<<30,dtype=torch.uint8,pin_memory=True); print('pin 4GiB s',time.time()-t)
PY
