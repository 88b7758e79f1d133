set -x
nproc; lscpu | head -30; free -g; df -h /dev/shm /tmp / ; mount | grep -E "shm|tmp|nvme| / " ; lsblk 2>/dev/null | head -40
nvidia-smi; nvidia-smi topo -m; numactl -H 2>/dev/null || cat /sys/devices/system/node/node*/cpulist
cat /proc/meminfo | head -20; cat /sys/kernel/mm/transparent_hugepage/enabled; cat /sys/kernel/mm/transparent_hugepage/shmem_enabled
uname -a; which fio; ulimit -a
python -c "import torch;print(torch.cuda.device_count())"
ls /dev/nvme* 2>/dev/null; cat /proc/mounts
python - <<'PY'
import torch, time
x = torch.empty(1<<30, dtype=torch.uint8, device='cuda')
h = torch.empty(1<<30, dtype=torch.uint8, pin_memory=True)
for _ in range(3): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
t=time.time()
for _ in range(5): h.copy_(x, non_blocking=True)
torch.cuda.synchronize(); print("D2H GB/s", 5*(1<<30)/(time.time()-t)/1e9)
t=time.time()
for _ in range(5): x.copy_(h, non_blocking=True)
torch.cuda.synchronize(); print("H2D GB/s", 5*(1<<30)/(time.time()-t)/1e9)
import os
t=time.time()
with open('/dev/shm/probe.bin','wb') as f:
    for _ in range(4): f.write(memoryview(h.numpy()))
print("tmpfs write 1 thread GB/s", 4*(1<<30)/(time.time()-t)/1e9)
t=time.time()
with open('/dev/shm/probe.bin','rb') as f:
    while f.readinto(memoryview(h.numpy())): pass
print("tmpfs read 1 thread GB/s", 4*(1<<30)/(time.time()-t)/1e9)
os.unlink('/dev/shm/probe.bin')
PY
