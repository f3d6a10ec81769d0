#!/bin/bash
# Probe the GPU box: host cores/RAM, disks, PCIe links and pinned-copy bandwidth.
out=gpurun_out/probe.txt
{
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== free"; free -g
echo "== df"; df -h / /tmp /root /dev/shm 2>/dev/null
echo "== mounts"; mount | grep -vE 'proc|sysfs|cgroup|devpts|mqueue' | head -40
echo "== lsblk"; lsblk -o NAME,SIZE,TYPE,ROTA,MOUNTPOINT,MODEL 2>/dev/null | head -40
echo "== nvme"; ls /dev/nvme* 2>/dev/null
echo "== nvidia-smi"; nvidia-smi; nvidia-smi topo -m
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current --format=csv
echo "== ulimit -l"; ulimit -l
echo "== torch pinned copy"
python - <<'PY'
import torch, time
torch.cuda.init()
for gib in (1,):
    n = gib << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device='cuda')
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        print(name, gib, "GiB", 5*n/ (e0.elapsed_time(e1)/1e3) / 1e9, "GB/s")
    # bidirectional
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("bidir each", 5*n/dt/1e9, "GB/s")
t=time.perf_counter(); x = torch.empty(8<<30, dtype=torch.uint8, pin_memory=True); print("pin 8GiB alloc s", time.perf_counter()-t)
PY
echo "== disk write/read O_DIRECT"
for d in /tmp /root /dev/shm; do
  f=$d/ddtest.bin
  echo "-- $d"; timeout 120 dd if=/dev/zero of=$f bs=4M count=1024 oflag=direct conv=fsync 2>&1 | tail -1
  timeout 120 dd if=$f of=/dev/null bs=4M iflag=direct 2>&1 | tail -1
  rm -f $f
done
} > $out 2>&1
cat $out | tail -80
