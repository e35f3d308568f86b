"""One-off probe of the GPU box: host memory, cores, NUMA, H2D link bandwidth."""
import os, time, json, subprocess
import torch

out = {}
out["cores_affinity"] = len(os.sched_getaffinity(0))
out["cpu_count"] = os.cpu_count()
with open("/proc/meminfo") as f:
    mi = {l.split(":")[0]: l.split(":")[1].strip() for l in f}
out["MemTotal"] = mi["MemTotal"]; out["MemAvailable"] = mi["MemAvailable"]
out["Hugepagesize"] = mi.get("Hugepagesize")
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
except Exception as e:
    out["lscpu"] = str(e)
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["smi"] = subprocess.run(["nvidia-smi", "-q", "-d", "PCI,CLOCK,MEMORY"], capture_output=True, text=True).stdout[:6000]
out["shm"] = subprocess.run(["df", "-h", "/dev/shm"], capture_output=True, text=True).stdout
out["numa"] = subprocess.run(["bash", "-c", "ls /sys/devices/system/node/; cat /sys/devices/system/node/node*/meminfo | grep MemTotal"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
res = {}
for gib in (0.25, 1, 4):
    n = int(gib * (1 << 30))
    t0 = time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); t_pin = time.time() - t0
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    best = 0; best_d2h = 0
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        e1.synchronize(); bw = n / (e0.elapsed_time(e1) * 1e-3) / 1e9; best = max(best, bw)
        with torch.cuda.stream(s):
            e0.record(); h.copy_(d, non_blocking=True); e1.record()
        e1.synchronize(); bw = n / (e0.elapsed_time(e1) * 1e-3) / 1e9; best_d2h = max(best_d2h, bw)
    res[str(gib)] = {"h2d_GBps": best, "d2h_GBps": best_d2h, "pin_alloc_s": t_pin}
    del h, d
out["copy"] = res
# big pinned alloc via cudaHostRegister of an mmap (simulate 32 GiB)
import ctypes, mmap
cudart = ctypes.CDLL("libcudart.so.12") if False else None
t0 = time.time()
big = torch.empty(32 << 30, dtype=torch.uint8)
t1 = time.time()
r = torch.cuda.cudart().cudaHostRegister(big.data_ptr(), big.numel(), 0)
t2 = time.time()
out["register_32GiB"] = {"alloc_s": t1 - t0, "register_s": t2 - t1, "rc": int(r)}
d = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(8):
    d.copy_(big[i * (4 << 30):(i + 1) * (4 << 30)], non_blocking=True)
e1.record(); e1.synchronize()
out["register_32GiB"]["h2d_GBps_32GiB"] = (32 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
