"""Box probe: host cores/RAM/topology, pinned H2D GB/s,
pin time, host DRAM bandwidth, device properties. Writes gpurun_out/box_probe.json."""
import ctypes, json, os, subprocess, sys, time, glob

out = {}
def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return f"ERR {e}"

out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
out["lscpu"] = sh("lscpu | head -30")
out["free_g"] = sh("free -g")
out["ulimit_l"] = sh("ulimit -l").strip()
out["topo"] = sh("nvidia-smi topo -m")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node/")
out["smi"] = sh("nvidia-smi --query-gpu=index,name,pci.bus_id,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current --format=csv")
print(out["free_g"], out["nproc"], out["ulimit_l"], flush=True)

import torch
p = torch.cuda.get_device_properties(0)
out["dev"] = dict(name=p.name, sms=p.multi_processor_count, total_mem=p.total_memory,
                  l2=getattr(p, "L2_cache_size", None))
cudart_path = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(cudart_path[0])
def host_alloc(nbytes):
    ptr = ctypes.c_void_p()
    t0 = time.time()
    err = rt.cudaHostAlloc(ctypes.byref(ptr), ctypes.c_size_t(nbytes), ctypes.c_uint(1))  # portable
    return err, ptr, time.time() - t0

torch.cuda.init(); torch.zeros(1, device="cuda")
# H2D bandwidth at chunk sizes, 352 MB expert
EXP = 352321536
err, hp, t_alloc = host_alloc(EXP)
out["pin_352MB_s"] = t_alloc
# touch
ctypes.memset(hp, 1, EXP)
dev = torch.empty(EXP, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
res = {}
for chunk_mb in [2, 8, 32, 128, 336]:
    chunk = chunk_mb << 20
    best = 0
    for rep in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            off = 0
            while off < EXP:
                n = min(chunk, EXP - off)
                rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr() + off), ctypes.c_void_p(hp.value + off), ctypes.c_size_t(n), 1, ctypes.c_void_p(s.cuda_stream))
                off += n
            e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, EXP / ms / 1e6)
    res[chunk_mb] = best
out["h2d_GBps_by_chunkMB"] = res
print("h2d", res, flush=True)
# D2H
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); rt.cudaMemcpyAsync(hp, ctypes.c_void_p(dev.data_ptr()), ctypes.c_size_t(EXP), 2, ctypes.c_void_p(0)); e1.record(); torch.cuda.synchronize()
out["d2h_GBps"] = EXP / e0.elapsed_time(e1) / 1e6
# two concurrent streams
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
half = EXP // 2
s.wait_event(e0); s2.wait_event(e0)
rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr()), hp, ctypes.c_size_t(half), 1, ctypes.c_void_p(s.cuda_stream))
rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr() + half), ctypes.c_void_p(hp.value + half), ctypes.c_size_t(half), 1, ctypes.c_void_p(s2.cuda_stream))
ee = torch.cuda.Event(); ee.record(s); torch.cuda.current_stream().wait_event(ee)
ee2 = torch.cuda.Event(); ee2.record(s2); torch.cuda.current_stream().wait_event(ee2)
e1.record(); torch.cuda.synchronize()
out["h2d_2streams_GBps"] = EXP / e0.elapsed_time(e1) / 1e6
rt.cudaFreeHost(hp)

# pin time for larger sizes, bounded by free RAM
import re
m = re.search(r"Mem:\s+(\d+)\s+(\d+)\s+(\d+)\s+\d+\s+\d+\s+(\d+)", out["free_g"])
avail_g = int(m.group(4)) if m else 0
out["avail_g"] = avail_g
pins = {}
for gb in [8, 32, 96]:
    if gb * 1.3 > avail_g:
        break
    err, p2, t = host_alloc(gb << 30)
    pins[gb] = dict(err=err, alloc_s=t)
    if err == 0:
        t0 = time.time(); ctypes.memset(p2, 0, gb << 30); pins[gb]["memset_s"] = time.time() - t0
        rt.cudaFreeHost(p2)
    print("pin", gb, pins[gb], flush=True)
out["pins"] = pins
# host DRAM bandwidth (torch CPU copy, all threads)
torch.set_num_threads(out["affinity"])
a = torch.empty(4 << 30, dtype=torch.uint8); b = torch.empty_like(a); a.fill_(1); b.fill_(2)
best = 0
for _ in range(3):
    t0 = time.time(); b.copy_(a); dt = time.time() - t0; best = max(best, 2 * a.numel() / dt / 1e9)
out["host_copy_GBps_rw"] = best
best = 0
af = a.view(torch.float32)
for _ in range(3):
    t0 = time.time(); s_ = af.sum(); dt = time.time() - t0; best = max(best, a.numel() / dt / 1e9)
out["host_read_GBps"] = best
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/box_probe.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "topo")}, indent=1))
print(out["lscpu"]); print(out["topo"])
