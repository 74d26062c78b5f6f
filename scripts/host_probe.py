"""Exploration probe of the GPU box's host side: CPU, NUMA, PCIe link
(pinned H2D / D2H / both directions at once) and host memory copy bandwidth
at 1..16 threads. Output: one JSON object (profiles/r2_host_probe.json)."""
import json, os, subprocess, threading, time, ctypes
import numpy as np
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = os.cpu_count()
out["sched_affinity"] = sorted(os.sched_getaffinity(0))
out["lscpu"] = sh("lscpu")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node")
out["meminfo"] = sh("head -5 /proc/meminfo")
out["topo"] = sh("nvidia-smi topo -m")
out["mps"] = sh("ls /tmp/nvidia-mps 2>&1; pgrep -l nvidia-cuda-mps 2>&1")
out["thp"] = sh("cat /sys/kernel/mm/transparent_hugepage/enabled")

dev = torch.device("cuda:0")
def pcie(nbytes, reps=10):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "bidir"):
        for _ in range(2):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            for _ in range(reps):
                if name in ("h2d", "bidir"):
                    with torch.cuda.stream(s1):
                        d.copy_(h, non_blocking=True)
                if name in ("d2h", "bidir"):
                    with torch.cuda.stream(s2):
                        h2.copy_(d2, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        res[name + "_gbs"] = (reps * nbytes * (2 if name == "bidir" else 1)) / dt / 1e9
    return res
for mb in (8, 64, 256):
    out[f"pcie_{mb}MiB"] = pcie(mb << 20)

# host memory copy bandwidth: numpy copyto releases the GIL
def hostcopy(threads, nbytes=256 << 20, reps=4):
    srcs = [np.ones(nbytes, dtype=np.uint8) for _ in range(threads)]
    dsts = [np.zeros(nbytes, dtype=np.uint8) for _ in range(threads)]
    def run(i):
        for _ in range(reps):
            np.copyto(dsts[i], srcs[i])
    ts = [threading.Thread(target=run, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts: t.start()
    for t in ts: t.join()
    dt = time.perf_counter() - t0
    return threads * reps * nbytes / dt / 1e9
out["host_memcpy_gbs_by_threads"] = {t: hostcopy(t) for t in (1, 2, 4, 8, 16)}
print(json.dumps(out, indent=1))
