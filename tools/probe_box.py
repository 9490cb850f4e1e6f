"""One-off probe of a GPU box: topology, VMM/multicast attributes, NCCL busbw (torch)."""
import ctypes, os, subprocess, sys, json
out = {}
def sh(c):
    try: return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e: return str(e)
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,memory.total --format=csv")
out["fabric"] = sh("nvidia-smi -q | grep -i -A3 fabric | head -20")
out["nvlink"] = sh("nvidia-smi nvlink -s -i 0 | head -24")
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = ctypes.c_int(); cu.cuDeviceGetCount(ctypes.byref(n))
attrs = {"vmm":102, "posix_fd":103, "fabric":128, "multicast":132}
for d in range(n.value):
    dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), d)
    r = {}
    for k, a in attrs.items():
        v = ctypes.c_int(); cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev); r[k] = v.value
    out[f"dev{d}"] = r
out["cpus"] = len(os.sched_getaffinity(0))
print(json.dumps(out, indent=1))
