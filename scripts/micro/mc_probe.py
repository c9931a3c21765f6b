"""Does this box support NVSwitch multicast (NVLS) objects? (dev probe)"""
import ctypes as C
cu = C.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
n = C.c_int()
cu.cuDeviceGetCount(C.byref(n))
for d in range(n.value):
    dev = C.c_int()
    cu.cuDeviceGet(C.byref(dev), d)
    vals = {}
    for name, attr in (("multicast", 132), ("fabric_handle", 128), ("posix_fd_handle", 103)):
        v = C.c_int()
        cu.cuDeviceGetAttribute(C.byref(v), attr, dev)
        vals[name] = v.value
    print(f"GPU {d}: {vals}")
