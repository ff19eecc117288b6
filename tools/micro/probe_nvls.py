"""Probe: does this box support NVLS multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED),
can a multicast object be created, and does NCCL pick NVLS? (one process)"""
import ctypes as C
import os
import sys

cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
n = C.c_int()
cu.cuDeviceGetCount(C.byref(n))
print("devices", n.value)
for d in range(n.value):
    dev = C.c_int()
    cu.cuDeviceGet(C.byref(dev), d)
    for name, attr in (("multicast", 132), ("fabric", 128), ("posix_fd", 125 if False else 0)):
        if attr == 0:
            continue
        v = C.c_int(-1)
        rc = cu.cuDeviceGetAttribute(C.byref(v), attr, dev)
        print(f"dev{d} {name} rc={rc} val={v.value}")


class McProp(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                ("flags", C.c_ulonglong)]


ctx = C.c_void_p()
dev = C.c_int()
cu.cuDeviceGet(C.byref(dev), 0)
cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev)
cu.cuCtxSetCurrent(ctx)
prop = McProp(max(1, n.value), 2 << 20, 1, 0)
gran = C.c_size_t()
rc = cu.cuMulticastGetGranularity(C.byref(gran), C.byref(prop), 0)
print("mc granularity min rc", rc, gran.value)
rc = cu.cuMulticastGetGranularity(C.byref(gran), C.byref(prop), 1)
print("mc granularity recommended rc", rc, gran.value)
h = C.c_ulonglong()
rc = cu.cuMulticastCreate(C.byref(h), C.byref(prop))
print("cuMulticastCreate rc", rc)
fd = C.c_int(-1)
rc = cu.cuMemExportToShareableHandle(C.byref(fd), h, 1, 0)
print("export fd rc", rc, fd.value)
try:
    import os
    pidfd = os.pidfd_open(os.getpid())
    print("pidfd_open ok", pidfd)
    SYS_pidfd_getfd = 438
    libc = C.CDLL(None, use_errno=True)
    r = libc.syscall(SYS_pidfd_getfd, pidfd, fd.value, 0)
    print("pidfd_getfd self", r, C.get_errno())
except Exception as e:
    print("pidfd err", e)
print("yama", open("/proc/sys/kernel/yama/ptrace_scope").read().strip() if os.path.exists("/proc/sys/kernel/yama/ptrace_scope") else "none")
