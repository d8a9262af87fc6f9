#!/usr/bin/env python
"""Diagnostics: multicast-object support on this box (driver API via ctypes): attributes, then
cuMulticastCreate for numDevices x handleTypes combinations."""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
cu.cuCtxSetCurrent(ctx)
for name, attr in [("MULTICAST", 132), ("FABRIC", 128), ("POSIX_FD", 103), ("VMM", 102)]:
    v = ctypes.c_int(-1)
    cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, v.value)


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


for nd in (1, 2):
    for ht, hn in ((0, "none"), (1, "posix_fd"), (8, "fabric")):
        p = Prop(nd, 0, ht, 0)
        g = ctypes.c_size_t()
        r1 = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 0)
        p.size = max(g.value, 1 << 21)
        h = ctypes.c_ulonglong()
        r2 = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        r3 = cu.cuMulticastAddDevice(h, dev) if r2 == 0 else -1
        print(f"numDevices={nd} handleTypes={hn}: granularity rc={r1} ({g.value}), create rc={r2}, add_device rc={r3}")
        if r2 == 0:
            cu.cuMemRelease(h)
