"""Probe NVLS multicast support on this device (tool): the attribute, the
multicast granularity, and which handle types cuMulticastCreate accepts for a
team of one.  Usage: python tools/probe_multicast.py"""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
for name, a in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128),
                ("HANDLE_TYPE_POSIX_FD_SUPPORTED", 100)):
    v = ctypes.c_int(-1)
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
    print(name, "rc", r, "value", v.value)
ctx = ctypes.c_void_p()
cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev)
cu.cuCtxSetCurrent(ctx)


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


for ht_name, ht in (("none", 0), ("posix_fd", 1), ("fabric", 8)):
    p = Prop(1, 1 << 21, ht, 0)
    g = ctypes.c_size_t(0)
    rg = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
    p.size = max(g.value, 1 << 21)
    h = ctypes.c_ulonglong(0)
    rc = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
    print(f"handleTypes={ht_name}: granularity rc {rg} = {g.value}, cuMulticastCreate rc {rc}")
    if rc == 0:
        cu.cuMemRelease(h)

err = ctypes.c_char_p()
for nd in (1, 2, 4, 8):
    for ht_name, ht in (("none", 0), ("fabric", 8)):
        p = Prop(nd, 1 << 21, ht, 0)
        g = ctypes.c_size_t(0)
        cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 0)
        p.size = max(g.value, 1 << 21)
        h = ctypes.c_ulonglong(0)
        rc = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        cu.cuGetErrorString(rc, ctypes.byref(err))
        print(f"numDevices={nd} handleTypes={ht_name} min-granularity {g.value}: rc {rc} ({err.value})")
        if rc == 0:
            ra = cu.cuMulticastAddDevice(h, dev)
            cu.cuGetErrorString(ra, ctypes.byref(err))
            print("   cuMulticastAddDevice", ra, err.value)
            cu.cuMemRelease(h)
