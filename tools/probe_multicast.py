"""Probe: does this GPU support NVLS multicast objects (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)
and which one-process multicast configurations can be created, bound and mapped?  (Plumbing.)"""
from cuda.bindings import driver as d


def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    return err == d.CUresult.CUDA_SUCCESS, err, (r[1] if isinstance(r, tuple) and len(r) > 1 else None)


d.cuInit(0)
_, _, dev = ok(d.cuDeviceGet(0))
_, _, ctx = ok(d.cuDevicePrimaryCtxRetain(dev))
d.cuCtxSetCurrent(ctx)
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    if hasattr(d.CUdevice_attribute, attr):
        print(attr, ok(d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, attr), dev))[2])
H = d.CUmemAllocationHandleType
for nd in (1, 2):
    for ht_name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR",
                    "CU_MEM_HANDLE_TYPE_FABRIC"):
        if not hasattr(H, ht_name):
            continue
        prop = d.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = getattr(H, ht_name)
        prop.flags = 0
        prop.size = 2 << 20
        g = ok(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        if g[0]:
            prop.size = max(int(g[2]), 2 << 20)
        c = ok(d.cuMulticastCreate(prop))
        msg = f"numDevices={nd} {ht_name}: gran={g[2] if g[0] else g[1]} create={c[1]}"
        if c[0]:
            a = ok(d.cuMulticastAddDevice(c[2], dev))
            msg += f" addDevice={a[1]}"
            if a[0] and nd == 1:
                ap = d.CUmemAllocationProp()
                ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
                ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
                ap.location.id = 0
                ap.requestedHandleTypes = getattr(H, ht_name)
                m = ok(d.cuMemCreate(prop.size, ap, 0))
                msg += f" memCreate={m[1]}"
                if m[0]:
                    b = ok(d.cuMulticastBindMem(c[2], 0, m[2], 0, prop.size, 0))
                    msg += f" bind={b[1]}"
        print(msg, flush=True)
