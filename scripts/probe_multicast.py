"""(GPU) Probe which multicast-object configurations the driver accepts on this box."""
from cuda.bindings import driver as d

print(d.cuInit(0))
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
print("ctx", d.cuCtxSetCurrent(ctx))
for attr in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    print(attr, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, attr), dev))
print("driver", d.cuDriverGetVersion())
for nd in (1, 2):
    for ht_name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
        prop = d.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = getattr(d.CUmemAllocationHandleType, ht_name)
        prop.size = 1 << 21
        e1, g = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        e0, gmin = d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        prop.size = max(g, 1 << 21)
        e2, mc = d.cuMulticastCreate(prop)
        print(nd, ht_name, "gran", e1, g, gmin, "create", e2)
        if e2 == d.CUresult.CUDA_SUCCESS:
            print("  add", d.cuMulticastAddDevice(mc, dev))
            d.cuMemRelease(mc)
