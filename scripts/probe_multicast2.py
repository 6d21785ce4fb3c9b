"""(GPU) More multicast-object probes: sizes, and what NCCL reports about NVLS."""
from cuda.bindings import driver as d

d.cuInit(0)
err, dev = d.cuDeviceGet(0)
err, ctx = d.cuDevicePrimaryCtxRetain(dev)
d.cuCtxSetCurrent(ctx)
for size in (1 << 21, 1 << 25, 1 << 29):
    prop = d.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = size
    prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    prop.flags = 0
    print(size, d.cuMulticastCreate(prop)[0])
print(d.cuGetErrorString(d.CUresult.CUDA_ERROR_INVALID_VALUE))
