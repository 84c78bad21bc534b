// NVLS multicast probe in C (driver API): create / add device / bind / map a one-device
// multicast object and run one multimem.ld_reduce over it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_mc tools/probe_mc.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_ldred(const float* mc, float* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i + 3 < n) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
        out[4 * i] = a; out[4 * i + 1] = b; out[4 * i + 2] = c; out[4 * i + 3] = d;
    }
}

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("%s -> %d %s\n", #x, (int)r_, s_); return 1; } } while (0)

int main() {
    cudaFree(0);
    CUdevice dev; CK(cuDeviceGet(&dev, 0));
    int sup = 0; cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    printf("multicast supported %d\n", sup);
    for (int ht : {0, (int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR}) {
        CUmulticastObjectProp prop = {};
        prop.numDevices = 1;
        prop.handleTypes = (unsigned long long)ht;
        prop.size = 2 << 20;
        size_t gran = 0;
        CUresult g = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        printf("handleTypes %d: granularity rc %d gran %zu\n", ht, (int)g, gran);
        if (gran) prop.size = gran;
        CUmemGenericAllocationHandle mc;
        CUresult c = cuMulticastCreate(&mc, &prop);
        const char* es; cuGetErrorString(c, &es);
        printf("  create rc %d %s\n", (int)c, es);
        if (c != CUDA_SUCCESS) continue;
        CK(cuMulticastAddDevice(mc, dev));
        CUmemAllocationProp ap = {};
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = 0;
        ap.requestedHandleTypes = (CUmemAllocationHandleType)ht;
        CUmemGenericAllocationHandle mem;
        CK(cuMemCreate(&mem, prop.size, &ap, 0));
        CK(cuMulticastBindMem(mc, 0, mem, 0, prop.size, 0));
        CUdeviceptr uc, mcp;
        CK(cuMemAddressReserve(&uc, prop.size, prop.size, 0, 0));
        CK(cuMemMap(uc, prop.size, 0, mem, 0));
        CK(cuMemAddressReserve(&mcp, prop.size, prop.size, 0, 0));
        CK(cuMemMap(mcp, prop.size, 0, mc, 0));
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = 0;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CK(cuMemSetAccess(uc, prop.size, &acc, 1));
        CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
        const int n = 1024;
        float h[n]; for (int i = 0; i < n; ++i) h[i] = (float)i;
        cudaMemcpy((void*)uc, h, sizeof h, cudaMemcpyHostToDevice);
        float* out; cudaMalloc(&out, sizeof h);
        k_ldred<<<1, 256>>>((const float*)mcp, out, n);
        cudaError_t e = cudaDeviceSynchronize();
        float o[n]; cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
        int bad = 0; for (int i = 0; i < n; ++i) bad += o[i] != h[i];
        printf("  ld_reduce kernel: %s, mismatches %d\n", cudaGetErrorString(e), bad);
    }
    return 0;
}
