#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
__global__ void red_kernel(double* mc, const double* src, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mc + i), "d"(src[i]) : "memory");
}
__global__ void ldred_kernel(const double* mc, double* dst, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v;
  if (i < n) { asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory"); dst[i] = v; }
}
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)
int main() {
  cudaFree(0);
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mcs = -1; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  int fab = -1; cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_supported=%d\n", mcs, fab);
  if (!mcs) return 0;
  for (int ht : {(int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC, 0}) {
    CUmulticastObjectProp p = {};
    p.numDevices = 1; p.handleTypes = ht; p.size = 0;
    size_t gran = 0;
    p.size = 2 << 20;
    CUresult r0 = cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("handle type %d: granularity rc=%d gran=%zu\n", ht, (int)r0, gran);
    if (r0 != CUDA_SUCCESS) continue;
    size_t sz = gran > (2u << 20) ? gran : (2u << 20);
    p.size = sz;
    CUmemGenericAllocationHandle mc;
    CUresult r1 = cuMulticastCreate(&mc, &p);
    printf("  create rc=%d\n", (int)r1);
    if (r1 != CUDA_SUCCESS) continue;
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)ht;
    CUmemGenericAllocationHandle mh; CK(cuMemCreate(&mh, sz, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mh, 0, sz, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, sz, gran, 0, 0)); CK(cuMemMap(uc, sz, 0, mh, 0));
    CK(cuMemAddressReserve(&mcp, sz, gran, 0, 0)); CK(cuMemMap(mcp, sz, 0, mc, 0));
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, sz, &ad, 1)); CK(cuMemSetAccess(mcp, sz, &ad, 1));
    const int n = 1000;
    double *src, *dst; cudaMalloc(&src, n * 8); cudaMalloc(&dst, n * 8);
    double h[n]; for (int i = 0; i < n; ++i) h[i] = i * 0.5;
    cudaMemcpy(src, h, n * 8, cudaMemcpyHostToDevice);
    cudaMemset((void*)uc, 0, n * 8);
    red_kernel<<<4, 256>>>((double*)mcp, src, n); red_kernel<<<4, 256>>>((double*)mcp, src, n);
    ldred_kernel<<<4, 256>>>((const double*)mcp, dst, n);
    cudaError_t e = cudaDeviceSynchronize();
    double o[n], u[n]; cudaMemcpy(o, dst, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(u, (void*)uc, n * 8, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < n; ++i) bad += (o[i] != 2 * h[i]) + (u[i] != 2 * h[i]);
    printf("  kernels: %s, mismatches %d (u[7]=%g ld[7]=%g)\n", cudaGetErrorString(e), bad, u[7], o[7]);
    return 0;
  }
  return 0;
}
