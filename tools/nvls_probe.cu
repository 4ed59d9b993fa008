// Probe: can this box create an NVLS multicast object (NVSwitch multimem) with one device bound,
// and do multimem.st / multimem.red.add.f64 / multimem.ld_reduce.add.f64 work through it?
// Also: POSIX-fd export of the multicast handle (how ranks would share it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("FAIL %s -> %d %s (line %d)\n", #x, (int)r, s, __LINE__); return 1; } } while (0)

__global__ void mm_kernel(double* mc, double* uc, int n, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 1.0 + i;
  asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(mc + i), "d"(v) : "memory");
  __threadfence_system();
  asm volatile("multimem.red.global.add.f64 [%0], %1;" ::"l"(mc + i), "d"(0.5) : "memory");
  __threadfence_system();
  double r;
  asm volatile("multimem.ld_reduce.global.add.f64 %0, [%1];" : "=d"(r) : "l"(mc + i) : "memory");
  out[i] = r;
}

int main() {
  CU(cuInit(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CU(cuDevicePrimaryCtxRetain(&ctx, dev));
  CU(cuCtxSetCurrent(ctx));
  int mc = -1, fabric = -1, posix = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handle=%d posix_fd=%d\n", mc, fabric, posix);
  if (!mc) { printf("no multicast on this box\n"); return 0; }
  const int n = 1 << 16;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  size_t gran = 0;
  CUmemGenericAllocationHandle mch;
  const char* names[3] = {"none", "posix_fd", "fabric"};
  CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                        CU_MEM_HANDLE_TYPE_FABRIC};
  int ok = -1;
  size_t size = 0;
  for (int ti = 2; ti >= 0; --ti) {
    mp.handleTypes = types[ti];
    mp.size = 0;
    CUresult rg = cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    size = ((n * 8 + gran - 1) / gran) * gran;
    mp.size = size;
    CUresult rc = cuMulticastCreate(&mch, &mp);
    printf("cuMulticastCreate handleTypes=%s gran_rc=%d gran=%zu -> %d\n", names[ti], (int)rg, gran, (int)rc);
    if (rc == CUDA_SUCCESS) { ok = ti; break; }
  }
  if (ok < 0) return 1;
  int fd = -1;
  if (ok == 1) {
    CUresult er = cuMemExportToShareableHandle(&fd, mch, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    printf("export mc handle as posix fd: rc=%d fd=%d\n", (int)er, fd);
  } else if (ok == 2) {
    CUmemFabricHandle fh;
    CUresult er = cuMemExportToShareableHandle(&fh, mch, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    printf("export mc handle as fabric handle: rc=%d\n", (int)er);
  }
  CU(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = types[ok];
  CUmemGenericAllocationHandle ph;
  CU(cuMemCreate(&ph, size, &ap, 0));
  CU(cuMulticastBindMem(mch, 0, ph, 0, size, 0));
  CUdeviceptr uc, mcp;
  CU(cuMemAddressReserve(&uc, size, gran, 0, 0));
  CU(cuMemMap(uc, size, 0, ph, 0));
  CU(cuMemAddressReserve(&mcp, size, gran, 0, 0));
  CU(cuMemMap(mcp, size, 0, mch, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(uc, size, &acc, 1));
  CU(cuMemSetAccess(mcp, size, &acc, 1));
  double* out;
  cudaMalloc(&out, n * 8);
  mm_kernel<<<n / 256, 256>>>((double*)mcp, (double*)uc, n, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double* h = (double*)malloc(n * 8);
  double* hu = (double*)malloc(n * 8);
  cudaMemcpy(h, out, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hu, (void*)uc, n * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i)
    if (h[i] != 1.5 + i || hu[i] != 1.5 + i) ++bad;
  printf("ld_reduce / unicast check: bad=%d (h[3]=%g hu[3]=%g, expect %g)\n", bad, h[3], hu[3], 4.5);
  return 0;
}
