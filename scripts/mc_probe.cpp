// Probe: does this box support CUDA multicast objects (NVLS) -- with one device bound?
//   g++ -O2 -I/usr/local/cuda/include scripts/mc_probe.cpp -o /tmp/mc_probe -L/usr/local/cuda/lib64/stubs -lcuda
#include <cuda.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); std::printf("%s -> %s\n", #x, s); return 1; } } while (0)
int main() {
  CK(cuInit(0));
  CUdevice d; CK(cuDeviceGet(&d, 0));
  int mc = -1, fab = -1, nvls = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
  std::printf("multicast_supported %d fabric %d\n", mc, fab);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, d)); CK(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp p = {};
  p.numDevices = 1; p.size = 2 << 20; p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  std::printf("mc granularity %zu\n", gran);
  p.size = gran;
  CUmemGenericAllocationHandle mch; CK(cuMulticastCreate(&mch, &p));
  CK(cuMulticastAddDevice(mch, d));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, gran, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mem, 0, gran, 0));
  CUdeviceptr va; CK(cuMemAddressReserve(&va, gran, gran, 0, 0)); CK(cuMemMap(va, gran, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location = ap.location; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, gran, &ad, 1));
  std::printf("multicast object mapped at %p: ok\n", (void*)va);
  return 0;
}
