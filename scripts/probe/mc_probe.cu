// Probe: NVLS multicast on this box (driver API) -- attribute, a 1-device multicast object bound to local
// cuMemCreate memory, multimem.ld_reduce / multimem.st through the multicast mapping.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)
__global__ void k_reduce(const __nv_bfloat16* mc_in, __nv_bfloat16* out, __nv_bfloat16* mc_out, int n) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i >= n) return;
  uint32_t a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mc_in + i) : "memory");
  uint4 v = make_uint4(a, b, c, d);
  *reinterpret_cast<uint4*>(out + i) = v;
  asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" :: "l"(mc_out + i), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("MULTICAST_SUPPORTED=%d\n", mc);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR; mp.size = 0;
  size_t gran = 0;
  mp.size = 2 << 20;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  printf("mc granularity %zu\n", gran);
  size_t size = ((4 << 20) + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mch;
  {
    const int hts[3] = {(int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC, 0};
    for (int nd = 1; nd <= 2; ++nd)
      for (int hi = 0; hi < 3; ++hi) {
        CUmulticastObjectProp q = mp; q.numDevices = nd; q.handleTypes = (unsigned long long)hts[hi];
        CUmemGenericAllocationHandle tmp;
        CUresult r = cuMulticastCreate(&tmp, &q);
        printf("cuMulticastCreate numDevices=%d handleTypes=%d -> %d\n", nd, hts[hi], (int)r);
        if (r == CUDA_SUCCESS) cuMemRelease(tmp);
      }
  }
  CUresult rr = cuMulticastCreate(&mch, &mp);
  if (rr != CUDA_SUCCESS) { mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC; rr = cuMulticastCreate(&mch, &mp); printf("fabric retry %d\n", (int)rr); }
  if (rr != CUDA_SUCCESS) { mp.handleTypes = 0; rr = cuMulticastCreate(&mch, &mp); printf("none retry %d\n", (int)rr); }
  if (rr != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  CUmemGenericAllocationHandle mh; CK(cuMemCreate(&mh, size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mh, 0, size, 0));
  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, size, gran, 0, 0)); CK(cuMemMap(uva, size, 0, mh, 0));
  CK(cuMemAddressReserve(&mva, size, gran, 0, 0)); CK(cuMemMap(mva, size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, size, &ad, 1)); CK(cuMemSetAccess(mva, size, &ad, 1));
  const int n = 1 << 16;
  __nv_bfloat16* h = new __nv_bfloat16[n];
  for (int i = 0; i < n; ++i) h[i] = __float2bfloat16((float)(i % 97) * 0.25f);
  CK(cuMemcpyHtoD(uva, h, n * 2));
  CUdeviceptr out; CK(cuMemAlloc(&out, n * 2));
  k_reduce<<<n / 8 / 256, 256>>>((const __nv_bfloat16*)mva, (__nv_bfloat16*)out, (__nv_bfloat16*)(mva + (2 << 20)), n);
  CK(cuCtxSynchronize());
  __nv_bfloat16* g = new __nv_bfloat16[n]; __nv_bfloat16* g2 = new __nv_bfloat16[n];
  CK(cuMemcpyDtoH(g, out, n * 2)); CK(cuMemcpyDtoH(g2, uva + (2 << 20), n * 2));
  int bad = 0, bad2 = 0;
  for (int i = 0; i < n; ++i) { if (__bfloat162float(g[i]) != __bfloat162float(h[i])) ++bad; if (__bfloat162float(g2[i]) != __bfloat162float(h[i])) ++bad2; }
  printf("ld_reduce mismatches %d, st mismatches %d (of %d)\n", bad, bad2, n);
  // a second "device" slot for the same GPU (how far can one GPU emulate a group?)
  CUmulticastObjectProp mp2 = mp; mp2.numDevices = 2;
  CUmemGenericAllocationHandle mch2; CK(cuMulticastCreate(&mch2, &mp2));
  CUresult r = cuMulticastAddDevice(mch2, dev); printf("add dev once: %d\n", (int)r);
  r = cuMulticastAddDevice(mch2, dev); printf("add same dev twice: %d\n", (int)r);
  printf("PROBE OK\n");
  return 0;
}
