#include <cuda.h>
#include <stdio.h>
#include <string.h>
#include <stdint.h>
#include <stdlib.h>
#define CK(x) do { CUresult r_ = (x); if (r_) { const char* s; cuGetErrorString(r_, &s); printf("%s -> %d %s\n", #x, r_, s); return 1; } } while (0)
int main(int argc, char** argv) {
  CUdevice dev; CUcontext ctx; CUmodule mod; CUfunction f;
  CK(cuInit(0)); CK(cuDeviceGet(&dev, 0)); CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CK(cuModuleLoad(&mod, argv[1])); CK(cuModuleGetFunction(&f, mod, "k2"));
  const int NX = 32, NY = 16; double h[32 * 16]; for (int i = 0; i < NX * NY; ++i) h[i] = i;
  CUdeviceptr d, o; CK(cuMemAlloc(&d, sizeof h)); CK(cuMemAlloc(&o, 64 * 8)); CK(cuMemcpyHtoD(d, h, sizeof h));
  CUtensorMap tm; memset(&tm, 0, sizeof tm);
  cuuint64_t dims[2] = {NX, NY}, strides[1] = {NX * 8};
  cuuint32_t box[2] = {12, 8}, es[2] = {1, 1};
  CK(cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)d, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  int x0 = argc > 2 ? atoi(argv[2]) : 3, y0 = 2;
  int dst_off = argc > 3 ? atoi(argv[3]) : 0;
  void* args[] = {&tm, &o, &x0, &y0, &dst_off};
  CK(cuLaunchKernel(f, 1, 1, 1, 32, 1, 1, 0, 0, args, 0));
  CUresult r = cuCtxSynchronize();
  double s[64] = {0};
  if (r == 0) cuMemcpyDtoH(s, o, sizeof s);
  const char* es_; cuGetErrorString(r, &es_);
  printf("x0 %d dst_off %d doubles: %s; s[0]=%g (want %d) s[13]=%g (want %d)\n", x0, dst_off, es_, s[0], 2 * NX + x0, s[13], 3 * NX + x0 + 1);
  return 0;
}
