// Host side of scripts/dispatch_probe.py: loads a probe cubin, runs a random op stream,
// prints warp-ops per clock per SM.  nvcc -O2 -o dh scripts/dispatch_host.cu -lcuda
// usage: dh probe.cubin NS W T blocks_per_sm mix   (mix: 0 register ops only; 1: 1/4 shared; 2: XRS-heavy)
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); \
  printf("%s failed: %s\n", #x, s); exit(1); } } while (0)

int main(int argc, char **argv) {
  const char *cubin = argv[1];
  int NS = atoi(argv[2]), W = atoi(argv[3]), T = atoi(argv[4]), bps = atoi(argv[5]), mix = atoi(argv[6]);
  int XR = 0, ST = NS, LD = 2 * NS, XS = 3 * NS, LS = XS + 1, SS = XS + 2, XRS = XS + 3, END = 4 * NS + 3;
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmodule mod; CK(cuModuleLoad(&mod, cubin));
  CUfunction f; CK(cuModuleGetFunction(&f, mod, "probe"));
  int regs; cuFuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
  int lmem; cuFuncGetAttribute(&lmem, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
  const int nops = 8192, iters = 40;
  std::vector<uint32_t> code;
  srand(7);
  for (int i = 0; i < nops; ++i) {
    int r = rand() % 100, h;
    if (mix == 0) h = rand() % (3 * NS);
    else if (mix == 1) h = r < 25 ? XS + rand() % 3 : rand() % (3 * NS);
    else h = r < 50 ? XRS + rand() % NS : r < 60 ? XS + rand() % 3 : rand() % (3 * NS);
    uint32_t row = rand() % 64;
    code.push_back((uint32_t)h | ((row * T * W * 4) << 9));
  }
  code.push_back(END);
  for (int k = 0; k < 8; ++k) code.push_back(END);
  CUdeviceptr dcode, dout, dcyc;
  int nsm = 148, grid = nsm * bps;
  CK(cuMemAlloc(&dcode, code.size() * 4));
  CK(cuMemcpyHtoD(dcode, code.data(), code.size() * 4));
  CK(cuMemAlloc(&dout, (size_t)grid * T * 4));
  CK(cuMemAlloc(&dcyc, (size_t)grid * 8));
  unsigned smem = (unsigned)(code.size() * 4 + 16 + 64 * T * W * 4);
  CK(cuFuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem));
  int ncode = (int)code.size(), it = 2;
  void *args[] = {&dcode, &ncode, &it, &dout, &dcyc};
  CK(cuLaunchKernel(f, grid, 1, 1, T, 1, 1, smem, 0, args, 0));
  CK(cuCtxSynchronize());
  it = iters;
  CUevent e0, e1; cuEventCreate(&e0, 0); cuEventCreate(&e1, 0);
  cuEventRecord(e0, 0);
  CK(cuLaunchKernel(f, grid, 1, 1, T, 1, 1, smem, 0, args, 0));
  cuEventRecord(e1, 0);
  CK(cuCtxSynchronize());
  float ms; cuEventElapsedTime(&ms, e0, e1);
  std::vector<long long> cyc(grid);
  CK(cuMemcpyDtoH(cyc.data(), dcyc, grid * 8));
  double avgc = 0; for (auto c : cyc) avgc += c; avgc /= grid;
  double warp_ops = (double)grid * (T / 32) * nops * iters;
  printf("NS=%d W=%d T=%d bps=%d mix=%d regs=%d lmem=%d ms=%.3f cyc/CTA=%.0f warp-ops/clk/SM=%.3f "
         "(per warp %.1f clk/op) GHz~%.2f wall-ops/ns/SM=%.3f\n", NS, W, T, bps, mix, regs, lmem, ms, avgc,
         warp_ops / nsm / avgc, avgc / ((double)nops * iters), avgc / (ms * 1e6),
         warp_ops / nsm / (ms * 1e6));
  return 0;
}
