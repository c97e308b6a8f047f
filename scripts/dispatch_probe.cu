// Probe: throughput of a switch-dispatched register-machine interpreter on sm_100a.
// Each thread owns W words; the interpreter has N register slots (static names inside the
// switch cases) and an accumulator; ops come warp-uniformly from shared memory, 4 per 128-bit
// load, prefetched one group ahead.  Reports ops per clock per SM for random programs.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dp scripts/dispatch_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#ifndef NS
#define NS 32
#endif
#ifndef WW
#define WW 2
#endif

enum { OP_XR = 0, OP_ST = NS, OP_LD = 2 * NS, OP_XS = 3 * NS, OP_LS, OP_SS, OP_END };

#define REP_W(stmt) _Pragma("unroll") for (int w = 0; w < WW; ++w) { stmt; }

template <int N>
__device__ __forceinline__ void noop() {}

__global__ void __launch_bounds__(256) probe(const uint32_t *__restrict__ gcode, int ncode,
                                             int iters, uint32_t *out, long long *cycles) {
  extern __shared__ uint4 sm4[];
  uint32_t *code = (uint32_t *)sm4;
  for (int i = threadIdx.x; i < ncode; i += blockDim.x) code[i] = gcode[i];
  uint32_t *rows = code + ncode;  // 64 rows x blockDim x W words
  const int T = blockDim.x;
  for (int i = threadIdx.x; i < 64 * T * WW; i += T) rows[i] = i * 2654435761u;
  __syncthreads();
  uint32_t R[NS][WW], acc[WW];
#pragma unroll
  for (int i = 0; i < NS; ++i) REP_W(R[i][w] = i + w + threadIdx.x)
  REP_W(acc[w] = 0)
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint4 *c4 = (const uint4 *)code;
    uint4 cur = c4[0];
    int g = 1;
    for (;;) {
      uint4 nxt = c4[g++];
      uint32_t ops[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t op = ops[q];
        const uint32_t h = op & 255u, a = op >> 8;
        uint32_t *row = rows + a * T * WW + threadIdx.x * WW;
        switch (h) {
#define XR(i) case OP_XR + i: REP_W(acc[w] ^= R[i][w]) break;
#define ST(i) case OP_ST + i: REP_W(R[i][w] = acc[w]) break;
#define LD(i) case OP_LD + i: REP_W(acc[w] = R[i][w]) break;
#define ALL(M) M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15)
#define ALL2(M) M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)
          ALL(XR) ALL(ST) ALL(LD)
#if NS > 16
          ALL2(XR) ALL2(ST) ALL2(LD)
#endif
          case OP_XS:
            if (WW == 2) { uint2 v = *(uint2 *)row; acc[0] ^= v.x; acc[WW - 1] ^= v.y; }
            else REP_W(acc[w] ^= row[w])
            break;
          case OP_LS:
            if (WW == 2) { uint2 v = *(uint2 *)row; acc[0] = v.x; acc[WW - 1] = v.y; }
            else REP_W(acc[w] = row[w])
            break;
          case OP_SS:
            if (WW == 2) { *(uint2 *)row = make_uint2(acc[0], acc[WW - 1]); }
            else REP_W(row[w] = acc[w])
            break;
          default:
            goto done;
        }
      }
      cur = nxt;
    }
  done:;
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NS; ++i) REP_W(s ^= R[i][w])
  REP_W(s ^= acc[w])
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main(int argc, char **argv) {
  int T = argc > 1 ? atoi(argv[1]) : 256;
  int blocks_per_sm = argc > 2 ? atoi(argv[2]) : 2;
  int mix = argc > 3 ? atoi(argv[3]) : 0;  // 0: register-only ops, 1: 1/4 shared ops
  const int nops = 4096, iters = 50;
  std::vector<uint32_t> code;
  srand(1);
  for (int i = 0; i < nops; ++i) {
    int r = rand();
    uint32_t h;
    if (mix && (r % 4) == 0) h = OP_XS + (r / 4) % 3;
    else h = (r / 4) % (3 * NS);
    code.push_back(h | ((uint32_t)(rand() % 64) << 8));
  }
  code.push_back(OP_END);
  while (code.size() % 4) code.push_back(OP_END);
  code.push_back(OP_END); code.push_back(OP_END); code.push_back(OP_END); code.push_back(OP_END);
  uint32_t *dcode, *dout;
  long long *dcyc;
  int nsm = 148, grid = nsm * blocks_per_sm;
  cudaMalloc(&dcode, code.size() * 4);
  cudaMemcpy(dcode, code.data(), code.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, grid * T * 4);
  cudaMalloc(&dcyc, grid * 8);
  size_t smem = code.size() * 4 + 64 * T * WW * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, probe);
  probe<<<grid, T, smem>>>(dcode, (int)code.size(), 2, dout, dcyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<<<grid, T, smem>>>(dcode, (int)code.size(), iters, dout, dcyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> cyc(grid);
  cudaMemcpy(cyc.data(), dcyc, grid * 8, cudaMemcpyDeviceToHost);
  double avgc = 0; for (auto c : cyc) avgc += c; avgc /= grid;
  double warp_ops = (double)grid * (T / 32) * nops * iters;
  double ops_per_clk_sm = warp_ops / nsm / avgc;
  printf("NS=%d W=%d T=%d bps=%d mix=%d regs=%d spill=%d err=%s ms=%.3f cyc=%.0f warp-ops/clk/SM=%.3f "
         "word-ops/s=%.3g\n", NS, WW, T, blocks_per_sm, mix, fa.numRegs, (int)fa.localSizeBytes,
         cudaGetErrorString(err), ms, avgc, ops_per_clk_sm, warp_ops * 32 * WW / (ms * 1e-3));
  return 0;
}
