// Probe (round 2): TMEM as an indexed per-thread store for the interpreter's variables.
// Measures tcgen05.ld / tcgen05.st throughput and latency from CUDA cores on sm_100a.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tp scripts/tmem_probe.cu
// usage: tp mode warps ctas_per_sm   mode 0: ld.x4 + wait per load (latency chain)
//        1: 4 x ld.x4 then one wait   2: ld.x16 + wait   3: st.x4 (wait::st every 4)
//        4: ld.x4 x4 + wait + xor + st.x4 (interpreter-like)   5: lds.128 x4 (smem reference)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smaddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD4(a, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" \
  : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a))
#define ST4(a, r) asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" \
  :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory")
#define WLD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define WST() asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory")

template <int mode>
__global__ void probe(int iters, uint32_t *out, long long *cyc) {
  __shared__ uint32_t taddr_s;
  extern __shared__ uint4 dsm[];
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smaddr(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) dsm[i] = make_uint4(i, i + 1, i + 2, i + 3);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = taddr_s + ((uint32_t)(warp & 3) * 32 << 16) + (warp >= 4 ? 256 : 0);
  uint32_t acc[4] = {threadIdx.x, 1, 2, 3}, r[4][4];
  for (int c = 0; c < 256; c += 4) ST4(tbase + c, acc);
  WST();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t c = (it * 28) & 240;
    if constexpr (mode == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { LD4(tbase + c + 4 * k, r[k]); WLD(); acc[0] ^= r[k][0]; acc[1] ^= r[k][1]; acc[2] ^= r[k][2]; acc[3] ^= r[k][3]; }
    } else if constexpr (mode == 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) LD4(tbase + c + 4 * k, r[k]);
      WLD();
#pragma unroll
      for (int k = 0; k < 4; ++k) { acc[0] ^= r[k][0]; acc[1] ^= r[k][1]; acc[2] ^= r[k][2]; acc[3] ^= r[k][3]; }
    } else if constexpr (mode == 2) {
      uint32_t q[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                     "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
                   : "r"(tbase + c));
      WLD();
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k & 3] ^= q[k];
    } else if constexpr (mode == 3) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { acc[k] += 1; ST4(tbase + c + 4 * k, acc); }
      WST();
    } else if constexpr (mode == 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) LD4(tbase + c + 4 * k, r[k]);
      WLD();
#pragma unroll
      for (int k = 0; k < 4; ++k) { acc[0] ^= r[k][0]; acc[1] ^= r[k][1]; acc[2] ^= r[k][2]; acc[3] ^= r[k][3]; }
      ST4(tbase + ((c + 64) & 252), acc);
      WST();
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint4 v = dsm[((it * 7 + k * 13) & 63) * 128 + (threadIdx.x & 127)];
        acc[0] ^= v.x; acc[1] ^= v.y; acc[2] ^= v.z; acc[3] ^= v.w;
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] ^ acc[1] ^ acc[2] ^ acc[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

int main(int argc, char **argv) {
  int mode = atoi(argv[1]), warps = atoi(argv[2]);
  const int iters = 20000, grid = 148;
  uint32_t *out; long long *cyc;
  cudaMalloc(&out, grid * warps * 32 * 4);
  cudaMalloc(&cyc, grid * 8);
  const int smem = 64 * 128 * 16;
  void (*fns[6])(int, uint32_t *, long long *) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>};
  auto fn = fns[mode];
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  fn<<<grid, warps * 32, smem>>>(10, out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fn<<<grid, warps * 32, smem>>>(iters, out, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c[148]; cudaMemcpy(c, cyc, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < grid; ++i) avg += c[i]; avg /= grid;
  // bytes moved per SM per clock (TMEM ld+st, or smem ld for mode 5)
  double per_it = mode == 3 ? 4 * 16 : mode == 4 ? 5 * 16 : mode == 2 ? 64 : 4 * 16;
  double bytes = per_it * iters * warps * 32;
  printf("mode=%d warps=%d err=%s ms=%.3f cyc=%.0f B/clk/SM=%.1f clk/iter/warp=%.1f\n", mode, warps,
         cudaGetErrorString(err), ms, avg, bytes / avg, avg / iters);
  return 0;
}
