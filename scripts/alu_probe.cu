// Integer-pipe and shared-memory microbenchmark for the roofline of SURVEY 8(d): the planning
// assumption was 64 LOP3 / clk / SM ("to be confirmed by a microbenchmark on the box").
// Measures, per SM per clock: LOP3.LUT (3-input XOR, the op the SLP kernels issue), PRMT (the
// nibble-table lookups of the approach-(1) kernel) and LDS.32 / LDS.64 bytes (the PIPE consumer's
// operand reads).  Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/alu_probe
// scripts/alu_probe.cu && /tmp/alu_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

constexpr int CHAINS = 8;      // independent dependency chains per thread (latency 4, rt 2)
constexpr int UNROLL = 16;

__global__ void k_lop3(uint32_t *out, long long *cyc, int iters) {
  uint32_t a[CHAINS];
  uint32_t b = threadIdx.x * 0x9e3779b9u, c = blockIdx.x * 0x85ebca6bu + 1;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = threadIdx.x + j * 0x01000193u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int j = 0; j < CHAINS; ++j)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(b), "r"(c));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) x ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_prmt(uint32_t *out, long long *cyc, int iters) {
  uint32_t a[CHAINS];
  uint32_t b = threadIdx.x * 0x9e3779b9u, c = blockIdx.x * 0x85ebca6bu + 1;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = threadIdx.x + j * 0x01000193u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < UNROLL; ++u)
#pragma unroll
      for (int j = 0; j < CHAINS; ++j)
        asm volatile("prmt.b32 %0, %1, %2, %0;" : "+r"(a[j]) : "r"(b), "r"(c));
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) x ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LDS bandwidth: W = 1 (LDS.32) or 2 (LDS.64) words per load, conflict-free, XOR-accumulated
template <int W>
__global__ void k_lds(uint32_t *out, long long *cyc, int iters) {
  extern __shared__ uint32_t sm[];
  const int N = 8192;    // 32 KiB
  for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = i * 0x9e3779b9u;
  __syncthreads();
  uint32_t acc[CHAINS] = {0};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) {
      int off = ((j * 32 + (i & 15) * 256) * W + threadIdx.x * W) & (N - 1);
      if (W == 1) {
        uint32_t v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm + off)));
        acc[j] ^= v;
      } else {
        uint32_t v0, v1;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1)
                     : "r"((uint32_t)__cvta_generic_to_shared(sm + off)));
        acc[j] ^= v0 ^ v1;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) x ^= acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
int run(const char *name, K kern, int threads, int blocks_per_sm, int iters, double per_thread_iter,
        const char *unit, size_t smem, int nsm) {
  int blocks = nsm * blocks_per_sm;
  uint32_t *out; long long *cyc;
  CK(cudaMalloc(&out, (size_t)blocks * threads * 4));
  CK(cudaMalloc(&cyc, blocks * sizeof(long long)));
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<blocks, threads, smem>>>(out, cyc, iters / 10);      // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads, smem>>>(out, cyc, iters);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(blocks);
  CK(cudaMemcpy(c.data(), cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
  std::sort(c.begin(), c.end());
  double med = (double)c[blocks / 2];
  double per_block = (double)threads * iters * per_thread_iter;
  double per_sm_clk = per_block * blocks_per_sm / med;       // blocks of one SM run concurrently
  double total_per_s = per_block * blocks / (ms / 1e3);
  double mhz = med / (ms * 1e3);                              // cycles per block / kernel time
  printf("{\"probe\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"per_sm_per_clk\": %.2f, "
         "\"unit\": \"%s\", \"chip_per_s\": %.4e, \"ms\": %.3f, \"sm_mhz_est\": %.0f}\n",
         name, threads, blocks_per_sm, per_sm_clk, unit, total_per_s, ms, mhz);
  cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("{\"sms\": %d}\n", nsm);
  const double ops = (double)UNROLL * CHAINS;
  for (int bps : {2, 4}) {
    if (run("lop3", k_lop3, 256, bps, 4096, ops, "LOP3 lane-ops", 0, nsm)) return 1;
    if (run("prmt", k_prmt, 256, bps, 4096, ops, "PRMT lane-ops", 0, nsm)) return 1;
  }
  for (int bps : {2, 4}) {
    if (run("lds32", k_lds<1>, 256, bps, 16384, CHAINS * 4.0, "bytes", 32768, nsm)) return 1;
    if (run("lds64", k_lds<2>, 256, bps, 16384, CHAINS * 8.0, "bytes", 32768, nsm)) return 1;
  }
  return 0;
}
