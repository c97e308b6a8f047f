// The paper's approach (1) on B200, as a comparison point (SURVEY §8(f) NEXT #3 alternative):
// Reed-Solomon as matrix multiplication over GF(2^8) with table-driven field multiplication
// ("tightly coupling sophisticated optimization methods for MM and finite field
// multiplication", ISA-L's nibble-table / PSHUFB method), instead of the XOR-based
// approach (2) that the rest of libxslp implements.
//
// Byte layout: output block i = sum_j coef[i][j] * input block j, byte by byte.
// Multiplication by a constant c is linear over GF(2), so c*x is the XOR of c*(bit groups of
// x): ISA-L splits x into two nibbles and looks each up in a 16-entry table with PSHUFB.  The
// GPU's byte permute PRMT indexes 8 bytes (two registers) with 3-bit selectors, so here x is
// split into three bit groups, bits [0,3), [3,6), [6,8), each looked up in an 8-entry table
// (c * (v << 3g), v = 0..7): one PRMT per group and 4 bytes, no select step.
//
// Selectors: PRMT reads four selectors from bits 0-15 (bit 3 of each must stay 0).  Two input
// words x, y are paired: lo = (group of x, at nibbles 0, 2, 4, 6) | (group of y, at nibbles 1,
// 3, 5, 7) and hi = lo >> 16, so PRMT(lo) yields the products of bytes (x0, y0, x1, y1) and
// PRMT(hi) those of (x2, y2, x3, y3); the accumulators stay interleaved and two PRMTs per word
// pair restore the byte order at the end.
//
// Work per (coefficient, 4 bytes): 3 PRMT + 1.5 LOP3 (two input blocks per step: six
// products per output word XORed into the accumulator by three LOP3); per input word about 6
// ALU ops for the selectors, shared by the m outputs.  A thread owns V x 16 bytes of every
// block; each CTA builds its tables in shared memory (24 B per coefficient) from the
// coefficient matrix (a kernel parameter) at start-up.  Still ALU-bound
// (profiles/r01_s2_gftable.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "xslp_api.h"

namespace xslp {



void count_launch();  // device.cu

constexpr int kMaxOut = 8, kMaxIn = 64;

struct GfCoef {
  uint8_t c[kMaxOut * kMaxIn];  // [m][n] row-major
};

// x * 2 in GF(2^8) / 0x11D
__device__ __forceinline__ uint32_t gf_x2(uint32_t a) { return ((a << 1) ^ ((a & 0x80) ? 0x11D : 0)) & 0xFF; }

__device__ uint32_t gf_mul_dev(uint32_t a, uint32_t b) {
  uint32_t r = 0;
  for (int k = 0; k < 8; ++k) {
    if (b & (1u << k)) r ^= a;
    a = gf_x2(a);
  }
  return r;
}

// selectors of bit group G for the word pair (x, y): see the header
template <int G>
__device__ __forceinline__ void pair_sel(uint32_t x, uint32_t y, uint32_t &lo, uint32_t &hi) {
  constexpr uint32_t kMask = G < 2 ? 0x07070707u : 0x03030303u;
  const uint32_t a = (x >> (3 * G)) & kMask;
  const uint32_t b = (G == 0 ? y << 4 : G == 1 ? y << 1 : y >> 2) & (kMask << 4);
  lo = a | b;
  hi = lo >> 16;
}

// the three selector sets [2 * pair + half] of the thread's V 16-byte chunks of one block
template <int V>
__device__ __forceinline__ void load_sel(const uint8_t *blk, uint64_t q0, uint64_t chunks, uint32_t *s0,
                                         uint32_t *s1, uint32_t *s2) {
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const uint64_t q = q0 + (uint64_t)v * blockDim.x;
    const uint4 x = q < chunks ? __ldcs(reinterpret_cast<const uint4 *>(blk) + q) : make_uint4(0, 0, 0, 0);
    pair_sel<0>(x.x, x.y, s0[4 * v], s0[4 * v + 1]);
    pair_sel<1>(x.x, x.y, s1[4 * v], s1[4 * v + 1]);
    pair_sel<2>(x.x, x.y, s2[4 * v], s2[4 * v + 1]);
    pair_sel<0>(x.z, x.w, s0[4 * v + 2], s0[4 * v + 3]);
    pair_sel<1>(x.z, x.w, s1[4 * v + 2], s1[4 * v + 3]);
    pair_sel<2>(x.z, x.w, s2[4 * v + 2], s2[4 * v + 3]);
  }
}

template <int M, int V>
__global__ void __launch_bounds__(256) xslp_gftable_kernel(const uint8_t *const *__restrict__ in_tbl,
                                                           uint8_t *const *__restrict__ out_tbl,
                                                           int n, uint64_t chunks, GfCoef coef) {
  // tables: [i][j][g] -> 8 bytes (c_ij * (v << 3g), v = 0..7)
  extern __shared__ uint2 tab[];
  for (int e = threadIdx.x; e < M * n * 24; e += blockDim.x) {
    const int pair = e / 24, g = (e % 24) / 8, v = e % 8;
    reinterpret_cast<uint8_t *>(tab)[e] = (uint8_t)gf_mul_dev(coef.c[pair], (uint32_t)(v << (3 * g)) & 0xFF);
  }
  __syncthreads();
  const uint64_t q0 = (uint64_t)blockIdx.x * blockDim.x * V + threadIdx.x;
  if (q0 >= chunks) return;
  const uint32_t stripe = blockIdx.y;
  const uint8_t *const *in = in_tbl + (uint64_t)stripe * n;
  uint8_t *const *out = out_tbl + (uint64_t)stripe * M;
  constexpr int W = 4 * V;               // words per thread = 2V word pairs, 2 selector words each
  uint32_t acc[M][W];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int k = 0; k < W; ++k) acc[i][k] = 0;
  // two input blocks per iteration: six products per (output, word) XORed by three LOP3
  int j = 0;
  for (; j + 1 < n; j += 2) {
    uint32_t a0[W], a1[W], a2[W], b0[W], b1[W], b2[W];
    load_sel<V>(in[j], q0, chunks, a0, a1, a2);
    load_sel<V>(in[j + 1], q0, chunks, b0, b1, b2);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const uint2 *ta = &tab[(i * n + j) * 3], *tb = ta + 3;
      const uint2 ta0 = ta[0], ta1 = ta[1], ta2 = ta[2], tb0 = tb[0], tb1 = tb[1], tb2 = tb[2];
#pragma unroll
      for (int k = 0; k < W; ++k)
        acc[i][k] ^= __byte_perm(ta0.x, ta0.y, a0[k]) ^ __byte_perm(ta1.x, ta1.y, a1[k]) ^
                     __byte_perm(ta2.x, ta2.y, a2[k]) ^ __byte_perm(tb0.x, tb0.y, b0[k]) ^
                     __byte_perm(tb1.x, tb1.y, b1[k]) ^ __byte_perm(tb2.x, tb2.y, b2[k]);
    }
  }
  if (j < n) {
    uint32_t a0[W], a1[W], a2[W];
    load_sel<V>(in[j], q0, chunks, a0, a1, a2);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const uint2 *ta = &tab[(i * n + j) * 3];
      const uint2 ta0 = ta[0], ta1 = ta[1], ta2 = ta[2];
#pragma unroll
      for (int k = 0; k < W; ++k)
        acc[i][k] ^= __byte_perm(ta0.x, ta0.y, a0[k]) ^ __byte_perm(ta1.x, ta1.y, a1[k]) ^
                     __byte_perm(ta2.x, ta2.y, a2[k]);
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const uint64_t q = q0 + (uint64_t)v * blockDim.x;
    if (q >= chunks) break;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const uint32_t *a = &acc[i][4 * v];   // (x0 y0 x1 y1) (x2 y2 x3 y3) per word pair
      __stcs(reinterpret_cast<uint4 *>(out[i]) + q,
             make_uint4(__byte_perm(a[0], a[1], 0x6420), __byte_perm(a[0], a[1], 0x7531),
                        __byte_perm(a[2], a[3], 0x6420), __byte_perm(a[2], a[3], 0x7531)));
    }
  }
}

template <int M>
static void launch_m(const uint8_t *const *in, uint8_t *const *out, int n, int nstripes, uint64_t chunks,
                     const GfCoef &c, cudaStream_t st) {
  const int T = 256;
  constexpr int V = M <= 4 ? 2 : 1;     // 16-byte chunks per thread
  const size_t smem = (size_t)M * n * 24;
  const dim3 grid((unsigned)((chunks + (uint64_t)T * V - 1) / ((uint64_t)T * V)), 1);
  for (int base = 0; base < nstripes; base += 65535) {
    const int cnt = std::min(65535, nstripes - base);
    xslp_gftable_kernel<M, V><<<dim3(grid.x, cnt), T, smem, st>>>(in + (size_t)base * n,
                                                                  out + (size_t)base * M, n, chunks, c);
    CUDA_OK(cudaGetLastError());
    count_launch();
  }
}

}  // namespace xslp

using namespace xslp;

extern "C" int xslp_gf_table_apply(const uint8_t *coef, int n, int m, const uint8_t *const *d_in_tbl,
                                   uint8_t *const *d_out_tbl, int nstripes, size_t block_bytes,
                                   void *stream) {
  API_BEGIN
  if (!coef || n < 1 || n > kMaxIn || m < 1 || m > kMaxOut || nstripes < 0)
    throw Error(XSLP_EINVAL, "bad arguments (1 <= n <= 64, 1 <= m <= 8)");
  if (!d_in_tbl || !d_out_tbl) throw Error(XSLP_EINVAL, "null pointer table");
  if (block_bytes % 16) throw Error(XSLP_EINVAL, "block_bytes must be a multiple of 16");
  if (nstripes == 0 || block_bytes == 0) return XSLP_OK;
  GfCoef c{};
  std::memcpy(c.c, coef, (size_t)m * n);
  const uint64_t chunks = block_bytes / 16;
  cudaStream_t st = (cudaStream_t)stream;
  switch (m) {
    case 1: launch_m<1>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 2: launch_m<2>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 3: launch_m<3>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 4: launch_m<4>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 5: launch_m<5>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 6: launch_m<6>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    case 7: launch_m<7>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
    default: launch_m<8>(d_in_tbl, d_out_tbl, n, nstripes, chunks, c, st); break;
  }
  API_END
}
