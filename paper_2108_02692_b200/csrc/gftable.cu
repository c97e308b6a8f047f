// The paper's approach (1) on B200, as a comparison point (SURVEY §8(f) NEXT #3 alternative):
// Reed-Solomon as matrix multiplication over GF(2^8) with table-driven field multiplication
// ("tightly coupling sophisticated optimization methods for MM and finite field
// multiplication", ISA-L's nibble-table / PSHUFB method), instead of the XOR-based
// approach (2) that the rest of libxslp implements.
//
// Byte layout: output block i = sum_j coef[i][j] * input block j, byte by byte.
// Multiplication by a constant c is linear over GF(2), so c*x = c*(x & 15) ^ c*(x & 0xF0):
// two 16-entry tables per coefficient.  On the GPU the PSHUFB step becomes PRMT (byte permute
// of two 32-bit registers by 4-bit selectors): entries 0-7 come from one PRMT, entries 8-15
// from another, and bit 3 of each nibble selects between them.  A thread owns 16 bytes of
// every block; each CTA builds its nibble tables in shared memory from the coefficient
// matrix (a kernel parameter) at start-up.
//
// Work per (coefficient, 4 bytes): 4 PRMT + 2 LOP3 on the ALU pipe, plus per input word the
// nibble split and selects; ALU-bound at roughly 10 instructions per data byte for RS(10,4)
// where the compiled XOR program needs about 0.8 (profiles/r01_s2_gftable.md).
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

// 16 table bytes as 4 words (entry e = byte e) -> product of the 4 packed nibbles in `nib`
// (byte k of nib holds a value 0..15) looked up byte by byte.
__device__ __forceinline__ uint32_t lookup16(const uint4 t, uint32_t nib) {
  // selectors: the 4 nibble values packed into the low 16 bits, bit 3 cleared (PRMT's
  // bit 3 would replicate the sign); bit 3 chooses the upper 8 entries
  uint32_t pk = __byte_perm(nib | (nib >> 4), 0, 0x4420) & 0x7777u;
  uint32_t lo = __byte_perm(t.x, t.y, pk);
  uint32_t hi = __byte_perm(t.z, t.w, pk);
  uint32_t m = ((nib >> 3) & 0x01010101u) * 0xFFu;
  return (hi & m) | (lo & ~m);
}

template <int M>
__global__ void __launch_bounds__(256) xslp_gftable_kernel(const uint8_t *const *__restrict__ in_tbl,
                                                           uint8_t *const *__restrict__ out_tbl,
                                                           int n, uint64_t chunks, GfCoef coef) {
  // tables: [i][j] -> lo (16 B) and hi (16 B) nibble tables
  extern __shared__ uint4 tab[];
  for (int e = threadIdx.x; e < M * n * 32; e += blockDim.x) {
    const int pair = e / 32, x = e % 32;
    const uint32_t c = coef.c[pair];
    const uint32_t v = x < 16 ? gf_mul_dev(c, x) : gf_mul_dev(c, (uint32_t)(x - 16) << 4);
    reinterpret_cast<uint8_t *>(tab)[pair * 32 + x] = (uint8_t)v;
  }
  __syncthreads();
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= chunks) return;
  const uint32_t stripe = blockIdx.y;
  const uint8_t *const *in = in_tbl + (uint64_t)stripe * n;
  uint8_t *const *out = out_tbl + (uint64_t)stripe * M;
  uint4 acc[M];
#pragma unroll
  for (int i = 0; i < M; ++i) acc[i] = make_uint4(0, 0, 0, 0);
  for (int j = 0; j < n; ++j) {
    const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(in[j]) + q);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      lo[k] = w[k] & 0x0F0F0F0Fu;
      hi[k] = (w[k] >> 4) & 0x0F0F0F0Fu;
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const uint4 tl = tab[(i * n + j) * 2], th = tab[(i * n + j) * 2 + 1];
      uint32_t *a = reinterpret_cast<uint32_t *>(&acc[i]);
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] ^= lookup16(tl, lo[k]) ^ lookup16(th, hi[k]);
    }
  }
#pragma unroll
  for (int i = 0; i < M; ++i) __stcs(reinterpret_cast<uint4 *>(out[i]) + q, acc[i]);
}

template <int M>
static void launch_m(const uint8_t *const *in, uint8_t *const *out, int n, int nstripes, uint64_t chunks,
                     const GfCoef &c, cudaStream_t st) {
  const int T = 256;
  const size_t smem = (size_t)M * n * 32;
  const dim3 grid((unsigned)((chunks + T - 1) / T), 1);
  for (int base = 0; base < nstripes; base += 65535) {
    const int cnt = std::min(65535, nstripes - base);
    xslp_gftable_kernel<M><<<dim3(grid.x, cnt), T, smem, st>>>(in + (size_t)base * n,
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
