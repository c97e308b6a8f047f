/* A plain C consumer of libxslp (no Python, no torch): the boundary as a C program sees it.
 *
 *   host mode (no GPU needed):  matrices, bitmatrix, compile, stats, dump, error reporting,
 *                               and a device call failing loudly without a device.
 *   device mode (argv[1] == "gpu"): RS(10,4) encode + a 4-erasure decode of 8 stripes of
 *                               1 MiB through xslp_encode_batch with cudaMalloc'd buffers;
 *                               checks parity block 0 = XOR of the data (the RAID-5 row of
 *                               [I; 2^ij]) and that decoding restores the erased blocks.
 * Prints "ok <mode>" and exits 0 on success. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "xslp.h"

#ifdef XSLP_WITH_CUDA
#include <cuda_runtime.h>
#endif

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ < 0) {                                                                \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,      \
              xslp_last_error());                                                 \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static int host_mode(void) {
  uint8_t g[14 * 10], bits[32 * 80], dbits[32 * 80];
  int32_t surv[10], er[4] = {2, 4, 5, 6};
  CHECK(xslp_coding_matrix(10, 4, XSLP_RS_ISAL, g));
  if (g[10 * 10 + 3] != 1 || g[11 * 10 + 1] != 2) return fprintf(stderr, "matrix\n"), 1;
  CHECK(xslp_encode_bitmatrix(g, 10, 4, bits));
  CHECK(xslp_decode_bitmatrix(g, 10, 4, er, 4, dbits, surv));
  xslp_opts o;
  xslp_default_opts(&o);
  o.specialise = 0;
  o.compress = XSLP_COMPRESS_NONE;
  o.fuse = 0;
  o.schedule = XSLP_SCHED_NONE;
  xslp_program *base = NULL, *enc = NULL;
  CHECK(xslp_compile(bits, 32, 80, &o, &base));
  xslp_stats st;
  CHECK(xslp_program_stats(base, &st));
  if (st.xor_count != 755) return fprintf(stderr, "P_enc #xor %lld != 755 (P:1652)\n", (long long)st.xor_count), 1;
  xslp_default_opts(&o);
  o.specialise = 0;
  CHECK(xslp_compile(bits, 32, 80, &o, &enc));
  CHECK(xslp_program_stats(enc, &st));
  if (st.xor_count >= 755 || st.n_goals != 32 || st.n_const != 80) return fprintf(stderr, "stats\n"), 1;
  int64_t need = xslp_program_dump(enc, 0, NULL, 0);
  char *txt = (char *)malloc((size_t)need + 1);
  if (xslp_program_dump(enc, 0, txt, (size_t)need + 1) != need || !strstr(txt, "return")) return 1;
  free(txt);
  /* errors are codes + a message, never an abort */
  int32_t bad[5] = {0, 1, 2, 3, 4};
  if (xslp_decode_bitmatrix(g, 10, 4, bad, 5, dbits, surv) != XSLP_EUNRECOVERABLE) return 1;
  if (strlen(xslp_last_error()) == 0) return 1;
  if (xslp_compile(NULL, 32, 80, &o, &base) != XSLP_EINVAL) return 1;
  xslp_free(base);
  xslp_free(enc);
  printf("ok host %s\n", xslp_version());
  return 0;
}

#ifdef XSLP_WITH_CUDA
static int gpu_mode(void) {
  enum { N = 10, P = 4, S = 8 };
  const size_t B = 1 << 20;
  uint8_t g[(N + P) * N], bits[8 * P * 8 * N], dbits[8 * P * 8 * N];
  int32_t er[P] = {0, 3, 11, 13}, surv[N];
  CHECK(xslp_coding_matrix(N, P, XSLP_RS_ISAL, g));
  CHECK(xslp_encode_bitmatrix(g, N, P, bits));
  CHECK(xslp_decode_bitmatrix(g, N, P, er, P, dbits, surv));
  xslp_opts o;
  xslp_default_opts(&o);
  o.block_bytes_hint = (int64_t)B;
  xslp_program *enc = NULL, *dec = NULL;
  CHECK(xslp_compile(bits, 8 * P, 8 * N, &o, &enc));
  CHECK(xslp_compile(dbits, 8 * P, 8 * N, &o, &dec));
  uint8_t *blocks, *rec;
  if (cudaMalloc((void **)&blocks, (size_t)S * (N + P) * B) || cudaMalloc((void **)&rec, (size_t)S * P * B)) return 1;
  CHECK(xslp_fill_random(blocks, S, N + P, B, 7, 0, NULL));
  const uint8_t **tin = (const uint8_t **)malloc(sizeof(void *) * S * N), **tdin = (const uint8_t **)malloc(sizeof(void *) * S * N);
  uint8_t **tout = (uint8_t **)malloc(sizeof(void *) * S * P), **trec = (uint8_t **)malloc(sizeof(void *) * S * P);
  for (int s = 0; s < S; ++s) {
    for (int j = 0; j < N; ++j) {
      tin[s * N + j] = blocks + ((size_t)s * (N + P) + j) * B;
      tdin[s * N + j] = blocks + ((size_t)s * (N + P) + surv[j]) * B;
    }
    for (int i = 0; i < P; ++i) {
      tout[s * P + i] = blocks + ((size_t)s * (N + P) + N + i) * B;
      trec[s * P + i] = rec + ((size_t)s * P + i) * B;
    }
  }
  void *d_tin, *d_tout, *d_tdin, *d_trec;
  const size_t ti = sizeof(void *) * S * N, to = sizeof(void *) * S * P;
  if (cudaMalloc(&d_tin, ti) || cudaMalloc(&d_tout, to) || cudaMalloc(&d_tdin, ti) || cudaMalloc(&d_trec, to)) return 1;
  cudaMemcpy(d_tin, tin, ti, cudaMemcpyHostToDevice);
  cudaMemcpy(d_tout, tout, to, cudaMemcpyHostToDevice);
  cudaMemcpy(d_tdin, tdin, ti, cudaMemcpyHostToDevice);
  cudaMemcpy(d_trec, trec, to, cudaMemcpyHostToDevice);
  CHECK(xslp_encode_batch(enc, (const uint8_t *const *)d_tin, (uint8_t *const *)d_tout, S, B, NULL));
  CHECK(xslp_encode_batch(dec, (const uint8_t *const *)d_tdin, (uint8_t *const *)d_trec, S, B, NULL));
  if (cudaDeviceSynchronize()) return fprintf(stderr, "cuda error\n"), 1;
  uint8_t *h = (uint8_t *)malloc((size_t)S * (N + P) * B), *hr = (uint8_t *)malloc((size_t)S * P * B);
  cudaMemcpy(h, blocks, (size_t)S * (N + P) * B, cudaMemcpyDeviceToHost);
  cudaMemcpy(hr, rec, (size_t)S * P * B, cudaMemcpyDeviceToHost);
  for (int s = 0; s < S; ++s) {
    const uint8_t *st = h + (size_t)s * (N + P) * B;
    for (size_t o2 = 0; o2 < B; ++o2) {
      uint8_t x = 0;
      for (int j = 0; j < N; ++j) x ^= st[(size_t)j * B + o2];
      if (x != st[(size_t)N * B + o2]) return fprintf(stderr, "parity0 stripe %d byte %zu\n", s, o2), 1;
    }
    for (int i = 0; i < P; ++i)
      if (memcmp(hr + ((size_t)s * P + i) * B, st + (size_t)er[i] * B, B))
        return fprintf(stderr, "decode stripe %d block %d\n", s, er[i]), 1;
  }
  printf("ok gpu launches=%lld\n", (long long)xslp_launch_count());
  return 0;
}
#endif

int main(int argc, char **argv) {
  if (argc > 1 && !strcmp(argv[1], "gpu")) {
#ifdef XSLP_WITH_CUDA
    return gpu_mode();
#else
    fprintf(stderr, "built without CUDA\n");
    return 2;
#endif
  }
  if (host_mode()) return 1;
  /* without a device every device call fails loudly */
  if (argc > 1 && !strcmp(argv[1], "nodevice")) {
    xslp_program *p = NULL;
    uint8_t g[14 * 10], bits[32 * 80];
    xslp_coding_matrix(10, 4, XSLP_RS_ISAL, g);
    xslp_encode_bitmatrix(g, 10, 4, bits);
    xslp_opts o;
    xslp_default_opts(&o);
    o.specialise = 0;
    CHECK(xslp_compile(bits, 32, 80, &o, &p));
    int rc = xslp_fill_random((uint8_t *)16, 1, 1, 64, 1, 0, NULL);
    if (rc != XSLP_ECUDA) return fprintf(stderr, "expected XSLP_ECUDA, got %d\n", rc), 1;
    xslp_free(p);
    printf("ok nodevice\n");
  }
  return 0;
}
