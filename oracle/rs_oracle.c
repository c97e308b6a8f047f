/* O3/O4 in C -- Reed-Solomon over the strip layout, multi-threaded (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library (through oracle/native.py).  It shares no code with the product
 * (paper_2108_02692_b200/): its own field, its own tables, its own input generator.
 *
 * What it computes is oracle/rs.py apply_rows, written in C so that whole BASELINE workloads
 * (10-40 GB of data) can be checked in seconds on the host cores:
 *   - field: GF(2^8) with x^8+x^4+x^3+x^2+1 ([Eval] §Dataset); multiplication is the
 *     carry-less product reduced mod the polynomial (gf_mul below), tabulated once;
 *   - layout: a block of B bytes is 8 strips of B/8 bytes, constant c_{8j+k} = strip k of
 *     block j (DESIGN reading R3 / R5);
 *   - the rows R (m x n over GF(2^8)) act on the 8n strips through their bitmatrix V~, cell
 *     (i, j) = x~(R_ij) with entry (r, k) = bit r of R_ij * 2^k (reading R3), and
 *     "MM over GF(2) is just array XORs": output strip (i, r) is the XOR of the
 *     input strips (j, k) whose bit is set -- the NAIVE product (no XorRePair, no sharing),
 *     i.e. oracle/rs.py bitmatrix_apply.  That this equals the table-driven byte RS on the
 *     bit-transposed view (oracle/rs.py apply_rows) is pinned byte for byte
 *     in tests/test_oracle_native.py.
 *   - inputs: the synth generator (synth/__init__.py), reimplemented here:
 *     word i of block j of stripe s = splitmix64(seed*0x9E3779B97F4A7C15 + ((s*64+j)<<40) + i).
 *
 * Pinned byte for byte to the numpy oracle (oracle/rs.py) and to synth on small inputs by
 * tests/test_oracle_native.py (-m "not gpu").
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- O1: GF(2^8) ------------------------------------------------------------------------ */
static uint8_t gf_mul(uint8_t a, uint8_t b) { /* polynomial product mod 0x11D */
  unsigned r = 0, x = a;
  while (b) {
    if (b & 1) r ^= x;
    b >>= 1;
    x <<= 1;
    if (x & 0x100) x ^= 0x11D;
  }
  return (uint8_t)r;
}

static uint8_t MUL[256][256];
static pthread_once_t mul_once = PTHREAD_ONCE_INIT;
static void mul_init(void) {
  for (int a = 0; a < 256; ++a)
    for (int b = 0; b < 256; ++b) MUL[a][b] = gf_mul((uint8_t)a, (uint8_t)b);
}

uint8_t oracle_gf_mul(uint8_t a, uint8_t b) { return gf_mul(a, b); }

/* ---- x~: the GF(2) lowering of a coefficient ----------------------------------- */
/* Reading R3 (LSB first): entry (r, k) of x~(c) is bit r of c * 2^k, so that
 * c * y = B^-1(x~(c) B(y)) -- pinned exhaustively in tests/test_oracle_native.py. */
int oracle_tilde_bit(uint8_t c, int r, int k) { return (gf_mul(c, (uint8_t)(1u << k)) >> r) & 1; }

/* ---- O3/O4: apply GF rows to one stripe in the strip layout ----------------------------- */
/* rows: m x n coefficients (row-major); in: n blocks of B bytes (block j at in + j*B);
 * out: m blocks of B bytes.  B % 8 == 0.
 *
 * MM over GF(2) "is just array XORs": with V~ the bitmatrix of the rows (cell
 * (i, j) = x~(R_ij)), output strip (i, r) = XOR of the input strips (j, k) whose bit in row
 * 8i + r of V~ is set -- the naive (uncompressed) product, one 64-bit word of every strip at a
 * time.  Words are processed 64 at a time through staging copies (the 8n input strips lie
 * B/8 bytes apart, which maps them onto the same L1 sets); a tail shorter than 8 bytes per
 * strip cannot occur because B % 8 == 0 leaves strips of B/8 bytes, handled bytewise below. */
#define CHUNK 64
void oracle_apply_rows(const uint8_t *rows, int m, int n, const uint8_t *in, uint8_t *out, size_t B) {
  pthread_once(&mul_once, mul_init);
  const size_t S = B / 8;          /* strip bytes */
  /* the bitmatrix rows as lists of input strips */
  int *lst = (int *)malloc(sizeof(int) * (size_t)(8 * m) * (size_t)(8 * n + 1));
  for (int i = 0; i < m; ++i)
    for (int r = 0; r < 8; ++r) {
      int *L = lst + (size_t)(8 * i + r) * (size_t)(8 * n + 1), cnt = 0;
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < 8; ++k)
          if ((MUL[rows[i * n + j]][1u << k] >> r) & 1) L[1 + cnt++] = 8 * j + k;
      L[0] = cnt;
    }
  const size_t W = S / 8;          /* whole 64-bit words per strip */
  uint64_t *sin = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(8 * n) * CHUNK);
  for (size_t w0 = 0; w0 < W; w0 += CHUNK) {
    const size_t cn = W - w0 < CHUNK ? W - w0 : CHUNK;
    for (int c = 0; c < 8 * n; ++c)
      memcpy(sin + (size_t)c * CHUNK, in + (size_t)(c / 8) * B + (size_t)(c % 8) * S + 8 * w0, 8 * cn);
    for (int g = 0; g < 8 * m; ++g) {
      const int *L = lst + (size_t)g * (size_t)(8 * n + 1);
      uint64_t acc[CHUNK];
      for (size_t w = 0; w < cn; ++w) acc[w] = 0;
      for (int q = 1; q <= L[0]; ++q) {
        const uint64_t *src = sin + (size_t)L[q] * CHUNK;
        for (size_t w = 0; w < cn; ++w) acc[w] ^= src[w];
      }
      memcpy(out + (size_t)(g / 8) * B + (size_t)(g % 8) * S + 8 * w0, acc, 8 * cn);
    }
  }
  for (size_t o = 8 * W; o < S; ++o)   /* strip bytes past the last whole word */
    for (int g = 0; g < 8 * m; ++g) {
      const int *L = lst + (size_t)g * (size_t)(8 * n + 1);
      uint8_t acc = 0;
      for (int q = 1; q <= L[0]; ++q) acc ^= in[(size_t)(L[q] / 8) * B + (size_t)(L[q] % 8) * S + o];
      out[(size_t)(g / 8) * B + (size_t)(g % 8) * S + o] = acc;
    }
  free(sin);
  free(lst);
}

/* Textbook byte-wise RS: out_i[t] = sum_j R_ij d_j[t] over GF(2^8), one byte
 * position at a time -- what the byte-compatible layout and the paper's approach (1) compute
 * (oracle/rs.py bytewise_apply). */
void oracle_apply_bytewise(const uint8_t *rows, int m, int n, const uint8_t *in, uint8_t *out, size_t B) {
  pthread_once(&mul_once, mul_init);
  for (int i = 0; i < m; ++i) {
    uint8_t *o = out + (size_t)i * B;
    memset(o, 0, B);
    for (int j = 0; j < n; ++j) {
      const uint8_t *mul = MUL[rows[i * n + j]], *d = in + (size_t)j * B;
      for (size_t t = 0; t < B; ++t) o[t] ^= mul[d[t]];
    }
  }
}

/* ---- the synth input generator ---------------------------------------------------------- */
static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* nblocks data blocks of stripe `stripe` into out (nblocks x B bytes, little-endian words) */
void oracle_fill(uint64_t seed, int64_t stripe, int nblocks, size_t B, uint8_t *out) {
  for (int j = 0; j < nblocks; ++j) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull + (((uint64_t)stripe * 64 + (uint64_t)j) << 40);
    for (size_t i = 0; i < B / 8; ++i) {
      const uint64_t v = splitmix64(base + i);
      for (int q = 0; q < 8; ++q) out[(size_t)j * B + 8 * i + q] = (uint8_t)(v >> (8 * q));
    }
  }
}

/* ---- whole-workload checks, threads over stripes ---------------------------------------- */
/* mode 0 (apply): the n input blocks of stripe s are oracle_fill(seed, stripe0+s, n, B); the
 *   expected m outputs are rows . inputs (encode: rows = R; decode of arbitrary survivor bytes:
 *   rows = the decode rows).
 * mode 1 (codeword): the data blocks are oracle_fill(seed, stripe0+s, n, B), the codeword is
 *   [data; rows . data] with rows = the p x n parity rows R, and the expected m outputs are
 *   the codeword blocks sel[s*m + k] (a decode's erased blocks, ascending).
 * mode 2 (bytewise): as mode 0 with the textbook byte-wise product instead of the strip layout.
 * got: nstripes x m x B host bytes.  bad: per stripe, 1 if any byte differs.  Returns the
 * number of differing stripes. */
typedef struct {
  int mode, m, n, p;
  const uint8_t *rows;
  const int32_t *sel;
  uint64_t seed;
  int64_t stripe0;
  size_t B;
  const uint8_t *got;
  uint8_t *bad;
  int s_lo, s_hi;
  int64_t nbad;
} job_t;

static void *check_worker(void *arg) {
  job_t *J = (job_t *)arg;
  const int nb_in = J->n;
  const int nout = J->mode == 1 ? J->p : J->m;
  uint8_t *in = (uint8_t *)malloc((size_t)nb_in * J->B);
  uint8_t *out = (uint8_t *)malloc((size_t)(nout > 0 ? nout : 1) * J->B);
  for (int s = J->s_lo; s < J->s_hi; ++s) {
    oracle_fill(J->seed, J->stripe0 + s, nb_in, J->B, in);
    if (J->mode == 2) oracle_apply_bytewise(J->rows, nout, nb_in, in, out, J->B);
    else oracle_apply_rows(J->rows, nout, nb_in, in, out, J->B);
    const uint8_t *g = J->got + (size_t)s * J->m * J->B;
    int diff = 0;
    for (int k = 0; k < J->m && !diff; ++k) {
      const uint8_t *want;
      if (J->mode != 1) {
        want = out + (size_t)k * J->B;
      } else {
        const int e = J->sel[(size_t)s * J->m + k];
        want = e < J->n ? in + (size_t)e * J->B : out + (size_t)(e - J->n) * J->B;
      }
      diff = memcmp(g + (size_t)k * J->B, want, J->B) != 0;
    }
    if (J->bad) J->bad[s] = (uint8_t)diff;
    J->nbad += diff;
  }
  free(in);
  free(out);
  return 0;
}

int64_t oracle_check(int mode, const uint8_t *rows, int m, int n, int p, const int32_t *sel,
                     uint64_t seed, int64_t stripe0, int nstripes, size_t B, const uint8_t *got,
                     uint8_t *bad, int nthreads) {
  pthread_once(&mul_once, mul_init);
  if (nstripes <= 0) return 0;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nstripes) nthreads = nstripes;
  job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    job_t *J = &jobs[t];
    J->mode = mode;
    J->m = m;
    J->n = n;
    J->p = p;
    J->rows = rows;
    J->sel = sel;
    J->seed = seed;
    J->stripe0 = stripe0;
    J->B = B;
    J->got = got;
    J->bad = bad;
    J->s_lo = (int)((int64_t)nstripes * t / nthreads);
    J->s_hi = (int)((int64_t)nstripes * (t + 1) / nthreads);
    pthread_create(&th[t], 0, check_worker, J);
  }
  int64_t nbad = 0;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], 0);
    nbad += jobs[t].nbad;
  }
  free(jobs);
  free(th);
  return nbad;
}

/* Throughput leg (bench.py cpu_baseline / --impl reference), the caller times it: apply the
 * rows of each stripe (rows + s * rows_stride; stride 0 = one matrix for all) to pre-generated
 * inputs (in = nstripes x n x B; the generator is not timed); bytewise selects the textbook
 * byte-wise product instead of the strip layout. */
typedef struct {
  const uint8_t *rows, *in;
  uint8_t *out;
  size_t rows_stride;
  int bytewise, m, n;
  size_t B;
  int s_lo, s_hi;
} app_job_t;

static void *app_worker(void *arg) {
  app_job_t *J = (app_job_t *)arg;
  for (int s = J->s_lo; s < J->s_hi; ++s) {
    const uint8_t *r = J->rows + (size_t)s * J->rows_stride;
    const uint8_t *x = J->in + (size_t)s * J->n * J->B;
    uint8_t *y = J->out + (size_t)s * J->m * J->B;
    if (J->bytewise) oracle_apply_bytewise(r, J->m, J->n, x, y, J->B);
    else oracle_apply_rows(r, J->m, J->n, x, y, J->B);
  }
  return 0;
}

void oracle_apply_each(int bytewise, const uint8_t *rows, size_t rows_stride, int m, int n,
                       const uint8_t *in, uint8_t *out, int nstripes, size_t B, int nthreads) {
  pthread_once(&mul_once, mul_init);
  if (nstripes <= 0) return;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nstripes) nthreads = nstripes;
  app_job_t *jobs = (app_job_t *)calloc((size_t)nthreads, sizeof(app_job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    app_job_t *J = &jobs[t];
    J->rows = rows;
    J->rows_stride = rows_stride;
    J->bytewise = bytewise;
    J->in = in;
    J->out = out;
    J->m = m;
    J->n = n;
    J->B = B;
    J->s_lo = (int)((int64_t)nstripes * t / nthreads);
    J->s_hi = (int)((int64_t)nstripes * (t + 1) / nthreads);
    pthread_create(&th[t], 0, app_worker, J);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], 0);
  free(jobs);
  free(th);
}
