// GF(2^8) and the coding matrices of the product path.
//
// Field: polynomial x^8+x^4+x^3+x^2+1 = 0x11D ([Eval] §Dataset), generator 2.
// Implemented with exp/log tables (the oracle uses shift-and-add; no code is shared).
// Matrices: [I; 2^{ij}] (reading R1, reproduces #xor(P_enc) = 755 of P:1652),
// [I; M V^-1] (the text's construction), Cauchy inv((n+i)^j) (R2).
// Lowering x~: block (i,j) row r column k = bit r of G_ij * 2^k (R3).
#include "xslp_internal.h"

namespace xslp {
namespace gf {

namespace {
struct Tables {
  uint8_t exp[512];
  int log[256];
  Tables() {
    int x = 1;
    for (int i = 0; i < 255; ++i) {
      exp[i] = (uint8_t)x;
      log[x] = i;
      x <<= 1;
      if (x & 0x100) x ^= 0x11D;
    }
    for (int i = 255; i < 512; ++i) exp[i] = exp[i - 255];
    log[0] = -1;
  }
};
const Tables &T() {
  static Tables t;
  return t;
}
}  // namespace

uint8_t mul(uint8_t a, uint8_t b) {
  if (!a || !b) return 0;
  return T().exp[T().log[a] + T().log[b]];
}

uint8_t inv(uint8_t a) {
  if (!a) throw Error(XSLP_ESINGULAR, "inverse of 0 in GF(2^8)");
  return T().exp[255 - T().log[a]];
}

uint8_t pow(uint8_t a, int e) {
  if (e == 0) return 1;
  if (!a) return 0;
  return T().exp[(int)(((int64_t)T().log[a] * e) % 255)];
}

std::vector<uint8_t> invert(const std::vector<uint8_t> &m, int n) {
  std::vector<uint8_t> a(m), r(n * n, 0);
  for (int i = 0; i < n; ++i) r[i * n + i] = 1;
  for (int c = 0; c < n; ++c) {
    int piv = -1;
    for (int i = c; i < n; ++i)
      if (a[i * n + c]) { piv = i; break; }
    if (piv < 0) throw Error(XSLP_ESINGULAR, "singular matrix");
    if (piv != c)
      for (int j = 0; j < n; ++j) {
        std::swap(a[piv * n + j], a[c * n + j]);
        std::swap(r[piv * n + j], r[c * n + j]);
      }
    uint8_t f = inv(a[c * n + c]);
    for (int j = 0; j < n; ++j) {
      a[c * n + j] = mul(f, a[c * n + j]);
      r[c * n + j] = mul(f, r[c * n + j]);
    }
    for (int i = 0; i < n; ++i) {
      if (i == c || !a[i * n + c]) continue;
      uint8_t g = a[i * n + c];
      for (int j = 0; j < n; ++j) {
        a[i * n + j] ^= mul(g, a[c * n + j]);
        r[i * n + j] ^= mul(g, r[c * n + j]);
      }
    }
  }
  return r;
}

std::vector<uint8_t> coding_matrix(int n, int p, int kind) {
  std::vector<uint8_t> g((size_t)(n + p) * n, 0);
  for (int i = 0; i < n; ++i) g[i * n + i] = 1;
  if (kind == XSLP_RS_ISAL) {
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < n; ++j) g[(n + i) * n + j] = pow(pow(2, i), j);
  } else if (kind == XSLP_CAUCHY) {
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < n; ++j) {
        int x = (n + i) ^ j;
        if (x == 0 || x > 255) throw Error(XSLP_EINVAL, "Cauchy matrix undefined for this (n,p)");
        g[(n + i) * n + j] = inv((uint8_t)x);
      }
  } else if (kind == XSLP_RS_SYSVAND) {
    // Vandermonde rows i = 1..n+p: (alpha^i)^j; reduce to [I; M V^-1].
    std::vector<uint8_t> V((size_t)n * n), M((size_t)p * n);
    for (int i = 1; i <= n + p; ++i)
      for (int j = 0; j < n; ++j) {
        uint8_t v = pow(pow(2, i), j);
        if (i <= n) V[(i - 1) * n + j] = v; else M[(i - 1 - n) * n + j] = v;
      }
    auto Vi = invert(V, n);
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < n; ++j) {
        uint8_t s = 0;
        for (int k = 0; k < n; ++k) s ^= mul(M[i * n + k], Vi[k * n + j]);
        g[(n + i) * n + j] = s;
      }
  } else {
    throw Error(XSLP_EINVAL, "unknown matrix kind");
  }
  return g;
}

std::vector<uint8_t> to_bits(const std::vector<uint8_t> &m, int a, int b) {
  std::vector<uint8_t> bits((size_t)64 * a * b, 0);
  const int cols = 8 * b;
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < b; ++j) {
      uint8_t x = m[i * b + j];
      for (int k = 0; k < 8; ++k) {
        uint8_t col = mul(x, (uint8_t)(1u << k));
        for (int r = 0; r < 8; ++r)
          bits[(size_t)(8 * i + r) * cols + 8 * j + k] = (col >> r) & 1;
      }
    }
  return bits;
}

}  // namespace gf
}  // namespace xslp
