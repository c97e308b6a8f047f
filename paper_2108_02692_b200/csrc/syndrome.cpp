// Syndrome-form decode (host side): a B200-specific restructuring of the paper's decode.
//
// The paper decodes an erasure pattern E with the rows of M^-1: one SLP per
// pattern over the n survivors.  With a distinct pattern per stripe, every stripe then runs
// its own large program and the GPU kernel becomes bound by fetching program code
// (profiles/r01_s2_heterogeneous_and_groups.md, cfg5h).  The same bytes follow from the
// parity-check form of the systematic code G = [I_n; R]:
//
//   H = [R | I_p]  (p x (n+p)),  H c = R d + p = 0 for every codeword c = [d; p] (char. 2).
//   With the erased blocks of a codeword replaced by zero blocks (c'),
//   s = H c' = H (c + c_E) = H_E c_E,   H_E = the columns of H at E (p x e).
//   Pick e rows J of H with H_E[J] invertible (MDS: one exists), then  c_E = H_E[J]^-1 s_J.
//
// So every stripe runs ONE shared syndrome program (H over all n+p blocks, erased ones read
// from a zero block) and then a small per-pattern solve program (e x |J| GF entries, lowered
// to an 8e x 8e bitmatrix over the syndrome words).  The solution is unique, so the bytes
// equal the M^-1 decode's bit for bit.
#include <algorithm>
#include <set>

#include "xslp_api.h"

namespace xslp {

// H = [R | I_p] of the (n+p) x n systematic coding matrix g (top n rows must be I_n).
std::vector<uint8_t> parity_check(const uint8_t *g, int n, int p) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (g[(size_t)i * n + j] != (i == j ? 1 : 0))
        throw Error(XSLP_EINVAL, "syndrome decode needs a systematic coding matrix [I; R]");
  std::vector<uint8_t> h((size_t)p * (n + p), 0);
  for (int i = 0; i < p; ++i) {
    for (int j = 0; j < n; ++j) h[(size_t)i * (n + p) + j] = g[(size_t)(n + i) * n + j];
    h[(size_t)i * (n + p) + n + i] = 1;
  }
  return h;
}

// e x p GF matrix mapping the syndrome to the erased blocks (ascending): rows J of H chosen
// lexicographically-first with H_E[J] invertible; entry (q, J[t]) = (H_E[J]^-1)[q][t].
std::vector<uint8_t> solve_rows(const std::vector<uint8_t> &h, int n, int p, const std::vector<int> &er) {
  const int e = (int)er.size(), w = n + p;
  std::vector<int> rows(e);
  for (int t = 0; t < e; ++t) rows[t] = t;
  for (;;) {
    std::vector<uint8_t> m((size_t)e * e);
    for (int a = 0; a < e; ++a)
      for (int b = 0; b < e; ++b) m[(size_t)a * e + b] = h[(size_t)rows[a] * w + er[b]];
    try {
      auto x = gf::invert(m, e);
      std::vector<uint8_t> out((size_t)e * p, 0);
      for (int q = 0; q < e; ++q)
        for (int t = 0; t < e; ++t) out[(size_t)q * p + rows[t]] = x[(size_t)q * e + t];
      return out;
    } catch (const Error &ex) {
      if (ex.code != XSLP_ESINGULAR) throw;
    }
    int i = e - 1;  // next e-subset of [0, p)
    while (i >= 0 && rows[i] == p - e + i) --i;
    if (i < 0) throw Error(XSLP_ESINGULAR, "no invertible row set: the code is not MDS for this pattern");
    ++rows[i];
    for (int k = i + 1; k < e; ++k) rows[k] = rows[k - 1] + 1;
  }
}

}  // namespace xslp

using namespace xslp;

extern "C" int xslp_syndrome_bitmatrices(const uint8_t *g, int n, int p, const int32_t *erased, int ne,
                                         uint8_t *syn_bits, uint8_t *solve_bits) {
  API_BEGIN
  if (!g || n < 1 || p < 1 || n + p > 255 || ne < 1 || !erased) throw Error(XSLP_EINVAL, "bad arguments");
  if (ne > p) throw Error(XSLP_EUNRECOVERABLE, "more erasures than parity blocks");
  std::set<int> es;
  for (int i = 0; i < ne; ++i) {
    if (erased[i] < 0 || erased[i] >= n + p) throw Error(XSLP_EINVAL, "erasure index out of range");
    if (!es.insert(erased[i]).second) throw Error(XSLP_EINVAL, "duplicate erasure index");
  }
  auto h = parity_check(g, n, p);
  if (syn_bits) {
    auto b = gf::to_bits(h, p, n + p);
    std::copy(b.begin(), b.end(), syn_bits);
  }
  if (solve_bits) {
    auto x = solve_rows(h, n, p, std::vector<int>(es.begin(), es.end()));
    auto b = gf::to_bits(x, ne, p);
    std::copy(b.begin(), b.end(), solve_bits);
  }
  API_END
}
