// Concurrent host-side stress of libxslp (no GPU needed), for the sanitizer builds
// (scripts/sanitize_host.sh: ASan+UBSan and TSan).  The header promises that compiled programs
// are immutable and shareable across threads and that codecs are thread-safe
// (include/xslp.h); this drives those paths from many threads at once:
//   * xslp_compile of seeded random bitmatrices (host compiler; every 4th with the in-process
//     PTX -> sm_100a JIT), stats, every dump form, the LRU cache measures, free;
//   * one shared program read by all threads (stats / dumps / cache measures);
//   * one shared codec with a small memo (forces LRU eviction) asked for decode programs of
//     random erasure patterns, each handed-out program then used (dumped) by its thread;
//   * error paths: the thread-local last-error message of each thread's own failing call.
// Prints "ok stress <threads> <iterations>" and exits 0; any failure exits non-zero.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "xslp.h"

static std::atomic<int> g_fail{0};

#define REQUIRE(c)                                                                   \
  do {                                                                               \
    if (!(c)) {                                                                      \
      std::fprintf(stderr, "%s:%d: %s (%s)\n", __FILE__, __LINE__, #c, xslp_last_error()); \
      g_fail++;                                                                      \
      return;                                                                        \
    }                                                                                \
  } while (0)

static void use_program(const xslp_program *p) {
  xslp_stats st;
  REQUIRE(xslp_program_stats(p, &st) == XSLP_OK);
  for (int form : {0, 1, 3, 4}) {
    const int64_t need = xslp_program_dump(p, form, nullptr, 0);
    REQUIRE(need > 0);
    std::string buf((size_t)need + 1, '\0');
    REQUIRE(xslp_program_dump(p, form, &buf[0], buf.size()) == need);
  }
  int64_t io = -1;
  int32_t ccap = 0;
  REQUIRE(xslp_program_cache(p, 0, nullptr, &ccap) == XSLP_OK);   // CCap
  REQUIRE(ccap >= 1);
  REQUIRE(xslp_program_cache(p, ccap, &io, nullptr) == XSLP_OK);  // IOcost at that capacity
  REQUIRE(io >= 0);
}

static void worker(int tid, int iters, const xslp_program *shared, xslp_codec *codec) {
  std::mt19937 rng(1234 + tid);
  for (int it = 0; it < iters; ++it) {
    // a random bitmatrix: 1-3 output blocks over 2-10 input blocks
    const int m = 8 * (1 + (int)(rng() % 3)), n = 8 * (2 + (int)(rng() % 9));
    std::vector<uint8_t> bits((size_t)m * n);
    for (auto &b : bits) b = (rng() % 3) == 0;
    xslp_opts o;
    xslp_default_opts(&o);
    o.specialise = (it % 4 == 0);
    o.schedule = (int)(rng() % 3);
    o.greedy_capacity = 8 + (int)(rng() % 32);
    o.compress = (int)(rng() % 3);
    xslp_program *p = nullptr;
    REQUIRE(xslp_compile(bits.data(), m, n, &o, &p) == XSLP_OK);
    use_program(p);
    xslp_free(p);
    use_program(shared);
    // the shared codec: decode programs of random 1-4 erasure patterns of RS(10,4)
    int32_t er[4];
    const int ne = 1 + (int)(rng() % 4);
    std::vector<int> pool(14);
    for (int i = 0; i < 14; ++i) pool[i] = i;
    for (int i = 0; i < ne; ++i) {
      std::swap(pool[i], pool[i + rng() % (14 - i)]);
      er[i] = pool[i];
    }
    const xslp_program *dp = nullptr;
    REQUIRE(xslp_codec_program(codec, er, ne, &dp) == XSLP_OK && dp);
    use_program(dp);
    REQUIRE(xslp_codec_cached(codec) >= 0);
    // error path: this thread's own message
    const int bad_n = 300 + tid;
    REQUIRE(xslp_coding_matrix(bad_n, 4, XSLP_RS_ISAL, nullptr) != XSLP_OK);
    REQUIRE(std::strlen(xslp_last_error()) > 0);
  }
}

int main(int argc, char **argv) {
  const int threads = argc > 1 ? std::atoi(argv[1]) : 8;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 40;
  uint8_t g[14 * 10], bits[32 * 80];
  if (xslp_coding_matrix(10, 4, XSLP_RS_ISAL, g) || xslp_encode_bitmatrix(g, 10, 4, bits)) return 1;
  xslp_opts o;
  xslp_default_opts(&o);
  o.specialise = 0;
  xslp_program *shared = nullptr;
  if (xslp_compile(bits, 32, 80, &o, &shared)) return 1;
  xslp_codec *codec = nullptr;
  if (xslp_codec_create(10, 4, XSLP_RS_ISAL, &o, 8, &codec)) return 1;   // memo of 8: evictions
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) ts.emplace_back(worker, t, iters, shared, codec);
  for (auto &t : ts) t.join();
  xslp_codec_free(codec);
  xslp_free(shared);
  if (g_fail) return 1;
  std::printf("ok stress %d %d\n", threads, iters);
  return 0;
}
