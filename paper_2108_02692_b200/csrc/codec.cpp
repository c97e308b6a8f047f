// Erasure-coding front end: RS(n,p) over arbitrary-length device
// data with zero padding, the 32-byte shard header, and a memo cache of compiled decode
// programs per erasure pattern (the paper precomputes all C(n+p,p) decode SLPs for its
// dataset; a bounded LRU cache is the serving-side equivalent).
//
// Layout: data of `len` bytes is zero-padded to n*B with B = block_bytes(len), a
// multiple of 128 (so every strip is 16-byte aligned and TMA-able); shard j < n is bytes
// [jB, (j+1)B) of the padded data, shard n+i is parity block i.
#include <cuda_runtime.h>

#include <algorithm>
#include <list>
#include <set>

#include "xslp_api.h"

namespace xslp {

struct Codec {
  int n, p, kind;
  xslp_opts opts;
  size_t cap;
  std::vector<uint8_t> G;  // (n+p) x n
  std::shared_ptr<Program> enc;
  std::mutex mu;
  std::list<std::vector<int>> lru;  // most recent at front
  std::map<std::vector<int>, std::pair<std::shared_ptr<Program>, std::list<std::vector<int>>::iterator>> memo;
  // encode-through programs, by the number f of whole data blocks in the caller's buffer:
  // goals = data shards 0..f-1 (copies) + the p parity shards, read straight from the data
  std::map<int, std::shared_ptr<Program>> thru;
  // decode-through programs, by (erasure pattern, f): goals = data blocks 0..f-1 (copies of
  // the surviving ones, M^-1 rows for the erased ones) written straight to the caller's buffer
  std::map<std::pair<std::vector<int>, int>, std::shared_ptr<Program>> dthru;
  // programs handed out by xslp_codec_program: kept alive until xslp_codec_free, so an LRU
  // eviction by another thread cannot free a program a caller still holds
  std::set<std::shared_ptr<Program>> handed_out;
};

std::shared_ptr<Program> compile_bits(const std::vector<uint8_t> &bits, int rows, int cols,
                                      const xslp_opts &o);

static void cuda_ok(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw Error(XSLP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static int64_t block_bytes_for(const Codec &c, int64_t len) {
  if (len < 0) throw Error(XSLP_EINVAL, "negative length");
  int64_t per = (len + c.n - 1) / c.n;
  int64_t B = (per + 127) / 128 * 128;
  return std::max<int64_t>(B, 128);
}

static std::shared_ptr<Program> decode_program(Codec &c, std::vector<int> er) {
  std::sort(er.begin(), er.end());
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.memo.find(er);
    if (it != c.memo.end()) {
      c.lru.splice(c.lru.begin(), c.lru, it->second.second);
      return it->second.first;
    }
  }
  // build outside the lock: compile may take ~0.1 s
  std::set<int> es(er.begin(), er.end());
  if ((int)er.size() > c.p) throw Error(XSLP_EUNRECOVERABLE, "more erasures than parity shards");
  if (es.size() != er.size()) throw Error(XSLP_EINVAL, "duplicate erasure index");
  for (int e : er)
    if (e < 0 || e >= c.n + c.p) throw Error(XSLP_EINVAL, "erasure index out of range");
  std::vector<int32_t> e32(er.begin(), er.end());
  std::vector<uint8_t> bits((size_t)64 * std::max<size_t>(1, er.size()) * c.n);
  std::vector<int32_t> surv(c.n);
  int rc = xslp_decode_bitmatrix(c.G.data(), c.n, c.p, e32.data(), (int)e32.size(), bits.data(),
                                 surv.data());
  if (rc) throw Error(rc, xslp_last_error());
  auto prog = compile_bits(bits, 8 * (int)er.size(), 8 * c.n, c.opts);
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.memo.find(er);
  if (it != c.memo.end()) return it->second.first;  // another thread won the race
  c.lru.push_front(er);
  c.memo[er] = {prog, c.lru.begin()};
  while (c.memo.size() > c.cap) {
    c.memo.erase(c.lru.back());
    c.lru.pop_back();
  }
  return prog;
}

// [I_8f rows of blocks 0..f-1 ; the 8p parity rows] over the 8n data strips
static std::shared_ptr<Program> thru_program(Codec &c, int f) {
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.thru.find(f);
    if (it != c.thru.end()) return it->second;
  }
  const int cols = 8 * c.n, rows = 8 * (f + c.p);
  std::vector<uint8_t> bits((size_t)rows * cols, 0);
  for (int r = 0; r < 8 * f; ++r) bits[(size_t)r * cols + r] = 1;
  std::vector<uint8_t> par((size_t)64 * c.p * c.n);
  int rc = xslp_encode_bitmatrix(c.G.data(), c.n, c.p, par.data());
  if (rc) throw Error(rc, xslp_last_error());
  std::copy(par.begin(), par.end(), bits.begin() + (size_t)8 * f * cols);
  auto prog = compile_bits(bits, rows, cols, c.opts);
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.thru.find(f);
  if (it != c.thru.end()) return it->second;
  c.thru[f] = prog;
  return prog;
}

static std::shared_ptr<Program> dthru_program(Codec &c, const std::vector<int> &er, int f) {
  const auto key = std::make_pair(er, f);
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.dthru.find(key);
    if (it != c.dthru.end()) return it->second;
  }
  const int cols = 8 * c.n;
  std::vector<int32_t> e32(er.begin(), er.end());
  std::vector<uint8_t> dec((size_t)64 * er.size() * c.n);
  std::vector<int32_t> surv(c.n);
  int rc = xslp_decode_bitmatrix(c.G.data(), c.n, c.p, e32.data(), (int)e32.size(), dec.data(),
                                 surv.data());
  if (rc) throw Error(rc, xslp_last_error());
  std::vector<uint8_t> bits((size_t)8 * f * cols, 0);
  for (int j = 0; j < f; ++j) {
    auto e = std::find(er.begin(), er.end(), j);
    if (e != er.end()) {                                   // erased: its M^-1 rows
      const size_t k = (size_t)(e - er.begin());
      std::copy(dec.begin() + 8 * k * cols, dec.begin() + 8 * (k + 1) * cols, bits.begin() + (size_t)8 * j * cols);
    } else {                                               // survivor: identity on its strips
      const int pos = (int)(std::find(surv.begin(), surv.end(), j) - surv.begin());
      for (int r = 0; r < 8; ++r) bits[(size_t)(8 * j + r) * cols + 8 * pos + r] = 1;
    }
  }
  auto prog = compile_bits(bits, 8 * f, cols, c.opts);
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.dthru.find(key);
  if (it != c.dthru.end()) return it->second;
  if (c.dthru.size() >= c.cap) c.dthru.clear();            // bounded, like the decode memo
  c.dthru[key] = prog;
  return prog;
}

}  // namespace xslp

using namespace xslp;


static Codec *C(const xslp_codec *c) {
  if (!c) throw Error(XSLP_EINVAL, "null codec");
  return reinterpret_cast<Codec *>(const_cast<xslp_codec *>(c));
}

extern "C" int xslp_codec_create(int n, int p, int kind, const xslp_opts *opts, int cache_entries,
                                 xslp_codec **out) {
  API_BEGIN
  if (!out || n < 1 || p < 0 || n + p > 64) throw Error(XSLP_EINVAL, "bad (n, p): 1 <= n, n + p <= 64");
  *out = nullptr;
  auto c = std::make_unique<Codec>();
  c->n = n;
  c->p = p;
  c->kind = kind;
  if (opts) c->opts = *opts; else xslp_default_opts(&c->opts);
  c->opts.block_bytes_hint = 0;  // shard sizes vary per call: generic strip addressing
  c->cap = cache_entries > 0 ? (size_t)cache_entries : 1024;
  c->G.resize((size_t)(n + p) * n);
  int rc = xslp_coding_matrix(n, p, kind, c->G.data());
  if (rc) throw Error(rc, xslp_last_error());
  if (p > 0) {
    std::vector<uint8_t> bits((size_t)64 * p * n);
    rc = xslp_encode_bitmatrix(c->G.data(), n, p, bits.data());
    if (rc) throw Error(rc, xslp_last_error());
    c->enc = compile_bits(bits, 8 * p, 8 * n, c->opts);
  }
  *out = reinterpret_cast<xslp_codec *>(c.release());
  API_END
}

extern "C" void xslp_codec_free(xslp_codec *c) { delete reinterpret_cast<Codec *>(c); }

extern "C" int64_t xslp_codec_block_bytes(const xslp_codec *c, int64_t len) {
  try {
    return block_bytes_for(*C(c), len);
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.code;
  }
}

extern "C" int xslp_codec_encode(const xslp_codec *cc, const uint8_t *d_data, int64_t len,
                                 uint8_t *d_shards, void *stream) {
  API_BEGIN
  Codec &c = *C(cc);
  if ((!d_data && len > 0) || !d_shards || ((uintptr_t)d_shards & 15))
    throw Error(XSLP_EINVAL, "bad buffers (shards must be 16-byte aligned)");
  const int64_t B = block_bytes_for(c, len);
  cudaStream_t st = (cudaStream_t)stream;
  const int f = (int)std::min<int64_t>(c.n, len / B);  // whole data blocks in the caller's buffer
  if (c.p > 0 && f > 0 && ((uintptr_t)d_data & 15) == 0) {
    // encode-through: one pass reads each data block once from the caller's buffer and writes
    // both its data shard (a copy goal) and the parity; only the partial / padding blocks are
    // staged into their shards first
    if (len > f * B)
      cuda_ok(cudaMemcpyAsync(d_shards + f * B, d_data + f * B, len - f * B, cudaMemcpyDeviceToDevice, st),
              "copy tail");
    if (c.n * B > len) cuda_ok(cudaMemsetAsync(d_shards + len, 0, c.n * B - len, st), "pad");
    auto prog = thru_program(c, f);
    std::vector<const uint8_t *> in(c.n);
    std::vector<uint8_t *> out(f + c.p);
    for (int j = 0; j < c.n; ++j) in[j] = j < f ? d_data + j * B : d_shards + j * B;
    for (int j = 0; j < f; ++j) out[j] = d_shards + j * B;
    for (int i = 0; i < c.p; ++i) out[f + i] = d_shards + (c.n + i) * B;
    int rc = xslp_encode(reinterpret_cast<const xslp_program *>(prog.get()), in.data(), out.data(),
                         (size_t)B, stream);
    if (rc) throw Error(rc, xslp_last_error());
    return XSLP_OK;
  }
  // systematic part: the padded data is the first n shards, contiguous
  if (len > 0) cuda_ok(cudaMemcpyAsync(d_shards, d_data, len, cudaMemcpyDeviceToDevice, st), "copy");
  if (c.n * B > len) cuda_ok(cudaMemsetAsync(d_shards + len, 0, c.n * B - len, st), "pad");
  if (c.p == 0) return XSLP_OK;
  std::vector<const uint8_t *> in(c.n);
  std::vector<uint8_t *> out(c.p);
  for (int j = 0; j < c.n; ++j) in[j] = d_shards + j * B;
  for (int i = 0; i < c.p; ++i) out[i] = d_shards + (c.n + i) * B;
  int rc = xslp_encode(reinterpret_cast<const xslp_program *>(c.enc.get()), in.data(), out.data(),
                       (size_t)B, stream);
  if (rc) throw Error(rc, xslp_last_error());
  API_END
}

extern "C" int xslp_codec_reconstruct(const xslp_codec *cc, uint8_t *d_shards, const int32_t *erased,
                                      int ne, int64_t len, void *stream) {
  API_BEGIN
  Codec &c = *C(cc);
  if (!d_shards || ((uintptr_t)d_shards & 15) || ne < 0 || (ne > 0 && !erased))
    throw Error(XSLP_EINVAL, "bad arguments");
  if (ne == 0) return XSLP_OK;
  const int64_t B = block_bytes_for(c, len);
  std::vector<int> er(erased, erased + ne);
  auto prog = decode_program(c, er);
  std::sort(er.begin(), er.end());
  std::vector<int> surv;
  for (int i = 0; i < c.n + c.p && (int)surv.size() < c.n; ++i)
    if (!std::binary_search(er.begin(), er.end(), i)) surv.push_back(i);
  std::vector<const uint8_t *> in(c.n);
  std::vector<uint8_t *> out(ne);
  for (int j = 0; j < c.n; ++j) in[j] = d_shards + surv[j] * B;
  for (int k = 0; k < ne; ++k) out[k] = d_shards + er[k] * B;
  int rc = xslp_decode(reinterpret_cast<const xslp_program *>(prog.get()), in.data(), out.data(),
                       (size_t)B, stream);
  if (rc) throw Error(rc, xslp_last_error());
  API_END
}

extern "C" int xslp_codec_decode(const xslp_codec *cc, uint8_t *d_shards, const int32_t *erased,
                                 int ne, int64_t len, uint8_t *d_data_out, void *stream) {
  API_BEGIN
  Codec &c = *C(cc);
  if (!d_data_out && len > 0) throw Error(XSLP_EINVAL, "null output");
  if (ne < 0 || (ne > 0 && !erased)) throw Error(XSLP_EINVAL, "bad erasure list");
  if (ne > c.p) throw Error(XSLP_EUNRECOVERABLE, "more erasures than parity shards");
  const int64_t B = block_bytes_for(c, len);
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> er(erased, erased + ne);
  std::sort(er.begin(), er.end());
  const int f = (int)std::min<int64_t>(c.n, len / B);   // whole data blocks of the output
  bool data_lost = false;
  for (int e : er) data_lost |= e < c.n;
  if (data_lost && f > 0 && ((uintptr_t)d_data_out & 15) == 0) {
    // decode-through: one pass reads the n survivors and writes blocks 0..f-1 of the data
    // straight to the caller's buffer (surviving ones copied, erased ones solved); the tail
    // block, if any, comes from its shard (rebuilt in place first if it was lost)
    if (std::set<int>(er.begin(), er.end()).size() != er.size())
      throw Error(XSLP_EINVAL, "duplicate erasure index");
    for (int e : er)
      if (e < 0 || e >= c.n + c.p) throw Error(XSLP_EINVAL, "erasure index out of range");
    auto prog = dthru_program(c, er, f);
    std::vector<int> surv;
    for (int i = 0; i < c.n + c.p && (int)surv.size() < c.n; ++i)
      if (!std::binary_search(er.begin(), er.end(), i)) surv.push_back(i);
    std::vector<const uint8_t *> in(c.n);
    std::vector<uint8_t *> out(f);
    for (int j = 0; j < c.n; ++j) in[j] = d_shards + surv[j] * B;
    for (int j = 0; j < f; ++j) out[j] = d_data_out + j * B;
    int rc = xslp_decode(reinterpret_cast<const xslp_program *>(prog.get()), in.data(), out.data(),
                         (size_t)B, stream);
    if (rc) throw Error(rc, xslp_last_error());
    if (len > f * B) {
      if (std::binary_search(er.begin(), er.end(), f)) {
        rc = xslp_codec_reconstruct(cc, d_shards, erased, ne, len, stream);
        if (rc) throw Error(rc, xslp_last_error());
      }
      cuda_ok(cudaMemcpyAsync(d_data_out + f * B, d_shards + f * B, len - f * B, cudaMemcpyDeviceToDevice, st),
              "copy tail");
    }
    return XSLP_OK;
  }
  // only erased data shards must be rebuilt to return the data: rebuild in place, copy out
  if (data_lost) {
    int rc = xslp_codec_reconstruct(cc, d_shards, erased, ne, len, stream);
    if (rc) throw Error(rc, xslp_last_error());
  }
  if (len > 0)
    cuda_ok(cudaMemcpyAsync(d_data_out, d_shards, len, cudaMemcpyDeviceToDevice, st), "copy out");
  API_END
}

extern "C" int xslp_codec_program(const xslp_codec *cc, const int32_t *erased, int ne,
                                  const xslp_program **out) {
  API_BEGIN
  Codec &c = *C(cc);
  if (!out || ne < 0 || (ne > 0 && !erased)) throw Error(XSLP_EINVAL, "bad arguments");
  if (ne == 0) {
    *out = reinterpret_cast<const xslp_program *>(c.enc.get());
    return XSLP_OK;
  }
  auto prog = decode_program(c, std::vector<int>(erased, erased + ne));
  {
    std::lock_guard<std::mutex> g(c.mu);
    c.handed_out.insert(prog);
  }
  *out = reinterpret_cast<const xslp_program *>(prog.get());
  API_END
}

extern "C" int xslp_codec_cached(const xslp_codec *cc) {
  Codec &c = *reinterpret_cast<Codec *>(const_cast<xslp_codec *>(cc));
  std::lock_guard<std::mutex> g(c.mu);
  std::set<std::vector<int>> pats;       // erasure patterns with a compiled decode program
  for (auto &kv : c.memo) pats.insert(kv.first);
  for (auto &kv : c.dthru) pats.insert(kv.first.first);
  return (int)pats.size();
}

// 32-byte shard header: "XSLP", version 1, n, p, shard index, original length (u64 LE),
// block size (u32 LE), 12 reserved zero bytes.
extern "C" int xslp_shard_header(uint8_t *out, int n, int p, int shard, uint64_t len, uint32_t block) {
  API_BEGIN
  if (!out || n < 1 || p < 0 || n + p > 255 || shard < 0 || shard >= n + p)
    throw Error(XSLP_EINVAL, "bad header fields");
  std::memset(out, 0, 32);
  std::memcpy(out, "XSLP", 4);
  out[4] = 1;
  out[5] = (uint8_t)n;
  out[6] = (uint8_t)p;
  out[7] = (uint8_t)shard;
  for (int i = 0; i < 8; ++i) out[8 + i] = (uint8_t)(len >> (8 * i));
  for (int i = 0; i < 4; ++i) out[16 + i] = (uint8_t)(block >> (8 * i));
  API_END
}

extern "C" int xslp_shard_header_parse(const uint8_t *in, int32_t *n, int32_t *p, int32_t *shard,
                                       uint64_t *len, uint32_t *block) {
  API_BEGIN
  if (!in || std::memcmp(in, "XSLP", 4) != 0 || in[4] != 1) throw Error(XSLP_EINVAL, "not an XSLP v1 shard");
  for (int i = 20; i < 32; ++i)
    if (in[i]) throw Error(XSLP_EINVAL, "reserved header bytes not zero");
  if (n) *n = in[5];
  if (p) *p = in[6];
  if (shard) *shard = in[7];
  uint64_t L = 0;
  for (int i = 0; i < 8; ++i) L |= (uint64_t)in[8 + i] << (8 * i);
  uint32_t Bk = 0;
  for (int i = 0; i < 4; ++i) Bk |= (uint32_t)in[16 + i] << (8 * i);
  if (in[7] >= in[5] + in[6] || in[5] == 0) throw Error(XSLP_EINVAL, "inconsistent header");
  if (len) *len = L;
  if (block) *block = Bk;
  API_END
}
