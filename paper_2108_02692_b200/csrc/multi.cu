// Heterogeneous decode in few launches: several compiled programs (one per erasure
// pattern) fused into persistent multi-program pipeline kernels (entry xslp_sl_multi,
// ptx.cpp body_multi).  The producer warp streams the union of the programs' constant
// strips by TMA; consumer warps look up their stripe's program and jump to its code
// through a branch table.  Programs are packed `per_module` to a module; modules are
// compiled in parallel host threads; a call launches one kernel per module that has
// stripes, each over its contiguous run of the caller's program-sorted stripe list.
//
// This replaces one small launch per pattern (xslp_decode_batch_grouped), whose per-launch
// ramp-up and tail dominate when a pattern owns one or two stripes (BASELINE cfg3: 644
// patterns over 1024 stripes; profiles/r01_s2_cfg3_launches.md).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <set>
#include <thread>

#include "xslp_api.h"

namespace xslp {



void count_launch();  // device.cu

struct MultiModule {
  int first = 0, count = 0;  // programs [first, first + count)
  int nused = 0;             // union of used constants (TMA rows per stage)
  std::vector<char> cubin;
  int regs = 0, spill = 0;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t k = nullptr;
  std::map<int, int> smem_set, occ;  // per device
};

struct Multi {
  int n_const = 0, n_goals = 0, threads = 128, stages = 2, lanes = 1, phases = 1, reuse = 16;
  int64_t baked_strip = 0;
  int nprogs = 0;
  std::vector<MultiModule> mods;
  double compile_ms = 0;
  std::mutex mu;
  ~Multi() {
    for (auto &m : mods)
      if (m.lib) cudaLibraryUnload(m.lib);
  }
};

static int cur_dev() {
  int d = -1;
  CUDA_OK(cudaGetDevice(&d));
  return d;
}

// Two internal streams per device: consecutive modules alternate between them (forked from
// and joined back into the caller's stream with events), so the tail of one module's
// persistent launch overlaps the start of the next.
struct MultiStreams {
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
};
static std::mutex g_ms_mu;
static std::map<int, MultiStreams> g_ms;

static void multi_launch(Multi &M, const int32_t *d_pos, const int32_t *d_ids, const int32_t *off,
                         const uint8_t *const *d_in, uint8_t *const *d_out, size_t B,
                         cudaStream_t user) {
  if (B % 32) throw Error(XSLP_EINVAL, "block_bytes must be a multiple of 32");
  uint64_t strip = B / 8;
  if (strip % 16) throw Error(XSLP_EINVAL, "TMA staging needs block_bytes % 128 == 0");
  if (M.baked_strip > 0 && (int64_t)strip != M.baked_strip)
    throw Error(XSLP_EINVAL, "block_bytes differs from the block_bytes_hint the kernels were built for");
  const int T = M.threads, L = M.lanes;
  uint32_t words = (uint32_t)(strip / (4 * L));
  uint32_t tps = (words + T - 1) / T;
  const int d = cur_dev();
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
  int active = 0;
  for (auto &m : M.mods) active += off[m.first + m.count] > off[m.first];
  MultiStreams *P = nullptr;
  std::unique_lock<std::mutex> lk(g_ms_mu, std::defer_lock);
  if (active > 1) {
    lk.lock();
    P = &g_ms[d];
    if (!P->fork) {
      for (int k = 0; k < 2; ++k) {
        CUDA_OK(cudaStreamCreateWithFlags(&P->st[k], cudaStreamNonBlocking));
        CUDA_OK(cudaEventCreateWithFlags(&P->join[k], cudaEventDisableTiming));
      }
      CUDA_OK(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming));
    }
    CUDA_OK(cudaEventRecord(P->fork, user));
    for (int k = 0; k < 2; ++k) CUDA_OK(cudaStreamWaitEvent(P->st[k], P->fork, 0));
  }
  int launched = 0;
  for (auto &m : M.mods) {
    const int a = m.first, b = m.first + m.count;
    if (off[b] < off[a]) throw Error(XSLP_EINVAL, "group offsets must be non-decreasing");
    const uint64_t nent = (uint64_t)(off[b] - off[a]);
    if (nent == 0) continue;
    if (nent * tps > 0xffffffffull) throw Error(XSLP_EINVAL, "too many tiles");
    uint32_t ntiles = (uint32_t)(nent * tps);
    // barriers + per-stage tile headers (ptx.cpp multi_hs / multi_rows) + the stage rows
    const int n_out = M.n_goals / 8;
    const size_t hs = (8 + 8 * (size_t)n_out + 15) / 16 * 16;
    const size_t rows = (128 + M.stages * hs + 127) / 128 * 128;
    const size_t smem = rows + (size_t)M.stages * m.nused * 4 * L * T;
    if (smem > 227 * 1024) throw Error(XSLP_EINVAL, "pipeline stages do not fit in shared memory");
    int per = 1;
    {
      std::lock_guard<std::mutex> g(M.mu);
      if (!m.lib) {
        CUDA_OK(cudaLibraryLoadData(&m.lib, m.cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
        CUDA_OK(cudaLibraryGetKernel(&m.k, m.lib, "xslp_sl_multi"));
      }
      if (m.smem_set[d] < (int)smem) {
        CUDA_OK(cudaKernelSetAttributeForDevice(m.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, d));
        m.smem_set[d] = (int)smem;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)m.k, T + 32, smem));
        m.occ[d] = std::max(1, per);
      }
      per = m.occ[d];
    }
    const int grid = (int)std::min<uint64_t>(ntiles, (uint64_t)sms * per);
    const int32_t *ids = d_ids + off[a];
    uint32_t first = (uint32_t)a;
    void *args[] = {(void *)&d_in, (void *)&d_out, (void *)&ids, &strip, &words, &tps, &ntiles,
                    (void *)&d_pos, &first};
    cudaStream_t st = P ? P->st[launched % 2] : user;
    CUDA_OK(cudaLaunchKernel((const void *)m.k, dim3(grid), dim3(T + 32), args, smem, st));
    count_launch();
    ++launched;
  }
  if (P)
    for (int k = 0; k < 2; ++k) {
      CUDA_OK(cudaEventRecord(P->join[k], P->st[k]));
      CUDA_OK(cudaStreamWaitEvent(user, P->join[k], 0));
    }
}

}  // namespace xslp

using namespace xslp;

extern "C" int xslp_multi_create(const xslp_program *const *progs, int nprogs, int per_module,
                                 const xslp_opts *opts, xslp_multi **out) {
  API_BEGIN
  if (!out || !progs || nprogs <= 0) throw Error(XSLP_EINVAL, "bad arguments");
  *out = nullptr;
  xslp_opts o;
  if (opts) o = *opts; else xslp_default_opts(&o);
  if (o.threads < 32 || o.threads > 992 || o.threads % 32) throw Error(XSLP_EINVAL, "bad threads");
  if (o.stages < 2 || o.stages > 8) throw Error(XSLP_EINVAL, "stages must be 2..8");
  if (o.lane_words != 1 && o.lane_words != 2 && o.lane_words != 4) throw Error(XSLP_EINVAL, "bad lane_words");
  if (per_module <= 0) per_module = 20;  // measured optimum for RS(10,4) decode (profiles)
  per_module = std::min(per_module, 256);
  auto t0 = std::chrono::steady_clock::now();
  auto M = std::make_unique<Multi>();
  std::vector<const Program *> ps;
  for (int i = 0; i < nprogs; ++i) {
    if (!progs[i]) throw Error(XSLP_EINVAL, "null program");
    ps.push_back(reinterpret_cast<const Program *>(progs[i]));
    if (ps[i]->opts.layout != XSLP_LAYOUT_STRIP) throw Error(XSLP_EINVAL, "strip layout only");
    if (ps[i]->n_const != ps[0]->n_const || ps[i]->n_goals != ps[0]->n_goals)
      throw Error(XSLP_EINVAL, "programs disagree on constants/goals");
  }
  M->n_const = ps[0]->n_const;
  M->n_goals = ps[0]->n_goals;
  M->threads = o.threads;
  M->stages = o.stages;
  M->lanes = o.lane_words;
  M->reuse = reuse_window(o.reuse, 64);   // full M^-1 programs: one CTA per SM, registers to spare
  M->nprogs = nprogs;
  M->baked_strip = o.block_bytes_hint > 0 && o.block_bytes_hint % 32 == 0 ? o.block_bytes_hint / 8 : 0;
  // input phases for wide codes (as the PIPE kernel's opts.phases; 0 = ceil(n/10) for n > 10)
  int nph = o.phases == 0 ? std::min(8, (M->n_const / 8 + 9) / 10) : std::max(1, o.phases);
  nph = std::min(nph, std::max(1, M->n_const / 8));
  M->phases = nph;
  std::vector<std::vector<Slp>> phased;  // phased[k][ph]
  if (nph > 1) {
    phased.resize(nprogs);
    std::atomic<int> nx{0};
    std::vector<std::string> perr(nprogs);
    auto pwork = [&]() {
      for (;;) {
        int k = nx++;
        if (k >= nprogs) return;
        try {
          phased[k] = phase_programs(evaluate(ps[k]->slp), M->n_const, nph, ps[k]->opts, nullptr);
        } catch (const std::exception &e) {
          perr[k] = e.what();
        }
      }
    };
    const int nt = (int)std::min<size_t>(nprogs, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(pwork);
    for (auto &t : th) t.join();
    for (auto &e : perr)
      if (!e.empty()) throw Error(XSLP_ECOMPILE, e);
  }
  for (int a = 0; a < nprogs; a += per_module) {
    MultiModule m;
    m.first = a;
    m.count = std::min(per_module, nprogs - a);
    // constants per stage fill: the union over the module's programs (per phase: the max)
    auto count_used = [&](const std::vector<const Slp *> &v) {
      std::vector<char> u(M->n_const, 0);
      for (const Slp *q : v) {
        for (auto &in : q->ins)
          for (int t : in.ops)
            if (t < M->n_const) u[t] = 1;
        for (int g : q->goal)
          if (g >= 0 && g < M->n_const) u[g] = 1;
      }
      return (int)std::count(u.begin(), u.end(), 1);
    };
    if (nph > 1) {
      m.nused = 1;
      for (int ph = 0; ph < nph; ++ph) {
        std::vector<const Slp *> v;
        for (int i = a; i < a + m.count; ++i) v.push_back(&phased[i][ph]);
        m.nused = std::max(m.nused, count_used(v));
      }
    } else {
      std::vector<const Slp *> v;
      for (int i = a; i < a + m.count; ++i) v.push_back(&ps[i]->slp);
      m.nused = count_used(v);
    }
    M->mods.push_back(std::move(m));
  }
  // compile the modules on host threads
  std::atomic<int> next{0};
  std::vector<std::string> errs(M->mods.size());
  auto work = [&]() {
    for (;;) {
      int i = next++;
      if (i >= (int)M->mods.size()) return;
      auto &m = M->mods[i];
      try {
        std::string ptx;
        if (nph > 1) {
          std::vector<std::vector<const Slp *>> v;
          for (int k = m.first; k < m.first + m.count; ++k) {
            v.emplace_back();
            for (auto &q : phased[k]) v.back().push_back(&q);
          }
          ptx = emit_ptx_multi_phases(v, M->lanes, M->baked_strip, M->threads, M->stages, M->reuse);
        } else {
          std::vector<const Slp *> v;
          for (int k = m.first; k < m.first + m.count; ++k) v.push_back(&ps[k]->slp);
          ptx = emit_ptx_multi(v, M->lanes, M->baked_strip, M->threads, M->stages, M->reuse);
        }
        m.cubin = ptx_to_cubin(ptx, nullptr, nullptr, nullptr, nullptr, &m.regs, &m.spill);
      } catch (const std::exception &e) {
        errs[i] = e.what();
      }
    }
  };
  const int nt = (int)std::min<size_t>(M->mods.size(), std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(work);
  for (auto &t : th) t.join();
  for (auto &e : errs)
    if (!e.empty()) throw Error(XSLP_ECOMPILE, e);
  M->compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = reinterpret_cast<xslp_multi *>(M.release());
  API_END
}

extern "C" int xslp_syndrome_create(const uint8_t *gf, int n, int p, const int32_t *patterns,
                                    int npat, int ne, int per_module, const xslp_opts *opts,
                                    xslp_multi **out) {
  API_BEGIN
  if (!out || !gf || !patterns || npat <= 0 || n < 1 || p < 1 || n + p > 255 || ne < 1)
    throw Error(XSLP_EINVAL, "bad arguments");
  if (ne > p) throw Error(XSLP_EUNRECOVERABLE, "more erasures than parity blocks");
  *out = nullptr;
  xslp_opts o;
  if (opts) o = *opts; else xslp_default_opts(&o);
  if (o.threads < 32 || o.threads > 992 || o.threads % 32) throw Error(XSLP_EINVAL, "bad threads");
  if (o.stages < 2 || o.stages > 8) throw Error(XSLP_EINVAL, "stages must be 2..8");
  if (o.lane_words != 1 && o.lane_words != 2 && o.lane_words != 4) throw Error(XSLP_EINVAL, "bad lane_words");
  if (per_module <= 0) per_module = 16;  // measured optimum for RS(10,4) / RS(20,4) (profiles/r01_s2_reuse.md)
  per_module = std::min(per_module, 256);
  auto t0 = std::chrono::steady_clock::now();
  auto M = std::make_unique<Multi>();
  const int nb = n + p;
  M->n_const = 8 * nb;
  M->n_goals = 8 * ne;
  M->threads = o.threads;
  M->stages = o.stages;
  M->lanes = o.lane_words;
  M->reuse = reuse_window(o.reuse, 16);   // 96 registers keep two CTAs per SM; 24+ drops to one
  M->nprogs = npat;
  M->baked_strip = o.block_bytes_hint > 0 && o.block_bytes_hint % 32 == 0 ? o.block_bytes_hint / 8 : 0;
  int nph = o.phases == 0 ? std::min(8, (nb + 9) / 10) : std::max(1, o.phases);
  nph = std::min(nph, nb);
  M->phases = nph;
  // the shared syndrome program (H over all n+p blocks), in input phases
  auto h = parity_check(gf, n, p);
  auto hb = gf::to_bits(h, p, nb);
  std::vector<Bits> sgoals(8 * p, Bits(8 * nb));
  for (int r = 0; r < 8 * p; ++r)
    for (int c = 0; c < 8 * nb; ++c)
      if (hb[(size_t)r * 8 * nb + c]) sgoals[r].set(c);
  xslp_opts so = o;
  so.specialise = 0;
  auto syn = phase_programs(sgoals, 8 * nb, nph, so, nullptr);
  // per-pattern solve programs (8e x 8p bitmatrices over the syndrome words)
  std::vector<std::shared_ptr<Program>> solve(npat);
  {
    std::atomic<int> nx{0};
    std::vector<std::string> perr(npat);
    auto work = [&]() {
      for (;;) {
        int k = nx++;
        if (k >= npat) return;
        try {
          std::set<int> es(patterns + (size_t)k * ne, patterns + (size_t)(k + 1) * ne);
          if ((int)es.size() != ne || *es.begin() < 0 || *es.rbegin() >= nb)
            throw Error(XSLP_EINVAL, "bad erasure pattern");
          auto x = solve_rows(h, n, p, std::vector<int>(es.begin(), es.end()));
          solve[k] = compile_bits(gf::to_bits(x, ne, p), 8 * ne, 8 * p, so);
        } catch (const std::exception &e) {
          perr[k] = e.what();
        }
      }
    };
    const int nt = (int)std::min<size_t>(npat, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(work);
    for (auto &t : th) t.join();
    for (auto &e : perr)
      if (!e.empty()) throw Error(XSLP_EINVAL, e);
  }
  int nused = 1;
  for (auto &q : syn) {
    std::vector<char> u(8 * nb, 0);
    for (auto &in : q.ins)
      for (int t : in.ops)
        if (t < 8 * nb) u[t] = 1;
    nused = std::max(nused, (int)std::count(u.begin(), u.end(), 1));
  }
  for (int a = 0; a < npat; a += per_module) {
    MultiModule m;
    m.first = a;
    m.count = std::min(per_module, npat - a);
    m.nused = nused;
    M->mods.push_back(std::move(m));
  }
  std::atomic<int> next{0};
  std::vector<std::string> errs(M->mods.size());
  auto work = [&]() {
    for (;;) {
      int i = next++;
      if (i >= (int)M->mods.size()) return;
      auto &m = M->mods[i];
      try {
        std::vector<const Slp *> v;
        for (int k = m.first; k < m.first + m.count; ++k) v.push_back(&solve[k]->slp);
        std::string ptx = emit_ptx_syndrome(syn, v, ne, M->lanes, M->baked_strip, M->threads, M->stages,
                                            M->reuse);
        m.cubin = ptx_to_cubin(ptx, nullptr, nullptr, nullptr, nullptr, &m.regs, &m.spill);
      } catch (const std::exception &e) {
        errs[i] = e.what();
      }
    }
  };
  const int nt = (int)std::min<size_t>(M->mods.size(), std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(work);
  for (auto &t : th) t.join();
  for (auto &e : errs)
    if (!e.empty()) throw Error(XSLP_ECOMPILE, e);
  M->compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  *out = reinterpret_cast<xslp_multi *>(M.release());
  API_END
}

extern "C" int xslp_multi_decode(const xslp_multi *multi, const int32_t *d_prog_of_stripe,
                                 const int32_t *d_stripe_ids, const int32_t *group_offsets,
                                 const uint8_t *const *d_in_tbl, uint8_t *const *d_out_tbl,
                                 size_t block_bytes, void *stream) {
  API_BEGIN
  if (!multi || !d_prog_of_stripe || !d_stripe_ids || !group_offsets || !d_in_tbl || !d_out_tbl)
    throw Error(XSLP_EINVAL, "null argument");
  if (group_offsets[0] < 0) throw Error(XSLP_EINVAL, "negative group offset");
  {
    const Multi &M = *reinterpret_cast<const Multi *>(multi);
    for (int i = 0; i < M.nprogs; ++i)
      if (group_offsets[i + 1] < group_offsets[i])
        throw Error(XSLP_EINVAL, "group offsets must be non-decreasing (nprogs + 1 entries)");
  }
  if (block_bytes == 0) return XSLP_OK;
  Multi &M = *reinterpret_cast<Multi *>(const_cast<xslp_multi *>(multi));
  multi_launch(M, d_prog_of_stripe, d_stripe_ids, group_offsets, d_in_tbl, d_out_tbl, block_bytes,
               (cudaStream_t)stream);
  API_END
}

extern "C" int xslp_multi_info(const xslp_multi *multi, int32_t *modules, int32_t *regs,
                               int32_t *spill_bytes, double *compile_ms) {
  API_BEGIN
  if (!multi) throw Error(XSLP_EINVAL, "null multi");
  const Multi &M = *reinterpret_cast<const Multi *>(multi);
  int r = 0, s = 0;
  for (auto &m : M.mods) {
    r = std::max(r, m.regs);
    s = std::max(s, m.spill);
  }
  if (modules) *modules = (int32_t)M.mods.size();
  if (regs) *regs = r;
  if (spill_bytes) *spill_bytes = s;
  if (compile_ms) *compile_ms = M.compile_ms;
  API_END
}

extern "C" void xslp_multi_free(xslp_multi *multi) { delete reinterpret_cast<Multi *>(multi); }
