// C ABI: host entry points (matrices, compile, stats, dump, errors).
// Device entry points live in device.cu.
#include <algorithm>
#include <chrono>
#include <set>

#include "xslp_api.h"

namespace xslp {
static thread_local std::string g_err;
void set_last_error(const std::string &m) { g_err = m; }
}  // namespace xslp

using namespace xslp;


extern "C" void xslp_default_opts(xslp_opts *o) {
  if (!o) return;
  o->compress = XSLP_COMPRESS_XORREPAIR;
  o->fuse = 1;
  o->schedule = XSLP_SCHED_DFS;
  o->specialise = 1;
  o->lane_words = 1;
  o->threads = 128;
  o->block_bytes_hint = 0;
  o->kernel = XSLP_KERNEL_AUTO;
  o->goal_order = 0;
  o->min_blocks = 0;
  o->stages = 2;
  o->greedy_capacity = 0;
  o->layout = XSLP_LAYOUT_STRIP;
  o->groups = 1;
  o->phases = 0;
  o->reuse = 0;
  o->interp = XSLP_INTERP_TMEM;
}

extern "C" int xslp_coding_matrix(int n, int p, int kind, uint8_t *gf_out) {
  API_BEGIN
  if (!gf_out || n < 1 || p < 0 || n + p > 255) throw Error(XSLP_EINVAL, "bad (n, p)");
  auto g = gf::coding_matrix(n, p, kind);
  std::copy(g.begin(), g.end(), gf_out);
  API_END
}

extern "C" int xslp_encode_bitmatrix(const uint8_t *gf_in, int n, int p, uint8_t *bits_out) {
  API_BEGIN
  if (!gf_in || !bits_out || n < 1 || p < 0 || n + p > 255) throw Error(XSLP_EINVAL, "bad (n, p)");
  std::vector<uint8_t> r(gf_in + (size_t)n * n, gf_in + (size_t)(n + p) * n);
  auto b = gf::to_bits(r, p, n);
  std::copy(b.begin(), b.end(), bits_out);
  API_END
}

// Goal rows of the erased blocks (ascending index) over the survivors surv (n distinct
// non-erased indices, in the column order the caller wants): M = the survivors'
// rows of g; data block e is row e of M^-1, parity block e is g[e] M^-1 (reading R4).
static std::vector<uint8_t> decode_bits(const uint8_t *g, int n, int p, const std::set<int> &es,
                                        const std::vector<int> &surv) {
  std::vector<uint8_t> M((size_t)n * n);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < n; ++c) M[r * n + c] = g[(size_t)surv[r] * n + c];
  auto Mi = gf::invert(M, n);
  std::vector<uint8_t> rows;
  for (int e : es) {
    if (e < n) {
      rows.insert(rows.end(), Mi.begin() + (size_t)e * n, Mi.begin() + (size_t)(e + 1) * n);
    } else {
      for (int c = 0; c < n; ++c) {
        uint8_t s = 0;
        for (int k = 0; k < n; ++k) s ^= gf::mul(g[(size_t)e * n + k], Mi[(size_t)k * n + c]);
        rows.push_back(s);
      }
    }
  }
  (void)p;
  return gf::to_bits(rows, (int)es.size(), n);
}

static std::set<int> erased_set(int n, int p, const int32_t *erased, int ne) {
  if (ne > p) throw Error(XSLP_EUNRECOVERABLE, "more erasures than parity blocks");
  std::set<int> es;
  for (int i = 0; i < ne; ++i) {
    if (erased[i] < 0 || erased[i] >= n + p) throw Error(XSLP_EINVAL, "erasure index out of range");
    if (!es.insert(erased[i]).second) throw Error(XSLP_EINVAL, "duplicate erasure index");
  }
  return es;
}

extern "C" int xslp_decode_bitmatrix(const uint8_t *g, int n, int p, const int32_t *erased, int ne,
                                     uint8_t *bits_out, int32_t *survivors_out) {
  API_BEGIN
  if (!g || !bits_out || !survivors_out || n < 1 || p < 0 || n + p > 255 || ne < 0 ||
      (ne > 0 && !erased))
    throw Error(XSLP_EINVAL, "bad arguments");
  auto es = erased_set(n, p, erased, ne);
  std::vector<int> surv;
  for (int i = 0; i < n + p && (int)surv.size() < n; ++i)
    if (!es.count(i)) surv.push_back(i);
  auto b = decode_bits(g, n, p, es, surv);
  std::copy(b.begin(), b.end(), bits_out);
  std::copy(surv.begin(), surv.end(), survivors_out);
  API_END
}

extern "C" int xslp_decode_bitmatrix_from(const uint8_t *g, int n, int p, const int32_t *erased,
                                          int ne, const int32_t *survivors, uint8_t *bits_out) {
  API_BEGIN
  if (!g || !bits_out || !survivors || n < 1 || p < 0 || n + p > 255 || ne < 0 ||
      (ne > 0 && !erased))
    throw Error(XSLP_EINVAL, "bad arguments");
  auto es = erased_set(n, p, erased, ne);
  std::set<int> seen;
  std::vector<int> surv(survivors, survivors + n);
  for (int s : surv) {
    if (s < 0 || s >= n + p) throw Error(XSLP_EINVAL, "survivor index out of range");
    if (es.count(s)) throw Error(XSLP_EINVAL, "survivor is erased");
    if (!seen.insert(s).second) throw Error(XSLP_EINVAL, "duplicate survivor index");
  }
  auto b = decode_bits(g, n, p, es, surv);
  std::copy(b.begin(), b.end(), bits_out);
  API_END
}

namespace xslp {
// Input-phase programs: the goal sets restricted to each of `nphases` contiguous input-block
// ranges (as equal as possible), each compressed, fused and DFS-scheduled as its own program
// over all goals, checked by evaluation.  xor_total (if given) accumulates the XORs the phases
// execute per word position, including each nonzero partial's XOR into its accumulator.
std::vector<Slp> phase_programs(const std::vector<Bits> &want, int n_const, int nphases,
                                const xslp_opts &o, int64_t *xor_total) {
  const int nb = n_const / 8, np = std::min(nphases, std::max(1, nb));
  std::vector<Slp> out;
  for (int k = 0; k < np; ++k) {
    const int lo = 8 * (k * nb / np), hi = 8 * ((k + 1) * nb / np);
    std::vector<Bits> g(want.size(), Bits(n_const));
    for (size_t r = 0; r < want.size(); ++r)
      for (int c = lo; c < hi; ++c)
        if (want[r].get(c)) g[r].set(c);
    Slp s = o.compress == XSLP_COMPRESS_NONE ? lift(g, n_const, o.fuse != 0)
                                             : compress(g, n_const, o.compress == XSLP_COMPRESS_XORREPAIR);
    if (o.fuse) fuse(s);
    if (o.schedule == XSLP_SCHED_GREEDY) {
      std::vector<int> peb;
      schedule_greedy(s, o.greedy_capacity, peb);
    } else if (o.schedule != XSLP_SCHED_NONE) {
      schedule_dfs(s, o.goal_order);
    }
    auto got = evaluate(s);
    for (size_t r = 0; r < g.size(); ++r)
      if (!(got[r] == g[r])) throw Error(XSLP_EINVAL, "internal: phase program differs from its goals");
    if (xor_total) {
      for (auto &in : s.ins) *xor_total += (int64_t)in.ops.size() - 1;
      for (int t : s.goal) *xor_total += t >= 0;
    }
    out.push_back(std::move(s));
  }
  return out;
}
}  // namespace xslp

namespace xslp {
// TMEM interpreter streams: the goal rows [0, R/2) and [R/2, R) each compressed, fused and
// scheduled as a program of its own (the same passes as the whole program), checked by
// evaluation.  Two consumer warps per TMEM lane quarter run one each, independently.
std::vector<Slp> stream_programs(const std::vector<Bits> &want, int n_const, const xslp_opts &o) {
  std::vector<Slp> out;
  const size_t half = want.size() / 2;
  for (int k = 0; k < 2; ++k) {
    std::vector<Bits> g(want.begin() + (k ? half : 0), k ? want.end() : want.begin() + half);
    Slp s = o.compress == XSLP_COMPRESS_NONE ? lift(g, n_const, o.fuse != 0)
                                             : compress(g, n_const, o.compress == XSLP_COMPRESS_XORREPAIR);
    if (o.fuse) fuse(s);
    if (o.schedule == XSLP_SCHED_GREEDY) {
      std::vector<int> peb;
      schedule_greedy(s, o.greedy_capacity, peb);
    } else if (o.schedule != XSLP_SCHED_NONE) {
      schedule_dfs(s, o.goal_order);
    }
    auto got = evaluate(s);
    for (size_t r = 0; r < g.size(); ++r)
      if (!(got[r] == g[r])) throw Error(XSLP_EINVAL, "internal: stream program differs from its goals");
    out.push_back(std::move(s));
  }
  return out;
}
}  // namespace xslp

namespace {

void build_phases(Program &P, const std::vector<Bits> &want) {
  P.phases = phase_programs(want, P.n_const, P.opts.phases, P.opts, &P.stats.group_xor);
  int used_max = 1;
  for (auto &s : P.phases) {
    std::vector<char> u(P.n_const, 0);
    for (auto &in : s.ins)
      for (int t : in.ops)
        if (t < P.n_const) u[t] = 1;
    for (int t : s.goal)
      if (t >= 0 && t < P.n_const) u[t] = 1;
    used_max = std::max(used_max, (int)std::count(u.begin(), u.end(), 1));
  }
  P.stage_used_const = used_max;
}

void finish(Program &P, const std::vector<Bits> *want, bool lifted) {
  auto t0 = std::chrono::steady_clock::now();
  const xslp_opts &o = P.opts;
  if (o.fuse) fuse(P.slp);
  if (o.schedule == XSLP_SCHED_DFS) schedule_dfs(P.slp, o.goal_order);
  std::vector<int> greedy_peb;
  int greedy_nvar = 0;
  if (o.schedule == XSLP_SCHED_GREEDY) greedy_nvar = schedule_greedy(P.slp, o.greedy_capacity, greedy_peb);
  if (want) {  // the compiler checks its own output against the goal sets
    auto got = evaluate(P.slp);
    if (got.size() != want->size()) throw Error(XSLP_EINVAL, "internal: goal count changed");
    for (size_t i = 0; i < got.size(); ++i)
      if (!(got[i] == (*want)[i])) throw Error(XSLP_EINVAL, "internal: compiled SLP differs from its input");
  }
  if (o.schedule == XSLP_SCHED_GREEDY) {
    P.pebble = greedy_peb;
    P.nvar = greedy_nvar;
  } else if (o.schedule == XSLP_SCHED_DFS || (lifted && o.compress == XSLP_COMPRESS_NONE && !o.fuse)) {
    // DFS pebbles; the unoptimised binary chains ("Base") are in place,
    // g <- g ^ c, which the same movable-pebble rule reproduces (NVar 32)
    P.nvar = paper_pebbles(P.slp, P.pebble);
  } else {
    P.pebble.clear();
    P.nvar = P.slp.n_vars;
  }
  if (want && o.interp == XSLP_INTERP_TMEM && (!o.specialise || o.kernel == XSLP_KERNEL_INTERP) &&
      want->size() >= 16)
    P.streams = stream_programs(*want, P.n_const, o);
  int maxlive = 0;
  build_bytecode(P.slp, P.code, P.nslots, maxlive);
  auto &st = P.stats;
  st.n_const = P.n_const;
  st.n_goals = P.n_goals;
  st.xor_count = st.mem_count = 0;
  for (auto &in : P.slp.ins) {
    st.xor_count += (int64_t)in.ops.size() - 1;
    st.mem_count += (int64_t)in.ops.size() + 1;
  }
  st.n_instr = (int)P.slp.ins.size();
  st.nvar = P.nvar;
  st.maxlive = maxlive;
  st.n_copy_goals = st.n_zero_goals = 0;
  for (int g : P.slp.goal) {
    if (g < 0) st.n_zero_goals++;
    else if (g < P.n_const) st.n_copy_goals++;
  }
  {
    std::vector<char> u(P.n_const, 0);
    for (auto &in : P.slp.ins)
      for (int t : in.ops)
        if (t < P.n_const) u[t] = 1;
    for (int g : P.slp.goal)
      if (g >= 0 && g < P.n_const) u[g] = 1;
    P.n_used_const = (int)std::count(u.begin(), u.end(), 1);
    P.stage_used_const = P.n_used_const;
    if (o.layout == XSLP_LAYOUT_BYTE) {  // PIPE stages hold whole 32-byte chunks of used blocks
      int nub = 0;
      for (int j = 0; j < P.n_const / 8; ++j) {
        bool any = false;
        for (int k = 0; k < 8; ++k) any |= u[8 * j + k] != 0;
        nub += any;
      }
      P.stage_used_const = 8 * std::max(1, nub);
    }
    // shared-memory reads of constants per word position in the TMA-staged kernels: the
    // emitter's rule (ptx.cpp compute) -- a constant used within the reuse window of its
    // previous use keeps its register, otherwise it is read again
    P.const_reads = 0;
    const int W = reuse_window(o.reuse, 64);
    std::vector<int> last(P.n_const, -1);
    for (size_t k = 0; k < P.slp.ins.size(); ++k)
      for (int t : P.slp.ins[k].ops) {
        if (t >= P.n_const) continue;
        if (W <= 0 || last[t] < 0 || (int)k - last[t] > W) P.const_reads++;
        last[t] = (int)k;
      }
  }
  st.regs = st.spill_bytes = st.regs_tma = st.spill_bytes_tma = st.regs_pipe = st.spill_bytes_pipe = 0;
  st.smem_reads = P.const_reads;
  st.group_xor = 0;
  const bool device_ok = P.n_const % 8 == 0 && P.n_goals % 8 == 0 && P.n_const > 0 &&
                         P.n_const / 8 + P.n_goals / 8 <= 128;
  if (o.specialise && device_ok) {
    int phases = o.phases;
    if (phases == 0)  // auto: at most 10 input blocks (80 strips) per stage fill
      phases = o.groups > 1 ? 1 : std::min(8, (P.n_const / 8 + 9) / 10);
    if (phases > 1 && o.layout == XSLP_LAYOUT_STRIP && want) {
      P.opts.phases = phases;
      build_phases(P, *want);
    }
    if (o.groups > 1 && o.layout == XSLP_LAYOUT_STRIP) {
      P.groups = split_goals(P.slp, o.groups);
      for (auto &g : P.groups)
        for (auto &in : g.ins) st.group_xor += (int64_t)in.ops.size() - 1;
    }
    const std::vector<Slp> *gp = P.groups.empty() ? nullptr : &P.groups;
    const std::vector<Slp> *ph = P.phases.empty() ? nullptr : &P.phases;
    P.ptx_generic = emit_ptx(P.slp, o.lane_words, 0, o.threads, o.min_blocks, o.stages, o.layout, gp, ph,
                             reuse_window(o.reuse, 64));
    P.cubin_generic = ptx_to_cubin(P.ptx_generic, &st.regs, &st.spill_bytes, &st.regs_tma, &st.spill_bytes_tma, &st.regs_pipe, &st.spill_bytes_pipe);
    if (o.block_bytes_hint > 0 && o.block_bytes_hint % 32 == 0) {
      P.baked_strip = o.block_bytes_hint / 8;
      P.ptx_baked = emit_ptx(P.slp, o.lane_words, P.baked_strip, o.threads, o.min_blocks, o.stages,
                           o.layout, gp, ph, reuse_window(o.reuse, 64));
      P.cubin_baked = ptx_to_cubin(P.ptx_baked, &st.regs, &st.spill_bytes, &st.regs_tma, &st.spill_bytes_tma, &st.regs_pipe, &st.spill_bytes_pipe);
    }
  }
  st.compile_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void check_opts(xslp_opts &o) {
  if (o.layout == XSLP_LAYOUT_BYTE) o.lane_words = 1;  // one 32-byte chunk per thread
  if (o.compress < 0 || o.compress > 2) throw Error(XSLP_EINVAL, "bad compress option");
  if (o.schedule < 0 || o.schedule > 2) throw Error(XSLP_EINVAL, "bad schedule option");
  if (o.schedule == XSLP_SCHED_GREEDY && o.greedy_capacity < 1)
    throw Error(XSLP_EINVAL, "greedy scheduling needs greedy_capacity >= 1");
  if (o.lane_words != 1 && o.lane_words != 2 && o.lane_words != 4)
    throw Error(XSLP_EINVAL, "lane_words must be 1, 2 or 4");
  if (o.threads < 32 || o.threads > 1024 || o.threads % 32) throw Error(XSLP_EINVAL, "bad threads");
  if (o.kernel < 0 || o.kernel > 4) throw Error(XSLP_EINVAL, "bad kernel option");
  if (o.min_blocks < 0 || o.min_blocks > 32) throw Error(XSLP_EINVAL, "bad min_blocks");
  if (o.stages < 1 || o.stages > 8) throw Error(XSLP_EINVAL, "stages must be 1..8");
  if (o.layout != XSLP_LAYOUT_STRIP && o.layout != XSLP_LAYOUT_BYTE) throw Error(XSLP_EINVAL, "bad layout");
  if (o.layout == XSLP_LAYOUT_BYTE && (o.kernel == XSLP_KERNEL_INTERP || o.kernel == XSLP_KERNEL_TMA))
    throw Error(XSLP_EINVAL, "the byte layout runs on the straight-line (LDG) or PIPE kernels only");
  if (o.layout == XSLP_LAYOUT_BYTE && !o.specialise)
    throw Error(XSLP_EINVAL, "the byte layout needs specialise = 1");
  if (o.groups < 1 || o.groups > 4) throw Error(XSLP_EINVAL, "groups must be 1..4");
  if (o.phases < 0 || o.phases > 8) throw Error(XSLP_EINVAL, "phases must be 0 (auto) or 1..8");
  if (o.phases > 1 && o.groups > 1) throw Error(XSLP_EINVAL, "phases and groups cannot be combined");
  if (o.reuse < -1 || o.reuse > 4096) throw Error(XSLP_EINVAL, "reuse must be -1, 0 (auto) or 1..4096");
  if (o.interp != XSLP_INTERP_LANES && o.interp != XSLP_INTERP_PAIRS && o.interp != XSLP_INTERP_TMEM)
    throw Error(XSLP_EINVAL, "interp must be XSLP_INTERP_LANES, XSLP_INTERP_PAIRS or XSLP_INTERP_TMEM");
  if (o.threads * o.groups > 992) throw Error(XSLP_EINVAL, "pipe kernel: threads * groups <= 992");
}

}  // namespace

namespace xslp {
// bitmatrix -> compiled program, in place (xslp_compile and the codec's memo cache)
static void build_from_bits(Program &P, const uint8_t *bits, int out_rows, int in_cols, const xslp_opts &o) {
  if (out_rows < 0 || in_cols <= 0 || in_cols > 512 || out_rows > 4096)
    throw Error(XSLP_EINVAL, "bitmatrix shape out of range");
  auto t0 = std::chrono::steady_clock::now();
  P.opts = o;
  check_opts(P.opts);
  P.n_const = in_cols;
  P.n_goals = out_rows;
  std::vector<Bits> goals(out_rows, Bits(in_cols));
  for (int r = 0; r < out_rows; ++r)
    for (int c = 0; c < in_cols; ++c) {
      uint8_t b = bits[(size_t)r * in_cols + c];
      if (b > 1) throw Error(XSLP_EINVAL, "bitmatrix entries must be 0 or 1");
      if (b) goals[r].set(c);
    }
  if (P.opts.compress == XSLP_COMPRESS_NONE)
    P.slp = lift(goals, in_cols, P.opts.fuse != 0);
  else
    P.slp = compress(goals, in_cols, P.opts.compress == XSLP_COMPRESS_XORREPAIR);
  P.stats.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  finish(P, &goals, true);
}

std::shared_ptr<Program> compile_bits(const std::vector<uint8_t> &bitv, int out_rows, int in_cols,
                                      const xslp_opts &o) {
  if (out_rows < 0 || in_cols <= 0 || bitv.size() < (size_t)out_rows * in_cols)
    throw Error(XSLP_EINVAL, "bitmatrix too short");
  auto P = std::make_shared<Program>();
  build_from_bits(*P, bitv.data(), out_rows, in_cols, o);
  return P;
}
}  // namespace xslp

extern "C" int xslp_compile(const uint8_t *bits, int out_rows, int in_cols, const xslp_opts *opts,
                            xslp_program **out) {
  API_BEGIN
  if (!out) throw Error(XSLP_EINVAL, "null out");
  *out = nullptr;
  if (!bits && out_rows * in_cols > 0) throw Error(XSLP_EINVAL, "null bitmatrix");
  xslp_opts o;
  if (opts) o = *opts; else xslp_default_opts(&o);
  auto P = std::make_unique<Program>();
  build_from_bits(*P, bits, out_rows, in_cols, o);
  *out = reinterpret_cast<xslp_program *>(P.release());
  API_END
}

extern "C" int xslp_compile_text(const char *text, int n_const, const xslp_opts *opts,
                                 xslp_program **out) {
  API_BEGIN
  if (!out || !text || n_const <= 0 || n_const > 512) throw Error(XSLP_EINVAL, "bad arguments");
  *out = nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto P = std::make_unique<Program>();
  if (opts) P->opts = *opts; else xslp_default_opts(&P->opts);
  check_opts(P->opts);
  Slp s = parse_text(text, n_const);
  auto goals = evaluate(s);
  P->n_const = n_const;
  P->n_goals = (int)goals.size();
  if (P->opts.compress == XSLP_COMPRESS_NONE) P->slp = s;
  else P->slp = compress(goals, n_const, P->opts.compress == XSLP_COMPRESS_XORREPAIR);
  P->stats.compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  finish(*P, &goals, P->opts.compress != XSLP_COMPRESS_NONE);
  *out = reinterpret_cast<xslp_program *>(P.release());
  API_END
}

extern "C" int xslp_program_stats(const xslp_program *prog, xslp_stats *st) {
  API_BEGIN
  if (!prog || !st) throw Error(XSLP_EINVAL, "null argument");
  *st = reinterpret_cast<const Program *>(prog)->stats;
  API_END
}

extern "C" int64_t xslp_program_dump(const xslp_program *prog, int form, char *buf, size_t cap) {
  try {
    if (!prog) throw Error(XSLP_EINVAL, "null program");
    const Program &P = *reinterpret_cast<const Program *>(prog);
    std::string s;
    if (form == 0) {
      s = "# xslp program: n_const=" + std::to_string(P.n_const) + " n_goals=" +
          std::to_string(P.n_goals) + " xor=" + std::to_string(P.stats.xor_count) + " mem=" +
          std::to_string(P.stats.mem_count) + " instr=" + std::to_string(P.stats.n_instr) +
          " nvar=" + std::to_string(P.stats.nvar) + " maxlive=" + std::to_string(P.stats.maxlive) + "\n";
      s += dump_pebbles(P.slp, P.pebble);
    } else if (form == 1) {
      s = dump_slots(P.code, P.n_const);
    } else if (form == 2) {
      s = P.ptx_baked.empty() ? P.ptx_generic : P.ptx_baked;
    } else if (form == 3) {
      // the pipelined interpreter's micro-op code (stage-0 variant) for this program's opts
      const int L = P.opts.lane_words == 2 || P.opts.lane_words == 4 ? P.opts.lane_words : 1;
      auto w = interp_code_dump(P.slp, P.opts.threads, L, P.opts.stages);
      for (size_t i = 0; i < w.size(); ++i) s += std::to_string(w[i]) + (i + 1 < w.size() ? " " : "\n");
    } else if (form == 4) {
      // the lane-parallel interpreter's code (stage-0 variant) for S = opts.stages
      auto w = interp_lanes_dump(&P, P.opts.stages);
      for (size_t i = 0; i < w.size(); ++i) s += std::to_string(w[i]) + (i + 1 < w.size() ? " " : "\n");
    } else if (form == 5 || form == 6 || form == 7) {
      // the TMEM interpreter's schedule (5) and the device code its kernel runs (6)
      auto w = interp_tmem_dump(&P, form);
      for (size_t i = 0; i < w.size(); ++i) s += std::to_string(w[i]) + (i + 1 < w.size() ? " " : "\n");
    } else {
      throw Error(XSLP_EINVAL, "bad dump form");
    }
    if (buf && cap) {
      size_t k = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
    return (int64_t)s.size();
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return XSLP_EINVAL;
  }
}

extern "C" int xslp_program_cache(const xslp_program *prog, int capacity, int64_t *iocost,
                                  int32_t *ccap) {
  API_BEGIN
  if (!prog) throw Error(XSLP_EINVAL, "null program");
  const Program &P = *reinterpret_cast<const Program *>(prog);
  if (ccap) *ccap = lru_ccap(P.slp, P.pebble);
  if (iocost) {
    if (capacity <= 0) throw Error(XSLP_EINVAL, "capacity must be positive");
    *iocost = lru_iocost(P.slp, P.pebble, capacity);
  }
  API_END
}

extern "C" void xslp_free(xslp_program *prog) { delete reinterpret_cast<Program *>(prog); }

extern "C" const char *xslp_last_error(void) { return g_err.c_str(); }

extern "C" const char *xslp_version(void) { return "xslp 0.1 (sm_100a)"; }
