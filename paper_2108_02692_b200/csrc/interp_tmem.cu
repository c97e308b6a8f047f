// TMEM interpreter: the paper's "interpreter style" with the SLP's constants and
// variables held in Blackwell tensor memory.  The default batched interpreter.
//
// Why: an interpreter cannot keep SLP variables in registers (their names are data, and an
// indirect branch per instruction costs ~150 cycles on sm_100a: scripts/dispatch_probe.py), so
// the shared-memory interpreters (interp.cu, interp_lanes.cu) read every operand from shared
// memory and are bound by its 128 B/clk/SM.  Tensor memory (256 KB per SM, 128 lanes x 512
// 32-bit columns) is addressed per thread by a warp-uniform column: exactly the "variable
// index is data" access an interpreter needs, at ~280-390 B/clk/SM of tcgen05.ld bandwidth and
// ~17 cycles latency (scripts/tmem_probe.cu).  Every thread runs the same instruction stream on
// its own words, so code reads are broadcasts and the data never crosses lanes.
//
// Work layout (persistent, one CTA per SM): 4 consumer warps (128 threads = the 128 TMEM
// lanes, warp w owns lane quarter w and all 512 columns) + 4 producer warps (one per SMSP).  A tile is 128*W
// consecutive 32-bit words of every strip of one stripe (W = 2 words per thread, 1 when the
// TMEM slots or shared-memory rows do not fit); thread t owns words t*W..t*W+W-1.  The producer
// streams each tile's constant strips by TMA (cp.async.bulk + mbarrier full/empty ring of S
// stages) and, when the program changes, the program's code into the code slot.  A consumer
// copies the tile's constant rows into its TMEM constant slots (8 slots per tcgen05.st) and
// releases the stage at once, then runs the batches out of TMEM.
//
// Two streams (when every program of the launch has Program::streams and their slots fit as
// many words per thread): the program's goal halves, compiled apart, run on 8 consumer warps,
// warps q and q + 4 sharing lane quarter q and its constant slots, each with variable slots of
// its own; the pair meets only after the tile's constant copies and at the tile's end, so two
// independent op streams hide each other's latencies on each SMSP.
//
// Code (host, build_tmem): the scheduled SLP's instructions (P:803-818 MultiSLP, DFS order
// P:1279-1303) become ops of at most four operands (wider instructions: a tree of partial ops
// into temporaries), list-scheduled into batches of kB (16) mutually independent ops: among
// the ready ops of a window of 400 in op order, the longest remaining chain first (critical-path
// priority; the batch count is the kernel's latency count), two-operand ops together where the
// window allows, ops that only store a goal deferred into a few goal batches.  A consumer issues all TMEM loads of a batch, waits once
// (tcgen05.wait::ld), XORs, stores the results to TMEM (tcgen05.st) and goals to HBM.  TMEM
// slots (W columns each) are assigned by liveness at batch granularity (a constant's slot is
// reused after the constant's last reader); a batch reading a slot
// stored since the last wait first waits for the stores (tcgen05.wait::st).  The device code
// has one variant per lane quarter with the quarter in every TMEM address, so an operand costs
// one R2UR and one tcgen05.ld.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <array>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>

#include "xslp_api.h"

namespace xslp {

void count_launch();  // device.cu

namespace tmem {

constexpr int kMaxB = 16;          // ops per batch: batch_size() (16; 4, 8, 12 for experiments)
constexpr int kH = 4;              // tile header slots (a ring longer than the S stages)
constexpr int kHead = 8;           // code header words
constexpr int kHdr = 16 + 8 * 256;  // tile header: stripe, prog, pad, a pointer per goal strip
constexpr int kCols = 512;         // TMEM columns allocated per CTA
constexpr int kNP = 4;             // producer warps
constexpr int kZero = 0, kJunk = 1, kConst0 = 2;  // TMEM slots: zero, write sink, constants
constexpr uint32_t kNone = 0xffff;

inline int batch_size() {
  static const int b = [] {
    const char *e = getenv("XSLP_TMEM_BATCH");
    // measured with the critical-path scheduler: 16 > 20 > 24 > 12 > 8 (profiles/r02/tmem)
    return e && (atoi(e) == 4 || atoi(e) == 8 || atoi(e) == 12) ? atoi(e) : 16;
  }();
  return b;
}

// two-stream code (Program::streams, 8 consumer warps) when available: XSLP_TMEM_STREAMS=1
// keeps one stream
inline bool streams_wanted() {
  static const bool v = [] {
    const char *e = getenv("XSLP_TMEM_STREAMS");
    return !(e && atoi(e) == 1);
  }();
  return v;
}
inline size_t sched_window() {
  static const size_t w = [] {
    const char *e = getenv("XSLP_TMEM_WINDOW");
    return e && atoi(e) > 0 ? (size_t)atoi(e) : (size_t)400;
  }();
  return w;
}
inline bool sched_recycle() {
  static const bool h = [] {
    const char *e = getenv("XSLP_TMEM_RECYCLE");
    return !e || atoi(e) > 0;
  }();
  return h;
}
inline bool sched_height() {
  static const bool h = [] {
    const char *e = getenv("XSLP_TMEM_HEIGHT");
    return !e || atoi(e) > 0;
  }();
  return h;
}
inline bool sched_mixed() {  // experiment: fill batches by priority only, ignoring the op class
  static const bool h = [] {
    const char *e = getenv("XSLP_TMEM_MIXED");
    return e && atoi(e) > 0;
  }();
  return h;
}

struct TOp {
  int t[4] = {-1, -1, -1, -1};  // operand terms: constant c (< n_const) or variable n_const + v
  int dst = -1;                 // variable defined (-1: none, the result is a goal only)
  int goal = -1;                // goal stored (-1: none)
  int arity() const { return (t[0] >= 0) + (t[1] >= 0) + (t[2] >= 0) + (t[3] >= 0); }
};

struct TSched {
  int n_const = 0;
  int B = 16;                                   // ops per batch
  std::vector<std::array<TOp, kMaxB>> batches;  // unused entries: no operands, dst = goal = -1
  std::vector<uint8_t> wait_st;              // batch first waits for earlier TMEM stores
  std::vector<int> consts;                   // constant row r (TMEM slot kConst0 + r) holds consts[r]
  std::vector<int> vslot;                    // variable -> TMEM slot
  int nslots = 0;                            // slots used (zero, sink, constants, variables)
};

// Lower the scheduled SLP into 4-operand ops and batches of kB independent ops.
TSched build_tmem(const Slp &s, bool recycle = true) {
  TSched out;
  out.n_const = s.n_const;
  const int kB = out.B = batch_size();
  int nv = s.n_vars;
  std::vector<TOp> ops;
  std::vector<std::vector<int>> goals_of(s.n_vars);  // variable -> goal indices
  for (size_t g = 0; g < s.goal.size(); ++g) {
    const int t = s.goal[g];
    if (t >= s.n_const) goals_of[t - s.n_const].push_back((int)g);
  }
  // an instruction of arity a > 4 becomes partial ops of 4 operands into temporaries
  auto emit = [&](std::vector<int> ts, int dst, int goal) {
    while (ts.size() > 4) {
      TOp p;
      for (int k = 0; k < 4; ++k, ts.pop_back()) p.t[k] = ts.back();
      p.dst = nv++;
      ops.push_back(p);
      ts.insert(ts.begin(), s.n_const + p.dst);
    }
    TOp o;
    for (size_t k = 0; k < ts.size(); ++k) o.t[k] = ts[k];
    o.dst = dst;
    o.goal = goal;
    ops.push_back(o);
  };
  std::vector<int> nuses(s.n_vars, 0);
  for (const auto &in : s.ins)
    for (int t : in.ops)
      if (t >= s.n_const) ++nuses[t - s.n_const];
  for (const auto &in : s.ins) {
    const auto &gl = goals_of[in.var];
    const int dst = nuses[in.var] > 0 ? in.var : -1;
    if (dst < 0 && gl.empty()) continue;  // dead (the compiler keeps none)
    emit(in.ops, dst, gl.empty() ? -1 : gl[0]);
    for (size_t k = 1; k < gl.size(); ++k) {  // duplicate goals: copy ops
      if (dst < 0) throw Error(XSLP_EINVAL, "tmem: duplicate goal of a dead variable");
      emit({s.n_const + in.var}, -1, gl[k]);
    }
  }
  for (size_t g = 0; g < s.goal.size(); ++g) {  // constant and zero goals
    const int t = s.goal[g];
    if (t >= s.n_const) continue;
    emit(t >= 0 ? std::vector<int>{t} : std::vector<int>{}, -1, (int)g);
  }
  // ---- batches: list scheduling in op order (the DFS order keeps lifetimes short); a batch
  // of ops with at most two operands skips the loads of operands 3-4, so such ops are batched
  // together when the window allows
  std::vector<int> batch_of(ops.size(), -1);
  std::vector<int> vbatch(nv, -1);  // batch that defines the variable
  auto ready = [&](size_t i, int nb) {
    for (int t : ops[i].t)
      if (t >= s.n_const && (vbatch[t - s.n_const] < 0 || vbatch[t - s.n_const] >= nb)) return false;
    return true;
  };
  // Ops that only store a goal (no later reader) are deferred and batched together, kB at a
  // time, so that only a few batches run the goal-store code.
  std::vector<size_t> gq;  // deferred goal-only ops, in order
  std::vector<uint8_t> deferred(ops.size(), 0);
  for (size_t i = 0; i < ops.size(); ++i)
    if (ops[i].dst < 0) {
      deferred[i] = 1;
      gq.push_back(i);
    }
  size_t first = 0, left = ops.size() - gq.size();
  int nb = 0;
  const size_t kWindow = sched_window();
  // height of an op: the longest chain of ops that read its result (critical-path priority)
  std::vector<int> height(ops.size(), 0);
  {
    std::vector<int> hv(nv, 0);  // variable -> height of its defining op
    for (size_t i = ops.size(); i-- > 0;) {
      int h = 0;
      if (ops[i].dst >= 0) h = hv[ops[i].dst];
      height[i] = h + 1;
      for (int t : ops[i].t)
        if (t >= s.n_const) hv[t - s.n_const] = std::max(hv[t - s.n_const], height[i]);
    }
  }
  const bool by_height = sched_height();
  auto skip = [&]() {
    while (first < ops.size() && (batch_of[first] >= 0 || deferred[first])) ++first;
  };
  skip();
  while (left > 0 || !gq.empty()) {
    std::array<TOp, kMaxB> b;
    int n = 0;
    std::vector<size_t> gready;
    for (size_t i : gq)
      if (ready(i, nb)) gready.push_back(i);
    if ((int)gready.size() >= kB || left == 0) {  // a batch of goal-only ops
      for (size_t i : gready) {
        if (n == kB) break;
        batch_of[i] = nb;
        b[n++] = ops[i];
      }
      std::vector<size_t> rest;
      for (size_t i : gq)
        if (batch_of[i] < 0) rest.push_back(i);
      gq.swap(rest);
    } else {
      // the oldest ready op decides the batch class; fill with ready ops of that class, then any
      int cls = -1;
      std::vector<size_t> cand;  // ready ops of the window, in priority order
      for (size_t i = first; i < ops.size() && i < first + kWindow; ++i)
        if (batch_of[i] < 0 && !deferred[i] && ready(i, nb)) cand.push_back(i);
      if (by_height)
        std::stable_sort(cand.begin(), cand.end(), [&](size_t x, size_t y) { return height[x] > height[y]; });
      for (int pass = 0; pass < 2 && n < kB; ++pass)
        for (size_t i : cand) {
          if (n == kB) break;
          if (batch_of[i] >= 0) continue;
          const int c = ops[i].arity() > 2;
          if (cls < 0) cls = c;
          if (pass == 0 && c != cls && !sched_mixed()) continue;
          batch_of[i] = nb;
          b[n++] = ops[i];
          --left;
        }
    }
    if (n == 0) throw Error(XSLP_EINVAL, "tmem: no ready op (bad schedule)");
    for (int k = 0; k < n; ++k)
      if (b[k].dst >= 0) vbatch[b[k].dst] = nb;
    out.batches.push_back(b);
    ++nb;
    skip();
  }
  // ---- constant rows in first-use order
  std::vector<int> row(s.n_const, -1);
  for (const auto &b : out.batches)
    for (const auto &o : b)
      for (int t : o.t)
        if (t >= 0 && t < s.n_const && row[t] < 0) {
          row[t] = (int)out.consts.size();
          out.consts.push_back(t);
        }
  // ---- variable slots by liveness at batch granularity, after the constant slots
  const int v0 = kConst0 + (int)out.consts.size();
  std::vector<int> last(nv, -1);
  for (int bi = 0; bi < nb; ++bi)
    for (const auto &o : out.batches[bi])
      for (int t : o.t)
        if (t >= s.n_const) last[t - s.n_const] = std::max(last[t - s.n_const], bi);
  out.vslot.assign(nv, -1);
  // slot kConst0 + k -> first batch that may overwrite it: a constant's slot is free after the
  // constant's last reader (the tile's constant copies come before batch 0 and after the
  // previous tile's last batch), a variable's after its last reader
  std::vector<int> free_at(out.consts.size(), 0);
  for (int bi = 0; bi < nb; ++bi)
    for (const auto &o : out.batches[bi])
      for (int t : o.t)
        if (t >= 0 && t < s.n_const) free_at[row[t]] = std::max(free_at[row[t]], bi + 1);
  if (!recycle || !sched_recycle()) std::fill(free_at.begin(), free_at.end(), nb + 1);
  for (int bi = 0; bi < nb; ++bi)
    for (const auto &o : out.batches[bi]) {
      if (o.dst < 0) continue;
      int k = 0;
      while (k < (int)free_at.size() && free_at[k] > bi) ++k;
      if (k == (int)free_at.size()) free_at.push_back(0);
      out.vslot[o.dst] = kConst0 + k;
      free_at[k] = std::max(last[o.dst], bi) + 1;  // read through batch last[dst]
    }
  out.nslots = std::max(v0, kConst0 + (int)free_at.size());
  // a wait::st at the start of batch w completes the stores of batches < w; the tile's
  // constant copies are waited for before batch 0
  out.wait_st.assign(nb, 0);
  int covered = 0;
  for (int bi = 1; bi < nb; ++bi) {
    bool need = false;
    for (const auto &o : out.batches[bi])
      for (int t : o.t)
        if (t >= s.n_const && vbatch[t - s.n_const] >= covered) need = true;
    if (need) {
      out.wait_st[bi] = 1;
      covered = bi;
    }
  }
  return out;
}

// Code (u32 words; TMEM columns = slot * W):
//   [0] nconst rows [1] nbatches [2] total words [3] slots used [4] kB [5] W [6..7] 0
//   batches: nbatches x kB ops x 4 words, then one padding batch (the consumer prefetches):
//     w0 = col(t0) | col(t1) << 16   w1 = col(t2) | col(t3) << 16   (absent operand: the zero slot)
//     w2 = col(dst) (absent: the sink slot) | (goal + 1) << 16
//     w3 (op 0 of a batch) = 1: wait for earlier TMEM stores first; 2: the batch has ops of
//        three or four operands (else operands 3-4 are not loaded); 4: the batch stores goals
//   loads: nconst x (constant index)   (row r = TMEM slot kConst0 + r)
std::vector<uint32_t> emit_code(const TSched &sc, int W) {
  const int kB = sc.B;
  std::vector<uint32_t> w(kHead, 0);
  std::vector<int> row(sc.n_const, -1);
  for (size_t r = 0; r < sc.consts.size(); ++r) row[sc.consts[r]] = (int)r;
  auto col = [&](int t) -> uint32_t {
    if (t < 0) return (uint32_t)(kZero * W);
    if (t < sc.n_const) return (uint32_t)((kConst0 + row[t]) * W);
    return (uint32_t)(sc.vslot[t - sc.n_const] * W);
  };
  w[0] = (uint32_t)sc.consts.size();
  w[1] = (uint32_t)sc.batches.size();
  w[3] = (uint32_t)sc.nslots;
  w[4] = kB;
  w[5] = (uint32_t)W;
  for (size_t bi = 0; bi < sc.batches.size(); ++bi) {
    bool quad = false, goals = false;
    for (int j = 0; j < kB; ++j) {
      quad |= sc.batches[bi][j].arity() > 2;
      goals |= sc.batches[bi][j].goal >= 0;
    }
    for (int j = 0; j < kB; ++j) {
      const TOp &o = sc.batches[bi][j];
      const uint32_t d = o.dst >= 0 ? (uint32_t)(sc.vslot[o.dst] * W) : (uint32_t)(kJunk * W);
      const uint32_t fl = j == 0 ? (sc.wait_st[bi] ? 1u : 0u) | (quad ? 2u : 0u) | (goals ? 4u : 0u) : 0u;
      w.insert(w.end(), {col(o.t[0]) | col(o.t[1]) << 16, col(o.t[2]) | col(o.t[3]) << 16,
                         d | (uint32_t)(o.goal + 1) << 16, fl});
    }
  }
  for (int j = 0; j < kB; ++j)  // padding batch
    w.insert(w.end(), {0u, 0u, (uint32_t)(kJunk * W), 0u});
  for (int c : sc.consts) w.push_back((uint32_t)c);
  while (w.size() % 4) w.push_back(0);
  w[2] = (uint32_t)w.size();
  return w;
}

inline int consumer_words(const TSched &sc) { return kHead + 4 * sc.B * ((int)sc.batches.size() + 1); }

// Device code (what the kernel runs; the form above is its compact, emulated twin): one
// variant per consumer warp with the warp's TMEM lane quarter in every address, so an operand
// costs one R2UR and one tcgen05.ld -- no decode.
//   [0] nconst [1] nbatches [2] total words [3] slots [4] kB [5] W [6] vw = words per variant
//   [7] batch 0's flags
//   4 variants of vw words; per batch: {flags (as w3 above), the next batch's flags (0 after the
//   last), 0, 0}, then the kB ops' operand addresses (flag 2, up to four operands: {a0, a1, a2,
//   a3} per op; else {a0, a1}), then kB dst addresses, then kB goal words (goal + 1)
//     (a = TMEM address: lane quarter << 16 | column; absent operand: the zero slot; absent
//      dst: the sink slot; goal + 1 = 0: none)
//   loads: nconst x (constant index)
// One stream's batches (the variant of lane quarter 0): col(t) = the TMEM column of operand
// term t, vcol(v) = the column of variable v, goals stored as goal + goal0 + 1.  adr marks the
// words that are TMEM addresses (the other variants add their lane quarter to them).
void emit_batches(const TSched &sc, int W, const std::vector<uint32_t> &ccol,
                  const std::vector<uint32_t> &vcol, int goal0, std::vector<uint32_t> &v,
                  std::vector<uint8_t> &adr, uint32_t &flags0) {
  const int kB = sc.B;
  auto col = [&](int t) -> uint32_t {
    if (t < 0) return (uint32_t)(kZero * W);
    return t < sc.n_const ? ccol[t] : vcol[t - sc.n_const];
  };
  auto bflags = [&](size_t bi) {
    bool quad = false, goals = false;
    for (int j = 0; j < kB; ++j) {
      quad |= sc.batches[bi][j].arity() > 2;
      goals |= sc.batches[bi][j].goal >= 0;
    }
    return (sc.wait_st[bi] ? 1u : 0u) | (quad ? 2u : 0u) | (goals ? 4u : 0u);
  };
  auto put = [&](uint32_t x, bool a) {
    v.push_back(x);
    adr.push_back(a);
  };
  for (size_t bi = 0; bi < sc.batches.size(); ++bi) {
    const bool quad = bflags(bi) & 2;
    put(bflags(bi), false);
    put(bi + 1 < sc.batches.size() ? bflags(bi + 1) : 0u, false);  // read ahead by the kernel
    for (int k = 0; k < 2; ++k) put(0, false);
    for (int j = 0; j < kB; ++j)
      for (int k = 0; k < (quad ? 4 : 2); ++k) put(col(sc.batches[bi][j].t[k]), true);
    for (int j = 0; j < kB; ++j) {
      const TOp &o = sc.batches[bi][j];
      put(o.dst >= 0 ? vcol[o.dst] : (uint32_t)(kJunk * W), true);
    }
    for (int j = 0; j < kB; ++j) {
      const int g = sc.batches[bi][j].goal;
      put(g >= 0 ? (uint32_t)(g + goal0 + 1) : 0u, false);
    }
  }
  flags0 = sc.batches.empty() ? 0u : bflags(0);
}

// lane quarter variants of a stream: the quarter in every TMEM address
inline void put_variants(std::vector<uint32_t> &w, const std::vector<uint32_t> &v,
                         const std::vector<uint8_t> &adr, int nvar) {
  for (int q = 0; q < nvar; ++q)
    for (size_t i = 0; i < v.size(); ++i) w.push_back(v[i] | (adr[i] ? (uint32_t)(q * 32) << 16 : 0u));
}

std::vector<uint32_t> emit_device(const TSched &sc, int W, int nvar = 4) {
  std::vector<uint32_t> ccol(sc.n_const, 0), vcol(sc.vslot.size(), 0);
  for (size_t r = 0; r < sc.consts.size(); ++r) ccol[sc.consts[r]] = (uint32_t)((kConst0 + r) * W);
  for (size_t x = 0; x < sc.vslot.size(); ++x) vcol[x] = (uint32_t)(sc.vslot[x] * W);
  std::vector<uint32_t> v;
  std::vector<uint8_t> adr;
  uint32_t f0 = 0;
  emit_batches(sc, W, ccol, vcol, 0, v, adr, f0);
  std::vector<uint32_t> w(kHead, 0);
  w[0] = (uint32_t)sc.consts.size();
  w[1] = (uint32_t)sc.batches.size();
  w[3] = (uint32_t)sc.nslots;
  w[4] = sc.B;
  w[5] = (uint32_t)W;
  w[6] = (uint32_t)v.size();
  w[7] = f0;
  put_variants(w, v, adr, nvar);
  for (int c : sc.consts) w.push_back((uint32_t)c);
  while (w.size() % 4) w.push_back(0);
  w[2] = (uint32_t)w.size();
  return w;
}

// Two streams (the program's goal halves compiled apart, Program::streams) sharing the
// constant rows: stream h's variables get slots of their own after the constants (no constant
// slot is reused: the streams run unsynchronised within a tile).
struct TStreams {
  std::shared_ptr<const TSched> sc[2];
  std::vector<int> consts;  // constant rows: the union, stream 0's first-use order first
  int base[2] = {0, 0};     // first variable slot of each stream
  int nslots = 0;
  int goal0[2] = {0, 0};    // goal offset of each stream
};

TStreams build_streams(const Program &p) {
  TStreams t;
  for (int h = 0; h < 2; ++h) t.sc[h] = std::make_shared<const TSched>(build_tmem(p.streams[h], false));
  std::vector<char> in(p.n_const, 0);
  for (int h = 0; h < 2; ++h)
    for (int c : t.sc[h]->consts)
      if (!in[c]) {
        in[c] = 1;
        t.consts.push_back(c);
      }
  int next = kConst0 + (int)t.consts.size();
  for (int h = 0; h < 2; ++h) {
    t.base[h] = next;
    next += t.sc[h]->nslots - (kConst0 + (int)t.sc[h]->consts.size());
  }
  t.nslots = next;
  t.goal0[1] = (int)p.streams[0].goal.size();
  return t;
}

// Two-stream device code: header (kHead2 words)
//   [0] constant rows [1] stream 0 batches [2] total words [3] slots [4] kB [5] W
//   [6] stream 0 words per variant [7] stream 0 batch 0 flags [8] stream 1 batches
//   [9] stream 1 words per variant [10] stream 1 batch 0 flags [11] stream 1 offset (words
//   after the header) [12..15] 0
// then stream 0's 4 variants, stream 1's 4 variants (as emit_device), the constant list.
constexpr int kHead2 = 16;
std::vector<uint32_t> emit_streams(const TStreams &t, int W, int nvar = 4) {
  std::vector<uint32_t> v[2];
  std::vector<uint8_t> adr[2];
  uint32_t f0[2] = {0, 0};
  for (int h = 0; h < 2; ++h) {
    const TSched &sc = *t.sc[h];
    std::vector<uint32_t> ccol(sc.n_const, 0), vcol(sc.vslot.size(), 0);
    for (size_t r = 0; r < t.consts.size(); ++r) ccol[t.consts[r]] = (uint32_t)((kConst0 + r) * W);
    const int v0 = kConst0 + (int)sc.consts.size();
    for (size_t x = 0; x < sc.vslot.size(); ++x)
      if (sc.vslot[x] >= 0) {
        if (sc.vslot[x] < v0) throw Error(XSLP_EINVAL, "tmem: stream variable in a constant slot");
        vcol[x] = (uint32_t)((t.base[h] + sc.vslot[x] - v0) * W);
      }
    emit_batches(sc, W, ccol, vcol, t.goal0[h], v[h], adr[h], f0[h]);
  }
  std::vector<uint32_t> w(kHead2, 0);
  w[0] = (uint32_t)t.consts.size();
  w[1] = (uint32_t)t.sc[0]->batches.size();
  w[3] = (uint32_t)t.nslots;
  w[4] = t.sc[0]->B;
  w[5] = (uint32_t)W;
  w[6] = (uint32_t)v[0].size();
  w[7] = f0[0];
  w[8] = (uint32_t)t.sc[1]->batches.size();
  w[9] = (uint32_t)v[1].size();
  w[10] = f0[1];
  w[11] = (uint32_t)(nvar * v[0].size());
  put_variants(w, v[0], adr[0], nvar);
  put_variants(w, v[1], adr[1], nvar);
  for (int c : t.consts) w.push_back((uint32_t)c);
  while (w.size() % 4) w.push_back(0);
  w[2] = (uint32_t)w.size();
  return w;
}

// words of the device code a consumer reads (header + 4 variants): the code slot size
inline int stream_words(const TSched &sc) {
  int per = 0;
  for (size_t bi = 0; bi < sc.batches.size(); ++bi) {
    bool quad = false;
    for (int j = 0; j < sc.B; ++j) quad |= sc.batches[bi][j].arity() > 2;
    per += 4 + sc.B * (quad ? 6 : 4);
  }
  return per;
}
inline int device_words(const TSched &sc) { return kHead + 4 * stream_words(sc); }
inline int device_words(const TStreams &t) {
  return kHead2 + 4 * (stream_words(*t.sc[0]) + stream_words(*t.sc[1]));
}

struct Layout {
  int W = 2, CW = 4, S = 2, NC = 1, capw = 0, B = 16;
  uint32_t code0 = 0, const0 = 0, RB = 0;
  size_t smem = 0;
};

size_t layout_smem(Layout &y) {
  y.RB = (uint32_t)(128 * y.W * 4);  // a row: 128 TMEM lanes x W words
  y.code0 = 128 + kH * kHdr;
  size_t c0 = y.code0 + (size_t)y.capw * 4;  // one code slot
  c0 = (c0 + 127) / 128 * 128;
  y.const0 = (uint32_t)c0;
  y.smem = c0 + (size_t)y.S * y.NC * y.RB;
  // at least half the SM's shared memory: one CTA per SM, so one TMEM allocation of 512 columns
  y.smem = std::max<size_t>(y.smem, 120 * 1024);
  return y.smem;
}

struct Args {
  const uint32_t *code;
  const int64_t *prog_off;
  const int32_t *prog_of_stripe;
  const int32_t *ids;
  const uint8_t *const *in_tbl;
  uint8_t *const *out_tbl;
  uint64_t strip;
  uint32_t words, tps, ntiles, tpos;  // tpos = consumer threads * W words per strip per tile
  int32_t n_in, n_out, S, nprogs;
  uint32_t code0, capw, const0, RB, NC;
};

__device__ __forceinline__ uint32_t sm_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}

template <int W>
struct Vec { uint32_t x[W]; };

template <int W>
__device__ __forceinline__ void lds_w(uint32_t a, Vec<W> &v) {
  if constexpr (W == 1) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v.x[0]) : "r"(a) : "memory");
  else asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x[0]), "=r"(v.x[1]) : "r"(a) : "memory");
}
template <int W>
__device__ __forceinline__ void ldtm_w(uint32_t ta, Vec<W> &v) {
  if constexpr (W == 1)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v.x[0]) : "r"(ta) : "memory");
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v.x[0]), "=r"(v.x[1]) : "r"(ta) : "memory");
}
template <int W>
__device__ __forceinline__ void sttm_w(uint32_t ta, const Vec<W> &v) {
  if constexpr (W == 1)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v.x[0]) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta), "r"(v.x[0]), "r"(v.x[1]) : "memory");
}
// 8 consecutive slots (8W columns) in one store
template <int W>
__device__ __forceinline__ void sttm_rows8(uint32_t ta, const Vec<W> (&v)[8]) {
  if constexpr (W == 1)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta), "r"(v[0].x[0]), "r"(v[1].x[0]), "r"(v[2].x[0]), "r"(v[3].x[0]), "r"(v[4].x[0]),
                 "r"(v[5].x[0]), "r"(v[6].x[0]), "r"(v[7].x[0]) : "memory");
  else
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                 "%11, %12, %13, %14, %15, %16};"
                 ::"r"(ta), "r"(v[0].x[0]), "r"(v[0].x[1]), "r"(v[1].x[0]), "r"(v[1].x[1]), "r"(v[2].x[0]),
                 "r"(v[2].x[1]), "r"(v[3].x[0]), "r"(v[3].x[1]), "r"(v[4].x[0]), "r"(v[4].x[1]),
                 "r"(v[5].x[0]), "r"(v[5].x[1]), "r"(v[6].x[0]), "r"(v[6].x[1]), "r"(v[7].x[0]),
                 "r"(v[7].x[1]) : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// W words per thread, CW consumer warps (4: each owns a 32-lane TMEM quarter and 512 columns;
// 8: warps w and w+4 share a quarter, 256 columns each)
template <int W, int CW, int kB>
__global__ void __launch_bounds__(CW * 32 + kNP * 32, 1) xslp_interp_tmem(Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t tid = threadIdx.x;
  const int S = a.S;
  const uint32_t base = sm_addr(sm);
  const uint32_t hdr0 = base + 128;
  const uint32_t warp = tid / 32, lane = tid & 31;
  // Tile it uses constant-row stage it % S and header slot it % kH; the program's code sits in
  // one code slot, rewritten when the program changes (after the previous tile is done).
  // Barriers: full[k] +8k (TMA bytes of stage k), rows_empty[k] +32+8k (stage k's rows
  // copied to TMEM), tile_done[h] +64+8h (the tile of header slot h is done); TMEM base
  // address at +120
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 8 * k), "n"(kNP));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 32 + 8 * k), "r"(CW));
    }
    for (int k = 0; k < kH; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 64 + 8 * k), "r"(CW));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(base + 120),
                 "n"(kCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tbase;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(base + 120) : "memory");
  if (tbase & 0xffffu) asm volatile("trap;");  // all 512 columns: the allocation starts at column 0
  const uint32_t chunk = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * chunk, t1 = min(a.ntiles, t0 + chunk);
  if (warp >= CW) {  // ---------------- producer warps (all lanes issue copies)
    // kNP producer warps, one per SMSP, so that the copy-issue work (the compiler serialises
    // the lanes' bulk copies) lands evenly on the four consumer warps' schedulers: producer pw
    // issues constant rows pw, pw + kNP, ... and arrives on the full barrier with its own bytes
    const uint32_t pw = warp - CW;
    int cur = -1;  // the program in the code slot
    for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
      const uint32_t st = it % S, ph = (it / S) & 1, hs = it % kH, hph = (it / kH) & 1;
      const uint32_t entry = tile / a.tps, tw = tile % a.tps;
      const uint32_t stripe = a.ids ? (uint32_t)a.ids[entry] : entry;
      const int prog = a.prog_of_stripe ? a.prog_of_stripe[stripe] : 0;
      if (prog < 0 || prog >= a.nprogs) asm volatile("trap;");
      const uint32_t *pc = a.code + a.prog_off[prog];
      const uint8_t *const *in = a.in_tbl + (size_t)stripe * a.n_in;
      uint8_t *const *out = a.out_tbl + (size_t)stripe * a.n_out;
      const uint32_t nl = pc[0], nw = pc[2];
      const uint32_t *ld = pc + nw - ((nl + 3) & ~3u);  // the constant list ends the code
      const size_t toff = (size_t)tw * a.tpos * 4;
      const bool newcode = cur != prog;
      // (each producer shares an SMSP with a consumer warp: sleep rather than spin)
      if (it >= (uint32_t)S)
        while (!try_wait(base + 32 + 8 * st, ph ^ 1)) __nanosleep(256);
      if (it >= (uint32_t)kH)  // the tile that last used this header slot is done
        while (!try_wait(base + 64 + 8 * hs, hph ^ 1)) __nanosleep(256);
      if (newcode && it >= 1) {  // every earlier tile is done with the code slot
        const uint32_t pit = it - 1;
        while (!try_wait(base + 64 + 8 * (pit % kH), (pit / kH) & 1)) __nanosleep(256);
      }
      const uint32_t h = hdr0 + hs * kHdr;
      // goal strip g of this tile starts at out[g / 8] + (g % 8) * strip + toff
      for (uint32_t g = pw * 32 + lane; g < 8u * a.n_out; g += 32 * kNP) {
        const uint64_t gp = (uint64_t)out[g >> 3] + (g & 7) * a.strip + toff;
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(h + 16 + 8 * g), "l"(gp) : "memory");
      }
      const uint32_t nbytes = min(a.tpos, a.words - tw * a.tpos) * 4;
      const uint32_t cbytes = newcode && pw == 0 ? (nw - ((nl + 3) & ~3u)) * 4 : 0;  // header + variants
      const uint32_t nmine = nl > pw ? (nl - pw + kNP - 1) / kNP : 0;  // rows this warp copies
      cur = prog;
      __syncwarp();
      if (lane == 0) {
        if (pw == 0) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(h), "r"(stripe) : "memory");
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(h + 4), "r"((uint32_t)prog) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(base + 8 * st),
                     "r"(nbytes * nmine + cbytes) : "memory");
        if (cbytes)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(base + a.code0), "l"(pc), "r"(cbytes), "r"(base + 8 * st) : "memory");
      }
      __syncwarp();
      const uint32_t rows = a.const0 + st * a.NC * a.RB;
      for (uint32_t i = pw + kNP * lane; i < nl; i += kNP * 32) {
        const uint32_t c = ld[i];
        const uint8_t *src = in[c >> 3] + (c & 7) * a.strip + toff;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(base + rows + i * a.RB), "l"(src), "r"(nbytes), "r"(base + 8 * st) : "memory");
      }
    }
  } else {
    // ---------------- consumer warps: every thread runs the op stream on its W words
    // CW = 4: warp q owns TMEM lane quarter q.  CW = 8 (two-stream code): warps q and q + 4 share
    // lane quarter q and its constant slots; warp q + 4h runs stream h (the program's goal half
    // h, variables in slots of its own) independently of the other; the pair meets after the
    // tile's constant copies and at the tile's end.
    static_assert(CW == 4 || CW == 8, "4 consumer warps, or 8 running two streams");
    constexpr int NH = CW / 4;
    const uint32_t q = warp & 3, h = warp >> 2;
    const uint32_t lt = tid & 127;  // TMEM lane = the thread's word position in the tile
    const uint32_t tl = tbase + ((q * 32u) << 16);
    auto pair_sync = [&]() {
      if constexpr (NH > 1) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    };
    if (h == 0) {
      Vec<W> z;
#pragma unroll
      for (int w = 0; w < W; ++w) z.x[w] = 0;
      sttm_w<W>(tl + kZero * W, z);
      wait_st();
    }
    for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
      const uint32_t st = it % S, ph = (it / S) & 1, hs = it % kH;
      while (!try_wait(base + 8 * st, ph)) {
      }
      const uint32_t tw = tile % a.tps;
      const uint32_t npos = min(a.tpos, a.words - tw * a.tpos);
      const bool live = lt * W < npos;  // ragged tail: no goal stores past the strip
      const uint32_t hdr = hdr0 + hs * kHdr;
      const uint32_t cp = base + a.code0;
      const uint4 head = lds128(cp), head2 = lds128(cp + 16);
      uint32_t nb = head.y, vw = head2.z, fln = head2.w, voff = 0;  // this warp's stream
      if constexpr (NH > 1) {
        const uint4 head3 = lds128(cp + 32);
        if (h) {
          nb = head3.x;
          vw = head3.y;
          fln = head3.z;
          voff = head3.w;
        }
      }
      const uint32_t nl = head.x;
      // the stage's constant rows -> this thread's TMEM constant slots (16-row chunks alternate
      // between the two warps of a lane quarter); then the rows are free
      {
        const uint32_t rs = base + a.const0 + st * a.NC * a.RB + lt * W * 4;
        uint32_t r = 16 * h;
        for (; r + 16 <= nl; r += 16 * NH) {  // 16 rows' loads in flight, then two stores
          Vec<W> v[8], u[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) lds_w<W>(rs + (r + k) * a.RB, v[k]);
#pragma unroll
          for (int k = 0; k < 8; ++k) lds_w<W>(rs + (r + 8 + k) * a.RB, u[k]);
          sttm_rows8<W>(tl + (kConst0 + r) * W, v);
          sttm_rows8<W>(tl + (kConst0 + r + 8) * W, u);
        }
        if (h == 0) {
          r = nl / 16 * 16;
          for (; r + 8 <= nl; r += 8) {  // 8 consecutive slots: one tcgen05.st of 8W columns
            Vec<W> v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) lds_w<W>(rs + (r + k) * a.RB, v[k]);
            sttm_rows8<W>(tl + (kConst0 + r) * W, v);
          }
          for (; r < nl; ++r) {
            Vec<W> v;
            lds_w<W>(rs + r * a.RB, v);
            sttm_w<W>(tl + (kConst0 + r) * W, v);
          }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(base + 32 + 8 * st) : "memory");
      wait_st();
      pair_sync();  // both warps' constant copies are done
      const uint32_t tofs = lt * W * 4;  // this thread's bytes within a goal strip of the tile
      // batches: a batch's code words (broadcast shared loads) -> its operand loads (TMEM), one
      // wait, XORs -> result stores (TMEM) and goal stores
      // this warp's code variant (its stream, its lane quarter)
      uint32_t p = cp + (NH > 1 ? kHead2 : kHead) * 4 + voff * 4 + q * vw * 4;
      for (uint32_t b = 0; b < nb; ++b) {
        // this batch's flags were read with the previous batch's header (off the critical path)
        const uint32_t fl = fln;
        fln = lds128(p).y;
        p += 16;
        if (fl & 1) wait_st();
        Vec<W> acc[kB];
        uint32_t dst[kB];
        uint32_t pg;  // the batch's goal words
        if (fl & 2) {  // ops of up to four operands: 4 address words each, then dst and goal words
          uint4 u[kB];
#pragma unroll
          for (int j = 0; j < kB; ++j) u[j] = lds128(p + 16 * j);
          Vec<W> x[kB][4];
#pragma unroll
          for (int j = 0; j < kB; ++j) {
            ldtm_w<W>(u[j].x, x[j][0]);
            ldtm_w<W>(u[j].y, x[j][1]);
            ldtm_w<W>(u[j].z, x[j][2]);
            ldtm_w<W>(u[j].w, x[j][3]);
          }
#pragma unroll
          for (int k = 0; k < kB / 4; ++k) {
            const uint4 t = lds128(p + 16 * kB + 16 * k);
            dst[4 * k] = t.x;
            dst[4 * k + 1] = t.y;
            dst[4 * k + 2] = t.z;
            dst[4 * k + 3] = t.w;
          }
          pg = p + 20 * kB;
          p += 24 * kB;
          wait_ld();
#pragma unroll
          for (int j = 0; j < kB; ++j)
#pragma unroll
            for (int w = 0; w < W; ++w) {
              uint32_t y;
              asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(y) : "r"(x[j][0].x[w]), "r"(x[j][1].x[w]), "r"(x[j][2].x[w]));
              acc[j].x[w] = y ^ x[j][3].x[w];
            }
        } else {  // binary ops: 2 address words each, then dst and goal words
          uint4 u[kB / 2];
#pragma unroll
          for (int k = 0; k < kB / 2; ++k) u[k] = lds128(p + 16 * k);
          Vec<W> x[kB][2];
#pragma unroll
          for (int k = 0; k < kB / 2; ++k) {
            ldtm_w<W>(u[k].x, x[2 * k][0]);
            ldtm_w<W>(u[k].y, x[2 * k][1]);
            ldtm_w<W>(u[k].z, x[2 * k + 1][0]);
            ldtm_w<W>(u[k].w, x[2 * k + 1][1]);
          }
#pragma unroll
          for (int k = 0; k < kB / 4; ++k) {
            const uint4 t = lds128(p + 8 * kB + 16 * k);
            dst[4 * k] = t.x;
            dst[4 * k + 1] = t.y;
            dst[4 * k + 2] = t.z;
            dst[4 * k + 3] = t.w;
          }
          pg = p + 12 * kB;
          p += 16 * kB;
          wait_ld();
#pragma unroll
          for (int j = 0; j < kB; ++j)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[j].x[w] = x[j][0].x[w] ^ x[j][1].x[w];
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) sttm_w<W>(dst[j], acc[j]);
        if (fl & 4) {  // goal stores (predicated: ops without a goal and the ragged tail skip)
          uint32_t gw[kB];
#pragma unroll
          for (int k = 0; k < kB / 4; ++k) {
            const uint4 t = lds128(pg + 16 * k);
            gw[4 * k] = t.x;
            gw[4 * k + 1] = t.y;
            gw[4 * k + 2] = t.z;
            gw[4 * k + 3] = t.w;
          }
#pragma unroll
          for (int j = 0; j < kB; ++j) {
            const uint32_t g = gw[j];
            uint64_t gp;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(gp) : "r"(hdr + 8 + 8 * g) : "memory");
            gp += tofs;
            const uint32_t doit = (g != 0) & live;
            if constexpr (W == 1)
              asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.global.cs.u32 [%0], %1;\n}"
                           ::"l"(gp), "r"(acc[j].x[0]), "r"(doit) : "memory");
            else
              asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n @p st.global.cs.v2.u32 [%0], {%1, %2};\n}"
                           ::"l"(gp), "r"(acc[j].x[0]), "r"(acc[j].x[1]), "r"(doit) : "memory");
          }
        }
      }
      // the next tile's constant copies overwrite slots this tile's last batches read/stored
      // (in either stream)
      wait_st();
      pair_sync();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(base + 64 + 8 * hs) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kCols) : "memory");
}

struct Pool {
  bool two = false;  // two-stream code (8 consumer warps)
  uint32_t *code = nullptr;
  int64_t *off = nullptr;
  Layout y;
};
std::mutex g_mu;
std::map<std::tuple<int, int, int, int, std::vector<const Program *>>, Pool> g_pools;  // (dev, S, W, CW, progs)

std::mutex g_smu;
std::map<const Program *, std::shared_ptr<const TSched>> g_scheds;

std::shared_ptr<const TSched> sched_of(const Program *p) {
  {
    std::lock_guard<std::mutex> g(g_smu);
    auto it = g_scheds.find(p);
    if (it != g_scheds.end()) return it->second;
  }
  auto sc = std::make_shared<const TSched>(build_tmem(p->slp));
  std::lock_guard<std::mutex> g(g_smu);
  return g_scheds.emplace(p, sc).first->second;
}

std::map<const Program *, std::shared_ptr<const TStreams>> g_streams;

// the two-stream schedule of a program (nullptr: the program has no stream programs)
std::shared_ptr<const TStreams> streams_of(const Program *p) {
  if (p->streams.size() != 2) return nullptr;
  {
    std::lock_guard<std::mutex> g(g_smu);
    auto it = g_streams.find(p);
    if (it != g_streams.end()) return it->second;
  }
  auto t = std::make_shared<const TStreams>(build_streams(*p));
  std::lock_guard<std::mutex> g(g_smu);
  return g_streams.emplace(p, t).first->second;
}

// schedules of a program set, built on all host cores: single-stream, and two-stream if `two`
void scheds_of(const Program *const *progs, int np, bool two, std::vector<std::shared_ptr<const TSched>> &out,
               std::vector<std::shared_ptr<const TStreams>> &out2) {
  out.assign(np, nullptr);
  out2.assign(np, nullptr);
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex em;
  auto work = [&]() {
    for (int i; (i = next++) < np;) {
      try {
        out[i] = sched_of(progs[i]);
        if (two) out2[i] = streams_of(progs[i]);
      } catch (...) {
        std::lock_guard<std::mutex> g(em);
        if (!err) err = std::current_exception();
      }
    }
  };
  const int nt = std::min<int>(np, std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::thread> ts;
  for (int t = 1; t < nt; ++t) ts.emplace_back(work);
  work();
  for (auto &t : ts) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace tmem

// Dump form 5: the TMEM interpreter's schedule in its compact form; form 6: the device code the
// kernel runs (both with W = 1: columns = slots).
std::vector<uint32_t> interp_tmem_dump(const Program *p, int form) {
  if (form == 7) {  // the two-stream device code
    auto t = tmem::streams_of(p);
    if (!t) throw Error(XSLP_EINVAL, "the program has no TMEM interpreter streams");
    return tmem::emit_streams(*t, 1);
  }
  return form == 5 ? tmem::emit_code(*tmem::sched_of(p), 1) : tmem::emit_device(*tmem::sched_of(p), 1);
}

void drop_tmem_of(const Program *p) {
  using namespace tmem;
  {
    std::lock_guard<std::mutex> g(g_smu);
    g_scheds.erase(p);
    g_streams.erase(p);
  }
  std::lock_guard<std::mutex> g(g_mu);
  for (auto it = g_pools.begin(); it != g_pools.end();) {
    const auto &progs = std::get<4>(it->first);
    if (std::find(progs.begin(), progs.end(), p) != progs.end()) {
      int cur = -1;
      const bool have = cudaGetDevice(&cur) == cudaSuccess;
      cudaSetDevice(std::get<0>(it->first));
      cudaFree(it->second.code);
      cudaFree(it->second.off);
      if (have) cudaSetDevice(cur);
      it = g_pools.erase(it);
    } else {
      ++it;
    }
  }
}

namespace tmem {
using KFn = void (*)(Args);
template <int W, int CW, int B>
const void *kfn() { return (const void *)(KFn)xslp_interp_tmem<W, CW, B>; }
template <int B>
const void *kernel_b(int W, int CW) {
  if constexpr (B == 16)
    if (CW == 8) return W == 2 ? kfn<2, 8, 16>() : kfn<1, 8, 16>();
  return W == 2 ? kfn<2, 4, B>() : kfn<1, 4, B>();
}
const void *kernel_of(int W, int CW, int B) {
  return B == 4 ? kernel_b<4>(W, CW) : B == 8 ? kernel_b<8>(W, CW) : B == 12 ? kernel_b<12>(W, CW) : kernel_b<16>(W, CW);
}
}  // namespace tmem

static bool tmem_finish_plan(int dev) {
  using namespace tmem;
  static std::mutex am;
  static std::map<int, bool> attr;
  std::lock_guard<std::mutex> g(am);
  if (!attr[dev]) {
    for (int W : {1, 2})
      for (int B : {4, 8, 12, 16})
        for (int CW : {4, 8})
          CUDA_OK(cudaFuncSetAttribute(kernel_of(W, CW, B), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    attr[dev] = true;
  }
  return true;
}

// Words per thread: the largest of {want, 1} whose TMEM slots (512 columns per lane) and
// shared-memory stages fit; 0 if neither fits.
static int tmem_words(int nc, int nslots, int S, int CW, int capw, int want) {
  using namespace tmem;
  for (int W : {2, 1}) {
    if (W > want) continue;
    if (nslots * W > kCols) continue;
    Layout y;
    y.W = W;
    y.CW = CW;
    y.S = S;
    y.NC = std::max(1, nc);
    y.capw = capw;
    if (layout_smem(y) <= 227 * 1024) return W;
  }
  return 0;
}

// The code pool and layout of a program set for strips of B/8 bytes on the current device;
// false if the TMEM interpreter does not apply (strip % 16, > 32 output blocks, or the slots /
// rows do not fit).  Four consumer warps (one per TMEM lane quarter, each with all 512 columns),
// or eight running the program's two goal-half streams.
static bool tmem_plan(const Program *const *progs, int np, size_t B, tmem::Pool &pool) {
  using namespace tmem;
  const xslp_opts &o = progs[0]->opts;
  const uint64_t strip = B / 8;
  if (strip % 16 || progs[0]->n_goals / 8 > 32) return false;
  const int S = std::max(1, std::min(4, o.stages));
  // two streams (8 consumer warps) when every program has stream programs and they fit at
  // least as many words per thread as the single stream
  bool try2 = streams_wanted() && batch_size() == 16;
  for (int i = 0; i < np && try2; ++i) try2 = progs[i]->streams.size() == 2;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  const int want = 2;  // 2 words per thread when they fit (tmem_words), else 1
  std::vector<const Program *> key(progs, progs + np);
  const auto k = std::make_tuple(dev, S, want, try2 ? 8 : 4, key);
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_pools.find(k);
    if (it != g_pools.end()) {
      pool = it->second;
      return tmem_finish_plan(dev);
    }
  }
  std::vector<std::shared_ptr<const TSched>> sc;
  std::vector<std::shared_ptr<const TStreams>> sc2;
  try {
    scheds_of(progs, np, try2, sc, sc2);
  } catch (const Error &) {
    return false;
  }
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_pools.find(k);
  if (it != g_pools.end()) {
    pool = it->second;
    return tmem_finish_plan(dev);
  }
  int nc = 1, ns = 0, cw = 0;
  for (int i = 0; i < np; ++i) {
    nc = std::max<int>(nc, (int)sc[i]->consts.size());
    ns = std::max(ns, sc[i]->nslots);
    cw = std::max(cw, device_words(*sc[i]));
  }
  Layout y;
  y.S = S;
  y.CW = 4;
  y.NC = nc;
  y.B = sc[0]->B;
  y.capw = (cw + 3) / 4 * 4;
  y.W = tmem_words(nc, ns, S, 4, y.capw, want);
  bool two = false;
  if (try2) {
    int nc2 = 1, ns2 = 0, cw2 = 0;
    for (int i = 0; i < np; ++i) {
      nc2 = std::max<int>(nc2, (int)sc2[i]->consts.size());
      ns2 = std::max(ns2, sc2[i]->nslots);
      cw2 = std::max(cw2, device_words(*sc2[i]));
    }
    const int capw2 = (cw2 + 3) / 4 * 4;
    const int W2 = tmem_words(nc2, ns2, S, 8, capw2, want);
    if (W2 > 0 && W2 >= y.W) {
      two = true;
      y.CW = 8;
      y.NC = nc2;
      y.capw = capw2;
      y.W = W2;
    }
  }
  if (y.W == 0) return false;
  layout_smem(y);
  std::vector<uint32_t> all;
  std::vector<int64_t> off;
  for (int i = 0; i < np; ++i) {
    off.push_back((int64_t)all.size());
    auto w = two ? emit_streams(*sc2[i], y.W) : emit_device(*sc[i], y.W);
    all.insert(all.end(), w.begin(), w.end());
  }
  Pool P;
  P.y = y;
  P.two = two;
  CUDA_OK(cudaMalloc(&P.code, all.size() * 4));
  CUDA_OK(cudaMemcpy(P.code, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMalloc(&P.off, off.size() * 8));
  CUDA_OK(cudaMemcpy(P.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  g_pools[k] = P;
  pool = P;
  return tmem_finish_plan(dev);
}

bool interp_tmem_prepare(const Program *p, size_t B) {
  const Program *ps[1] = {p};
  tmem::Pool pool;
  return tmem_plan(ps, 1, B, pool);
}

bool interp_tmem_launch(const Program *const *progs, int np, const int32_t *d_pos,
                        const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                        int nstripes, size_t B, cudaStream_t st) {
  using namespace tmem;
  if (!in || !out || nstripes <= 0) return false;
  Pool pool;
  if (!tmem_plan(progs, np, B, pool)) return false;
  const Layout &y = pool.y;
  Args a{};
  a.code = pool.code;
  a.prog_off = pool.off;
  a.prog_of_stripe = d_pos;
  a.ids = d_ids;
  a.in_tbl = in;
  a.out_tbl = out;
  a.strip = B / 8;
  a.words = (uint32_t)(a.strip / 4);
  a.tpos = (uint32_t)(128 * y.W);
  a.tps = (a.words + a.tpos - 1) / a.tpos;
  if ((uint64_t)a.tps * nstripes > 0xffffffffull) throw Error(XSLP_EINVAL, "too many tiles");
  a.ntiles = a.tps * (uint32_t)nstripes;
  a.n_in = progs[0]->n_const / 8;
  a.n_out = progs[0]->n_goals / 8;
  a.S = y.S;
  a.nprogs = np;
  a.code0 = y.code0;
  a.capw = (uint32_t)y.capw;
  a.const0 = y.const0;
  a.RB = y.RB;
  a.NC = (uint32_t)y.NC;
  int dev = 0, sms = 148;
  CUDA_OK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<uint64_t>(a.ntiles, (uint64_t)sms);
  void *args[] = {&a};
  CUDA_OK(cudaLaunchKernel(kernel_of(y.W, y.CW, y.B), dim3(grid), dim3(y.CW * 32 + kNP * 32), args, y.smem, st));
  count_launch();
  return true;
}

}  // namespace xslp
