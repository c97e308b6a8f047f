// Generic SLP interpreter, pipelined (the paper's "interpreter style", on B200).
// Used for batched interpreter launches (xslp_encode_batch / xslp_decode_batch_multi when no
// straight-line kernel runs); single-stripe calls keep the one-tile xslp_interp_kernel.
//
// One kernel runs ANY compiled program from a host-built micro-op code -- no JIT -- and one
// launch can run a different program per stripe.  Work layout is the PIPE kernel's: persistent
// CTAs, each walking a contiguous run of tiles (a tile = T*L consecutive 32-bit words of every
// strip of one stripe); a producer warp streams each tile's constant strips by TMA
// (cp.async.bulk + mbarrier full/empty ring of S stages) while T consumer threads, L words
// each, run the program over the previous stage.
//
// Shared memory (one CTA per SM):
//   [0,128) barriers | S tile headers | S code buffers | variable rows | S x NC constant rows
// A "row" holds T*L words, thread t owning words t*L..t*L+L-1.  Constants are TMA'd into the
// stage's constant rows; SLP variables live in ONE set of variable rows shared by all stages
// (a thread only ever touches its own column, and the tiles of a CTA run one after another),
// so the footprint is S*NC + V rows instead of S*(NC + V).  Row 0 of the variable rows is the
// zero row that pads short operand lists.
//
// Code: the program's instructions (P:803-818 MultiSLP, in the compiler's DFS order,
// P:1279-1303) become micro-ops (mops) of exactly four operands XORed into an accumulator
// (arity a -> ceil(a/4) mops; 3-input XORs in LOP3), executed in PAIRS: a consumer issues the
// eight shared-memory operand loads of a pair back to back, then computes and stores both.
// The host schedules the mops so the second of a pair never reads the variable the first one
// stores (list scheduling over the SSA dependences, falling back to a no-op), then assigns
// variable rows by liveness at pair granularity.  Operand addresses are pre-baked byte offsets
// (constant rows of stage s differ per stage, so the code holds S variants; the producer copies
// a stage's variant into that stage's code buffer with the tile whenever the program changes),
// so an operand costs one add and one load.  The consumer prefetches the next pair's mops while
// the current pair's loads are in flight.
#include <cuda_runtime.h>

#include <algorithm>
#include <set>

#include "xslp_api.h"

namespace xslp {

void count_launch();  // device.cu

// ---- host: micro-op schedule ---------------------------------------------------------------
namespace {

// operand term of a mop: constant c (>= 0), variable v (-(v + 2)), zero row (-1)
struct Mop {
  int op[4] = {-1, -1, -1, -1};
  int flags = 0;     // 1 = reset the accumulator first, 2 = store to dst var, 4 = store goal
  int dst = -1;      // variable stored (flags & 2)
  int goal = -1;     // goal index stored (flags & 4)
};

struct Sched {
  std::vector<Mop> mops;          // even length: pairs (2k, 2k+1)
  std::vector<int> consts;        // constant row r holds constant consts[r]
  std::vector<int> crow;          // constant -> row (or -1)
  std::vector<int> vrow;          // variable -> variable row (1-based; row 0 = zero row)
  int nvrows = 1;                 // variable rows including the zero row
};

Sched schedule_pairs(const Slp &s) {
  const int nc = s.n_const, nv = s.n_vars;
  // defining instruction of each variable, and the goals each term feeds
  std::vector<int> def(nv, -1);
  for (size_t k = 0; k < s.ins.size(); ++k) def[s.ins[k].var] = (int)k;
  std::vector<std::vector<int>> goals_of_var(nv), goals_of_const(nc);
  std::vector<int> zero_goals;
  for (size_t g = 0; g < s.goal.size(); ++g) {
    const int t = s.goal[g];
    if (t < 0) zero_goals.push_back((int)g);
    else if (t < nc) goals_of_const[t].push_back((int)g);
    else goals_of_var[t - nc].push_back((int)g);
  }
  // live instructions (backwards): a variable is needed if it is a goal or a needed
  // instruction reads it; var_used = read by a needed instruction
  std::vector<char> needed(nv, 0), var_used(nv, 0);
  for (int v = 0; v < nv; ++v) needed[v] = !goals_of_var[v].empty();
  for (size_t k = s.ins.size(); k-- > 0;) {
    if (!needed[s.ins[k].var]) continue;
    for (int t : s.ins[k].ops)
      if (t >= nc) needed[t - nc] = var_used[t - nc] = 1;
  }
  // units: a run of mops that must stay consecutive (the accumulator flows through them)
  struct Unit {
    std::vector<Mop> mops;
    std::vector<int> deps;   // variables read
    int stores = -1;         // variable stored by the last operand mop
  };
  std::vector<Unit> units;
  auto make = [&](const std::vector<int> &ops, int dstvar, const std::vector<int> &goals) {
    Unit u;
    const int chunks = std::max<int>(1, ((int)ops.size() + 3) / 4);
    for (int c = 0; c < chunks; ++c) {
      Mop m;
      for (int q = 0; q < 4; ++q) {
        const size_t i = 4 * (size_t)c + q;
        if (i < ops.size()) m.op[q] = ops[i] < nc ? ops[i] : -(ops[i] - nc + 2);
      }
      if (c == 0) m.flags |= 1;
      if (c == chunks - 1) {
        if (dstvar >= 0) { m.flags |= 2; m.dst = dstvar; }
        if (!goals.empty()) { m.flags |= 4; m.goal = goals[0]; }
      }
      u.mops.push_back(m);
    }
    for (size_t g = 1; g < goals.size(); ++g) {  // extra goals of the same value
      Mop m;
      m.flags = 4;
      m.goal = goals[g];
      u.mops.push_back(m);
    }
    for (int t : ops)
      if (t >= nc) u.deps.push_back(t - nc);
    u.stores = dstvar;
    units.push_back(std::move(u));
  };
  if (!zero_goals.empty()) make({}, -1, zero_goals);
  for (int c = 0; c < nc; ++c)
    if (!goals_of_const[c].empty()) make({c}, -1, goals_of_const[c]);
  std::vector<int> unit_of_var(nv, -1);
  for (size_t k = 0; k < s.ins.size(); ++k) {
    const int v = s.ins[k].var;
    const bool keep = var_used[v];
    if (!needed[v]) continue;  // dead instruction
    make(s.ins[k].ops, keep ? v : -1, goals_of_var[v]);
    unit_of_var[v] = (int)units.size() - 1;
  }
  // list scheduling: the earliest (compiler order) ready unit none of whose mops reads a
  // variable stored by a mop of its own pair or of the pair before -- the consumer issues the
  // operand loads of pair k+1 before it computes and stores pair k (software pipelining), and
  // those of both mops of a pair before either stores; a no-op when nothing fits
  Sched out;
  std::vector<int> stored_at;  // per position: variable stored there, or -1
  std::vector<char> placed(units.size(), 0);
  std::vector<char> var_done(nv, 0);
  size_t first_open = 0, nplaced = 0;
  const size_t kWindow = 64;
  auto ready = [&](const Unit &u) {
    for (int v : u.deps)
      if (!var_done[v]) return false;
    return true;
  };
  auto reads = [&](const Mop &m, int v) {
    for (int q = 0; q < 4; ++q)
      if (m.op[q] == -(v + 2)) return true;
    return false;
  };
  auto window_lo = [](size_t pos) { return pos >= 2 ? 2 * (pos / 2 - 1) : 0; };
  auto conflict = [&](const Unit &u) {
    const size_t P = out.mops.size();
    for (size_t j = 0; j < u.mops.size(); ++j)
      for (size_t q = window_lo(P + j); q < P; ++q)  // the unit's own mops store only last
        if (stored_at[q] >= 0 && reads(u.mops[j], stored_at[q])) return true;
    return false;
  };
  while (nplaced < units.size()) {
    while (first_open < units.size() && placed[first_open]) ++first_open;
    int pick = -1;
    for (size_t i = first_open, seen = 0; i < units.size() && seen < kWindow; ++i) {
      if (placed[i]) continue;
      ++seen;
      if (!ready(units[i]) || conflict(units[i])) continue;
      pick = (int)i;
      break;
    }
    if (pick < 0) {
      out.mops.push_back(Mop{});  // no-op: no operands, no flags
      stored_at.push_back(-1);
      continue;
    }
    for (auto &m : units[pick].mops) {
      out.mops.push_back(m);
      stored_at.push_back(m.flags & 2 ? m.dst : -1);
    }
    placed[pick] = 1;
    ++nplaced;
    if (units[pick].stores >= 0) var_done[units[pick].stores] = 1;
  }
  while (out.mops.size() % 6) {  // a multiple of 3 pairs (the consumer runs three per iteration)
    out.mops.push_back(Mop{});
    stored_at.push_back(-1);
  }
  // hazard check (the property the kernel relies on)
  for (size_t i = 0; i < out.mops.size(); ++i)
    for (size_t q = window_lo(i); q < i; ++q)
      if (stored_at[q] >= 0 && reads(out.mops[i], stored_at[q]))
        throw Error(XSLP_EINVAL, "interpreter schedule: pipeline hazard");
  // constant rows: in order of first use
  out.crow.assign(nc, -1);
  for (auto &m : out.mops)
    for (int q = 0; q < 4; ++q)
      if (m.op[q] >= 0 && out.crow[m.op[q]] < 0) {
        out.crow[m.op[q]] = (int)out.consts.size();
        out.consts.push_back(m.op[q]);
      }
  // variable rows by liveness, per pair: pair k's stores happen after the loads of pairs k and
  // k+1, and pair k+1 reads nothing stored or last read in pair k... so rows whose last read is
  // in pair k are free for pair k's stores (rows read later are still held)
  std::vector<int> last_pair(nv, -1);
  for (size_t i = 0; i < out.mops.size(); ++i)
    for (int q = 0; q < 4; ++q)
      if (out.mops[i].op[q] < -1) last_pair[-out.mops[i].op[q] - 2] = (int)(i / 2);
  out.vrow.assign(nv, -1);
  std::set<int> free_rows;
  int next = 1;  // row 0 is the zero row (empty operand slots 0/1 read it)
  for (size_t p = 0; p < out.mops.size() / 2; ++p) {
    for (int h = 0; h < 2; ++h) {
      const Mop &m = out.mops[2 * p + h];
      for (int q = 0; q < 4; ++q)
        if (m.op[q] < -1) {
          const int v = -m.op[q] - 2;
          if (out.vrow[v] < 0) throw Error(XSLP_EINVAL, "interpreter schedule: read before store");
          if (last_pair[v] == (int)p && out.vrow[v] < (1 << 30)) {
            free_rows.insert(out.vrow[v]);
            out.vrow[v] = 1 << 30;   // released
          }
        }
    }
    for (int h = 0; h < 2; ++h) {
      const Mop &m = out.mops[2 * p + h];
      if (!(m.flags & 2)) continue;
      int r;
      if (!free_rows.empty()) { r = *free_rows.begin(); free_rows.erase(free_rows.begin()); }
      else r = next++;
      out.vrow[m.dst] = r;
    }
  }
  out.nvrows = next;
  return out;
}

struct Layout {
  int T = 0, L = 1, S = 2, NC = 0, V = 0, capw = 0;
  uint32_t code0 = 0, var0 = 0, const0 = 0, RB = 0;
  size_t smem = 0;
};

constexpr int kHdr = 16 + 8 * 32;  // per-stage tile header: stripe, prog, pad, up to 32 output ptrs
constexpr int kPairWords = 12, kHeadWords = 8, kSlackPairs = 2;

size_t layout_smem(Layout &y) {
  y.RB = (uint32_t)y.T * y.L * 4;
  y.code0 = 128 + y.S * kHdr;                                  // 16-byte aligned (kHdr = 17*16)
  size_t var0 = y.code0 + (size_t)y.S * y.capw * 4;
  var0 = (var0 + 127) / 128 * 128;
  y.var0 = (uint32_t)var0;
  y.const0 = (uint32_t)(var0 + (size_t)y.V * y.RB);
  y.smem = (size_t)y.const0 + (size_t)y.S * y.NC * y.RB;
  return y.smem;
}

// One code variant (stage st): header, pairs (+ kSlackPairs empty pairs, so the consumer's
// prefetch two pairs ahead reads valid empty code), then the producer's load list.
//   [0] nloads [1] npairs [2] words of this variant [3] variable rows (incl. the zero row 0)
//   [4] row bytes [5] variable rows offset [6] this stage's constant rows offset [7] 8
//   pair: 12 words = A's 4 operand offsets, B's 4 operand offsets, A.dst, A.ctl, B.dst, B.ctl
//     operand slots 0 and 1 are always loaded (an empty one names the zero row); slots 2 and 3
//     only with the HI flag (then an empty slot 3 names the zero row)
//     ctl = flags << 24 | (goal & 7) << 16 | header offset of the goal's block pointer;
//     flags: 1 reset acc, 2 store to dst, 4 store goal, 8 HI (slots 2 and 3 present)
//   loads: nloads x (constant index, byte offset of its row)
// Offsets are from the start of dynamic shared memory; the consumer adds its column.
std::vector<uint32_t> emit_variant(const Slp &s, const Sched &sc, const Layout &y, int st) {
  const uint32_t cst = y.const0 + (uint32_t)st * y.NC * y.RB;
  std::vector<uint32_t> w(kHeadWords, 0);
  w[0] = (uint32_t)sc.consts.size();
  w[1] = (uint32_t)(sc.mops.size() / 2);
  w[3] = (uint32_t)sc.nvrows;
  w[4] = y.RB;
  w[5] = y.var0;
  w[6] = cst;
  w[7] = kHeadWords;
  // replay the row allocation of schedule_pairs to know each variable's row at each use
  const int nv = s.n_vars;
  std::vector<int> last_pair(nv, -1), row(nv, -1);
  for (size_t i = 0; i < sc.mops.size(); ++i)
    for (int q = 0; q < 4; ++q)
      if (sc.mops[i].op[q] < -1) last_pair[-sc.mops[i].op[q] - 2] = (int)(i / 2);
  std::set<int> free_rows;
  int next = 1;
  auto off_of = [&](int t) -> uint32_t {
    if (t >= 0) return cst + (uint32_t)sc.crow[t] * y.RB;
    if (t == -1) return y.var0;  // the zero row
    return y.var0 + (uint32_t)row[-t - 2] * y.RB;
  };
  for (size_t p = 0; p < sc.mops.size() / 2; ++p) {
    uint32_t ops[2][4], dst[2], ctl[2];
    for (int h = 0; h < 2; ++h) {
      const Mop &m = sc.mops[2 * p + h];
      const bool hi = m.op[2] != -1 || m.op[3] != -1;
      for (int q = 0; q < 4; ++q) ops[h][q] = q < 2 || hi ? off_of(m.op[q]) : 0u;
    }
    for (int h = 0; h < 2; ++h)
      for (int q = 0; q < 4; ++q) {
        const int t = sc.mops[2 * p + h].op[q];
        if (t < -1 && last_pair[-t - 2] == (int)p && row[-t - 2] < (1 << 30)) {
          free_rows.insert(row[-t - 2]);
          row[-t - 2] = 1 << 30;
        }
      }
    for (int h = 0; h < 2; ++h) {
      const Mop &m = sc.mops[2 * p + h];
      uint32_t flags = (uint32_t)m.flags;
      if (m.op[2] != -1 || m.op[3] != -1) flags |= 8;
      dst[h] = 0;
      if (m.flags & 2) {
        int r;
        if (!free_rows.empty()) { r = *free_rows.begin(); free_rows.erase(free_rows.begin()); }
        else r = next++;
        row[m.dst] = r;
        dst[h] = y.var0 + (uint32_t)r * y.RB;
      }
      ctl[h] = flags << 24;
      if (m.flags & 4) ctl[h] |= (uint32_t)(16 + 8 * (m.goal >> 3)) | ((uint32_t)(m.goal & 7) << 16);
    }
    w.insert(w.end(), {ops[0][0], ops[0][1], ops[0][2], ops[0][3], ops[1][0], ops[1][1],
                       ops[1][2], ops[1][3], dst[0], ctl[0], dst[1], ctl[1]});
  }
  if (next != sc.nvrows) throw Error(XSLP_EINVAL, "interpreter code: row replay mismatch");
  // slack pairs: operand slots 0/1 name the zero row, so prefetched loads stay in bounds
  for (int k = 0; k < kSlackPairs; ++k)
    w.insert(w.end(), {y.var0, y.var0, 0u, 0u, y.var0, y.var0, 0u, 0u, 0u, 0u, 0u, 0u});
  for (size_t r = 0; r < sc.consts.size(); ++r) {
    w.push_back((uint32_t)sc.consts[r]);
    w.push_back(cst + (uint32_t)r * y.RB);
  }
  while (w.size() % 8) w.push_back(0);
  w[2] = (uint32_t)w.size();
  return w;
}

// words the consumers need in shared memory: header + pairs + the empty slack pairs
inline int consumer_words(const Sched &sc) {
  return kHeadWords + kPairWords * ((int)sc.mops.size() / 2 + kSlackPairs);
}

}  // namespace

// Dump form 3: the stage-0 code variant for this program alone at T = opts.threads,
// L = opts.lane_words, S = opts.stages (clamped to the kernel's 1..4).
std::vector<uint32_t> interp_code_dump(const Slp &s, int T, int L, int S) {
  Sched sc = schedule_pairs(s);
  Layout y;
  y.T = T;
  y.L = L;
  y.S = std::max(1, std::min(4, S));
  y.NC = std::max<int>(1, (int)sc.consts.size());
  y.V = sc.nvrows;
  y.capw = (consumer_words(sc) + 3) / 4 * 4;
  layout_smem(y);
  return emit_variant(s, sc, y, 0);
}

struct InterpArgs {
  const uint32_t *code;          // code pool: per program, S variants of code words
  const int64_t *prog_off;       // word offset of each program's variant 0 in the pool
  const int32_t *prog_of_stripe; // nullable: program 0 for every stripe
  const int32_t *ids;            // nullable: tile stripe = ids[entry]
  const uint8_t *const *in_tbl;
  uint8_t *const *out_tbl;
  uint64_t strip;
  uint32_t words, tps, ntiles;   // words = strip / 4; tps = tiles per stripe (T*L words each)
  int32_t n_in, n_out, S, nprogs;
  uint32_t code0, capw;          // code buffers: code0 + st * capw * 4
  uint32_t var0, RB;             // variable rows, row bytes
};

__device__ __forceinline__ uint32_t sm_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}

// L consecutive 32-bit words of one row, as one shared-memory access
template <int L> struct Vec;
template <> struct Vec<1> {
  uint32_t x;
  __device__ void zero() { x = 0; }
};
template <> struct Vec<2> {
  uint2 x;
  __device__ void zero() { x = make_uint2(0, 0); }
};
template <> struct Vec<4> {
  uint4 x;
  __device__ void zero() { x = make_uint4(0, 0, 0, 0); }
};
__device__ __forceinline__ uint32_t vxor3(uint32_t a, uint32_t b, uint32_t c) { return xor3(a, b, c); }
__device__ __forceinline__ uint2 vxor3(uint2 a, uint2 b, uint2 c) {
  return make_uint2(xor3(a.x, b.x, c.x), xor3(a.y, b.y, c.y));
}
__device__ __forceinline__ uint4 vxor3(uint4 a, uint4 b, uint4 c) {
  return make_uint4(xor3(a.x, b.x, c.x), xor3(a.y, b.y, c.y), xor3(a.z, b.z, c.z), xor3(a.w, b.w, c.w));
}
// predicated shared-memory load of L words at 32-bit shared address a (v untouched when !p)
__device__ __forceinline__ void lds_if(uint32_t a, bool p, Vec<1> &v) {
  if (p) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v.x) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds_if(uint32_t a, bool p, Vec<2> &v) {
  if (p) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x.x), "=r"(v.x.y) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds_if(uint32_t a, bool p, Vec<4> &v) {
  if (p)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x.x), "=r"(v.x.y), "=r"(v.x.z), "=r"(v.x.w) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, const Vec<1> &v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v.x) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, const Vec<2> &v) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x.x), "r"(v.x.y) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, const Vec<4> &v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x.x), "r"(v.x.y),
               "r"(v.x.z), "r"(v.x.w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// a pair's code: A's operands, B's operands, (A.df, A.gsel, B.df, B.gsel)
struct PairCode {
  uint4 a, b, f;
};
__device__ __forceinline__ PairCode fetch_pair(uint32_t a) {
  return PairCode{lds128(a), lds128(a + 16), lds128(a + 32)};
}
// the operands of a pair at this thread's column: slots 0/1 always, 2/3 with the HI flag
template <int L>
__device__ __forceinline__ void load_pair(uint32_t col, const PairCode &c, Vec<L> (&v)[8]) {
  lds_if(col + c.a.x, true, v[0]);
  lds_if(col + c.a.y, true, v[1]);
  lds_if(col + c.b.x, true, v[4]);
  lds_if(col + c.b.y, true, v[5]);
  const bool ha = (c.f.y >> 27) & 1, hb = (c.f.w >> 27) & 1;
  lds_if(col + c.a.z, ha, v[2]);
  lds_if(col + c.a.w, ha, v[3]);
  lds_if(col + c.b.z, hb, v[6]);
  lds_if(col + c.b.w, hb, v[7]);
}
template <int L>
__device__ __forceinline__ void st_goal(uint64_t p, const Vec<L> &v) {
  using T = decltype(v.x);
  __stcs(reinterpret_cast<T *>(p), v.x);
}
template <int L>
__device__ __forceinline__ void run_mop(Vec<L> &acc, const Vec<L> *v, uint32_t dst, uint32_t ctl,
                                        uint32_t col, uint32_t hdr, uint64_t strip, uint64_t off) {
  const uint32_t fl = ctl >> 24;
  Vec<L> x = acc;
  if (fl & 1) x.zero();
  x.x = vxor3(x.x, v[0].x, v[1].x);
  if (fl & 8) x.x = vxor3(x.x, v[2].x, v[3].x);
  acc = x;
  if (fl & 2) sts(col + dst, acc);
  if (fl & 4) {
    uint64_t p;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(p) : "r"(hdr + (ctl & 0xffffu)) : "memory");
    st_goal<L>(p + (uint64_t)((ctl >> 16) & 7) * strip + off, acc);
  }
}
template <int L>
__device__ __forceinline__ void run_pair(Vec<L> &acc, const Vec<L> (&v)[8], const PairCode &c,
                                         uint32_t col, uint32_t hdr, uint64_t strip, uint64_t off) {
  run_mop<L>(acc, v, c.f.x, c.f.y, col, hdr, strip, off);
  run_mop<L>(acc, v + 4, c.f.z, c.f.w, col, hdr, strip, off);
}

template <int L>
__global__ void __launch_bounds__(512, 1) xslp_interp_pipe(InterpArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t T = blockDim.x - 32, tid = threadIdx.x;
  const int S = a.S;
  const uint32_t base = sm_addr(sm);
  const uint32_t hdr0 = base + 128;  // S tile headers
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(base + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 64 + 8 * k), "r"(T / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < T) {  // the zero row (row 0 of the variable rows), this thread's column
    Vec<L> z;
    z.zero();
    sts(base + a.var0 + tid * 4 * L, z);
  }
  __syncthreads();
  // contiguous tile run of this CTA
  const uint32_t chunk = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * chunk, t1 = min(a.ntiles, t0 + chunk);
  if (tid >= T) {  // ---------------- producer warp
    // All 32 lanes issue: lane i copies constant rows i, i+32, ... so the dependent global
    // reads of each copy's source (load list entry, then the block pointer) overlap across
    // lanes instead of serialising ~2 cache round trips per row in one thread.
    const uint32_t pl = tid - T;
    int cur[4] = {-1, -1, -1, -1};  // program whose code sits in each stage's code buffer
    for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
      const uint32_t st = it % S, ph = (it / S) & 1;
      const uint32_t entry = tile / a.tps, tw = tile % a.tps;
      const uint32_t stripe = a.ids ? (uint32_t)a.ids[entry] : entry;
      const int prog = a.prog_of_stripe ? a.prog_of_stripe[stripe] : 0;
      if (prog < 0 || prog >= a.nprogs) asm volatile("trap;");
      const uint32_t *pc0 = a.code + a.prog_off[prog];
      const uint32_t *pc = pc0 + (size_t)st * pc0[2];  // this stage's variant
      const uint8_t *const *in = a.in_tbl + (size_t)stripe * a.n_in;
      uint8_t *const *out = a.out_tbl + (size_t)stripe * a.n_out;
      const uint32_t nl = pc[0], np = pc[1];
      const uint32_t *ld = pc + kHeadWords + kPairWords * (np + kSlackPairs);
      // this lane's first two copies' sources, fetched before the wait for the stage
      const size_t toff = (size_t)tw * T * L * 4;
      const uint8_t *src0 = nullptr, *src1 = nullptr;
      uint32_t dst0 = 0, dst1 = 0;
      if (pl < nl) {
        const uint32_t c = ld[2 * pl];
        dst0 = ld[2 * pl + 1];
        src0 = in[c >> 3] + (c & 7) * a.strip + toff;
      }
      if (pl + 32 < nl) {
        const uint32_t c = ld[2 * (pl + 32)];
        dst1 = ld[2 * (pl + 32) + 1];
        src1 = in[c >> 3] + (c & 7) * a.strip + toff;
      }
      const uint64_t optr = pl < (uint32_t)a.n_out ? (uint64_t)out[pl] : 0;
      if (it >= (uint32_t)S)
        while (!try_wait(base + 64 + 8 * st, ph ^ 1)) __nanosleep(64);  // keep issue slots free
      const uint32_t h = hdr0 + st * kHdr;
      if (pl < (uint32_t)a.n_out) asm volatile("st.shared.u64 [%0], %1;" ::"r"(h + 16 + 8 * pl), "l"(optr) : "memory");
      const uint32_t nb = min(T * L, a.words - tw * T * L) * 4;
      const uint32_t cbytes = cur[st] != prog ? (kHeadWords + kPairWords * (np + kSlackPairs)) * 4 : 0;
      cur[st] = prog;
      __syncwarp();  // header stores of every lane before lane 0's arrive (release)
      if (pl == 0) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(h), "r"(stripe) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(h + 4), "r"((uint32_t)prog) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(base + 8 * st),
                     "r"(nb * nl + cbytes) : "memory");
        if (cbytes)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(base + a.code0 + st * a.capw * 4), "l"(pc), "r"(cbytes), "r"(base + 8 * st) : "memory");
      }
      __syncwarp();  // expect_tx before any complete_tx
      if (pl < nl)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(base + dst0), "l"(src0), "r"(nb), "r"(base + 8 * st) : "memory");
      if (pl + 32 < nl)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(base + dst1), "l"(src1), "r"(nb), "r"(base + 8 * st) : "memory");
      for (uint32_t i = pl + 64; i < nl; i += 32) {  // wide codes: more than 64 rows
        const uint32_t c = ld[2 * i], off = ld[2 * i + 1];
        const uint8_t *src = in[c >> 3] + (c & 7) * a.strip + toff;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(base + off), "l"(src), "r"(nb), "r"(base + 8 * st) : "memory");
      }
    }
    return;
  }
  // ---------------- consumers
  const uint32_t lane = tid & 31;
  const uint32_t col = base + tid * 4 * L;  // this thread's column of every row
  for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
    const uint32_t st = it % S, ph = (it / S) & 1;
    while (!try_wait(base + 8 * st, ph)) {
    }
    const uint32_t tw = tile % a.tps;
    const uint32_t w = tw * T * L + tid * L;
    if (w < a.words) {
      const uint32_t hdr = hdr0 + st * kHdr;
      const uint32_t cp = base + a.code0 + st * a.capw * 4;
      uint32_t np;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(np) : "r"(cp + 4) : "memory");
      const uint64_t off = (uint64_t)w * 4;
      uint32_t pc = cp + kHeadWords * 4;  // address of the next pair's code to fetch
      Vec<L> acc;
      acc.zero();
      // software pipeline (np is a multiple of 3, two empty pairs follow): the operands of
      // pair q+1 are loaded before pair q computes and stores, and the code of pair q+2 is
      // fetched before pair q computes; three register sets rotate with the 3x unrolled loop
      PairCode c0 = fetch_pair(pc), c1 = fetch_pair(pc + 48), c2;
      pc += 96;
      Vec<L> va[8], vb[8], vc[8];
      load_pair<L>(col, c0, va);
      for (uint32_t q = 0; q < np; q += 3) {
        load_pair<L>(col, c1, vb);
        c2 = fetch_pair(pc);
        run_pair<L>(acc, va, c0, col, hdr, a.strip, off);
        load_pair<L>(col, c2, vc);
        c0 = fetch_pair(pc + 48);
        run_pair<L>(acc, vb, c1, col, hdr, a.strip, off);
        load_pair<L>(col, c0, va);
        c1 = fetch_pair(pc + 96);
        pc += 144;
        run_pair<L>(acc, vc, c2, col, hdr, a.strip, off);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(base + 64 + 8 * st) : "memory");
  }
}

// ---- host launch -----------------------------------------------------------------------
struct CodePool {
  uint32_t *code = nullptr;
  int64_t *off = nullptr;
  Layout y;
};
static std::mutex g_pool_mu;
static std::map<std::tuple<int, int, int, int, std::vector<const Program *>>, CodePool> g_pools;

// Build (or find) the code pool of a program set for (T, L, S) on device `dev`: the layout is
// chosen from the largest program, T lowered until the shared memory fits.  False if no T fits.
static bool code_pool(const Program *const *progs, int np, int want_T, int L, int S, int dev,
                      CodePool &out) {
  std::vector<const Program *> key(progs, progs + np);
  std::lock_guard<std::mutex> g(g_pool_mu);
  auto it = g_pools.find({dev, want_T, L, S, key});
  if (it != g_pools.end()) {
    out = it->second;
    return true;
  }
  std::vector<Sched> sc(np);
  Layout y;
  y.L = L;
  y.S = S;
  int cw = 0;
  for (int i = 0; i < np; ++i) {
    sc[i] = schedule_pairs(progs[i]->slp);
    y.NC = std::max<int>(y.NC, (int)sc[i].consts.size());
    y.V = std::max(y.V, sc[i].nvrows);
    cw = std::max(cw, consumer_words(sc[i]));
  }
  y.NC = std::max(1, y.NC);
  y.capw = (cw + 3) / 4 * 4;
  int T = std::min(480, std::max(32, want_T / 32 * 32));  // + the producer warp <= 512
  for (; T >= 32; T -= 32) {
    y.T = T;
    if (layout_smem(y) <= 227 * 1024) break;
  }
  if (T < 32) return false;
  std::vector<uint32_t> all;
  std::vector<int64_t> off;
  for (int i = 0; i < np; ++i) {
    off.push_back((int64_t)all.size());
    for (int st = 0; st < S; ++st) {
      auto w = emit_variant(progs[i]->slp, sc[i], y, st);
      all.insert(all.end(), w.begin(), w.end());
    }
  }
  CodePool P;
  P.y = y;
  CUDA_OK(cudaMalloc(&P.code, all.size() * 4));
  CUDA_OK(cudaMemcpy(P.code, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMalloc(&P.off, off.size() * 8));
  CUDA_OK(cudaMemcpy(P.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  g_pools[{dev, want_T, L, S, key}] = P;
  out = P;
  return true;
}

// Programs are freed by their owners; a pool must not outlive a member program (a later
// program allocated at the same address would otherwise find it).  Called by ~Program.
void drop_code32_of(const Program *p) {
  std::lock_guard<std::mutex> g(g_pool_mu);
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

struct InterpPlan {
  CodePool pool;
  int grid_per_sm = 1;
  const void *fn = nullptr;
};

template <int L>
static const void *kernel_of() { return (const void *)xslp_interp_pipe<L>; }

// Everything a launch needs that is not capturable in a CUDA graph (pool allocation and upload,
// the function attribute, the occupancy query), done once per (programs, T, L, S, device).
static bool interp_pipe_plan(const Program *const *progs, int np, size_t B, InterpPlan &out) {
  const xslp_opts &o = progs[0]->opts;
  const int L = o.lane_words == 2 || o.lane_words == 4 ? o.lane_words : 1;
  const int S = std::max(1, std::min(4, o.stages));
  const uint64_t strip = B / 8;
  if (strip % 16 || strip % (4 * L) || progs[0]->n_goals / 8 > 32) return false;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  CodePool pool;
  if (!code_pool(progs, np, o.threads, L, S, dev, pool)) return false;
  const void *fn = L == 1 ? kernel_of<1>() : L == 2 ? kernel_of<2>() : kernel_of<4>();
  static std::mutex m;
  static std::map<std::pair<int, const void *>, bool> attr;
  static std::map<std::tuple<int, const void *, int, size_t>, int> occ;
  int per = 1;
  {
    std::lock_guard<std::mutex> g(m);
    if (!attr[{dev, fn}]) {
      CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr[{dev, fn}] = true;
    }
    auto key = std::make_tuple(dev, fn, pool.y.T, pool.y.smem);
    auto it = occ.find(key);
    if (it == occ.end()) {
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, pool.y.T + 32, pool.y.smem));
      occ[key] = std::max(1, per);
    }
    per = occ[key];
  }
  out.pool = pool;
  out.grid_per_sm = per;
  out.fn = fn;
  return true;
}

bool interp_lanes_prepare(const Program *p, size_t B);  // interp_lanes.cu

bool interp_tmem_prepare(const Program *p, size_t B);  // interp_tmem.cu

bool interp_pipe_prepare(const Program *p, size_t B) {
  if (p->opts.interp == XSLP_INTERP_LANES) return interp_lanes_prepare(p, B);
  if (p->opts.interp == XSLP_INTERP_TMEM)
    return interp_tmem_prepare(p, B) || interp_lanes_prepare(p, B);
  const Program *ps[1] = {p};
  InterpPlan plan;
  return interp_pipe_plan(ps, 1, B, plan);
}

bool interp_lanes_launch(const Program *const *progs, int np, const int32_t *d_pos,
                         const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                         int nstripes, size_t B, cudaStream_t st);  // interp_lanes.cu
bool interp_tmem_launch(const Program *const *progs, int np, const int32_t *d_pos,
                        const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                        int nstripes, size_t B, cudaStream_t st);  // interp_tmem.cu

bool interp_pipe_launch(const Program *const *progs, int np, const int32_t *d_pos,
                        const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                        int nstripes, size_t B, cudaStream_t st, int /*want_T: opts.threads*/) {
  if (!in || !out || nstripes <= 0) return false;
  if (progs[0]->opts.interp == XSLP_INTERP_LANES)
    return interp_lanes_launch(progs, np, d_pos, d_ids, in, out, nstripes, B, st);
  if (progs[0]->opts.interp == XSLP_INTERP_TMEM)  // the lane interpreter when TMEM does not fit
    return interp_tmem_launch(progs, np, d_pos, d_ids, in, out, nstripes, B, st) ||
           interp_lanes_launch(progs, np, d_pos, d_ids, in, out, nstripes, B, st);
  InterpPlan plan;
  if (!interp_pipe_plan(progs, np, B, plan)) return false;
  const Layout &y = plan.pool.y;
  InterpArgs a{};
  a.code = plan.pool.code;
  a.prog_off = plan.pool.off;
  a.prog_of_stripe = d_pos;
  a.ids = d_ids;
  a.in_tbl = in;
  a.out_tbl = out;
  a.strip = B / 8;
  a.words = (uint32_t)(a.strip / 4);
  a.tps = (a.words + y.T * y.L - 1) / (y.T * y.L);
  if ((uint64_t)a.tps * nstripes > 0xffffffffull) throw Error(XSLP_EINVAL, "too many tiles");
  a.ntiles = a.tps * (uint32_t)nstripes;
  a.n_in = progs[0]->n_const / 8;
  a.n_out = progs[0]->n_goals / 8;
  a.S = y.S;
  a.nprogs = np;
  a.code0 = y.code0;
  a.capw = (uint32_t)y.capw;
  a.var0 = y.var0;
  a.RB = y.RB;
  int dev = 0, sms = 148;
  CUDA_OK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<uint64_t>(a.ntiles, (uint64_t)sms * plan.grid_per_sm);
  void *args[] = {&a};
  CUDA_OK(cudaLaunchKernel(plan.fn, dim3(grid), dim3(y.T + 32), args, y.smem, st));
  count_launch();
  return true;
}

}  // namespace xslp
