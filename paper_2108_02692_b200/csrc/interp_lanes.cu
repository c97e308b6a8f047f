// Lane-parallel SLP interpreter (the paper's "interpreter style", organised for B200).
//
// The pipelined interpreter of interp.cu gives every thread its own data word and runs the
// micro-op stream warp-uniformly: every SLP operand then costs a warp-wide address add, load
// and code fetch for 32 words.  Here the roles are swapped: the 32 lanes of a warp run 32
// DIFFERENT instructions of the SLP (a "round" of mutually independent lane-ops) over the same
// four consecutive words ("quad", 16 bytes) of the tile, each lane reading its operands with
// 128-bit shared-memory loads.  One warp-wide load then moves 32 operands x 4 words, the
// per-lane code is a plain coalesced load, and -- the point -- the number of warps no longer
// depends on the positions held in shared memory: a tile of T_pos words (its constant and
// variable rows fill shared memory) is processed quad by quad by any number of warps.
//
// Host side (build_lanes): the scheduled SLP's instructions (P:803-818 MultiSLP, DFS order,
// P:1279-1303) become lane-ops of at most four operands (wider instructions split into a tree
// of partial XORs into temporaries), list-scheduled into rounds of <= 32 ops whose operands
// were all produced in earlier rounds (critical path first); variable rows are assigned by
// liveness at round granularity (every lane of a round loads before any lane stores, and a
// __syncwarp separates rounds).  Goals are stored straight to HBM by their lane (16 bytes).
//
// Shared memory: [0,128) barriers | S tile headers | S code buffers | variable rows |
// S x NC constant rows; a row is T_pos words + 16 bytes (rows start 16 bytes apart modulo 128,
// so the 8 lanes of a quarter-warp reading different rows at one column hit different banks
// when their rows differ modulo 8).  Constants are TMA'd into the stage's rows by a producer
// warp (cp.async.bulk + mbarrier full/empty ring), the code variant of the stage with them when
// the program changes.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <iterator>
#include <map>
#include <memory>
#include <set>
#include <thread>

#include "xslp_api.h"

namespace xslp {

void count_launch();  // device.cu

namespace lanes {

constexpr int kK = 4;                      // operands per lane-op
constexpr int kOpWords = 8;                // 4 operand offsets; dst, goal select, ctl, 0
constexpr int kRoundWords = 32 * kOpWords; // one round of 32 lane-ops (1 KB)
constexpr int kHead = 8;
constexpr int kHdr = 16 + 8 * 32;          // per-stage tile header: stripe, prog, pad, 32 out ptrs

// operand term: constant c (>= 0), variable v (-(v + 2))
struct LOp {
  int op[kK] = {-1, -1, -1, -1};
  int zg[kK] = {0, 0, 0, 0};  // a loaded slot with op -1 reads zero row zg (one per bank group)
  int cnt = 0;
  int dst = -1;   // variable stored to a row (-1: none)
  int goal = -1;  // goal stored to HBM (-1: none)
};

struct LSched {
  std::vector<std::vector<LOp>> rounds;  // 32 lanes each after dealing (slots positional)
  std::vector<int> consts, crow;  // constant row r holds constant consts[r] (-1: padding)
  int nvars = 0;                  // variables incl. split temporaries
  std::vector<int> vrow;          // variable -> its row (SSA: one row for its lifetime)
  int nvrows = 16;                // variable rows incl. the zero rows 0-7, a multiple of 8
};

// Lane order of one round.  A 128-bit shared load is served a quarter-warp (8 lanes) at a
// time, and a row's 16-byte bank group is (offset / 16) mod 8 (row bytes = 16 mod 128), so for
// every operand slot the 8 lanes of a quarter should read rows of 8 different groups.  The ops
// are dealt to the 4 quarters and each op's operands permuted over its loaded slots (XOR is
// commutative; a 3-operand op may put its zero-row read in any slot, and a zero read may use
// any of the 8 zero rows, one per bank group), greedily by the number of reads already sharing
// the group, then improved by annealing on the exact wavefront count.
template <class Grp, class DGrp>
std::vector<LOp> deal_round(std::vector<LOp> in, Grp grp, DGrp dgrp) {
  const int n = (int)in.size();
  for (auto &o : in) {  // terms first (an op dealt before has positional slots with zero reads)
    int t[kK], m = 0;
    for (int k = 0; k < kK; ++k)
      if (o.op[k] != -1) t[m++] = o.op[k];
    for (int k = 0; k < kK; ++k) o.op[k] = k < m ? t[k] : -1;
  }
  // candidate slot layouts of an op: term index per slot (-1 = zero row / not loaded)
  std::vector<std::vector<std::array<int, kK>>> cand(n);
  std::vector<std::array<int, kK>> g(n);
  for (int i = 0; i < n; ++i) {
    const LOp &o = in[i];
    for (int k = 0; k < kK; ++k) g[i][k] = k < o.cnt ? grp(o.op[k]) : -1;
    std::vector<int> idx;
    for (int k = 0; k < o.cnt; ++k) idx.push_back(k);
    const int slots = o.cnt == 0 ? 0 : o.cnt <= 2 ? 2 : 4;   // loaded slots
    while ((int)idx.size() < slots) idx.push_back(-1);       // zero-row reads
    std::sort(idx.begin(), idx.end());
    do {
      std::array<int, kK> c = {-1, -1, -1, -1};
      for (int k = 0; k < slots; ++k) c[k] = idx[k];
      cand[i].push_back(c);
    } while (std::next_permutation(idx.begin(), idx.end()));
  }
  // per quarter and slot (slot kK: the dst store): the rows already read (a row read by several
  // lanes of a quarter is a broadcast) and the distinct rows per bank group
  struct Cell {  // <= 8 lanes read a cell: a flat list of (row key, readers)
    int key[8], cnt[8], n = 0;
    int *find(int t) {
      for (int i = 0; i < n; ++i)
        if (key[i] == t) return &cnt[i];
      return nullptr;
    }
  };
  Cell rows[4][kK + 1];
  int distinct[4][kK + 1][8] = {};
  std::vector<int> qof(n, -1), cof(n, 0), fill(4, 0);
  std::vector<int> dg(n);
  for (int i = 0; i < n; ++i) dg[i] = dgrp(in[i]);
  std::vector<std::array<int, kK>> zsel(n);  // zero row group of each applied zero read
  const int kZeroKey = -1000000;             // row key of zero row g: kZeroKey + g
  auto slots_of = [&](int i) { return in[i].cnt == 0 ? 0 : in[i].cnt <= 2 ? 2 : 4; };
  auto term_cost = [&](int q, int k, int t, int gr) {
    if (gr < 0) return 0;
    const int *c = rows[q][k].find(t);
    return c && *c > 0 ? 0 : distinct[q][k][gr];
  };
  auto zero_pick = [&](int q, int k) {  // the zero row adding fewest wavefronts to this cell
    int bg = 0, bv = 1 << 30;
    for (int g = 0; g < 8; ++g) {
      const int v = term_cost(q, k, kZeroKey + g, g);
      if (v < bv) { bv = v; bg = g; }
    }
    return bg;
  };
  auto term_apply = [&](int q, int k, int t, int gr, int d) {
    if (gr < 0) return;
    Cell &cl = rows[q][k];
    int *c = cl.find(t);
    if (!c) {  // a new key (entries are never removed: a count may fall back to 0)
      if (cl.n == 8) {  // recycle an entry no lane reads any more
        int i = 0;
        while (cl.cnt[i] != 0) ++i;
        cl.key[i] = t;
        c = &cl.cnt[i];
      } else {
        cl.key[cl.n] = t;
        cl.cnt[cl.n] = 0;
        c = &cl.cnt[cl.n++];
      }
    }
    if (d > 0 && (*c)++ == 0) ++distinct[q][k][gr];
    if (d < 0 && --(*c) == 0) --distinct[q][k][gr];
  };
  auto cost = [&](int i, int q, int c) {
    int v = in[i].dst >= 0 ? term_cost(q, kK, -(in[i].dst + 2), dg[i]) : 0;
    for (int k = 0; k < kK; ++k) {
      const int t = cand[i][c][k];
      if (t >= 0) v += term_cost(q, k, in[i].op[t], g[i][t]);
      else if (k < slots_of(i)) {
        const int z = zero_pick(q, k);
        v += term_cost(q, k, kZeroKey + z, z);
      }
    }
    return v;
  };
  auto apply = [&](int i, int q, int c, int d) {
    if (in[i].dst >= 0) term_apply(q, kK, -(in[i].dst + 2), dg[i], d);
    for (int k = 0; k < kK; ++k) {
      const int t = cand[i][c][k];
      if (t >= 0) term_apply(q, k, in[i].op[t], g[i][t], d);
      else if (k < slots_of(i)) {
        if (d > 0) zsel[i][k] = zero_pick(q, k);
        term_apply(q, k, kZeroKey + zsel[i][k], zsel[i][k], d);
      }
    }
    fill[q] += d;
  };
  auto place = [&](int i) {
    int bq = -1, bc = 0, bv = 1 << 30;
    for (int q = 0; q < 4; ++q) {
      if (fill[q] == 8) continue;
      for (int c = 0; c < (int)cand[i].size(); ++c) {
        const int v = cost(i, q, c);
        if (v < bv) { bv = v; bq = q; bc = c; }
      }
    }
    qof[i] = bq;
    cof[i] = bc;
    apply(i, bq, bc, +1);
  };
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return in[a].cnt > in[b].cnt; });
  for (int i : order) place(i);
  for (int pass = 0; pass < 2; ++pass)
    for (int i : order) {
      apply(i, qof[i], cof[i], -1);
      place(i);
    }
  // local search on the exact measure -- wavefronts = sum over (quarter, slot) of the largest
  // number of distinct rows in one bank group -- by re-slotting one op or swapping two ops of
  // different quarters; a fixed-seed generator keeps compiles deterministic
  auto qcost = [&](int q) {
    int v = 0;
    for (int k = 0; k <= kK; ++k) v += *std::max_element(distinct[q][k], distinct[q][k] + 8);
    return v;
  };
  uint64_t rng = 0x9E3779B97F4A7C15ull ^ (uint64_t)n;
  auto rnd = [&](int m) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return (int)(rng % (uint64_t)m);
  };
  // simulated annealing: a worse move is kept with probability exp(-delta / temp), temp
  // falling linearly to zero; the best arrangement seen is the result
  int cur_cost = 0;
  for (int q = 0; q < 4; ++q) cur_cost += qcost(q);
  int best_cost = cur_cost;
  std::vector<int> best_q = qof, best_c = cof;
  const int iters = 400 * n;
  auto accept = [&](int delta, int iter) {
    if (delta <= 0) return true;
    const double temp = 1.5 * (1.0 - (double)iter / iters);
    if (temp <= 0.0) return false;
    const double u = (double)(rnd(1 << 20) + 1) / (1 << 20);
    return u < std::exp(-delta / temp);
  };
  for (int iter = 0; iter < iters && n > 1; ++iter) {
    const int i = rnd(n);
    if (rnd(2) == 0) {  // another slot layout for op i
      const int c = rnd((int)cand[i].size()), q = qof[i], old = cof[i];
      if (c == old) continue;
      const int before = qcost(q);
      apply(i, q, old, -1);
      apply(i, q, c, +1);
      const int delta = qcost(q) - before;
      if (accept(delta, iter)) { cof[i] = c; cur_cost += delta; }
      else { apply(i, q, c, -1); apply(i, q, old, +1); }
    } else {            // swap op i with op j of another quarter
      const int j = rnd(n), qi = qof[i], qj = qof[j];
      if (qi == qj) continue;
      const int before = qcost(qi) + qcost(qj);
      apply(i, qi, cof[i], -1);
      apply(j, qj, cof[j], -1);
      apply(i, qj, cof[i], +1);
      apply(j, qi, cof[j], +1);
      const int delta = qcost(qi) + qcost(qj) - before;
      if (accept(delta, iter)) { qof[i] = qj; qof[j] = qi; cur_cost += delta; }
      else {
        apply(i, qj, cof[i], -1);
        apply(j, qi, cof[j], -1);
        apply(i, qi, cof[i], +1);
        apply(j, qj, cof[j], +1);
      }
    }
    if (cur_cost < best_cost) { best_cost = cur_cost; best_q = qof; best_c = cof; }
  }
  // replay the best arrangement, then re-pick every zero row against the final neighbours
  for (int i = 0; i < n; ++i) apply(i, qof[i], cof[i], -1);
  qof = best_q;
  cof = best_c;
  for (int i = 0; i < n; ++i) apply(i, qof[i], cof[i], +1);
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < n; ++i) {
      apply(i, qof[i], cof[i], -1);
      apply(i, qof[i], cof[i], +1);
    }
  std::vector<LOp> rd(32);
  std::vector<int> lane = {0, 8, 16, 24};
  for (int i = 0; i < n; ++i) {
    LOp o = in[i];
    for (int k = 0; k < kK; ++k) {
      const int t = cand[i][cof[i]][k];
      o.op[k] = t >= 0 ? in[i].op[t] : -1;
      o.zg[k] = t >= 0 ? 0 : zsel[i][k];
    }
    // slots are now positional: cnt keeps its meaning (2 slots loaded if <= 2, else 4)
    rd[lane[qof[i]]++] = o;
  }
  return rd;
}

// Row polish.  After dealing, every (round, quarter, slot) cell's wavefronts -- the largest
// number of distinct rows one bank group serves in it (slot kK: the dst stores) -- depend only
// on which row each constant and variable got.  Constant rows may be permuted freely (the
// producer's load list names each constant's row); a variable may move to any variable row free
// for its whole lifetime [round stored, round last read] (a row is reused only from the round
// after its last read).  Moves that do not raise the total are kept; deterministic.

int cell_wavefronts(const LSched &sc, int r, int q, int k) {
  int rows[8], n = 0;
  for (int l = 8 * q; l < 8 * q + 8; ++l) {
    const LOp &o = sc.rounds[r][l];
    int key;  // a row: zero row g -> g, variable row -> its index, constant row -> 1e6 + index
    if (k == kK) {
      if (o.dst < 0) continue;
      key = sc.vrow[o.dst];
    } else {
      if (!((k < 2 && o.cnt > 0) || (k >= 2 && o.cnt > 2))) continue;
      const int t = o.op[k];
      key = t == -1 ? o.zg[k] : t >= 0 ? 1000000 + sc.crow[t] : sc.vrow[-t - 2];
    }
    bool seen = false;
    for (int i = 0; i < n; ++i) seen |= rows[i] == key;
    if (!seen) rows[n++] = key;
  }
  int cnt[8] = {}, m = 0;
  for (int i = 0; i < n; ++i) m = std::max(m, ++cnt[(rows[i] % 1000000) % 8]);
  return m;
}

int round_wavefronts(const LSched &sc, int r) {
  int v = 0;
  for (int q = 0; q < 4; ++q)
    for (int k = 0; k <= kK; ++k) v += cell_wavefronts(sc, r, q, k);
  return v;
}

int total_wavefronts(const LSched &sc) {
  int v = 0;
  for (int r = 0; r < (int)sc.rounds.size(); ++r) v += round_wavefronts(sc, r);
  return v;
}

struct RowPolish {
  LSched &sc;
  int R;
  std::vector<std::vector<int>> cells_of_c, cells_of_v;  // cells reading / storing each row user
  std::vector<int> def, last;                             // variable lifetime in rounds
  std::vector<std::vector<int>> on_row;                   // variables on each variable row
  explicit RowPolish(LSched &s) : sc(s), R((int)s.rounds.size()) {
    const int nv = (int)sc.vrow.size();
    cells_of_c.assign(sc.consts.size(), {});
    cells_of_v.assign(nv, {});
    def.assign(nv, -1);
    last.assign(nv, -1);
    on_row.assign(sc.nvrows, {});
    for (int r = 0; r < R; ++r)
      for (int l = 0; l < 32; ++l) {
        const LOp &o = sc.rounds[r][l];
        for (int k = 0; k < kK; ++k) {
          if (!loaded(o, k) || o.op[k] == -1) continue;
          const int t = o.op[k];
          if (t >= 0) cells_of_c[sc.crow[t]].push_back(cell(r, l / 8, k));
          else {
            cells_of_v[-t - 2].push_back(cell(r, l / 8, k));
            last[-t - 2] = std::max(last[-t - 2], r);
          }
        }
        if (o.dst >= 0) {
          cells_of_v[o.dst].push_back(cell(r, l / 8, kK));
          def[o.dst] = r;
        }
      }
    for (auto *vv : {&cells_of_c, &cells_of_v})
      for (auto &v : *vv) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
      }
    for (int v = 0; v < nv; ++v)
      if (def[v] >= 0) {
        last[v] = std::max(last[v], def[v]);
        on_row[sc.vrow[v]].push_back(v);
      }
  }
  static bool loaded(const LOp &o, int k) { return (k < 2 && o.cnt > 0) || (k >= 2 && o.cnt > 2); }
  static int cell(int r, int q, int k) { return (r * 4 + q) * (kK + 1) + k; }
  int cell_cost(int c) const {
    return cell_wavefronts(sc, c / (kK + 1) / 4, (c / (kK + 1)) % 4, c % (kK + 1));
  }
  std::vector<int> scratch;
  int cost_of(const std::vector<int> &a, const std::vector<int> &b) {  // over a u b (both sorted)
    scratch.clear();
    std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(scratch));
    int v = 0;
    for (int c : scratch) v += cell_cost(c);
    return v;
  }
  bool row_free(int row, int v) const {
    for (int u : on_row[row])
      if (u != v && !(last[u] < def[v] || last[v] < def[u])) return false;
    return true;
  }
  void move(int v, int row) {
    auto &from = on_row[sc.vrow[v]];
    from.erase(std::find(from.begin(), from.end(), v));
    on_row[row].push_back(v);
    sc.vrow[v] = row;
  }
  void run(uint64_t seed) {
    const int nused = (int)sc.consts.size(), nv = (int)sc.vrow.size();
    std::vector<int> vars;
    for (int v = 0; v < nv; ++v)
      if (def[v] >= 0) vars.push_back(v);
    uint64_t rng = seed;
    auto rnd = [&](int m) {
      rng ^= rng << 13;
      rng ^= rng >> 7;
      rng ^= rng << 17;
      return (int)(rng % (uint64_t)m);
    };
    const int iters = 60 * (nused + (int)vars.size());
    const std::vector<int> none;
    for (int iter = 0; iter < iters; ++iter) {
      if (rnd(2) == 0 && nused >= 2) {  // swap two constants' rows
        const int i = rnd(nused), j = rnd(nused);
        if (i % 8 == j % 8) continue;  // same bank group: no change
        const int before = cost_of(cells_of_c[i], cells_of_c[j]);
        auto swap_rows = [&]() {
          const int a = sc.consts[i], b = sc.consts[j];
          if (a >= 0) sc.crow[a] = j;
          if (b >= 0) sc.crow[b] = i;
          std::swap(sc.consts[i], sc.consts[j]);
          std::swap(cells_of_c[i], cells_of_c[j]);
        };
        swap_rows();
        if (cost_of(cells_of_c[i], cells_of_c[j]) > before) swap_rows();
      } else if (!vars.empty() && sc.nvrows > 8) {  // a variable to a free row of another group
        const int v = vars[rnd((int)vars.size())];
        const int row = 8 + rnd(sc.nvrows - 8), old = sc.vrow[v];
        if (row % 8 == old % 8 || !row_free(row, v)) continue;
        const int before = cost_of(cells_of_v[v], none);
        move(v, row);
        if (cost_of(cells_of_v[v], none) > before) move(v, old);
      }
    }
  }
};

LSched build_lanes(const Slp &s) {
  const int nc = s.n_const;
  int nv = s.n_vars;
  std::vector<std::vector<int>> goals_of_var(nv), goals_of_const(nc);
  std::vector<int> zero_goals;
  for (size_t g = 0; g < s.goal.size(); ++g) {
    const int t = s.goal[g];
    if (t < 0) zero_goals.push_back((int)g);
    else if (t < nc) goals_of_const[t].push_back((int)g);
    else goals_of_var[t - nc].push_back((int)g);
  }
  std::vector<char> needed(nv, 0), used(nv, 0);
  for (int v = 0; v < nv; ++v) needed[v] = !goals_of_var[v].empty();
  for (size_t k = s.ins.size(); k-- > 0;) {
    if (!needed[s.ins[k].var]) continue;
    for (int t : s.ins[k].ops)
      if (t >= nc) needed[t - nc] = used[t - nc] = 1;
  }
  std::vector<LOp> ops;
  auto term = [&](int t) { return t < nc ? t : -(t - nc + 2); };
  // one lane-op per <= 4 operands; wider instructions become a tree of partial XORs
  auto emit = [&](std::vector<int> terms, int dstvar, const std::vector<int> &goals) {
    while (terms.size() > (size_t)kK) {
      std::vector<int> next;
      for (size_t i = 0; i < terms.size(); i += kK) {
        if (terms.size() - i == 1) { next.push_back(terms[i]); continue; }
        LOp o;
        for (size_t q = 0; q < (size_t)kK && i + q < terms.size(); ++q) o.op[o.cnt++] = terms[i + q];
        o.dst = nv++;
        ops.push_back(o);
        next.push_back(-(o.dst + 2));
      }
      terms.swap(next);
    }
    LOp o;
    for (int t : terms) o.op[o.cnt++] = t;
    const bool copies = goals.size() > 1;
    o.dst = dstvar >= 0 ? dstvar : (copies ? nv++ : -1);
    if (!goals.empty()) o.goal = goals[0];
    ops.push_back(o);
    for (size_t g = 1; g < goals.size(); ++g) {  // the same value for further goals
      LOp c;
      c.op[c.cnt++] = -(o.dst + 2);
      c.goal = goals[g];
      ops.push_back(c);
    }
  };
  if (!zero_goals.empty()) emit({}, -1, zero_goals);
  for (int c = 0; c < nc; ++c)
    if (!goals_of_const[c].empty()) emit({c}, -1, goals_of_const[c]);
  for (size_t k = 0; k < s.ins.size(); ++k) {
    const int v = s.ins[k].var;
    if (!needed[v]) continue;
    std::vector<int> terms;
    for (int t : s.ins[k].ops) terms.push_back(term(t));
    emit(terms, used[v] ? v : -1, goals_of_var[v]);
  }
  // dependences
  const int n = (int)ops.size();
  std::vector<int> prod(nv, -1);
  for (int i = 0; i < n; ++i)
    if (ops[i].dst >= 0) prod[ops[i].dst] = i;
  std::vector<std::vector<int>> succ(n);
  std::vector<int> indeg(n, 0);
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < ops[i].cnt; ++q)
      if (ops[i].op[q] < -1) {
        const int p = prod[-ops[i].op[q] - 2];
        if (p < 0) throw Error(XSLP_EINVAL, "lane interpreter: operand without producer");
        succ[p].push_back(i);
        ++indeg[i];
      }
  // rounds: up to 32 ready ops in creation order
  LSched out;
  std::vector<int> ready;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push_back(i);
  int done = 0;
  while (done < n) {
    // the compiler's (DFS) order: fewer live variables -> more positions per tile
    // (critical path first gave the same number of rounds with ~15% more variable rows)
    std::sort(ready.begin(), ready.end());
    const size_t take = std::min<size_t>(32, ready.size());
    if (take == 0) throw Error(XSLP_EINVAL, "lane interpreter: cyclic program");
    std::vector<int> now(ready.begin(), ready.begin() + take);
    ready.erase(ready.begin(), ready.begin() + take);
    std::vector<LOp> round;
    for (int i : now) round.push_back(ops[i]);
    out.rounds.push_back(round);
    done += (int)take;
    for (int i : now)
      for (int j : succ[i])
        if (--indeg[j] == 0) ready.push_back(j);
  }
  out.nvars = nv;
  // Bank groups.  Every region starts on a multiple of 8 rows and a row is 16 bytes longer than
  // a multiple of 128, so row i of any region lies in 16-byte bank group i mod 8 (deal_round
  // uses it).  Constant rows in order of first use; variable rows by liveness at round
  // granularity: a row whose last read is in round r is reused from round r+1 on (the lanes of a
  // warp may diverge inside a round, so a store of round r must not race another lane's load of
  // round r).
  const int R = (int)out.rounds.size();
  out.crow.assign(nc, -1);
  for (auto &rd : out.rounds)
    for (auto &o : rd)
      for (int q = 0; q < o.cnt; ++q)
        if (o.op[q] >= 0 && out.crow[o.op[q]] < 0) {
          out.crow[o.op[q]] = (int)out.consts.size();
          out.consts.push_back(o.op[q]);
        }
  std::vector<int> last(nv, -1);
  for (int r = 0; r < R; ++r)
    for (auto &o : out.rounds[r])
      for (int q = 0; q < o.cnt; ++q)
        if (o.op[q] < -1) last[-o.op[q] - 2] = r;
  out.vrow.assign(nv, -1);
  // round by round: deal the ops to lanes (their operands' rows are known), then give each
  // stored variable a row whose bank group no other store of its quarter uses -- a free row of
  // that group, else a fresh one -- so the 128-bit stores of a quarter-warp do not conflict
  std::array<std::vector<int>, 8> free_rows;
  std::array<int, 8> fresh;  // next unused row of each group (rows 0-7: the zero rows)
  for (int g = 0; g < 8; ++g) fresh[g] = 8 + g;
  std::vector<int> freed_now;
  auto grp = [&](int t) { return t == -1 ? -1 : t >= 0 ? out.crow[t] % 8 : out.vrow[-t - 2] % 8; };
  for (int r = 0; r < R; ++r) {
    auto &rd = out.rounds[r];
    rd = deal_round(rd, grp, [](const LOp &) { return -1; });
    for (int q = 0; q < 4; ++q) {
      bool used_g[8] = {};
      for (int l = 8 * q; l < 8 * q + 8; ++l) {
        const LOp &o = rd[l];
        if (o.dst < 0) continue;
        int bg = -1;
        for (int g = 0; g < 8 && bg < 0; ++g)  // an unused group with a free row
          if (!used_g[g] && !free_rows[g].empty()) bg = g;
        for (int g = 0; g < 8 && bg < 0; ++g)  // an unused group, fresh row
          if (!used_g[g]) bg = g;
        int rr;
        if (!free_rows[bg].empty()) { rr = free_rows[bg].back(); free_rows[bg].pop_back(); }
        else { rr = fresh[bg]; fresh[bg] += 8; }
        used_g[bg] = true;
        out.vrow[o.dst] = rr;
      }
    }
    for (auto &o : rd)
      for (int q = 0; q < kK; ++q)
        if (o.op[q] < -1) {
          const int v = -o.op[q] - 2;
          if (out.vrow[v] < 0) throw Error(XSLP_EINVAL, "lane interpreter: read before store");
          if (last[v] == r) freed_now.push_back(out.vrow[v]);
        }
    std::sort(freed_now.begin(), freed_now.end());
    freed_now.erase(std::unique(freed_now.begin(), freed_now.end()), freed_now.end());
    for (int x : freed_now) free_rows[x % 8].push_back(x);
    freed_now.clear();
  }
  int maxrow = 0;
  for (int g = 0; g < 8; ++g) maxrow = std::max(maxrow, fresh[g] - 8);
  out.nvrows = (maxrow / 8 + 1) * 8;
  // alternate row polish and re-dealing each round against the polished rows (the deal now also
  // sees each store's group), a round's new deal kept only if it is cheaper
  for (int pass = 0; pass < 3; ++pass) {
    RowPolish(out).run(0x243F6A8885A308D3ull + (uint64_t)pass);
    auto dgrp = [&](const LOp &o) { return o.dst >= 0 ? out.vrow[o.dst] % 8 : -1; };
    for (int r = 0; r < R; ++r) {
      const int before = round_wavefronts(out, r);
      std::vector<LOp> live, keep = out.rounds[r];
      for (const auto &o : keep)
        if (o.cnt > 0 || o.dst >= 0 || o.goal >= 0) live.push_back(o);
      out.rounds[r] = deal_round(live, grp, dgrp);
      if (round_wavefronts(out, r) > before) out.rounds[r] = keep;
    }
  }
  LSched &best = out;
  return best;
}

struct Layout {
  int Tpos = 0, S = 2, NC = 8, V = 8, capw = 0;  // NC, V multiples of 8 (regions on group 0)
  uint32_t code0 = 0, var0 = 0, const0 = 0, RB = 0;
  size_t smem = 0;
};

size_t layout_smem(Layout &y) {
  y.RB = (uint32_t)y.Tpos * 4 + 16;
  y.code0 = 128 + y.S * kHdr;
  size_t var0 = y.code0 + (size_t)y.S * y.capw * 4;
  var0 = (var0 + 127) / 128 * 128;
  y.var0 = (uint32_t)var0;
  y.const0 = (uint32_t)(var0 + (size_t)y.V * y.RB);
  y.smem = (size_t)y.const0 + (size_t)y.S * y.NC * y.RB;
  return y.smem;
}

// One code variant (stage st):
//   [0] nloads [1] nrounds [2] words of this variant [3] variable rows (incl. zero rows 0-7)
//   [4] row bytes [5] variable rows offset [6] this stage's constant rows offset [7] 8
//   rounds: nrounds x 256 words: 32 lanes x 4 operand byte offsets (unused slots: a zero
//           row), then 32 lanes x (dst byte offset, goal select (header offset | (goal & 7) <<
//           16), ctl (count | flags << 8; flags 1 = store dst, 2 = store goal), 0)
//   one empty slack round (the consumer prefetches the next round's code)
//   loads: nloads x (constant index, byte offset of its row)
std::vector<uint32_t> emit_variant(const LSched &sc, const Layout &y, int st) {
  const uint32_t cst = y.const0 + (uint32_t)st * y.NC * y.RB;
  std::vector<uint32_t> w(kHead, 0);
  w[0] = (uint32_t)sc.consts.size();
  w[1] = (uint32_t)sc.rounds.size();
  w[3] = (uint32_t)sc.nvrows;
  w[4] = y.RB;
  w[5] = y.var0;
  w[6] = cst;
  w[7] = kHead;
  auto off_of = [&](const LOp &o, int k) -> uint32_t {
    const int t = o.op[k];
    if (t >= 0) return cst + (uint32_t)sc.crow[t] * y.RB;
    if (t == -1) return y.var0 + (uint32_t)o.zg[k] * y.RB;  // zero row zg (group zg)
    return y.var0 + (uint32_t)sc.vrow[-t - 2] * y.RB;
  };
  for (const auto &rd : sc.rounds) {
    // [32 lanes x (4 operand offsets)] then [32 lanes x (dst, goal select, ctl, 0)]: each of
    // the two 128-bit code loads of a round is one contiguous 512-byte warp access
    for (int l = 0; l < 32; ++l)
      w.insert(w.end(), {off_of(rd[l], 0), off_of(rd[l], 1), off_of(rd[l], 2), off_of(rd[l], 3)});
    for (int l = 0; l < 32; ++l) {
      const LOp &o = rd[l];
      uint32_t flags = 0, dst = 0, gsel = 0;
      if (o.dst >= 0) {
        dst = y.var0 + (uint32_t)sc.vrow[o.dst] * y.RB;
        flags |= 1;
      }
      if (o.goal >= 0) {
        gsel = (uint32_t)(16 + 8 * (o.goal >> 3)) | ((uint32_t)(o.goal & 7) << 16);
        flags |= 2;
      }
      w.insert(w.end(), {dst, gsel, (uint32_t)o.cnt | flags << 8, 0u});
    }
  }
  for (int l = 0; l < 32; ++l) w.insert(w.end(), {y.var0, y.var0, y.var0, y.var0});
  for (int l = 0; l < 32; ++l) w.insert(w.end(), {0u, 0u, 0u, 0u});
  for (size_t r = 0; r < sc.consts.size(); ++r) {
    if (sc.consts[r] < 0) continue;  // a padding row of the group layout: nothing to load
    w.push_back((uint32_t)sc.consts[r]);
    w.push_back(cst + (uint32_t)r * y.RB);
  }
  w[0] = (uint32_t)((w.size() - kHead - kRoundWords * (sc.rounds.size() + 1)) / 2);
  while (w.size() % 8) w.push_back(0);
  w[2] = (uint32_t)w.size();
  return w;
}

inline int consumer_words(const LSched &sc) { return kHead + kRoundWords * ((int)sc.rounds.size() + 1); }

struct Args {
  const uint32_t *code;
  const int64_t *prog_off;
  const int32_t *prog_of_stripe;
  const int32_t *ids;
  const uint8_t *const *in_tbl;
  uint8_t *const *out_tbl;
  uint64_t strip;
  uint32_t words, tps, ntiles, tpos;   // words = strip / 4; tps = tiles per stripe (tpos words each)
  int32_t n_in, n_out, S, nprogs;
  uint32_t code0, capw, var0, RB;
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
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 xor3v(uint4 a, uint4 b, uint4 c) {
  uint4 d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d.x) : "r"(a.x), "r"(b.x), "r"(c.x));
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d.y) : "r"(a.y), "r"(b.y), "r"(c.y));
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d.z) : "r"(a.z), "r"(b.z), "r"(c.z));
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d.w) : "r"(a.w), "r"(b.w), "r"(c.w));
  return d;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}

// kJ: quads a warp runs per round (the round's code is read once for them)
template <int kJ>
__global__ void __launch_bounds__(1024, 1) xslp_interp_lanes(Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t W = nthr / 32 - 1;  // consumer warps; the last warp produces
  const int S = a.S;
  const uint32_t base = sm_addr(sm);
  const uint32_t hdr0 = base + 128;
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(base + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 64 + 8 * k), "r"(W));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the zero rows (unused operand slots read them): every column of variable rows 0-7
  for (uint32_t i = tid; i < a.RB / 2; i += nthr) sts128(base + a.var0 + 16 * i, make_uint4(0, 0, 0, 0));
  __syncthreads();
  const uint32_t chunk = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * chunk, t1 = min(a.ntiles, t0 + chunk);
  const uint32_t warp = tid / 32, lane = tid & 31;
  if (warp == W) {  // ---------------- producer warp (all 32 lanes issue copies)
    int cur[4] = {-1, -1, -1, -1};
    for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
      const uint32_t st = it % S, ph = (it / S) & 1;
      const uint32_t entry = tile / a.tps, tw = tile % a.tps;
      const uint32_t stripe = a.ids ? (uint32_t)a.ids[entry] : entry;
      const int prog = a.prog_of_stripe ? a.prog_of_stripe[stripe] : 0;
      if (prog < 0 || prog >= a.nprogs) asm volatile("trap;");
      const uint32_t *pc0 = a.code + a.prog_off[prog];
      const uint32_t *pc = pc0 + (size_t)st * pc0[2];
      const uint8_t *const *in = a.in_tbl + (size_t)stripe * a.n_in;
      uint8_t *const *out = a.out_tbl + (size_t)stripe * a.n_out;
      const uint32_t nl = pc[0], nr = pc[1];
      const uint32_t *ld = pc + kHead + kRoundWords * (nr + 1);
      const size_t toff = (size_t)tw * a.tpos * 4;
      const uint64_t optr = lane < (uint32_t)a.n_out ? (uint64_t)out[lane] : 0;
      if (it >= (uint32_t)S)
        while (!try_wait(base + 64 + 8 * st, ph ^ 1)) __nanosleep(64);
      const uint32_t h = hdr0 + st * kHdr;
      if (lane < (uint32_t)a.n_out) asm volatile("st.shared.u64 [%0], %1;" ::"r"(h + 16 + 8 * lane), "l"(optr) : "memory");
      const uint32_t nb = min(a.tpos, a.words - tw * a.tpos) * 4;
      const uint32_t cbytes = cur[st] != prog ? (kHead + kRoundWords * (nr + 1)) * 4 : 0;
      cur[st] = prog;
      __syncwarp();
      if (lane == 0) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(h), "r"(stripe) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(h + 4), "r"((uint32_t)prog) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(base + 8 * st),
                     "r"(nb * nl + cbytes) : "memory");
        if (cbytes)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(base + a.code0 + st * a.capw * 4), "l"(pc), "r"(cbytes), "r"(base + 8 * st) : "memory");
      }
      __syncwarp();
      for (uint32_t i = lane; i < nl; i += 32) {
        const uint32_t c = ld[2 * i], off = ld[2 * i + 1];
        const uint8_t *src = in[c >> 3] + (c & 7) * a.strip + toff;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(base + off), "l"(src), "r"(nb), "r"(base + 8 * st) : "memory");
      }
    }
    return;
  }
  // ---------------- consumer warps: a group of kJ quads per warp, each round's code once
  for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
    const uint32_t st = it % S, ph = (it / S) & 1;
    while (!try_wait(base + 8 * st, ph)) {
    }
    const uint32_t tw = tile % a.tps;
    const uint32_t nq = min(a.tpos, a.words - tw * a.tpos) / 4;
    const uint32_t hdr = hdr0 + st * kHdr;
    const uint32_t cp = base + a.code0 + st * a.capw * 4;
    const uint32_t nr = lds128(cp).y;
    const uint32_t lc = cp + kHead * 4 + lane * 16;  // this lane's operands in round 0 (+512: ctl)
    for (uint32_t q0 = warp * kJ; q0 < nq; q0 += W * kJ) {
      const uint32_t nj = min((uint32_t)kJ, nq - q0);   // quads of this group (ragged tile end)
      const uint32_t col0 = base + q0 * 16;
      const uint64_t off0 = ((uint64_t)tw * a.tpos + (uint64_t)q0 * 4) * 4;
      uint4 o = lds128(lc), c = lds128(lc + 512);
      for (uint32_t r = 0; r < nr; ++r) {
        const uint32_t nx = lc + (r + 1) * kRoundWords * 4;
        const uint4 on = lds128(nx), cn = lds128(nx + 512);  // prefetch (the slack round at the end)
        const uint32_t cnt = c.z & 0xffu, fl = c.z >> 8;
        if (fl) {  // idle lanes (a partly filled round) issue no loads
          uint64_t gp = 0;
          if (fl & 2) {
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(gp) : "r"(hdr + (c.y & 0xffffu)) : "memory");
            gp += (uint64_t)(c.y >> 16) * a.strip + off0;
          }
#pragma unroll
          for (int j = 0; j < kJ; ++j) {
            if ((uint32_t)j >= nj) break;
            const uint32_t col = col0 + 16 * j;
            uint4 acc = make_uint4(0, 0, 0, 0);
            if (cnt > 0) {  // an unused slot 1 / 3 names the zero row
              const uint4 v0 = lds128(col + o.x), v1 = lds128(col + o.y);
              acc = make_uint4(v0.x ^ v1.x, v0.y ^ v1.y, v0.z ^ v1.z, v0.w ^ v1.w);
            }
            if (cnt > 2) {
              const uint4 v2 = lds128(col + o.z), v3 = lds128(col + o.w);
              acc = xor3v(acc, v2, v3);
            }
            if (fl & 1) sts128(col + c.x, acc);
            if (fl & 2)
              asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(gp + 16 * j), "r"(acc.x),
                           "r"(acc.y), "r"(acc.z), "r"(acc.w) : "memory");
          }
        }
        __syncwarp();
        o = on;
        c = cn;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(base + 64 + 8 * st) : "memory");
  }
}

struct Pool {
  uint32_t *code = nullptr;
  int64_t *off = nullptr;
  Layout y;
};
std::mutex g_mu;
std::map<std::tuple<int, int, int, std::vector<const Program *>>, Pool> g_pools;  // (dev, S, max T_pos, progs)

// Lane schedules are built once per program (untimed host work, ~0.1-0.3 s for an RS(10,4)
// decode) and cached until the program is freed; a batch of programs is built on all host cores.
std::mutex g_smu;
std::map<const Program *, std::shared_ptr<const LSched>> g_scheds;

std::shared_ptr<const LSched> sched_of(const Program *p) {
  {
    std::lock_guard<std::mutex> g(g_smu);
    auto it = g_scheds.find(p);
    if (it != g_scheds.end()) return it->second;
  }
  auto sc = std::make_shared<const LSched>(build_lanes(p->slp));
  std::lock_guard<std::mutex> g(g_smu);
  return g_scheds.emplace(p, sc).first->second;  // a racing builder's equal schedule may win
}

std::vector<std::shared_ptr<const LSched>> scheds_of(const Program *const *progs, int np) {
  std::vector<std::shared_ptr<const LSched>> out(np);
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex em;
  auto work = [&]() {
    for (int i; (i = next++) < np;) {
      try {
        out[i] = sched_of(progs[i]);
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
  return out;
}

}  // namespace lanes

// Dump form 4: the lane interpreter's stage-0 code variant for this program alone (T_pos = the
// largest multiple of 32 words that fits with S = opts.stages).
std::vector<uint32_t> interp_lanes_dump(const Program *p, int S) {
  using namespace lanes;
  const LSched &sc = *sched_of(p);
  Layout y;
  y.S = std::max(1, std::min(4, S));
  y.NC = std::max<int>(8, ((int)sc.consts.size() + 7) / 8 * 8);  // regions start on group 0
  y.V = sc.nvrows;
  y.capw = (consumer_words(sc) + 3) / 4 * 4;
  for (y.Tpos = 2048; y.Tpos > 32; y.Tpos -= 32)
    if (layout_smem(y) <= 227 * 1024) break;
  layout_smem(y);
  return emit_variant(sc, y, 0);
}

void drop_lanes_of(const Program *p) {
  using namespace lanes;
  {
    std::lock_guard<std::mutex> g(g_smu);
    g_scheds.erase(p);
  }
  std::lock_guard<std::mutex> g(g_mu);
  for (auto it = g_pools.begin(); it != g_pools.end();) {
    const auto &progs = std::get<3>(it->first);
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

// the kernel's shared-memory opt-in, once per device
static bool finish_plan(int dev) {
  using namespace lanes;
  static std::mutex am;
  static std::map<int, bool> attr;
  std::lock_guard<std::mutex> g(am);
  if (!attr[dev]) {
    for (const void *f : {(const void *)xslp_interp_lanes<4>})
      CUDA_OK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr[dev] = true;
  }
  return true;
}

// The code pool and layout of a program set for strips of B/8 bytes on the current device, built
// once (everything a launch needs that cannot be captured in a CUDA graph); false if the
// interpreter does not apply (strip % 16, > 32 output blocks, or the rows do not fit).
static bool lanes_plan(const Program *const *progs, int np, size_t B, lanes::Pool &pool) {
  using namespace lanes;
  const xslp_opts &o = progs[0]->opts;
  const uint64_t strip = B / 8;
  if (strip % 16 || progs[0]->n_goals / 8 > 32) return false;
  const int S = std::max(1, std::min(4, o.stages));
  // the largest tile (a multiple of 32 words) whose rows fit; T_pos <= the strip
  const int maxpos = (int)std::min<uint64_t>(2048, (strip / 4 + 31) / 32 * 32);
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  {
    std::vector<const Program *> key(progs, progs + np);
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_pools.find({dev, S, maxpos, key});
    if (it != g_pools.end()) {
      pool = it->second;
      return finish_plan(dev);
    }
  }
  // schedules outside the pool lock (parallel, cached per program)
  const auto sc = scheds_of(progs, np);
  {
    std::vector<const Program *> key(progs, progs + np);
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_pools.find({dev, S, maxpos, key});
    if (it != g_pools.end()) {
      pool = it->second;
    } else {
      Layout y;
      y.S = S;
      int cw = 0;
      for (int i = 0; i < np; ++i) {
        y.NC = std::max<int>(y.NC, ((int)sc[i]->consts.size() + 7) / 8 * 8);  // group-aligned
        y.V = std::max(y.V, sc[i]->nvrows);
        cw = std::max(cw, consumer_words(*sc[i]));
      }
      y.capw = (cw + 3) / 4 * 4;
      for (y.Tpos = maxpos; y.Tpos >= 32; y.Tpos -= 32)
        if (layout_smem(y) <= 227 * 1024) break;
      if (y.Tpos < 32) return false;
      std::vector<uint32_t> all;
      std::vector<int64_t> off;
      for (int i = 0; i < np; ++i) {
        off.push_back((int64_t)all.size());
        for (int s_ = 0; s_ < S; ++s_) {
          auto w = emit_variant(*sc[i], y, s_);
          all.insert(all.end(), w.begin(), w.end());
        }
      }
      Pool P;
      P.y = y;
      CUDA_OK(cudaMalloc(&P.code, all.size() * 4));
      CUDA_OK(cudaMemcpy(P.code, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMalloc(&P.off, off.size() * 8));
      CUDA_OK(cudaMemcpy(P.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
      g_pools[{dev, S, maxpos, key}] = P;
      pool = P;
    }
  }
  return finish_plan(dev);
}

bool interp_lanes_prepare(const Program *p, size_t B) {
  const Program *ps[1] = {p};
  lanes::Pool pool;
  return lanes_plan(ps, 1, B, pool);
}

// Launch the lane-parallel interpreter; false if it does not apply.  Consumer warps:
// max(16, opts.threads / 32), at most 31 (plus the producer warp).
bool interp_lanes_launch(const Program *const *progs, int np, const int32_t *d_pos,
                         const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                         int nstripes, size_t B, cudaStream_t st) {
  using namespace lanes;
  if (!in || !out || nstripes <= 0) return false;
  Pool pool;
  if (!lanes_plan(progs, np, B, pool)) return false;
  const uint64_t strip = B / 8;
  constexpr int J = 4;  // quads per warp per round (measured: 2 slower, 8 slower)
  // consumer warps: max(16, threads / 32), but no more than a full tile has 4-quad groups
  const int groups = (int)((pool.y.Tpos / 4 + J - 1) / J);
  const int W = std::max(1, std::min(groups, std::max(16, std::min(31, progs[0]->opts.threads / 32))));
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  const Layout &y = pool.y;
  Args a{};
  a.code = pool.code;
  a.prog_off = pool.off;
  a.prog_of_stripe = d_pos;
  a.ids = d_ids;
  a.in_tbl = in;
  a.out_tbl = out;
  a.strip = strip;
  a.words = (uint32_t)(strip / 4);
  a.tpos = (uint32_t)y.Tpos;
  a.tps = (a.words + a.tpos - 1) / a.tpos;
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
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<uint64_t>(a.ntiles, (uint64_t)sms);
  void *args[] = {&a};
  const void *fn = (const void *)xslp_interp_lanes<J>;
  CUDA_OK(cudaLaunchKernel(fn, dim3(grid), dim3(32 * (W + 1)), args, y.smem, st));
  count_launch();
  return true;
}

}  // namespace xslp
