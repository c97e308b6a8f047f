// Host compiler: bitmatrix -> SLP -> RePair/XorRePair -> XOR fusion -> DFS schedule
// -> pebble names (paper NVar) and interpreter slots (device bytecode).
//
// Paper: SLP_xor and its set semantics ([SLP]); Pair / RePair with the
// total order; Rebuild / XorRePair; MultiSLP, #M and XOR
// fusion ([Fus]); computation graph, pebble game and the DFS
// heuristic ([Peb]).  Readings of silent points are in DESIGN.md
// (R8-R12).  The product shares no code with oracle/.
#include <algorithm>
#include <functional>
#include <set>
#include <sstream>
#include <unordered_map>

#include "xslp_internal.h"

namespace xslp {

// ---------------------------------------------------------------------------------------
// Lifting: goal g = XOR of the constants at the set bits of row g.
// multi = true gives one variadic instruction per goal (P^{+F}); false gives the
// in-place binary chain per goal ("Base", reading R17).  Rows with one bit are copy
// goals and all-zero rows zero goals; neither needs an instruction.
Slp lift(const std::vector<Bits> &goals, int n_const, bool multi) {
  Slp s;
  s.n_const = n_const;
  s.goal.assign(goals.size(), -1);
  for (size_t g = 0; g < goals.size(); ++g) {
    std::vector<int> cs;
    for (int c = 0; c < n_const; ++c)
      if (goals[g].get(c)) cs.push_back(c);
    if (cs.empty()) continue;
    if (cs.size() == 1) { s.goal[g] = cs[0]; continue; }
    if (multi) {
      s.ins.push_back({s.n_vars, cs});
      s.goal[g] = s.term_of_var(s.n_vars++);
    } else {
      int acc = cs[0];
      for (size_t i = 1; i < cs.size(); ++i) {
        s.ins.push_back({s.n_vars, {acc, cs[i]}});
        acc = s.term_of_var(s.n_vars++);
      }
      s.goal[g] = acc;
    }
  }
  return s;
}

// ---------------------------------------------------------------------------------------
// RePair / XorRePair.
//
// Terms inside the compressor: temporal k -> key k, constant j -> key CB + j, so the
// total order "temporals by generation order, t < c, constants by index"
// is integer order, and the lexicographic order on pairs is the order of
// (lo << 32 | hi).  Pair frequency counts each original definition once (reading R8).
namespace {
constexpr int CB = 1 << 30;

struct PairCounter {
  std::unordered_map<uint64_t, int> cnt;
  std::vector<std::set<uint64_t>> bucket;  // bucket[c] = pairs with count c
  int maxc = 0;
  explicit PairCounter(int max_count) : bucket(max_count + 2) {}
  void add(uint64_t k, int d) {
    int &c = cnt[k];
    if (c) bucket[c].erase(k);
    c += d;
    if (c) {
      bucket[c].insert(k);
      if (c > maxc) maxc = c;
    } else {
      cnt.erase(k);
    }
  }
  // most frequent pair, smallest in the lexicographic order on ties
  bool best(uint64_t &k) {
    while (maxc > 0 && bucket[maxc].empty()) --maxc;
    if (maxc == 0) return false;
    k = *bucket[maxc].begin();
    return true;
  }
};

inline uint64_t pkey(int a, int b) {
  if (a > b) std::swap(a, b);
  return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
}

void pairs_of(PairCounter &pc, const std::vector<int> &def, int d) {
  for (size_t i = 0; i < def.size(); ++i)
    for (size_t j = i + 1; j < def.size(); ++j) pc.add(pkey(def[i], def[j]), d);
}
}  // namespace

Slp compress(const std::vector<Bits> &goals, int n_const, bool xor_rebuild) {
  const int W = (n_const + 63) / 64;
  const int m = (int)goals.size();
  Slp out;
  out.n_const = n_const;
  out.goal.assign(m, -1);

  // An original with its cached Rebuild trajectory.  Temporal values never change and
  // every outer iteration adds one temporal with the largest index, so a cached greedy
  // trajectory stays valid unless the new temporal is strictly better at some step
  // (ties go to the smaller index); then it is recomputed from that step.
  // The result is identical to recomputing Rebuild from scratch.
  struct Orig {
    std::vector<int> def;
    int goal;
    bool alive;
    std::vector<uint64_t> val;        // val(v), W words
    std::vector<uint64_t> step_rem;   // rem before step i, [steps][W]
    std::vector<int> step_c;          // |rem| after step i
    std::vector<int> S;               // chosen temporals
    std::vector<uint64_t> final_rem;
    int final_c = 0;
    int seen = -1;                    // temporals considered so far (-1: none computed)
  };
  std::vector<Orig> orig;
  int64_t mass = 0;
  for (int g = 0; g < m; ++g) {
    std::vector<int> cs;
    for (int c = 0; c < n_const; ++c)
      if (goals[g].get(c)) cs.push_back(CB + c);
    if (cs.empty()) continue;
    if (cs.size() == 1) { out.goal[g] = cs[0] - CB; continue; }
    mass += (int64_t)cs.size();
    Orig o;
    o.def = cs;
    o.goal = g;
    o.alive = true;
    o.val = goals[g].w;
    o.val.resize(W, 0);
    orig.push_back(std::move(o));
  }
  // temporals
  std::vector<std::pair<int, int>> tops;  // operand keys
  std::vector<uint64_t> tval;             // [T][W]
  auto val_of = [&](int key, uint64_t *dst) {
    if (key >= CB) {
      std::fill(dst, dst + W, 0);
      int c = key - CB;
      dst[c >> 6] |= 1ull << (c & 63);
    } else {
      std::copy(tval.begin() + (size_t)key * W, tval.begin() + (size_t)(key + 1) * W, dst);
    }
  };
  auto popx = [&](const uint64_t *x, const uint64_t *y) {
    int c = 0;
    for (int i = 0; i < W; ++i) c += __builtin_popcountll(x[i] ^ y[i]);
    return c;
  };
  // Greedy Rebuild continued from step `from` with temporals 0..T-1.
  auto extend = [&](Orig &o, size_t from, int T) {
    o.step_rem.resize(from * W);
    o.step_c.resize(from);
    o.S.resize(from);
    std::vector<uint64_t> rem(W);
    if (from == 0) rem = o.val;
    else {
      const uint64_t *pr = &o.step_rem[(from - 1) * W];
      const uint64_t *tv = &tval[(size_t)o.S[from - 1] * W];
      for (int i = 0; i < W; ++i) rem[i] = pr[i] ^ tv[i];
    }
    int remc = 0;
    for (int i = 0; i < W; ++i) remc += __builtin_popcountll(rem[i]);
    for (;;) {
      int bt = -1, bc = remc;
      for (int k = 0; k < T; ++k) {
        int c = popx(rem.data(), &tval[(size_t)k * W]);
        if (c < bc) { bc = c; bt = k; }  // strict: ties keep the smallest t
      }
      if (bt < 0) break;  // cannot shorten rem
      o.step_rem.insert(o.step_rem.end(), rem.begin(), rem.end());
      o.step_c.push_back(bc);
      o.S.push_back(bt);
      const uint64_t *tv = &tval[(size_t)bt * W];
      for (int i = 0; i < W; ++i) rem[i] ^= tv[i];
      remc = bc;
    }
    o.final_rem = rem;
    o.final_c = remc;
  };
  auto rebuild = [&](Orig &o, int T) {
    if (o.seen < 0) {
      extend(o, 0, T);
    } else {
      for (int tn = o.seen; tn < T; ++tn) {
        const uint64_t *tv = &tval[(size_t)tn * W];
        const size_t steps = o.S.size();
        size_t redo = SIZE_MAX;
        for (size_t i = 0; i <= steps && redo == SIZE_MAX; ++i) {
          const uint64_t *r = i < steps ? &o.step_rem[i * W] : o.final_rem.data();
          const int bc = i < steps ? o.step_c[i] : o.final_c;
          if (popx(r, tv) < bc) redo = i;
        }
        if (redo != SIZE_MAX) { extend(o, redo, T); break; }
      }
    }
    o.seen = T;
  };
  PairCounter pc((int)orig.size());
  for (auto &o : orig) pairs_of(pc, o.def, +1);

  std::vector<uint64_t> rem(W), tmp(W);
  uint64_t best;
  (void)rem;
  while (pc.best(best)) {
    const int a = (int)(best >> 32), b = (int)(best & 0xffffffffu);
    const int t = (int)tops.size();
    tops.push_back({a, b});
    tval.resize((size_t)(t + 1) * W);
    val_of(a, rem.data());
    val_of(b, tmp.data());
    for (int i = 0; i < W; ++i) tval[(size_t)t * W + i] = rem[i] ^ tmp[i];
    // Pair(a, b): replace every co-occurrence in an original definition
    for (auto &o : orig) {
      if (!o.alive) continue;
      auto &d = o.def;
      if (!std::binary_search(d.begin(), d.end(), a) || !std::binary_search(d.begin(), d.end(), b))
        continue;
      // incremental pair counts: pairs with a or b leave, pairs with t arrive
      for (int x : d) {
        if (x == a || x == b) continue;
        pc.add(pkey(a, x), -1);
        pc.add(pkey(b, x), -1);
      }
      pc.add(pkey(a, b), -1);
      d.erase(std::find(d.begin(), d.end(), a));
      d.erase(std::find(d.begin(), d.end(), b));
      d.insert(std::lower_bound(d.begin(), d.end(), t), t);
      if (d.size() == 1) {  // the original becomes the temporal (reading R10)
        o.alive = false;
        out.goal[o.goal] = n_const + d[0];
      } else {
        for (int x : d)
          if (x != t) pc.add(pkey(t, x), +1);
      }
    }
    if (!xor_rebuild) continue;
    // XorRePair step (3): Rebuild every original, in definition order (R9)
    const int T = (int)tops.size();
    for (auto &o : orig) {
      if (!o.alive) continue;
      rebuild(o, T);
      const auto &S = o.S;
      const uint64_t *remf = o.final_rem.data();
      const int remc = o.final_c;
      std::vector<uint64_t> rem(remf, remf + W);
      if ((int)S.size() + remc >= (int)o.def.size()) continue;  // must be strictly smaller
      std::vector<int> nd(S.begin(), S.end());
      std::sort(nd.begin(), nd.end());
      for (int c = 0; c < n_const; ++c)
        if ((rem[c >> 6] >> (c & 63)) & 1) nd.push_back(CB + c);
      pairs_of(pc, o.def, -1);
      o.def = nd;
      if (nd.size() == 1) {
        o.alive = false;
        out.goal[o.goal] = nd[0] >= CB ? nd[0] - CB : n_const + nd[0];
      } else {
        pairs_of(pc, o.def, +1);
      }
    }
  }
  (void)mass;
  for (auto &o : orig)
    if (o.alive) throw Error(XSLP_EINVAL, "internal: RePair left an original");
  auto term = [&](int key) { return key >= CB ? key - CB : n_const + key; };
  for (size_t k = 0; k < tops.size(); ++k)
    out.ins.push_back({(int)k, {term(tops[k].first), term(tops[k].second)}});
  out.n_vars = (int)tops.size();
  return out;
}

// ---------------------------------------------------------------------------------------
// Renumber variables densely in instruction order; drop instructions not reachable
// from a goal.
static void compact(Slp &s) {
  std::vector<int> idx(s.n_vars, -1);
  for (size_t i = 0; i < s.ins.size(); ++i) idx[s.ins[i].var] = (int)i;
  std::vector<char> live(s.ins.size(), 0);
  std::vector<int> st;
  for (int g : s.goal)
    if (g >= s.n_const) st.push_back(idx[g - s.n_const]);
  while (!st.empty()) {
    int i = st.back();
    st.pop_back();
    if (i < 0 || live[i]) continue;
    live[i] = 1;
    for (int t : s.ins[i].ops)
      if (t >= s.n_const) st.push_back(idx[t - s.n_const]);
  }
  std::vector<int> ren(s.n_vars, -1);
  std::vector<Ins> ni;
  for (size_t i = 0; i < s.ins.size(); ++i)
    if (live[i]) {
      ren[s.ins[i].var] = (int)ni.size();
      ni.push_back(s.ins[i]);
    }
  for (auto &in : ni) {
    in.var = ren[in.var];
    for (auto &t : in.ops)
      if (t >= s.n_const) t = s.n_const + ren[t - s.n_const];
  }
  for (auto &g : s.goal)
    if (g >= s.n_const) g = s.n_const + ren[g - s.n_const];
  s.ins.swap(ni);
  s.n_vars = (int)s.ins.size();
}

// ---------------------------------------------------------------------------------------
// XOR fusion: repeatedly unfold a variable used exactly once and not
// returned.  Splicing can create x ^ x; set semantics cancels the pair (reading R11).
// Variables used more than once are never unfolded.
void fuse(Slp &s) {
  compact(s);
  const int nc = s.n_const;
  const int nv = s.n_vars;
  std::vector<int> uses(nv, 0);
  std::vector<char> isgoal(nv, 0), alive(nv, 1);
  for (auto &in : s.ins)
    for (int t : in.ops)
      if (t >= nc) uses[t - nc]++;
  for (int g : s.goal)
    if (g >= nc) isgoal[g - nc] = 1;
  // var ids equal instruction positions after compact()
  bool changed = true;
  while (changed) {
    changed = false;
    for (int k = 0; k < nv; ++k) {
      if (!alive[k]) continue;
      auto &ops = s.ins[k].ops;
      size_t i = 0;
      while (i < ops.size()) {
        int t = ops[i];
        int u = t - nc;
        if (t < nc || uses[u] != 1 || isgoal[u] || !alive[u]) { ++i; continue; }
        std::vector<int> sp = s.ins[u].ops;
        std::vector<int> merged(ops.begin(), ops.begin() + i);
        merged.insert(merged.end(), sp.begin(), sp.end());
        merged.insert(merged.end(), ops.begin() + i + 1, ops.end());
        // cancel duplicate pairs, keeping first-occurrence order
        std::vector<int> res;
        std::unordered_map<int, int> cntm;
        for (int x : merged) cntm[x]++;
        std::set<int> done;
        for (int x : merged) {
          if (done.count(x)) continue;
          done.insert(x);
          int c = cntm[x];
          if (c % 2) res.push_back(x);
          if (x >= nc && c > 1) uses[x - nc] -= (c - (c % 2));
        }
        alive[u] = 0;
        uses[u] = 0;
        ops = res;
        changed = true;
        // rescan from i: spliced operands may themselves be unfoldable
      }
    }
    // degenerate instructions (cancellation left < 2 operands): substitute
    for (int k = 0; k < nv; ++k) {
      if (!alive[k] || s.ins[k].ops.size() >= 2) continue;
      int rep = s.ins[k].ops.empty() ? -1 : s.ins[k].ops[0];
      alive[k] = 0;
      changed = true;
      const int tk = nc + k;
      for (auto &g : s.goal)
        if (g == tk) g = rep;
      for (int j = 0; j < nv; ++j) {
        if (!alive[j]) continue;
        auto &o = s.ins[j].ops;
        auto it = std::find(o.begin(), o.end(), tk);
        if (it == o.end()) continue;
        o.erase(it);
        if (rep >= 0) {
          auto it2 = std::find(o.begin(), o.end(), rep);
          if (it2 != o.end()) {
            o.erase(it2);
            if (rep >= nc) uses[rep - nc] -= 1;
          } else {
            o.push_back(rep);
            if (rep >= nc) uses[rep - nc] += 1;
          }
        }
      }
      if (rep >= nc) {
        uses[rep - nc] -= 1;  // k's own use of rep is gone
        for (int g : s.goal)
          if (g == rep) isgoal[rep - nc] = 1;
      }
    }
  }
  std::vector<Ins> ni;
  for (int k = 0; k < nv; ++k)
    if (alive[k]) ni.push_back(s.ins[k]);
  s.ins.swap(ni);
  compact(s);
}

// ---------------------------------------------------------------------------------------
// DFS scheduling: post-order traversal of the computation graph from
// the goal nodes, children visited in the total order (variables by creation, then
// constants); operands are emitted in that order.  goal_order 0 visits the roots in
// the term order of the goal nodes, 1 in goal-index order.
void schedule_dfs(Slp &s, int goal_order) {
  compact(s);
  const int nc = s.n_const, nv = s.n_vars;
  for (auto &in : s.ins) std::sort(in.ops.begin(), in.ops.end(), [&](int x, int y) {
      bool vx = x >= nc, vy = y >= nc;
      if (vx != vy) return vx;  // variables (temporals) precede constants
      return x < y;
    });
  std::vector<int> roots;
  for (int g : s.goal)
    if (g >= nc) roots.push_back(g - nc);
  if (goal_order == 0) std::sort(roots.begin(), roots.end());
  std::vector<char> vis(nv, 0);
  std::vector<int> order;
  for (int r : roots) {
    if (vis[r]) continue;
    std::vector<std::pair<int, size_t>> st{{r, 0}};
    vis[r] = 1;
    while (!st.empty()) {
      auto &[v, ci] = st.back();
      const auto &ops = s.ins[v].ops;
      if (ci < ops.size()) {
        int t = ops[ci++];
        if (t >= nc && !vis[t - nc]) {
          vis[t - nc] = 1;
          st.push_back({t - nc, 0});
        }
      } else {
        order.push_back(v);
        st.pop_back();
      }
    }
  }
  std::vector<Ins> ni;
  for (int v : order) ni.push_back(s.ins[v]);
  s.ins.swap(ni);
  compact(s);
}

// ---------------------------------------------------------------------------------------
// Bottom-up greedy scheduling with cache capacity c ([Peb]):
//  (i)   choose a computable node maximising |H|/|C|, C = its children, H = the children
//        whose block is in the (LRU) cache; ties by the node order (creation order);
//  (ii)  access H, then the rest of C (operands emitted in that order, each part in the
//        term order);
//  (iii) move a movable cached pebble to the node if there is one, else a movable pebble,
//        else a fresh one; the smallest pebble first.
// A pebble is movable when its node is not a goal and all its parents are computed (R12).
// The cache model is the abstract LRU of P:1007-1022 over constants and pebbles.
// Reorders s.ins in place and returns NVar; pebble[v] receives the pebble of variable v
// (indices after the reordering).
int schedule_greedy(Slp &s, int cap, std::vector<int> &pebble) {
  compact(s);
  const int nc = s.n_const, nv = s.n_vars;
  if (cap < 1) throw Error(XSLP_EINVAL, "greedy capacity must be positive");
  auto ord_less = [&](int x, int y) {  // variables (temporals) before constants
    bool vx = x >= nc, vy = y >= nc;
    if (vx != vy) return vx;
    return x < y;
  };
  std::vector<int> nparents(nv, 0), waiting(nv, 0), remaining(nv, 0);
  std::vector<std::vector<int>> users(nv);
  std::vector<char> goal(nv, 0), done(nv, 0);
  for (int k = 0; k < nv; ++k)
    for (int t : s.ins[k].ops)
      if (t >= nc) { users[t - nc].push_back(k); nparents[t - nc]++; waiting[k]++; }
  for (int g : s.goal)
    if (g >= nc) goal[g - nc] = 1;
  remaining = nparents;
  std::set<int> ready;
  for (int k = 0; k < nv; ++k)
    if (!waiting[k]) ready.insert(k);
  std::vector<int> peb(nv, -1);
  std::set<int> movable;  // pebbles of movable nodes
  std::vector<int> node_of_peb;
  std::vector<int> cache;  // LRU names: constant c -> c, pebble q -> nc + q; front = LRU
  auto in_cache = [&](int name) { return std::find(cache.begin(), cache.end(), name) != cache.end(); };
  auto touch = [&](int name) {
    auto it = std::find(cache.begin(), cache.end(), name);
    if (it != cache.end()) cache.erase(it);
    else if ((int)cache.size() >= cap) cache.erase(cache.begin());
    cache.push_back(name);
  };
  auto name_of = [&](int t) { return t < nc ? t : nc + peb[t - nc]; };
  std::vector<Ins> out;
  std::vector<int> order;
  while (!ready.empty()) {
    int best = -1;
    int64_t bh = -1, bc = 1;
    for (int k : ready) {
      int h = 0;
      for (int t : s.ins[k].ops)
        if (in_cache(name_of(t))) ++h;
      const int64_t c = (int64_t)s.ins[k].ops.size();
      if (best < 0 || h * bc > bh * c) { best = k; bh = h; bc = c; }  // ties keep the smaller node
    }
    ready.erase(best);
    auto ops = s.ins[best].ops;
    std::vector<int> H, R;
    for (int t : ops) (in_cache(name_of(t)) ? H : R).push_back(t);
    std::sort(H.begin(), H.end(), ord_less);
    std::sort(R.begin(), R.end(), ord_less);
    ops = H;
    ops.insert(ops.end(), R.begin(), R.end());
    for (int t : ops) touch(name_of(t));
    // children whose last parent is this node become movable (non-goals)
    for (int t : s.ins[best].ops)
      if (t >= nc && --remaining[t - nc] == 0 && !goal[t - nc]) movable.insert(peb[t - nc]);
    int q = -1;
    for (int m : movable)
      if (in_cache(nc + m)) { q = m; break; }
    if (q < 0 && !movable.empty()) q = *movable.begin();
    if (q >= 0) movable.erase(q);
    else { q = (int)node_of_peb.size(); node_of_peb.push_back(-1); }
    peb[best] = q;
    node_of_peb[q] = best;
    touch(nc + q);
    out.push_back({best, ops});
    order.push_back(best);
    done[best] = 1;
    for (int u : users[best])
      if (--waiting[u] == 0) ready.insert(u);
  }
  if ((int)out.size() != nv) throw Error(XSLP_EINVAL, "internal: greedy schedule incomplete");
  s.ins.swap(out);
  // compact() renumbers variables in the new order; carry the pebbles along
  std::vector<int> new_peb(nv);
  for (int i = 0; i < nv; ++i) new_peb[i] = peb[order[i]];
  compact(s);
  pebble = new_peb;
  return (int)node_of_peb.size();
}

// ---------------------------------------------------------------------------------------
// Pebble assignment of the DFS heuristic: "If we have a pebble on G
// that can move, we reuse it; otherwise, we put a fresh pebble."  A pebble can move
// when its node is not a goal and all its parents are pebbled (reading R12); among
// the current instruction's movable operands the most recently computed wins; other
// released pebbles are reused smallest-first.  Returns NVar.
int paper_pebbles(const Slp &s, std::vector<int> &pebble) {
  const int nc = s.n_const, nv = s.n_vars;
  std::vector<int> rem(nv, 0);
  std::vector<char> goal(nv, 0);
  for (auto &in : s.ins)
    for (int t : in.ops)
      if (t >= nc) rem[t - nc]++;
  for (int g : s.goal)
    if (g >= nc) goal[g - nc] = 1;
  pebble.assign(nv, -1);
  std::set<int> freep;
  int next = 0;
  for (int k = 0; k < nv; ++k) {
    int cand = -1;
    std::vector<int> released;
    for (int t : s.ins[k].ops) {
      if (t < nc) continue;
      int u = t - nc;
      if (--rem[u] == 0 && !goal[u]) released.push_back(u);
    }
    for (int u : released)
      if (u > cand) cand = u;
    for (int u : released)
      if (u != cand) freep.insert(pebble[u]);
    if (cand >= 0) {
      pebble[k] = pebble[cand];
    } else if (!freep.empty()) {
      pebble[k] = *freep.begin();
      freep.erase(freep.begin());
    } else {
      pebble[k] = next++;
    }
  }
  return next;
}

// ---------------------------------------------------------------------------------------
// Device bytecode for the interpreter kernel, with GPU slot allocation: every used
// constant is loaded into a slot first; a goal is stored as soon as it is computed
// (eager stores) and its slot is released after its last operand use (reading R12).
// Slots are assigned by a linear scan over the straight-line order (exact max-live).
//
// Format (uint16 words; the whole program is padded to a multiple of 8 words so it
// can be staged with 16-byte copies):
//   [0] nloads  [1] ninstr  [2] total words  [3] nslots
//   nloads x {const, slot}
//   per instruction: hdr = arity (bits 0-9) | ngoals << 10 (bits 10-13) | has_dst << 15,
//   [dst], goals[ngoals], pad to an even index, operand slots[arity], pad to even.
//   Copy goals are arity-1 instructions without dst; zero goals arity-0 ones.
void build_bytecode(const Slp &s, std::vector<uint16_t> &code, int &nslots, int &maxlive) {
  const int nc = s.n_const, nv = s.n_vars;
  std::vector<int> last_c(nc, -2), last_v(nv, -2);
  for (int k = 0; k < nv; ++k)
    for (int t : s.ins[k].ops) (t < nc ? last_c[t] : last_v[t - nc]) = k;
  std::vector<std::vector<int>> goals_of_var(nv);
  std::vector<int> zero_goals;
  std::vector<std::vector<int>> copies_of_const(nc);
  for (size_t g = 0; g < s.goal.size(); ++g) {
    int t = s.goal[g];
    if (t < 0) zero_goals.push_back((int)g);
    else if (t < nc) copies_of_const[t].push_back((int)g);
    else goals_of_var[t - nc].push_back((int)g);
  }
  std::set<int> freeslots;
  int next = 0, live = 0;
  maxlive = 0;
  auto alloc = [&]() {
    int sl;
    if (!freeslots.empty()) { sl = *freeslots.begin(); freeslots.erase(freeslots.begin()); }
    else sl = next++;
    ++live;
    maxlive = std::max(maxlive, live);
    return sl;
  };
  auto release = [&](int sl) { freeslots.insert(sl); --live; };
  std::vector<int> cslot(nc, -1), vslot(nv, -1);
  std::vector<uint16_t> loads, body;
  int nloads = 0, nins = 0;
  for (int c = 0; c < nc; ++c) {
    if (last_c[c] < -1 && copies_of_const[c].empty()) continue;
    cslot[c] = alloc();
    loads.push_back((uint16_t)c);
    loads.push_back((uint16_t)cslot[c]);
    ++nloads;
  }
  // body offsets are relative to the header + loads (an even number of words)
  auto emit1 = [&](int dst, const std::vector<int> &gl, const std::vector<int> &ops) {
    body.push_back((uint16_t)(ops.size() | (gl.size() << 10) | (dst >= 0 ? 0x8000 : 0)));
    if (dst >= 0) body.push_back((uint16_t)dst);
    for (int g : gl) body.push_back((uint16_t)g);
    if (body.size() & 1) body.push_back(0);
    for (int o : ops) body.push_back((uint16_t)o);
    if (body.size() & 1) body.push_back(0);
    ++nins;
  };
  auto emit = [&](int dst, const std::vector<int> &gl, const std::vector<int> &ops) {
    if (ops.size() > 1023) throw Error(XSLP_EINVAL, "instruction arity > 1023");
    // at most 15 goals per instruction: extra goals recompute the same XOR first
    size_t i = 15;
    for (; i < gl.size(); i += 15)
      emit1(-1, std::vector<int>(gl.begin() + i, gl.begin() + std::min(gl.size(), i + 15)), ops);
    emit1(dst, std::vector<int>(gl.begin(), gl.begin() + std::min<size_t>(gl.size(), 15)), ops);
  };
  if (!zero_goals.empty()) emit(-1, zero_goals, {});
  for (int c = 0; c < nc; ++c) {
    if (copies_of_const[c].empty()) continue;
    emit(-1, copies_of_const[c], {cslot[c]});
    if (last_c[c] < -1) { release(cslot[c]); cslot[c] = -1; }
  }
  for (int k = 0; k < nv; ++k) {
    std::vector<int> ops;
    for (int t : s.ins[k].ops) ops.push_back(t < nc ? cslot[t] : vslot[t - nc]);
    for (int t : s.ins[k].ops) {
      if (t < nc) { if (last_c[t] == k) release(cslot[t]); }
      else if (last_v[t - nc] == k) release(vslot[t - nc]);
    }
    int dst = -1;
    if (last_v[k] > k) dst = vslot[k] = alloc();
    emit(dst, goals_of_var[k], ops);
  }
  nslots = std::max(next, 1);
  code.assign(4, 0);
  code.insert(code.end(), loads.begin(), loads.end());
  code.insert(code.end(), body.begin(), body.end());
  while (code.size() % 8) code.push_back(0);
  code[0] = (uint16_t)nloads;
  code[1] = (uint16_t)nins;
  if (code.size() > 0xffff || nc > 0xffff || nslots > 0x7fff || nins > 0xffff)
    throw Error(XSLP_EINVAL, "program too large for the interpreter bytecode");
  code[2] = (uint16_t)code.size();
  code[3] = (uint16_t)nslots;
}

// ---------------------------------------------------------------------------------------
// Set semantics of a compiled program: the compiler checks its own output.
std::vector<Bits> evaluate(const Slp &s) {
  std::vector<Bits> val(s.n_vars, Bits(s.n_const));
  auto term = [&](int t) {
    if (t < s.n_const) { Bits b(s.n_const); b.set(t); return b; }
    return val[t - s.n_const];
  };
  for (auto &in : s.ins) {
    Bits v(s.n_const);
    for (int t : in.ops) v ^= term(t);
    val[in.var] = v;
  }
  std::vector<Bits> out;
  for (int g : s.goal) out.push_back(g < 0 ? Bits(s.n_const) : term(g));
  return out;
}

static std::string tname(const Slp &s, const std::vector<int> &peb, int t) {
  if (t < 0) return "0";
  if (t < s.n_const) return "c" + std::to_string(t);
  return "p" + std::to_string(peb.empty() ? t - s.n_const : peb[t - s.n_const]);
}

// ---------------------------------------------------------------------------------------
// Abstract LRU cache of P:1007-1022 over the program as dumped (pebble names when
// present): per instruction, touch-or-load the operands in order, then touch-or-allocate
// the target, evicting the least recently used block when full.  Returns loads,
// evictions and reloads (a load of a block that was in the cache before).
struct LruResult { int64_t loads = 0, evictions = 0, reloads = 0; };

static LruResult lru_run(const Slp &s, const std::vector<int> &peb, int cap) {
  const int nc = s.n_const;
  auto name = [&](int t) { return t < nc ? t : nc + (peb.empty() ? t - nc : peb[t - nc]); };
  std::vector<int> cache;  // front = LRU
  std::vector<char> seen;
  LruResult r;
  auto find = [&](int x) { return std::find(cache.begin(), cache.end(), x); };
  auto room = [&]() {
    if ((int)cache.size() >= cap) { cache.erase(cache.begin()); r.evictions++; }
  };
  for (auto &in : s.ins) {
    for (int t : in.ops) {
      int x = name(t);
      if ((int)seen.size() <= x) seen.resize(x + 1, 0);
      auto it = find(x);
      if (it != cache.end()) { cache.erase(it); cache.push_back(x); continue; }
      room();
      r.loads++;
      if (seen[x]) r.reloads++;
      seen[x] = 1;
      cache.push_back(x);
    }
    int x = name(nc + in.var);
    if ((int)seen.size() <= x) seen.resize(x + 1, 0);
    auto it = find(x);
    if (it != cache.end()) { cache.erase(it); cache.push_back(x); continue; }
    room();
    seen[x] = 1;
    cache.push_back(x);
  }
  return r;
}

int64_t lru_iocost(const Slp &s, const std::vector<int> &peb, int cap) {
  for (auto &in : s.ins)
    if ((int)in.ops.size() + 1 > cap) throw Error(XSLP_EINVAL, "capacity smaller than one instruction");
  auto r = lru_run(s, peb, cap);
  return r.loads + r.evictions;
}

// CCap: least capacity without reloads.  LRU has the inclusion property,
// so reload-freedom is monotone in the capacity and a binary search is exact.
int lru_ccap(const Slp &s, const std::vector<int> &peb) {
  int lo = 1, hi = 1;
  std::set<int> names;
  const int nc = s.n_const;
  for (auto &in : s.ins) {
    lo = std::max(lo, (int)in.ops.size() + 1);
    for (int t : in.ops) names.insert(t < nc ? t : nc + (peb.empty() ? t - nc : peb[t - nc]));
    names.insert(nc + (peb.empty() ? in.var : peb[in.var]));
  }
  hi = std::max(lo, (int)names.size());
  if (s.ins.empty()) return 0;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (lru_run(s, peb, mid).reloads == 0) hi = mid; else lo = mid + 1;
  }
  return lo;
}

std::string dump_pebbles(const Slp &s, const std::vector<int> &peb) {
  std::ostringstream o;
  for (auto &in : s.ins) {
    o << tname(s, peb, s.n_const + in.var) << " =";
    for (size_t i = 0; i < in.ops.size(); ++i) o << (i ? " ^ " : " ") << tname(s, peb, in.ops[i]);
    o << "\n";
  }
  o << "return";
  for (int g : s.goal) o << " " << tname(s, peb, g);
  o << "\n";
  return o.str();
}

std::string dump_slots(const std::vector<uint16_t> &code, int n_const) {
  (void)n_const;
  std::ostringstream o;
  const int nl = code[0], ni = code[1];
  size_t pc = 4;
  for (int i = 0; i < nl; ++i, pc += 2) o << "s" << code[pc + 1] << " = c" << code[pc] << "\n";
  for (int k = 0; k < ni; ++k) {
    const int hdr = code[pc++];
    const int arity = hdr & 1023, ng = (hdr >> 10) & 15;
    const int dst = (hdr & 0x8000) ? code[pc++] : -1;
    std::vector<int> gl(code.begin() + pc, code.begin() + pc + ng);
    pc += ng;
    pc += pc & 1;
    std::string name = dst >= 0 ? "s" + std::to_string(dst) : "g" + std::to_string(k);
    std::string rhs;
    for (int a = 0; a < arity; ++a) rhs += (a ? " ^ s" : "s") + std::to_string(code[pc + a]);
    pc += arity + (arity & 1);
    if (arity == 0) {
      for (int g : gl) o << "out " << g << " = 0\n";
      continue;
    }
    o << name << " = " << rhs << "\n";
    for (int g : gl) o << "out " << g << " = " << name << "\n";
  }
  return o.str();
}

// ---------------------------------------------------------------------------------------
// Text format (include/xslp.h) -> SSA Slp.
Slp parse_text(const std::string &text, int n_const) {
  Slp s;
  s.n_const = n_const;
  std::map<std::string, int> cur;  // name -> term
  std::map<int, int> outs;
  std::vector<int> ret;
  bool has_ret = false;
  std::istringstream in(text);
  std::string line;
  auto term = [&](const std::string &w) -> int {
    if (w == "0") return -1;
    if (w.size() > 1 && w[0] == 'c' && std::all_of(w.begin() + 1, w.end(), ::isdigit)) {
      int c = std::stoi(w.substr(1));
      if (c >= n_const) throw Error(XSLP_EINVAL, "constant " + w + " out of range");
      return c;
    }
    auto it = cur.find(w);
    if (it == cur.end()) throw Error(XSLP_EINVAL, "undefined variable " + w);
    return it->second;
  };
  while (std::getline(in, line)) {
    auto h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    std::string w;
    while (ls >> w) tok.push_back(w);
    if (tok.empty() || tok[0] == "slp") continue;
    if (tok[0] == "return") {
      has_ret = true;
      for (size_t i = 1; i < tok.size(); ++i) ret.push_back(term(tok[i]));
      continue;
    }
    if (tok[0] == "out") {
      if (tok.size() != 4 || tok[2] != "=") throw Error(XSLP_EINVAL, "bad out line: " + line);
      outs[std::stoi(tok[1])] = term(tok[3]);
      continue;
    }
    if (tok.size() < 3 || tok[1] != "=") throw Error(XSLP_EINVAL, "bad line: " + line);
    std::vector<int> ops;
    for (size_t i = 2; i < tok.size(); ++i) {
      if (tok[i] == "^") continue;
      int t = term(tok[i]);
      if (t < 0) continue;  // XOR with the empty set
      auto it = std::find(ops.begin(), ops.end(), t);
      if (it != ops.end()) ops.erase(it); else ops.push_back(t);  // x ^ x cancels
    }
    int v = s.n_vars++;
    s.ins.push_back({v, ops});
    cur[tok[0]] = s.term_of_var(v);
  }
  if (has_ret) {
    for (size_t g = 0; g < ret.size(); ++g) outs[(int)g] = ret[g];
  }
  for (size_t g = 0; g < outs.size(); ++g) {
    if (!outs.count((int)g)) throw Error(XSLP_EINVAL, "goals must be numbered 0..m-1");
    s.goal.push_back(outs[(int)g]);
  }
  // single-operand / empty instructions become aliases
  std::vector<int> alias(s.n_vars, -2);
  for (auto &in : s.ins) {
    for (auto &t : in.ops)
      if (t >= n_const && alias[t - n_const] != -2) t = alias[t - n_const];
    std::vector<int> ops;
    for (int t : in.ops) {
      if (t < 0) continue;
      auto it = std::find(ops.begin(), ops.end(), t);
      if (it != ops.end()) ops.erase(it); else ops.push_back(t);
    }
    in.ops = ops;
    if (in.ops.size() < 2) alias[in.var] = in.ops.empty() ? -1 : in.ops[0];
  }
  for (auto &g : s.goal)
    if (g >= n_const && alias[g - n_const] != -2) g = alias[g - n_const];
  std::vector<Ins> ni;
  for (auto &in : s.ins)
    if (alias[in.var] == -2) ni.push_back(in);
  s.ins.swap(ni);
  compact(s);
  return s;
}

}  // namespace xslp

namespace xslp {

// ---------------------------------------------------------------------------------
// Goal split for the PIPE kernel's consumer groups.  The goals [0, m) are cut into k
// contiguous ranges; a range's cost is the issue count of the instructions its goals reach
// (ceil((arity-1)/2) LOP3s + one shared-memory read per constant operand) plus its stores.
// Cut points (every goal for m <= 64, else evenly spaced block boundaries) are chosen by a
// DP minimising the largest range cost; shared temporaries are recomputed per group.
std::vector<Slp> split_goals(const Slp &s, int k) {
  const int m = (int)s.goal.size(), nc = s.n_const;
  if (k < 1) throw Error(XSLP_EINVAL, "split_goals: k < 1");
  std::vector<int> def(s.n_vars, -1);
  for (size_t i = 0; i < s.ins.size(); ++i) def[s.ins[i].var] = (int)i;
  auto reach = [&](int lo, int hi) {
    std::vector<char> keep(s.ins.size(), 0);
    std::vector<int> st;
    for (int g = lo; g < hi; ++g)
      if (s.goal[g] >= nc) st.push_back(def[s.goal[g] - nc]);
    while (!st.empty()) {
      int i = st.back();
      st.pop_back();
      if (i < 0 || keep[i]) continue;
      keep[i] = 1;
      for (int t : s.ins[i].ops)
        if (t >= nc) st.push_back(def[t - nc]);
    }
    return keep;
  };
  auto cost = [&](int lo, int hi) {
    auto keep = reach(lo, hi);
    int64_t c = hi - lo;
    for (size_t i = 0; i < s.ins.size(); ++i) {
      if (!keep[i]) continue;
      const auto &ops = s.ins[i].ops;
      c += ((int64_t)ops.size() - 1 + 1) / 2;
      for (int t : ops) c += t < nc;
    }
    return c;
  };
  std::vector<int> pos;  // candidate cut positions, including 0 and m
  if (m <= 64) {
    for (int g = 0; g <= m; ++g) pos.push_back(g);
  } else {
    const int step = std::max(8, (m / 64 + 7) / 8 * 8);
    for (int g = 0; g < m; g += step) pos.push_back(g);
    pos.push_back(m);
  }
  const int P = (int)pos.size() - 1;  // segments between consecutive positions
  k = std::min(k, std::max(1, P));
  std::map<std::pair<int, int>, int64_t> memo;
  auto C = [&](int a, int b) {  // cost of goals [pos[a], pos[b])
    auto key = std::make_pair(a, b);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int64_t v = cost(pos[a], pos[b]);
    memo[key] = v;
    return v;
  };
  const int64_t INF = INT64_MAX / 4;
  // best[j][b]: min over splits of [0, pos[b]) into j non-empty ranges of the max range cost
  std::vector<std::vector<int64_t>> best(k + 1, std::vector<int64_t>(P + 1, INF));
  std::vector<std::vector<int>> arg(k + 1, std::vector<int>(P + 1, -1));
  best[0][0] = 0;
  for (int j = 1; j <= k; ++j)
    for (int b = j; b <= P; ++b)
      for (int a = j - 1; a < b; ++a) {
        if (best[j - 1][a] >= INF) continue;
        int64_t v = std::max(best[j - 1][a], C(a, b));
        if (v < best[j][b]) { best[j][b] = v; arg[j][b] = a; }
      }
  std::vector<int> cuts(k + 1);
  cuts[k] = P;
  for (int j = k; j >= 1; --j) cuts[j - 1] = arg[j][cuts[j]];
  std::vector<Slp> out;
  for (int j = 0; j < k; ++j) {
    const int lo = pos[cuts[j]], hi = pos[cuts[j + 1]];
    auto keep = reach(lo, hi);
    Slp r;
    r.n_const = s.n_const;
    r.n_vars = s.n_vars;
    for (size_t i = 0; i < s.ins.size(); ++i)
      if (keep[i]) r.ins.push_back(s.ins[i]);
    r.goal = s.goal;
    for (int g = 0; g < m; ++g)
      if (g < lo || g >= hi) r.goal[g] = -2;
    out.push_back(std::move(r));
  }
  return out;
}

}  // namespace xslp
