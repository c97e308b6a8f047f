// Internal declarations of libxslp (product side; shares nothing with oracle/).
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/xslp.h"

namespace xslp {

// ---- errors -------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string &msg);

// ---- GF(2^8) ---------------------------------------------------------
namespace gf {
uint8_t mul(uint8_t a, uint8_t b);
uint8_t inv(uint8_t a);
uint8_t pow(uint8_t a, int e);
// (n+p) x n row-major coding matrix of the given family.
std::vector<uint8_t> coding_matrix(int n, int p, int kind);
// Gauss-Jordan inverse of an n x n matrix; throws Error(XSLP_ESINGULAR).
std::vector<uint8_t> invert(const std::vector<uint8_t> &m, int n);
// x~ lowering of an a x b matrix into (8a) x (8b) bits.
std::vector<uint8_t> to_bits(const std::vector<uint8_t> &m, int a, int b);
}  // namespace gf

// ---- bitset over constants ----------------------------------------------------------
struct Bits {
  std::vector<uint64_t> w;
  Bits() = default;
  explicit Bits(int nbits) : w((nbits + 63) / 64, 0) {}
  void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
  bool get(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
  void flip(int i) { w[i >> 6] ^= 1ull << (i & 63); }
  int count() const {
    int c = 0;
    for (auto x : w) c += __builtin_popcountll(x);
    return c;
  }
  Bits &operator^=(const Bits &o) {
    for (size_t i = 0; i < w.size(); ++i) w[i] ^= o.w[i];
    return *this;
  }
  bool operator==(const Bits &o) const { return w == o.w; }
  bool any() const {
    for (auto x : w)
      if (x) return true;
    return false;
  }
};

// ---- the multi-ary SLP (MultiSLP) -----------------------------------------
// Terms: t < n_const is constant c_t; t >= n_const is variable (t - n_const), i.e.
// the value defined by instruction (t - n_const) of `ins` before scheduling.
struct Ins {
  int var;               // variable id defined here (SSA)
  std::vector<int> ops;  // operand terms
};

struct Slp {
  int n_const = 0;
  int n_vars = 0;                // variables ids are 0..n_vars-1
  std::vector<Ins> ins;          // topologically ordered
  std::vector<int> goal;         // per goal: term (constant, variable+n_const) or -1 = zero
  int term_of_var(int v) const { return n_const + v; }
  bool is_const(int t) const { return t >= 0 && t < n_const; }
};

// A compiled device program.
struct Program {
  xslp_opts opts;
  int n_const = 0, n_goals = 0;
  int n_used_const = 0;           // constants read by the program (TMA rows)
  int64_t const_reads = 0;        // constant operand occurrences (smem reads per word, TMA kernels)
  Slp slp;                         // scheduled program (SSA)
  std::vector<int> pebble;         // paper pebble id per variable
  int nvar = 0;
  xslp_stats stats{};
  // interpreter bytecode (uint16 words) and slot count
  std::vector<Slp> groups;         // PIPE consumer groups: goal-restricted sub-programs (opts.groups > 1)
  std::vector<Slp> phases;         // PIPE input phases: programs over contiguous input-block ranges
  std::vector<Slp> streams;        // TMEM interpreter: goals [0, R/2) and [R/2, R) compiled apart
  int stage_used_const = 0;        // constants per PIPE stage fill (max over phases, or n_used_const)
  std::vector<uint16_t> code;
  int nslots = 0;
  // straight-line kernel(s): generic addressing + optional baked strip size
  std::string ptx_generic, ptx_baked;
  std::vector<char> cubin_generic, cubin_baked;
  int64_t baked_strip = 0;
  // device state, per device ordinal
  struct Dev;
  mutable std::mutex mu;
  mutable std::map<int, std::shared_ptr<Dev>> dev;
  ~Program();
};

// compiler passes (compiler.cpp)
Slp lift(const std::vector<Bits> &goals, int n_const, bool multi);
Slp compress(const std::vector<Bits> &goals, int n_const, bool xor_rebuild);
void fuse(Slp &s);
void schedule_dfs(Slp &s, int goal_order);
int paper_pebbles(const Slp &s, std::vector<int> &pebble);
int schedule_greedy(Slp &s, int cap, std::vector<int> &pebble);
void build_bytecode(const Slp &s, std::vector<uint16_t> &code, int &nslots, int &maxlive);
std::vector<Bits> evaluate(const Slp &s);
std::string dump_pebbles(const Slp &s, const std::vector<int> &pebble);
int64_t lru_iocost(const Slp &s, const std::vector<int> &peb, int cap);
int lru_ccap(const Slp &s, const std::vector<int> &peb);
std::string dump_slots(const std::vector<uint16_t> &code, int n_const);
Slp parse_text(const std::string &text, int n_const);

// PTX (ptx.cpp).  `reuse`: constant register reuse window of the TMA-staged kernels in
// instructions (0 = a fresh shared-memory read at every use); see xslp_opts.reuse.
std::string emit_ptx(const Slp &s, int lanes, int64_t baked_strip, int threads, int min_blocks,
                     int stages, int layout, const std::vector<Slp> *groups = nullptr,
                     const std::vector<Slp> *phases = nullptr, int reuse = 0);
// xslp_opts.reuse -> window: 0 = auto (the kernel family's default), -1 = off
inline int reuse_window(int opt, int auto_window) { return opt == 0 ? auto_window : opt < 0 ? 0 : opt; }
// Split the goals into k contiguous sets balanced by issue cost; each result keeps the
// instructions its goals reach (original order and variable ids) and marks the other goals -2.
std::vector<Slp> split_goals(const Slp &s, int k);
// Paired micro-op code of the pipelined interpreter (interp.cu): the stage-0 code variant of
// this program alone for T consumers, L words per thread, S stages (xslp_program_dump form 3).
std::vector<uint32_t> interp_code_dump(const Slp &s, int T, int L, int S);
// The lane-parallel interpreter's code (interp_lanes.cu; xslp_program_dump form 4).
std::vector<uint32_t> interp_lanes_dump(const Program *p, int S);
// The TMEM interpreter's code (interp_tmem.cu; xslp_program_dump form 5).
std::vector<uint32_t> interp_tmem_dump(const Program *p, int form);
// Input-phase programs of a goal set (capi.cpp; PIPE input phases and the phased multi kernel).
std::vector<Slp> stream_programs(const std::vector<Bits> &want, int n_const, const xslp_opts &o);
std::vector<Slp> phase_programs(const std::vector<Bits> &want, int n_const, int nphases,
                                const xslp_opts &o, int64_t *xor_total);
// One persistent pipeline kernel (entry xslp_sl_multi) over several programs with the same
// constants/goals, dispatching per stripe through a branch table.
std::string emit_ptx_multi(const std::vector<const Slp *> &progs, int lanes, int64_t baked_strip,
                           int threads, int stages, int reuse = 0);
// bitmatrix -> compiled program (capi.cpp)
std::shared_ptr<Program> compile_bits(const std::vector<uint8_t> &bits, int out_rows, int in_cols,
                                      const xslp_opts &o);
// syndrome-form decode math (syndrome.cpp)
std::vector<uint8_t> parity_check(const uint8_t *g, int n, int p);
std::vector<uint8_t> solve_rows(const std::vector<uint8_t> &h, int n, int p, const std::vector<int> &er);
// Syndrome-form decode kernel (entry xslp_sl_multi): the shared syndrome program in input
// phases `syn`, then per-pattern solve programs (constants = the 8p syndrome words).
std::string emit_ptx_syndrome(const std::vector<Slp> &syn, const std::vector<const Slp *> &solves,
                              int n_out, int lanes, int64_t baked_strip, int threads, int stages,
                              int reuse = 0);
// The same with input phases: phased[k][ph] = phase ph's program of table entry k.
std::string emit_ptx_multi_phases(const std::vector<std::vector<const Slp *>> &phased, int lanes,
                                  int64_t baked_strip, int threads, int stages, int reuse = 0);
std::vector<char> ptx_to_cubin(const std::string &ptx, int *regs, int *spill, int *regs_tma,
                               int *spill_tma, int *regs_pipe, int *spill_pipe);

}  // namespace xslp
