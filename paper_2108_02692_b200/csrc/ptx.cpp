// Straight-line specialisation: the scheduled MultiSLP emitted as PTX for sm_100a and
// compiled in-process to a cubin (nvPTXCompiler, no GPU needed).
//
// Execution model: a thread owns `lanes` consecutive 32-bit
// words at one offset of every strip of its stripe (coalesced: a warp reads
// 128*lanes contiguous bytes of each strip).  Constants are loaded from HBM once,
// every variable of the SLP is a register, each variadic XOR of arity a becomes
// ceil((a-1)/2) 3-input XORs (lop3.b32 with truth table 0x96), and each goal is stored
// as soon as it is computed.  This is the paper's blocked interpreter loop
// ([Peb]) with the block = one thread's words and "cache" = registers.
//
// Two entries per module:
//   xslp_sl_batch(in_tbl, out_tbl, stripe_ids, strip_bytes, words, stripe_base)
//     stripe = stripe_ids ? stripe_ids[ctaid.y + stripe_base] : ctaid.y + stripe_base;
//     block pointers from the device tables in_tbl[stripe*n_in + j], out_tbl[stripe*n_out + i]
//   xslp_sl_one(ptrs[128], strip_bytes, words)
//     one stripe, pointers passed by value (in[0..n_in), out[n_in..n_in+n_out))
// With a baked strip size the 8 strips of a block are addressed by immediate offsets.
#include <functional>
#include <map>
#include <sstream>

#include <nvPTXCompiler.h>

#include "xslp_internal.h"

namespace xslp {

namespace {

struct Emitter {
  const Slp *sp;                  // the program being emitted (a group's sub-program in PIPE)
  const Slp &full;                // the whole program (declarations, other entries)
  const std::vector<Slp> *groups; // PIPE consumer groups, or nullptr
  const std::vector<Slp> *phases = nullptr; // PIPE input phases (K-split), or nullptr
  int L;
  int64_t baked;
  int threads;
  int min_blocks;
  int stages;
  int layout;
  int n_in, n_out;
  std::ostringstream o;
  Emitter(const Slp &s_, int L_, int64_t baked_, int threads_, int min_blocks_, int stages_,
          int layout_, const std::vector<Slp> *groups_)
      : sp(&s_), full(s_), groups(groups_), L(L_), baked(baked_), threads(threads_), min_blocks(min_blocks_), stages(stages_),
        layout(layout_),
        n_in(s_.n_const / 8),
        n_out((int)(s_.goal.size() / 8)) {}
  const Slp &cur() const { return *sp; }
  int decl_vars = -1, decl_nq = -1;  // register declaration sizes when several programs share a body

  std::string creg(int c, int l) {
    if (acc_consts) return "%acc" + std::to_string(c * L + l);  // syndrome solve: constants = %acc
    return "%c" + std::to_string(c * L + l);
  }
  bool acc_consts = false;
  std::string vreg(int v, int l) { return "%v" + std::to_string(v * L + l); }
  std::string treg(int t, int l) { return t < cur().n_const ? creg(t, l) : vreg(t - cur().n_const, l); }

  const char *vsuf() { return L == 1 ? ".u32" : (L == 2 ? ".v2.u32" : ".v4.u32"); }
  std::string vec(const std::vector<std::string> &r) {
    if (L == 1) return r[0];
    std::string x = "{";
    for (int l = 0; l < L; ++l) x += (l ? ", " : "") + r[l];
    return x + "}";
  }

  // address of strip k of block register `base` (already offset by the thread's word)
  std::string addr(const std::string &base, int k, int &tmpctr) {
    if (k == 0) return "[" + base + "]";
    if (baked > 0) return "[" + base + "+" + std::to_string((int64_t)k * baked) + "]";
    std::string t = "%ta" + std::to_string(tmpctr++);
    o << "  add.s64 " << t << ", " << base << ", %sk" << k << ";\n";
    return "[" + t + "]";
  }

  // mode 0: batch, constants loaded from HBM into registers (LDG)
  // mode 1: one stripe, pointers in the parameter block (LDG)
  // mode 2: batch, the CTA's tile of every constant strip staged into shared memory by
  //         TMA bulk copies (cp.async.bulk, one mbarrier), constants read from smem at use
  void body(int mode) {
    const bool one = mode == 1, tma = mode == 2;
    const int nc = cur().n_const;
    std::vector<char> used(nc, 0);
    for (size_t k = 0; k < cur().ins.size(); ++k)
      for (int t : cur().ins[k].ops)
        if (t < nc) used[t] = 1;
    for (int g : cur().goal)
      if (g >= 0 && g < nc) used[g] = 1;
    std::vector<char> blk_used(n_in, 0);
    std::vector<int> slot(nc, -1);
    int nused = 0;
    for (int c = 0; c < nc; ++c)
      if (used[c]) { blk_used[c / 8] = 1; slot[c] = nused++; }
    const int rowb = 4 * L * threads;  // smem bytes per constant row (TMA mode)

    o << "  mov.u32 %s0, %ctaid.x;\n  mov.u32 %s1, %ntid.x;\n  mov.u32 %s2, %tid.x;\n";
    o << "  mad.lo.u32 %s3, %s0, %s1, %s2;\n";
    o << "  ld.param.u32 %s4, [p_words];\n";
    if (!tma) o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $DONE;\n";
    o << "  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    if (!one) {
      o << "  mov.u32 %s5, %ctaid.y;\n  ld.param.u32 %s6, [p_base];\n  add.u32 %s5, %s5, %s6;\n";
      o << "  ld.param.u64 %rd0, [p_ids];\n  setp.eq.u64 %p1, %rd0, 0;\n  @%p1 bra $NOIDS;\n";
      o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n";
      o << "  ld.global.nc.u32 %s5, [%rd1];\n$NOIDS:\n";
      o << "  ld.param.u64 %rd2, [p_in];\n  ld.param.u64 %rd3, [p_out];\n";
      o << "  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
      o << "  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    }
    int tmp = 0;
    if (tma) {
      // tile = words [ctaid.x*T, +T) of every strip; bytes per strip this tile
      o << "  mul.lo.u32 %s7, %s0, " << threads << ";\n";          // first group of the tile
      o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << threads << ";\n";
      o << "  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
      o << "  mov.u32 %sb, dsm;\n";
      o << "  setp.ne.u32 %p2, %s2, 0;\n  @%p2 bra $INIT;\n";
      o << "  mbarrier.init.shared::cta.b64 [%sb], 1;\n  fence.mbarrier_init.release.cluster;\n";
      o << "$INIT:\n  bar.sync 0;\n  @%p2 bra $WAIT;\n";
      o << "  mul.lo.u32 %s6, %nb, " << nused << ";\n";
      o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%sb], %s6;\n";
      o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
      for (int j = 0; j < n_in; ++j) {
        if (!blk_used[j]) continue;
        o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
        o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
      }
      for (int c = 0; c < nc; ++c) {
        if (!used[c]) continue;
        std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
        o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%sb+"
          << 128 + slot[c] * rowb << "], " << a << ", %nb, [%sb];\n";
      }
      o << "$WAIT:\n  mbarrier.try_wait.parity.shared::cta.b64 %p3, [%sb], 0;\n  @!%p3 bra $WAIT;\n";
      o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $DONE;\n";
      o << "  mul.lo.u32 %sth, %s2, " << 4 * L << ";\n  add.u32 %sth, %sth, %sb;\n";
    } else {
      for (int j = 0; j < n_in; ++j) {
        if (!blk_used[j]) continue;
        if (one) o << "  ld.param.u64 %ib" << j << ", [p_ptrs+" << 8 * j << "];\n";
        else o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
        o << "  add.s64 %ib" << j << ", %ib" << j << ", %off;\n";
      }
    }
    for (int i = 0; i < n_out; ++i) {
      if (one) o << "  ld.param.u64 %ob" << i << ", [p_ptrs+" << 8 * (n_in + i) << "];\n";
      else o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
      o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
    }
    compute(tma, 128, slot, used, tmp);
    o << "$DONE:\n  ret;\n";
  }

  // ---- pieces shared by the pipelined kernels (a producer warp + consumer warps) ----------
  // Shared memory [0, 8S): full barriers (one arrival: the producer's expect_tx, completed by
  // the TMA bytes); [8S, 16S): empty barriers (one arrival per consumer warp).  Stage use %it
  // of a CTA lives in stage %it % S with phase parity (%it / S) & 1.
  void pipe_barriers(int S, int consumer_warps) {
    o << "  mov.u32 %s2, %tid.x;\n  mov.u32 %sb, dsm;\n";
    o << "  setp.ne.u32 %p2, %s2, 0;\n  @%p2 bra $INIT;\n";
    for (int k = 0; k < S; ++k) {
      o << "  mbarrier.init.shared::cta.b64 [%sb+" << 8 * k << "], 1;\n";
      o << "  mbarrier.init.shared::cta.b64 [%sb+" << 8 * S + 8 * k << "], " << consumer_warps << ";\n";
    }
    o << "  fence.mbarrier_init.release.cluster;\n$INIT:\n  bar.sync 0;\n";
  }
  // %st, %ph (raw phase count) and %fb (full barrier) of stage use %it
  void stage_regs(int S) {
    o << "  rem.u32 %st, %it, " << S << ";\n  div.u32 %ph, %it, " << S << ";\n";
    o << "  mad.lo.u32 %fb, %st, 8, %sb;\n";
  }
  // consumer: wait until the producer's fill of this stage use has landed
  void consumer_wait(int S, const std::string &x) {
    stage_regs(S);
    o << "  and.b32 %ph, %ph, 1;\n";
    o << "$CW" << x << ":\n  mbarrier.try_wait.parity.shared::cta.b64 %p3, [%fb], %ph;\n  @!%p3 bra $CW" << x << ";\n";
  }
  // consumer: $CSKIP<x> (threads without a word jump here), then one arrival per warp on the
  // stage's empty barrier; ends at $CNEXT<x>
  void consumer_release(int S, const std::string &x) {
    o << "$CSKIP" << x << ":\n  bar.warp.sync -1;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $CNEXT" << x << ";\n";
    o << "  add.u32 %eb, %fb, " << 8 * S << ";\n  mbarrier.arrive.shared::cta.b64 _, [%eb];\n";
    o << "$CNEXT" << x << ":\n";
  }
  // producer (after stage_regs): from the second round on, wait until the consumers drained
  // the stage's previous fill
  void producer_wait(int S, const std::string &x) {
    o << "  setp.lt.u32 %p5, %it, " << S << ";\n  @%p5 bra $PNW" << x << ";\n";
    o << "  sub.u32 %ph, %ph, 1;\n  and.b32 %ph, %ph, 1;\n  add.u32 %eb, %fb, " << 8 * S << ";\n";
    o << "$PW" << x << ":\n  mbarrier.try_wait.parity.shared::cta.b64 %p3, [%eb], %ph;\n  @!%p3 bra $PW" << x << ";\n";
    o << "$PNW" << x << ":\n";
  }

  // Persistent, warp-specialised TMA pipeline (entry xslp_sl_pipe).  threads = consumer
  // threads TC (NCW warps) plus one producer warp.  Each CTA walks tiles
  // tile = ctaid.x + i*nctaid.x (tile -> stripe = tile / tps, tw = tile % tps; a tile is
  // TC lane-groups of every strip); S shared-memory stages of nused rows x 4*L*TC bytes.
  // Producer (lane 0 of the last warp): wait empty[st] -> expect_tx on full[st] ->
  // cp.async.bulk every used strip segment into the stage.  Consumers: wait full[st] ->
  // run the program reading the stage -> stores -> one arrive per warp on empty[st].
  void body_pipe(int S) {
    const int nc = cur().n_const;
    const int TC = threads, NCW = threads / 32;
    const int G = groups ? (int)groups->size() : 1;  // consumer groups, NCW warps each
    std::vector<char> used(nc, 0);
    for (size_t k = 0; k < cur().ins.size(); ++k)
      for (int t : cur().ins[k].ops)
        if (t < nc) used[t] = 1;
    for (int g : cur().goal)
      if (g >= 0 && g < nc) used[g] = 1;
    std::vector<char> blk_used(n_in, 0);
    std::vector<int> slot(nc, -1);
    int nused = 0;
    for (int c = 0; c < nc; ++c)
      if (used[c]) { blk_used[c / 8] = 1; slot[c] = nused++; }
    const int rowb = 4 * L * TC;
    const int64_t STAGE = (int64_t)nused * rowb;
    pipe_barriers(S, G * NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n  setp.ne.u64 %pids, %rd0, 0;\n";
    o << "  mov.u32 %nct, %nctaid.x;\n";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << G * NCW << ";\n  @%pprod bra $PROD;\n";
    // consumer group of this warp and the thread's column within the group
    o << "  div.u32 %grp, %wid, " << NCW << ";\n  mul.lo.u32 %ltid, %grp, " << TC << ";\n";
    o << "  sub.u32 %ltid, %s2, %ltid;\n";
    for (int g = 1; g < G; ++g)
      o << "  setp.eq.u32 %p5, %grp, " << g << ";\n  @%p5 bra $C" << g << "START;\n";
    // helper: stripe of %tile -> %s5, tile-in-strip -> %tw
    auto stripe_of = [&](const char *lab) {
      o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
      o << "  @!%pids bra " << lab << ";\n";
      o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
      o << lab << ":\n";
    };
    // ---------------- consumers (one loop per group; group g runs its sub-program)
    for (int g = 0; g < G; ++g) {
      const std::string x = std::to_string(g);
      if (groups) sp = &(*groups)[g];
      o << "$C" << x << "START:\n";
      o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n  mov.u32 %lane, %laneid;\n";
      o << "$CLOOP" << x << ":\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
      consumer_wait(S, x);
      stripe_of(("$CID" + x).c_str());
      o << "  mad.lo.u32 %s3, %tw, " << TC << ", %ltid;\n";
      o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $CSKIP" << x << ";\n";
      o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
      o << "  mad.lo.u32 %sth, %ltid, " << 4 * L << ", %sth;\n  add.u32 %sth, %sth, 128;\n";
      if (pipe_one)   // single stripe: the block pointers are kernel parameters (p_ptrs)
        o << "  mov.u64 %rd3, p_ptrs;\n  cvta.param.u64 %rd3, %rd3;\n  add.s64 %rd3, %rd3, " << 8 * n_in << ";\n";
      else
        o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
      o << "  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
      std::vector<char> oused(n_out, 0);
      for (int q = 0; q < (int)cur().goal.size(); ++q)
        if (cur().goal[q] != -2) oused[q / 8] = 1;
      for (int i = 0; i < n_out; ++i) {
        if (!oused[i]) continue;
        o << (pipe_one ? "  ld.u64 %ob" : "  ld.global.nc.u64 %ob") << i << ", [%rd3+" << 8 * i << "];\n";
        o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
      }
      int tmp = 0;
      compute(true, 0, slot, used, tmp);
      consumer_release(S, x);
      o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, %nct;\n  bra.uni $CLOOP" << x << ";\n";
    }
    sp = &full;
    int tmp = 0;
    // ---------------- producer
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
    stage_regs(S);
    producer_wait(S, "");
    stripe_of("$PID");
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
    o << "  mul.lo.u32 %s6, %nb, " << nused << ";\n";
    o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
    if (pipe_one)
      o << "  mov.u64 %rd2, p_ptrs;\n  cvta.param.u64 %rd2, %rd2;\n";
    else
      o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
    for (int j = 0; j < n_in; ++j) {
      if (!blk_used[j]) continue;
      o << (pipe_one ? "  ld.u64 %ib" : "  ld.global.nc.u64 %ib") << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
    }
    o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
    for (int c = 0; c < nc; ++c) {
      if (!used[c]) continue;
      std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
      o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
        << 128 + (int64_t)slot[c] * rowb << "], " << a << ", %nb, [%fb];\n";
    }
    o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, %nct;\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  // Byte-compatible layout: blocks are plain byte arrays and the
  // output equals textbook byte-wise RS.  The SLP runs on bit-planes: a
  // thread owns a 32-byte chunk of every block (one 256-bit load), and an in-register 8x8
  // bit transpose per byte lane turns the 8 words W_i into 8 plane words P_k with
  // P_k bit (8m+i) = bit k of byte 4i+m (so constant c_{8j+k} is plane k of block j).
  // Goals are transposed back per output block (the network is an involution) and
  // stored with one 256-bit store when the block's 8 planes are complete.
  void transpose8(const std::vector<std::string> &w) {
    static const int S[3] = {4, 2, 1};
    static const char *MASK[3] = {"0x0F0F0F0F", "0x33333333", "0x55555555"};
    static const int PAIRS[3][4][2] = {{{0, 4}, {1, 5}, {2, 6}, {3, 7}},
                                       {{0, 2}, {1, 3}, {4, 6}, {5, 7}},
                                       {{0, 1}, {2, 3}, {4, 5}, {6, 7}}};
    for (int st = 0; st < 3; ++st)
      for (int q = 0; q < 4; ++q) {
        const std::string &a = w[PAIRS[st][q][0]], &b = w[PAIRS[st][q][1]];
        o << "  shr.b32 %tx0, " << a << ", " << S[st] << ";\n";
        o << "  xor.b32 %tx0, %tx0, " << b << ";\n  and.b32 %tx0, %tx0, " << MASK[st] << ";\n";
        o << "  xor.b32 " << b << ", " << b << ", %tx0;\n";
        o << "  shl.b32 %tx0, %tx0, " << S[st] << ";\n  xor.b32 " << a << ", " << a << ", %tx0;\n";
      }
  }

  // constants read by the program: per input block, any of its 8 planes used
  std::vector<char> byte_blocks_used() {
    const int nc = cur().n_const;
    std::vector<char> used(nc, 0), blk(n_in, 0);
    for (auto &in : cur().ins)
      for (int t : in.ops)
        if (t < nc) used[t] = 1;
    for (int g : cur().goal)
      if (g >= 0 && g < nc) used[g] = 1;
    for (int c = 0; c < nc; ++c)
      if (used[c]) blk[c / 8] = 1;
    return blk;
  }

  // The byte-layout program on one 32-byte chunk of every block: `load(j, w)` brings block
  // j's 8 words into registers w; they are transposed into bit-planes, the SLP runs, and each
  // output block is transposed back and stored (256-bit) once its 8 goals exist.  %ob<i> must
  // address the thread's chunk of output block i.
  void byte_compute(const std::function<void(int, const std::vector<std::string> &)> &load) {
    const int nc = cur().n_const;
    auto blk = byte_blocks_used();
    for (int j = 0; j < n_in; ++j) {
      if (!blk[j]) continue;
      std::vector<std::string> w;
      for (int k = 0; k < 8; ++k) w.push_back(creg(8 * j + k, 0));
      load(j, w);
      transpose8(w);
    }
    // when is each output block complete?
    std::vector<int> ready_at(n_out, -1);  // instruction index after which all 8 goals exist
    for (int g = 0; g < (int)cur().goal.size(); ++g) {
      int t = cur().goal[g], at = -1;
      if (t >= nc) at = t - nc;  // var ids equal instruction positions (compacted)
      ready_at[g / 8] = std::max(ready_at[g / 8], at);
    }
    auto gval = [&](int g) {
      int t = cur().goal[g];
      if (t < 0) return std::string("%zero");
      return treg(t, 0);
    };
    auto store_block = [&](int i) {
      std::vector<std::string> y;
      for (int r = 0; r < 8; ++r) {
        std::string reg = "%y" + std::to_string(r);
        o << "  mov.b32 " << reg << ", " << gval(8 * i + r) << ";\n";
        y.push_back(reg);
      }
      transpose8(y);
      o << "  st.global.v8.u32 [%ob" << i << "], {";
      for (int r = 0; r < 8; ++r) o << (r ? ", " : "") << y[r];
      o << "};\n";
    };
    for (int i = 0; i < n_out; ++i)
      if (ready_at[i] < 0) store_block(i);
    for (size_t k = 0; k < cur().ins.size(); ++k) {
      const auto &in = cur().ins[k];
      const auto &ops = in.ops;
      std::string d = vreg(in.var, 0);
      size_t i;
      if (ops.size() == 2) {
        o << "  xor.b32 " << d << ", " << treg(ops[0], 0) << ", " << treg(ops[1], 0) << ";\n";
      } else {
        o << "  lop3.b32 " << d << ", " << treg(ops[0], 0) << ", " << treg(ops[1], 0) << ", "
          << treg(ops[2], 0) << ", 0x96;\n";
        for (i = 3; i + 1 < ops.size(); i += 2)
          o << "  lop3.b32 " << d << ", " << d << ", " << treg(ops[i], 0) << ", " << treg(ops[i + 1], 0)
            << ", 0x96;\n";
        if (i < ops.size()) o << "  xor.b32 " << d << ", " << d << ", " << treg(ops[i], 0) << ";\n";
      }
      for (int b = 0; b < n_out; ++b)
        if (ready_at[b] == (int)k) store_block(b);
    }
  }

  void body_byte(bool one) {
    o << "  mov.u32 %s0, %ctaid.x;\n  mov.u32 %s1, %ntid.x;\n  mov.u32 %s2, %tid.x;\n";
    o << "  mad.lo.u32 %s3, %s0, %s1, %s2;\n  ld.param.u32 %s4, [p_words];\n";
    o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $DONE;\n  mul.wide.u32 %off, %s3, 32;\n";
    if (!one) {
      o << "  mov.u32 %s5, %ctaid.y;\n  ld.param.u32 %s6, [p_base];\n  add.u32 %s5, %s5, %s6;\n";
      o << "  ld.param.u64 %rd0, [p_ids];\n  setp.eq.u64 %p1, %rd0, 0;\n  @%p1 bra $NOIDS;\n";
      o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n";
      o << "  ld.global.nc.u32 %s5, [%rd1];\n$NOIDS:\n";
      o << "  ld.param.u64 %rd2, [p_in];\n  ld.param.u64 %rd3, [p_out];\n";
      o << "  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
      o << "  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    }
    auto blk = byte_blocks_used();
    for (int j = 0; j < n_in; ++j) {
      if (!blk[j]) continue;
      if (one) o << "  ld.param.u64 %ib" << j << ", [p_ptrs+" << 8 * j << "];\n";
      else o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %off;\n";
    }
    for (int i = 0; i < n_out; ++i) {
      if (one) o << "  ld.param.u64 %ob" << i << ", [p_ptrs+" << 8 * (n_in + i) << "];\n";
      else o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
      o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
    }
    byte_compute([&](int j, const std::vector<std::string> &w) {
      o << "  ld.global.nc.L1::no_allocate.v8.u32 {";
      for (int k = 0; k < 8; ++k) o << (k ? ", " : "") << w[k];
      o << "}, [%ib" << j << "];\n";
    });
    o << "$DONE:\n  ret;\n";
  }

  // Byte layout through the TMA pipeline (entry xslp_sl_pipe of a byte-layout module): the
  // producer warp copies the tile's T 32-byte chunks of every used input block (one bulk copy
  // per block) into a stage row; consumers read their chunk with two 128-bit shared loads and
  // run byte_compute.  "words" are 32-byte chunks here.
  void body_pipe_byte(int S) {
    const int TC = threads, NCW = threads / 32;
    auto blk = byte_blocks_used();
    std::vector<int> bslot(n_in, -1);
    int nub = 0;
    for (int j = 0; j < n_in; ++j)
      if (blk[j]) bslot[j] = nub++;
    const int ROWB = 32 * TC;
    const int64_t STAGE = (int64_t)std::max(1, nub) * ROWB;
    pipe_barriers(S, NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n  setp.ne.u64 %pids, %rd0, 0;\n";
    o << "  mov.u32 %nct, %nctaid.x;\n";
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << NCW << ";\n  @%pprod bra $PROD;\n";
    auto stripe_of = [&](const std::string &lab) {
      o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
      o << "  @!%pids bra " << lab << ";\n";
      o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
      o << lab << ":\n";
    };
    // ---------------- consumers
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n  mov.u32 %lane, %laneid;\n";
    o << "$CLOOP:\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
    consumer_wait(S, "");
    stripe_of("$CID");
    o << "  mad.lo.u32 %s3, %tw, " << TC << ", %s2;\n";
    o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $CSKIP;\n";
    o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
    o << "  mad.lo.u32 %sth, %s2, 32, %sth;\n  add.u32 %sth, %sth, 128;\n";
    o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    o << "  mul.wide.u32 %off, %s3, 32;\n";
    for (int i = 0; i < n_out; ++i) {
      o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
      o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
    }
    byte_compute([&](int j, const std::vector<std::string> &w) {
      const int64_t at = (int64_t)bslot[j] * ROWB;
      o << "  ld.shared.v4.u32 {" << w[0] << ", " << w[1] << ", " << w[2] << ", " << w[3] << "}, [%sth+" << at << "];\n";
      o << "  ld.shared.v4.u32 {" << w[4] << ", " << w[5] << ", " << w[6] << ", " << w[7] << "}, [%sth+" << at + 16 << "];\n";
    });
    consumer_release(S, "");
    o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, %nct;\n  bra.uni $CLOOP;\n";
    // ---------------- producer
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
    stage_regs(S);
    producer_wait(S, "");
    stripe_of("$PID");
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, 32;\n";
    o << "  mul.lo.u32 %s6, %nb, " << nub << ";\n";
    o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
    o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.wide.u32 %toff, %s7, 32;\n";
    o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
    for (int j = 0; j < n_in; ++j) {
      if (!blk[j]) continue;
      o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
      o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
        << 128 + (int64_t)bslot[j] * ROWB << "], [%ib" << j << "], %nb, [%fb];\n";
    }
    o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, %nct;\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  // The straight-line program over this thread's words: constants come from HBM (LDG,
  // all issued up front) or, when `smem`, from shared-memory rows at [%sth + off0 +
  // slot*rowb] with a fresh volatile read per use; goals are stored when computed.
  void compute(bool tma, int off0, const std::vector<int> &slot, const std::vector<char> &used,
               int &tmp) {
    const int nc = cur().n_const;
    const int rowb = 4 * L * threads;
    std::vector<char> loaded(nc, 0);
    auto need = [&](int c) {  // make constant c available in registers
      if (acc_consts) return;   // already in %acc
      if (loaded[c]) return;
      loaded[c] = 1;
      std::vector<std::string> r;
      for (int l = 0; l < L; ++l) r.push_back(creg(c, l));
      if (tma)
        o << "  ld.shared" << vsuf() << " " << vec(r) << ", [%sth+" << off0 + slot[c] * rowb << "];\n";
      else {
        std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);  // may emit an add
        o << "  ld.global.nc.L1::no_allocate" << vsuf() << " " << vec(r) << ", " << a << ";\n";
      }
    };
    // LDG: every used constant up front (maximum memory-level parallelism; ptxas
    // schedules them against register pressure).  TMA: smem reads at first use.
    if (!tma)
      for (int c = 0; c < nc; ++c)
        if (used[c]) need(c);
    // goals that are constants or zero
    std::vector<std::vector<int>> goals_of_var(cur().n_vars);
    for (size_t g = 0; g < cur().goal.size(); ++g) {
      int t = cur().goal[g];
      if (t == -2) continue;  // another consumer group's goal (PIPE split)
      if (t >= nc) { goals_of_var[t - nc].push_back((int)g); continue; }
      if (t >= 0) need(t);
      std::vector<std::string> r;
      for (int l = 0; l < L; ++l) r.push_back(t < 0 ? std::string("%zero") : creg(t, l));
      store((int)g, r, tmp);
    }
    // the program
    int qn = 0;
    // TMA: a constant read within the last `reuse` instructions keeps its register instead of
    // a fresh shared-memory read (0 = a fresh read at every use)
    std::map<int, std::pair<int, int>> lastq;  // constant -> (register index, last use)
    for (size_t k = 0; k < cur().ins.size(); ++k) {
      const auto &in = cur().ins[k];
      const auto &ops = in.ops;
      std::map<int, int> q;  // TMA: constant -> register for this instruction
      for (int t : ops) {
        if (t >= nc) continue;
        if (!tma) { need(t); continue; }
        auto lq = lastq.find(t);
        if (reuse > 0 && lq != lastq.end() && (int)k - lq->second.second <= reuse) {
          q[t] = lq->second.first;
          lq->second.second = (int)k;
          continue;
        }
        lastq[t] = {qn, (int)k};
        q[t] = qn;
        std::vector<std::string> r;
        for (int l = 0; l < L; ++l) r.push_back("%q" + std::to_string(qn * L + l));
        ++qn;
        // volatile: ptxas must not merge repeated reads and keep constants live in
        // registers (that would recreate the register pressure TMA staging removes)
        o << "  ld.volatile.shared" << vsuf() << " " << vec(r) << ", [%sth+" << off0 + slot[t] * rowb << "];\n";
      }
      auto treg = [&](int t, int l) {
        if (tma && t < nc) return "%q" + std::to_string(q[t] * L + l);
        return this->treg(t, l);
      };
      for (int l = 0; l < L; ++l) {
        std::string d = vreg(in.var, l);
        size_t i;
        if (ops.size() == 2) {
          o << "  xor.b32 " << d << ", " << treg(ops[0], l) << ", " << treg(ops[1], l) << ";\n";
          continue;
        }
        o << "  lop3.b32 " << d << ", " << treg(ops[0], l) << ", " << treg(ops[1], l) << ", "
          << treg(ops[2], l) << ", 0x96;\n";
        for (i = 3; i + 1 < ops.size(); i += 2)
          o << "  lop3.b32 " << d << ", " << d << ", " << treg(ops[i], l) << ", "
            << treg(ops[i + 1], l) << ", 0x96;\n";
        if (i < ops.size()) o << "  xor.b32 " << d << ", " << d << ", " << treg(ops[i], l) << ";\n";
      }
      for (int g : goals_of_var[in.var]) {
        std::vector<std::string> r;
        for (int l = 0; l < L; ++l) r.push_back(vreg(in.var, l));
        store(g, r, tmp);
      }
    }
  }

  void store(int g, const std::vector<std::string> &r, int &tmp) {
    if (accumulate) {  // input phases: goal partials are XORed into %acc, stored after the last
      if (r[0] == "%zero") return;
      for (int l = 0; l < L; ++l) {
        const std::string acc = "%acc" + std::to_string(g * L + l);
        o << "  xor.b32 " << acc << ", " << acc << ", " << r[l] << ";\n";
      }
      return;
    }
    std::string a = addr("%ob" + std::to_string(g / 8), g % 8, tmp);
    o << "  st.global" << vsuf() << " " << a << ", " << vec(r) << ";\n";
  }
  bool accumulate = false;
  bool pipe_one = false;   // body_pipe for one stripe: block pointers in the p_ptrs parameter
  bool multi_acc = false;  // phased multi-program kernel: declare the accumulators
  int reuse = 0;   // constant register reuse window in instructions (xslp_opts.reuse)

  void decls(int ntmp_guess) {
    o << "  .reg .pred %p<5>;\n  .reg .b32 %s<8>;\n  .reg .b64 %rd<8>;\n  .reg .b64 %off;\n";
    o << "  .reg .b32 %zero;\n";
    o << "  .reg .b64 %sk<8>;\n";
    o << "  .reg .b64 %ib<" << std::max(1, n_in) << ">;\n  .reg .b64 %ob<" << std::max(1, n_out) << ">;\n";
    o << "  .reg .b32 %c<" << std::max(1, cur().n_const * L) << ">;\n";
    o << "  .reg .b32 %v<" << std::max(1, (decl_vars >= 0 ? decl_vars : cur().n_vars) * L) << ">;\n";
    o << "  .reg .b64 %ta<" << std::max(1, ntmp_guess) << ">;\n";
    o << "  .reg .b32 %sb, %sth, %nb;\n  .reg .b64 %toff;\n";
    o << "  .reg .b32 %tps, %nt, %nct, %wid, %it, %tile, %lane, %st, %ph, %fb, %eb, %tw, %dst;\n";
    o << "  .reg .pred %pids, %pprod, %p5;\n  .reg .b32 %grp, %ltid, %pk, %pfirst, %t1, %chunk;\n";
    o << "  .reg .b64 %rpm;\n";
    if (phases || multi_acc)
      o << "  .reg .b32 %acc<" << std::max<size_t>(1, full.goal.size() * L) << ">;\n";
    o << "  .reg .b32 %tx0;\n  .reg .b32 %y<8>;\n";
    int nq = 0;
    for (auto &in : cur().ins)
      for (int t : in.ops)
        if (t < cur().n_const) ++nq;
    if (decl_nq >= 0) nq = decl_nq;
    o << "  .reg .b32 %q<" << std::max(1, nq * L) << ">;\n";
    o << "  mov.u32 %zero, 0;\n";
  }

  // Multi-program persistent pipeline (entry xslp_sl_multi): like body_pipe, but every stripe
  // names its own program (p_pos[stripe] - p_first indexes `progs`) and the consumers jump to
  // that program's code through a branch table (brx.idx).  The producer streams the union of
  // the programs' constants.  Each CTA owns a contiguous run of tiles (stripes are grouped by
  // program by the caller), so a CTA changes program rarely and its code stays in cache.
  // The producer also resolves each tile's metadata -- the program index and the output
  // block pointers -- into a per-stage header before it arrives on the stage's full barrier,
  // so consumers start computing without a dependent global load.
  // Shared memory: [0,128) barriers | S headers of HS bytes | stage rows from multi_rows().
  static int multi_hs(int n_out) { return (8 + 8 * n_out + 15) / 16 * 16; }
  static int multi_rows(int S, int n_out) { return (128 + S * multi_hs(n_out) + 127) / 128 * 128; }

  void body_multi(int S, const std::vector<const Slp *> &progs) {
    const int nc = full.n_const;
    const int TC = threads, NCW = threads / 32;
    std::vector<char> used(nc, 0);
    for (const Slp *q : progs) {
      for (auto &in : q->ins)
        for (int t : in.ops)
          if (t < nc) used[t] = 1;
      for (int g : q->goal)
        if (g >= 0 && g < nc) used[g] = 1;
    }
    std::vector<char> blk_used(n_in, 0);
    std::vector<int> slot(nc, -1);
    int nused = 0;
    for (int c = 0; c < nc; ++c)
      if (used[c]) { blk_used[c / 8] = 1; slot[c] = nused++; }
    const int rowb = 4 * L * TC;
    const int64_t STAGE = (int64_t)nused * rowb;
    const int HS = multi_hs(n_out), ROWS = multi_rows(S, n_out);
    pipe_barriers(S, NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n";
    o << "  ld.param.u64 %rpm, [p_pos];\n  ld.param.u32 %pfirst, [p_first];\n";
    // contiguous tile range of this CTA: [ctaid*chunk, min(nt, (ctaid+1)*chunk))
    o << "  mov.u32 %nct, %nctaid.x;\n  add.u32 %chunk, %nt, %nct;\n  sub.u32 %chunk, %chunk, 1;\n";
    o << "  div.u32 %chunk, %chunk, %nct;\n  mov.u32 %s0, %ctaid.x;\n";
    o << "  mul.lo.u32 %s1, %s0, %chunk;\n  add.u32 %t1, %s1, %chunk;\n  min.u32 %t1, %t1, %nt;\n";
    // (a strided tile order -- tile = ctaid + i * nctaid, the PIPE kernel's -- measured 0.61
    // here against 0.96: neighbouring CTAs then run different programs and instruction fetch
    // thrashes; profiles/r01_s2_heterogeneous_and_groups.md)
    const char *step = "1";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << NCW << ";\n  @%pprod bra $PROD;\n";
    // ---------------- consumers
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n  mov.u32 %lane, %laneid;\n";
    o << "$CLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    consumer_wait(S, "");
    o << "  rem.u32 %tw, %tile, %tps;\n";
    o << "  mad.lo.u32 %s3, %tw, " << TC << ", %s2;\n";
    o << "  setp.ge.u32 %p0, %s3, %s4;\n  @%p0 bra $CSKIP;\n";
    o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";   // header
    o << "  ld.shared.u32 %pk, [%dst+4];\n";
    o << "  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
    for (int i = 0; i < n_out; ++i) {
      o << "  ld.shared.u64 %ob" << i << ", [%dst+" << 8 + 8 * i << "];\n";
      o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
    }
    o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
    o << "  mad.lo.u32 %sth, %s2, " << 4 * L << ", %sth;\n";
    o << "  $TBL: .branchtargets ";
    for (size_t k = 0; k < progs.size(); ++k) o << (k ? ", " : "") << "$K" << k;
    o << ";\n  brx.idx %pk, $TBL;\n";
    for (size_t k = 0; k < progs.size(); ++k) {
      sp = progs[k];
      o << "$K" << k << ":\n";
      int tmp = 0;
      compute(true, ROWS, slot, used, tmp);
      o << "  bra.uni $CSKIP;\n";
    }
    sp = &full;
    consumer_release(S, "");
    o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, " << step << ";\n  bra.uni $CLOOP;\n";
    // ---------------- producer
    int tmp = 0;
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    o << "  rem.u32 %st, %it, " << S << ";\n  div.u32 %ph, %it, " << S << ";\n";
    o << "  mad.lo.u32 %fb, %st, 8, %sb;\n";
    // tile metadata first (global loads overlap the wait for the stage to drain)
    o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
    o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
    o << "  mul.wide.u32 %rd6, %s5, 4;\n  add.s64 %rd6, %rpm, %rd6;\n  ld.global.nc.u32 %pk, [%rd6];\n";
    o << "  sub.u32 %pk, %pk, %pfirst;\n";
    // a table entry outside this module would send brx.idx out of its branch table: trap
    // (the launch fails with an error) instead of jumping to an arbitrary address
    o << "  setp.ge.u32 %p0, %pk, " << progs.size() << ";\n  @%p0 trap;\n";
    o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    for (int i = 0; i < n_out; ++i) o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
    o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
    for (int j = 0; j < n_in; ++j) {
      if (!blk_used[j]) continue;
      o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
    }
    producer_wait(S, "");
    o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";
    o << "  st.shared.u32 [%dst], %s5;\n  st.shared.u32 [%dst+4], %pk;\n";
    for (int i = 0; i < n_out; ++i) o << "  st.shared.u64 [%dst+" << 8 + 8 * i << "], %ob" << i << ";\n";
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
    o << "  mul.lo.u32 %s6, %nb, " << nused << ";\n";
    o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
    o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
    for (int c = 0; c < nc; ++c) {
      if (!used[c]) continue;
      std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
      o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
        << ROWS + (int64_t)slot[c] * rowb << "], " << a << ", %nb, [%fb];\n";
    }
    o << "  add.u32 %it, %it, 1;\n  add.u32 %tile, %tile, " << step << ";\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  // PIPE with input phases (K-split): the constants are cut into P contiguous block ranges,
  // each compiled as its own program over all goals; a word-tile is streamed as P stage fills
  // (phase k's strips only), the consumers run phase k's program on fill k and XOR its goal
  // values into accumulators %acc that live across the phases, stored after the last one.
  // A stage holds one phase's strips, so wide codes (RS(20,4): 160 strips) keep T=256
  // consumers with two stages in shared memory.
  void body_pipe_phases(int S) {
    const int nc = full.n_const, P = (int)phases->size();
    const int TC = threads, NCW = threads / 32;
    std::vector<std::vector<char>> used(P, std::vector<char>(nc, 0));
    std::vector<std::vector<int>> slot(P, std::vector<int>(nc, -1));
    std::vector<int> nused(P, 0);
    std::vector<std::vector<char>> blk(P, std::vector<char>(n_in, 0));
    int maxused = 1;
    for (int k = 0; k < P; ++k) {
      const Slp &q = (*phases)[k];
      for (auto &in : q.ins)
        for (int t : in.ops)
          if (t < nc) used[k][t] = 1;
      for (int g : q.goal)
        if (g >= 0 && g < nc) used[k][g] = 1;
      for (int c = 0; c < nc; ++c)
        if (used[k][c]) { blk[k][c / 8] = 1; slot[k][c] = nused[k]++; }
      maxused = std::max(maxused, nused[k]);
    }
    const int rowb = 4 * L * TC;
    const int64_t STAGE = (int64_t)maxused * rowb;
    pipe_barriers(S, NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n  setp.ne.u64 %pids, %rd0, 0;\n";
    o << "  mov.u32 %nct, %nctaid.x;\n";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << NCW << ";\n  @%pprod bra $PROD;\n";
    auto stripe_of = [&](const std::string &lab) {
      o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
      o << "  @!%pids bra " << lab << ";\n";
      o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
      o << lab << ":\n";
    };
    // ---------------- consumers: per word-tile, P phases
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n  mov.u32 %lane, %laneid;\n";
    o << "$CLOOP:\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
    stripe_of("$CID");
    o << "  mad.lo.u32 %s3, %tw, " << TC << ", %s2;\n";
    o << "  setp.lt.u32 %p5, %s3, %s4;\n";  // this thread has a word in the tile
    o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    o << "  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
    for (size_t g = 0; g < full.goal.size() * L; ++g) o << "  mov.b32 %acc" << g << ", 0;\n";
    accumulate = true;
    for (int k = 0; k < P; ++k) {
      const std::string x = std::to_string(k);
      consumer_wait(S, x);
      o << "  @!%p5 bra $CSKIP" << x << ";\n";
      o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
      o << "  mad.lo.u32 %sth, %s2, " << 4 * L << ", %sth;\n  add.u32 %sth, %sth, 128;\n";
      sp = &(*phases)[k];
      int tmp = 0;
      compute(true, 0, slot[k], used[k], tmp);
      consumer_release(S, x);
      o << "  add.u32 %it, %it, 1;\n";
    }
    accumulate = false;
    sp = &full;
    {  // the goals, once per word-tile
      o << "  @!%p5 bra $CSTORED;\n";
      for (int i = 0; i < n_out; ++i) {
        o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
        o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
      }
      int tmp = 0;
      for (size_t g = 0; g < full.goal.size(); ++g) {
        std::vector<std::string> r;
        for (int l = 0; l < L; ++l) r.push_back("%acc" + std::to_string(g * L + l));
        store((int)g, r, tmp);
      }
      o << "$CSTORED:\n";
    }
    o << "  add.u32 %tile, %tile, %nct;\n  bra.uni $CLOOP;\n";
    // ---------------- producer: per word-tile, P stage fills
    int tmp = 0;
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %ctaid.x;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %nt;\n  @%p0 bra $DONE;\n";
    stripe_of("$PID");
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
    o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
    for (int j = 0; j < n_in; ++j) {
      bool any = false;
      for (int k = 0; k < P; ++k) any |= blk[k][j] != 0;
      if (!any) continue;
      o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
    }
    for (int k = 0; k < P; ++k) {
      const std::string x = std::to_string(k);
      stage_regs(S);
      producer_wait(S, x);
      o << "  mul.lo.u32 %s6, %nb, " << nused[k] << ";\n";
      o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
      o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
      for (int c = 0; c < nc; ++c) {
        if (!used[k][c]) continue;
        std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
        o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
          << 128 + (int64_t)slot[k][c] * rowb << "], " << a << ", %nb, [%fb];\n";
      }
      o << "  add.u32 %it, %it, 1;\n";
    }
    o << "  add.u32 %tile, %tile, %nct;\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  // Multi-program pipeline with input phases (wide codes): program k is given as P phase
  // programs progs[k][ph] over contiguous input-block ranges.  A word-tile is streamed as P
  // stage fills (phase ph's strips only); on each fill the consumers jump through phase ph's
  // branch table to their stripe's phase program and XOR the goal partials into %acc, stored
  // after the last phase.  The program index and output pointers are taken from the header of
  // the tile's first fill into registers (that stage may be refilled before the last phase).
  void body_multi_phases(int S, const std::vector<std::vector<const Slp *>> &progs) {
    const int nc = full.n_const, P = (int)progs[0].size();
    const int TC = threads, NCW = threads / 32;
    std::vector<std::vector<char>> used(P, std::vector<char>(nc, 0));
    std::vector<std::vector<int>> slot(P, std::vector<int>(nc, -1));
    std::vector<int> nused(P, 0);
    std::vector<char> blk(n_in, 0);
    int maxused = 1;
    for (int ph = 0; ph < P; ++ph) {
      for (auto &pk : progs) {
        const Slp *q = pk[ph];
        for (auto &in : q->ins)
          for (int t : in.ops)
            if (t < nc) used[ph][t] = 1;
        for (int g : q->goal)
          if (g >= 0 && g < nc) used[ph][g] = 1;
      }
      for (int c = 0; c < nc; ++c)
        if (used[ph][c]) { blk[c / 8] = 1; slot[ph][c] = nused[ph]++; }
      maxused = std::max(maxused, nused[ph]);
    }
    const int rowb = 4 * L * TC;
    const int64_t STAGE = (int64_t)maxused * rowb;
    const int HS = multi_hs(n_out), ROWS = multi_rows(S, n_out);
    pipe_barriers(S, NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n";
    o << "  ld.param.u64 %rpm, [p_pos];\n  ld.param.u32 %pfirst, [p_first];\n";
    // contiguous tile range of this CTA (see body_multi)
    o << "  mov.u32 %nct, %nctaid.x;\n  add.u32 %chunk, %nt, %nct;\n  sub.u32 %chunk, %chunk, 1;\n";
    o << "  div.u32 %chunk, %chunk, %nct;\n  mov.u32 %s0, %ctaid.x;\n";
    o << "  mul.lo.u32 %s1, %s0, %chunk;\n  add.u32 %t1, %s1, %chunk;\n  min.u32 %t1, %t1, %nt;\n";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << NCW << ";\n  @%pprod bra $PROD;\n";
    // ---------------- consumers
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n  mov.u32 %lane, %laneid;\n";
    o << "$CLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    o << "  rem.u32 %tw, %tile, %tps;\n  mad.lo.u32 %s3, %tw, " << TC << ", %s2;\n";
    o << "  setp.lt.u32 %p5, %s3, %s4;\n  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
    for (size_t g = 0; g < full.goal.size() * L; ++g) o << "  mov.b32 %acc" << g << ", 0;\n";
    accumulate = true;
    for (int ph = 0; ph < P; ++ph) {
      const std::string x = std::to_string(ph);
      consumer_wait(S, x);
      if (ph == 0) {  // tile metadata from the first fill's header
        o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";
        o << "  ld.shared.u32 %pk, [%dst+4];\n";
        for (int i = 0; i < n_out; ++i) {
          o << "  ld.shared.u64 %ob" << i << ", [%dst+" << 8 + 8 * i << "];\n";
          o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
        }
      }
      o << "  @!%p5 bra $CSKIP" << x << ";\n";
      o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
      o << "  mad.lo.u32 %sth, %s2, " << 4 * L << ", %sth;\n";
      o << "  $TBL" << x << ": .branchtargets ";
      for (size_t k = 0; k < progs.size(); ++k) o << (k ? ", " : "") << "$K" << k << "_" << x;
      o << ";\n  brx.idx %pk, $TBL" << x << ";\n";
      for (size_t k = 0; k < progs.size(); ++k) {
        sp = progs[k][ph];
        o << "$K" << k << "_" << x << ":\n";
        int tmp = 0;
        compute(true, ROWS, slot[ph], used[ph], tmp);
        o << "  bra.uni $CSKIP" << x << ";\n";
      }
      consumer_release(S, x);
      o << "  add.u32 %it, %it, 1;\n";
    }
    accumulate = false;
    sp = &full;
    {
      o << "  @!%p5 bra $CSTORED;\n";
      int tmp = 0;
      for (size_t g = 0; g < full.goal.size(); ++g) {
        std::vector<std::string> r;
        for (int l = 0; l < L; ++l) r.push_back("%acc" + std::to_string(g * L + l));
        store((int)g, r, tmp);
      }
      o << "$CSTORED:\n";
    }
    o << "  add.u32 %tile, %tile, 1;\n  bra.uni $CLOOP;\n";
    // ---------------- producer
    int tmp = 0;
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
    o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
    o << "  mul.wide.u32 %rd6, %s5, 4;\n  add.s64 %rd6, %rpm, %rd6;\n  ld.global.nc.u32 %pk, [%rd6];\n";
    o << "  sub.u32 %pk, %pk, %pfirst;\n";
    // a table entry outside this module would send brx.idx out of its branch table: trap
    // (the launch fails with an error) instead of jumping to an arbitrary address
    o << "  setp.ge.u32 %p0, %pk, " << progs.size() << ";\n  @%p0 trap;\n";
    o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    for (int i = 0; i < n_out; ++i) o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
    o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
    for (int j = 0; j < n_in; ++j) {
      if (!blk[j]) continue;
      o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
    }
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
    for (int ph = 0; ph < P; ++ph) {
      const std::string x = std::to_string(ph);
      stage_regs(S);
      producer_wait(S, "P" + x);
      if (ph == 0) {
        o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";
        o << "  st.shared.u32 [%dst], %s5;\n  st.shared.u32 [%dst+4], %pk;\n";
        for (int i = 0; i < n_out; ++i) o << "  st.shared.u64 [%dst+" << 8 + 8 * i << "], %ob" << i << ";\n";
      }
      o << "  mul.lo.u32 %s6, %nb, " << nused[ph] << ";\n";
      o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
      o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
      for (int c = 0; c < nc; ++c) {
        if (!used[ph][c]) continue;
        std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
        o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
          << ROWS + (int64_t)slot[ph][c] * rowb << "], " << a << ", %nb, [%fb];\n";
      }
      o << "  add.u32 %it, %it, 1;\n";
    }
    o << "  add.u32 %tile, %tile, 1;\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  // Syndrome-form decode (csrc/syndrome.cpp): every stripe runs the ONE syndrome program over
  // all n+p blocks (erased ones read from a zero block), streamed in input phases with the
  // syndrome words accumulated in %acc, then jumps through a branch table to its pattern's
  // small solve program, whose constants are the %acc registers and whose goals (the erased
  // blocks) are stored.  The shared code stays hot in the instruction cache; per pattern only
  // the solve code (~e x p GF entries) differs.
  void body_syndrome(int S, const std::vector<Slp> &syn, const std::vector<const Slp *> &solves) {
    const int nc = full.n_const, P = (int)syn.size();
    const int TC = threads, NCW = threads / 32;
    std::vector<std::vector<char>> used(P, std::vector<char>(nc, 0));
    std::vector<std::vector<int>> slot(P, std::vector<int>(nc, -1));
    std::vector<int> nused(P, 0);
    std::vector<char> blk(n_in, 0);
    int maxused = 1;
    for (int ph = 0; ph < P; ++ph) {
      for (auto &in : syn[ph].ins)
        for (int t : in.ops)
          if (t < nc) used[ph][t] = 1;
      for (int g : syn[ph].goal)
        if (g >= 0 && g < nc) used[ph][g] = 1;
      for (int c = 0; c < nc; ++c)
        if (used[ph][c]) { blk[c / 8] = 1; slot[ph][c] = nused[ph]++; }
      maxused = std::max(maxused, nused[ph]);
    }
    const int rowb = 4 * L * TC;
    const int64_t STAGE = (int64_t)maxused * rowb;
    const int HS = multi_hs(n_out), ROWS = multi_rows(S, n_out);
    const int nsyn = (int)full.goal.size();  // syndrome words (8p)
    pipe_barriers(S, NCW);
    o << "  ld.param.u32 %s4, [p_words];\n  ld.param.u32 %tps, [p_tps];\n  ld.param.u32 %nt, [p_ntiles];\n";
    o << "  ld.param.u64 %rd0, [p_ids];\n";
    o << "  ld.param.u64 %rpm, [p_pos];\n  ld.param.u32 %pfirst, [p_first];\n";
    o << "  mov.u32 %nct, %nctaid.x;\n  add.u32 %chunk, %nt, %nct;\n  sub.u32 %chunk, %chunk, 1;\n";
    o << "  div.u32 %chunk, %chunk, %nct;\n  mov.u32 %s0, %ctaid.x;\n";
    o << "  mul.lo.u32 %s1, %s0, %chunk;\n  add.u32 %t1, %s1, %chunk;\n  min.u32 %t1, %t1, %nt;\n";
    if (baked <= 0) {
      o << "  ld.param.u64 %sk1, [p_strip];\n";
      for (int k = 2; k < 8; ++k) o << "  mul.lo.u64 %sk" << k << ", %sk1, " << k << ";\n";
    }
    o << "  shr.u32 %wid, %s2, 5;\n  setp.eq.u32 %pprod, %wid, " << NCW << ";\n  @%pprod bra $PROD;\n";
    // ---------------- consumers
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n  mov.u32 %lane, %laneid;\n";
    o << "$CLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    o << "  rem.u32 %tw, %tile, %tps;\n  mad.lo.u32 %s3, %tw, " << TC << ", %s2;\n";
    o << "  setp.lt.u32 %p5, %s3, %s4;\n  mul.wide.u32 %off, %s3, " << 4 * L << ";\n";
    for (int g = 0; g < nsyn * L; ++g) o << "  mov.b32 %acc" << g << ", 0;\n";
    accumulate = true;
    for (int ph = 0; ph < P; ++ph) {
      const std::string x = std::to_string(ph);
      consumer_wait(S, x);
      if (ph == 0) {
        o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";
        o << "  ld.shared.u32 %pk, [%dst+4];\n";
        for (int i = 0; i < n_out; ++i) {
          o << "  ld.shared.u64 %ob" << i << ", [%dst+" << 8 + 8 * i << "];\n";
          o << "  add.s64 %ob" << i << ", %ob" << i << ", %off;\n";
        }
      }
      o << "  @!%p5 bra $CSKIP" << x << ";\n";
      o << "  mul.lo.u32 %sth, %st, " << STAGE << ";\n  add.u32 %sth, %sth, %sb;\n";
      o << "  mad.lo.u32 %sth, %s2, " << 4 * L << ", %sth;\n";
      sp = &syn[ph];
      int tmp = 0;
      compute(true, ROWS, slot[ph], used[ph], tmp);
      consumer_release(S, x);
      o << "  add.u32 %it, %it, 1;\n";
    }
    accumulate = false;
    // the pattern's solve program on the syndrome words
    o << "  @!%p5 bra $CSOLVED;\n";
    o << "  $TBL: .branchtargets ";
    for (size_t k = 0; k < solves.size(); ++k) o << (k ? ", " : "") << "$K" << k;
    o << ";\n  brx.idx %pk, $TBL;\n";
    acc_consts = true;
    for (size_t k = 0; k < solves.size(); ++k) {
      sp = solves[k];
      o << "$K" << k << ":\n";
      int tmp = 0;
      std::vector<int> noslot(nsyn, -1);
      std::vector<char> nouse(nsyn, 0);
      compute(false, 0, noslot, nouse, tmp);
      o << "  bra.uni $CSOLVED;\n";
    }
    acc_consts = false;
    sp = &full;
    o << "$CSOLVED:\n  add.u32 %tile, %tile, 1;\n  bra.uni $CLOOP;\n";
    // ---------------- producer
    int tmp = 0;
    o << "$PROD:\n  mov.u32 %lane, %laneid;\n  setp.ne.u32 %p4, %lane, 0;\n  @%p4 bra $DONE;\n";
    o << "  mov.u32 %it, 0;\n  mov.u32 %tile, %s1;\n";
    o << "$PLOOP:\n  setp.ge.u32 %p0, %tile, %t1;\n  @%p0 bra $DONE;\n";
    o << "  div.u32 %s5, %tile, %tps;\n  rem.u32 %tw, %tile, %tps;\n";
    o << "  mul.wide.u32 %rd1, %s5, 4;\n  add.s64 %rd1, %rd0, %rd1;\n  ld.global.nc.u32 %s5, [%rd1];\n";
    o << "  mul.wide.u32 %rd6, %s5, 4;\n  add.s64 %rd6, %rpm, %rd6;\n  ld.global.nc.u32 %pk, [%rd6];\n";
    o << "  sub.u32 %pk, %pk, %pfirst;\n";
    // a table entry outside this module would send brx.idx out of its branch table: trap
    // (the launch fails with an error) instead of jumping to an arbitrary address
    o << "  setp.ge.u32 %p0, %pk, " << solves.size() << ";\n  @%p0 trap;\n";
    o << "  ld.param.u64 %rd3, [p_out];\n  mul.wide.u32 %rd5, %s5, " << 8 * n_out << ";\n  add.s64 %rd3, %rd3, %rd5;\n";
    for (int i = 0; i < n_out; ++i) o << "  ld.global.nc.u64 %ob" << i << ", [%rd3+" << 8 * i << "];\n";
    o << "  ld.param.u64 %rd2, [p_in];\n  mul.wide.u32 %rd4, %s5, " << 8 * n_in << ";\n  add.s64 %rd2, %rd2, %rd4;\n";
    o << "  mul.lo.u32 %s7, %tw, " << TC << ";\n";
    o << "  mul.wide.u32 %toff, %s7, " << 4 * L << ";\n";
    for (int j = 0; j < n_in; ++j) {
      if (!blk[j]) continue;
      o << "  ld.global.nc.u64 %ib" << j << ", [%rd2+" << 8 * j << "];\n";
      o << "  add.s64 %ib" << j << ", %ib" << j << ", %toff;\n";
    }
    o << "  sub.u32 %nb, %s4, %s7;\n  min.u32 %nb, %nb, " << TC << ";\n  mul.lo.u32 %nb, %nb, " << 4 * L << ";\n";
    for (int ph = 0; ph < P; ++ph) {
      const std::string x = std::to_string(ph);
      stage_regs(S);
      producer_wait(S, "P" + x);
      if (ph == 0) {
        o << "  mad.lo.u32 %dst, %st, " << HS << ", %sb;\n  add.u32 %dst, %dst, 128;\n";
        o << "  st.shared.u32 [%dst], %s5;\n  st.shared.u32 [%dst+4], %pk;\n";
        for (int i = 0; i < n_out; ++i) o << "  st.shared.u64 [%dst+" << 8 + 8 * i << "], %ob" << i << ";\n";
      }
      o << "  mul.lo.u32 %s6, %nb, " << nused[ph] << ";\n";
      o << "  mbarrier.arrive.expect_tx.shared::cta.b64 _, [%fb], %s6;\n";
      o << "  mul.lo.u32 %dst, %st, " << STAGE << ";\n  add.u32 %dst, %dst, %sb;\n";
      for (int c = 0; c < nc; ++c) {
        if (!used[ph][c]) continue;
        std::string a = addr("%ib" + std::to_string(c / 8), c % 8, tmp);
        o << "  cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%dst+"
          << ROWS + (int64_t)slot[ph][c] * rowb << "], " << a << ", %nb, [%fb];\n";
      }
      o << "  add.u32 %it, %it, 1;\n";
    }
    o << "  add.u32 %tile, %tile, 1;\n  bra.uni $PLOOP;\n";
    o << "$DONE:\n  ret;\n";
  }

  std::string run_syndrome(const std::vector<Slp> &syn, const std::vector<const Slp *> &solves) {
    int mv = 0, mq = 0;
    std::vector<const Slp *> all(solves);
    for (auto &q : syn) all.push_back(&q);
    for (const Slp *q : all) {
      mv = std::max(mv, q->n_vars);
      int nq = 0;
      for (auto &in : q->ins)
        for (int t : in.ops)
          if (t < q->n_const) ++nq;
      mq = std::max(mq, nq);
    }
    decl_vars = mv;
    decl_nq = mq;
    multi_acc = true;
    o << "//\n// xslp syndrome-form decode kernel: " << solves.size() << " patterns, "
      << full.n_const << " constants, " << full.goal.size() << " syndrome words\n//\n";
    o << ".version 8.8\n.target sm_100a\n.address_size 64\n\n";
    o << ".extern .shared .align 128 .b8 dsm[];\n\n";
    o << ".visible .entry xslp_sl_multi(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
         "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
         "  .param .u32 p_tps,\n  .param .u32 p_ntiles,\n  .param .u64 p_pos,\n"
         "  .param .u32 p_first)\n.maxntid "
      << threads + 32 << ", 1, 1\n{\n";
    decls(full.n_const + (int)full.goal.size() + 8);
    body_syndrome(stages, syn, solves);
    o << "}\n";
    return o.str();
  }

  // progs: one program per table entry; with input phases (phased non-empty) the entries'
  // phase programs are phased[k][ph] and progs is unused by the body.
  std::string run_multi(const std::vector<const Slp *> &progs,
                        const std::vector<std::vector<const Slp *>> &phased = {}) {
    int mv = 0, mq = 0;
    std::vector<const Slp *> all(progs);
    for (auto &pk : phased) all.insert(all.end(), pk.begin(), pk.end());
    for (const Slp *q : all) {
      mv = std::max(mv, q->n_vars);
      int nq = 0;
      for (auto &in : q->ins)
        for (int t : in.ops)
          if (t < q->n_const) ++nq;
      mq = std::max(mq, nq);
    }
    decl_vars = mv;
    decl_nq = mq;
    multi_acc = !phased.empty();
    o << "//\n// xslp multi-program pipeline kernel: " << progs.size() << " programs, "
      << full.n_const << " constants, " << full.goal.size() << " goals, lanes=" << L << "\n//\n";
    o << ".version 8.8\n.target sm_100a\n.address_size 64\n\n";
    o << ".extern .shared .align 128 .b8 dsm[];\n\n";
    o << ".visible .entry xslp_sl_multi(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
         "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
         "  .param .u32 p_tps,\n  .param .u32 p_ntiles,\n  .param .u64 p_pos,\n"
         "  .param .u32 p_first)\n.maxntid "
      << threads + 32 << ", 1, 1\n{\n";
    decls(full.n_const + (int)full.goal.size() + 8);
    if (phased.empty()) body_multi(stages, progs); else body_multi_phases(stages, phased);
    o << "}\n";
    return o.str();
  }

  std::string run() {
    o << "//\n// xslp straight-line kernel: " << cur().n_const << " constants, " << cur().goal.size()
      << " goals, " << cur().ins.size() << " instructions, lanes=" << L << ", strip="
      << (baked > 0 ? std::to_string(baked) : std::string("runtime")) << "\n//\n";
    o << ".version 8.8\n.target sm_100a\n.address_size 64\n\n";
    o << ".extern .shared .align 128 .b8 dsm[];\n\n";
    const int ntmp = cur().n_const + (int)cur().goal.size() + 8;
    o << ".visible .entry xslp_sl_batch(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
         "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
         "  .param .u32 p_base)\n.maxntid "
      << threads << ", 1, 1\n";
    if (min_blocks > 0) o << ".minnctapersm " << min_blocks << "\n";
    o << "{\n";
    decls(ntmp);
    if (layout == XSLP_LAYOUT_BYTE) body_byte(false); else body(0);
    o << "}\n\n";
    o << ".visible .entry xslp_sl_one(\n  .param .align 8 .b8 p_ptrs[1024],\n"
         "  .param .u64 p_strip,\n  .param .u32 p_words)\n.maxntid "
      << threads << ", 1, 1\n{\n";
    decls(ntmp);
    if (layout == XSLP_LAYOUT_BYTE) body_byte(true); else body(1);
    o << "}\n\n";
    if (layout == XSLP_LAYOUT_BYTE) {  // byte layout: the TMA pipeline only (no xslp_sl_tma)
      o << ".visible .entry xslp_sl_pipe(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
           "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
           "  .param .u32 p_tps,\n  .param .u32 p_ntiles)\n.maxntid "
        << threads + 32 << ", 1, 1\n{\n";
      decls(ntmp);
      body_pipe_byte(stages);
      o << "}\n";
      return o.str();
    }
    o << ".visible .entry xslp_sl_tma(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
         "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
         "  .param .u32 p_base)\n.maxntid "
      << threads << ", 1, 1\n";
    if (min_blocks > 0) o << ".minnctapersm " << min_blocks << "\n";
    o << "{\n";
    decls(ntmp);
    body(2);
    o << "}\n\n";
    o << ".visible .entry xslp_sl_pipe(\n  .param .u64 p_in,\n  .param .u64 p_out,\n"
         "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
         "  .param .u32 p_tps,\n  .param .u32 p_ntiles)\n.maxntid "
      << threads * (groups ? (int)groups->size() : 1) + 32 << ", 1, 1\n";
    o << "{\n";
    decls(ntmp);
    if (phases) body_pipe_phases(stages); else body_pipe(stages);
    o << "}\n";
    if (!phases && !groups) {  // one stripe, pointers by value (xslp_encode / xslp_decode)
      o << "\n.visible .entry xslp_sl_pipe_one(\n  .param .align 8 .b8 p_ptrs[1024],\n"
           "  .param .u64 p_ids,\n  .param .u64 p_strip,\n  .param .u32 p_words,\n"
           "  .param .u32 p_tps,\n  .param .u32 p_ntiles)\n.maxntid "
        << threads + 32 << ", 1, 1\n{\n";
      decls(ntmp);
      pipe_one = true;
      body_pipe(stages);
      pipe_one = false;
      o << "}\n";
    }
    return o.str();
  }
};

}  // namespace

std::string emit_ptx(const Slp &s, int lanes, int64_t baked_strip, int threads, int min_blocks,
                     int stages, int layout, const std::vector<Slp> *groups,
                     const std::vector<Slp> *phases, int reuse) {
  if (s.n_const % 8 || s.goal.size() % 8)
    throw Error(XSLP_EINVAL, "device programs need whole blocks (constants and goals multiples of 8)");
  if (s.n_const / 8 + s.goal.size() / 8 > 128)
    throw Error(XSLP_EINVAL, "too many blocks for one kernel (n + m > 128)");
  if (layout == XSLP_LAYOUT_BYTE) lanes = 1;
  Emitter e(s, lanes, baked_strip, threads, min_blocks, stages, layout, groups);
  e.phases = phases;
  e.reuse = reuse;
  return e.run();
}

std::string emit_ptx_multi(const std::vector<const Slp *> &progs, int lanes, int64_t baked_strip,
                           int threads, int stages, int reuse) {
  if (progs.empty()) throw Error(XSLP_EINVAL, "no programs");
  const Slp &f = *progs[0];
  for (const Slp *q : progs)
    if (q->n_const != f.n_const || q->goal.size() != f.goal.size())
      throw Error(XSLP_EINVAL, "programs disagree on constants/goals");
  if (f.n_const % 8 || f.goal.size() % 8 || f.n_const / 8 + f.goal.size() / 8 > 128)
    throw Error(XSLP_EINVAL, "device programs need whole blocks (n + m <= 128)");
  Emitter e(f, lanes, baked_strip, threads, 0, stages, XSLP_LAYOUT_STRIP, nullptr);
  e.reuse = reuse;
  return e.run_multi(progs);
}

std::string emit_ptx_multi_phases(const std::vector<std::vector<const Slp *>> &phased, int lanes,
                                  int64_t baked_strip, int threads, int stages, int reuse) {
  if (phased.empty() || phased[0].empty()) throw Error(XSLP_EINVAL, "no programs");
  const Slp &f = *phased[0][0];
  for (auto &pk : phased) {
    if (pk.size() != phased[0].size()) throw Error(XSLP_EINVAL, "programs disagree on phases");
    for (const Slp *q : pk)
      if (q->n_const != f.n_const || q->goal.size() != f.goal.size())
        throw Error(XSLP_EINVAL, "programs disagree on constants/goals");
  }
  if (f.n_const % 8 || f.goal.size() % 8 || f.n_const / 8 + f.goal.size() / 8 > 128)
    throw Error(XSLP_EINVAL, "device programs need whole blocks (n + m <= 128)");
  Emitter e(f, lanes, baked_strip, threads, 0, stages, XSLP_LAYOUT_STRIP, nullptr);
  e.reuse = reuse;
  return e.run_multi({}, phased);
}

std::string emit_ptx_syndrome(const std::vector<Slp> &syn, const std::vector<const Slp *> &solves,
                              int n_out, int lanes, int64_t baked_strip, int threads, int stages,
                              int reuse) {
  if (syn.empty() || solves.empty()) throw Error(XSLP_EINVAL, "no programs");
  for (const Slp *q : solves)
    if (q->n_const != (int)syn[0].goal.size() || (int)q->goal.size() != 8 * n_out)
      throw Error(XSLP_EINVAL, "solve programs do not match the syndrome");
  if (syn[0].n_const % 8 || syn[0].goal.size() % 8 || syn[0].n_const / 8 + n_out > 128)
    throw Error(XSLP_EINVAL, "device programs need whole blocks (n + p + e <= 128)");
  Emitter e(syn[0], lanes, baked_strip, threads, 0, stages, XSLP_LAYOUT_STRIP, nullptr);
  e.n_out = n_out;  // outputs are the erased blocks, not the syndrome
  e.reuse = reuse;
  return e.run_syndrome(syn, solves);
}

std::vector<char> ptx_to_cubin(const std::string &ptx, int *regs, int *spill, int *regs_tma,
                               int *spill_tma, int *regs_pipe, int *spill_pipe) {
  nvPTXCompilerHandle h = nullptr;
  if (nvPTXCompilerCreate(&h, ptx.size(), ptx.c_str()) != NVPTXCOMPILE_SUCCESS)
    throw Error(XSLP_ECOMPILE, "nvPTXCompilerCreate failed");
  const char *opts[] = {"--gpu-name=sm_100a", "-O3", "--verbose"};
  nvPTXCompileResult r = nvPTXCompilerCompile(h, 3, opts);
  if (r != NVPTXCOMPILE_SUCCESS) {
    size_t n = 0;
    nvPTXCompilerGetErrorLogSize(h, &n);
    std::string log(n + 1, '\0');
    if (n) nvPTXCompilerGetErrorLog(h, &log[0]);
    nvPTXCompilerDestroy(&h);
    throw Error(XSLP_ECOMPILE, "ptx compile failed (" + std::to_string((int)r) + "): " + log);
  }
  size_t n = 0;
  nvPTXCompilerGetCompiledProgramSize(h, &n);
  std::vector<char> bin(n);
  nvPTXCompilerGetCompiledProgram(h, bin.data());
  size_t ln = 0;
  nvPTXCompilerGetInfoLogSize(h, &ln);
  std::string info(ln + 1, '\0');
  if (ln) nvPTXCompilerGetInfoLog(h, &info[0]);
  nvPTXCompilerDestroy(&h);
  // per-entry "Used N registers" / "N bytes spill stores" from the ptxas info log
  auto entry_info = [&](const std::string &name, int *r, int *sp) {
    if (r) *r = 0;
    if (sp) *sp = 0;
    auto p = info.find("'" + name + "'");
    if (p == std::string::npos) return;
    auto nxt = info.find("Compiling entry function", p + 1);
    std::string blk = info.substr(p, nxt == std::string::npos ? std::string::npos : nxt - p);
    auto u = blk.find("Used ");
    if (u != std::string::npos && r) *r = std::atoi(blk.c_str() + u + 5);
    auto q = blk.find("bytes spill stores");
    if (q != std::string::npos && sp) {
      auto c = blk.rfind(',', q);
      *sp = std::atoi(blk.c_str() + (c == std::string::npos ? 0 : c + 1));
    }
  };
  entry_info("xslp_sl_batch", regs, spill);
  entry_info("xslp_sl_tma", regs_tma, spill_tma);
  entry_info("xslp_sl_pipe", regs_pipe, spill_pipe);
  if (info.find("'xslp_sl_multi'") != std::string::npos) entry_info("xslp_sl_multi", regs_pipe, spill_pipe);
  return bin;
}

}  // namespace xslp
