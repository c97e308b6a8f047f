// Generic SLP interpreter, pipelined (the paper's "interpreter style", on B200).
// Used for batched interpreter launches (xslp_encode_batch / xslp_decode_batch_multi when no
// straight-line kernel runs); single-stripe calls keep the one-tile xslp_interp_kernel.
//
// One kernel runs ANY compiled program from its bytecode -- no JIT -- and one launch can run a
// different program per stripe.  Layout of the work is the PIPE kernel's: persistent CTAs,
// a producer warp streaming each tile's constant strips by TMA (cp.async.bulk + mbarrier
// full/empty ring) into the tile's slot region, T consumer threads running the program
// over the region while the producer fills the next one.  Each CTA walks a contiguous run of
// tiles, so with program-sorted stripes it rarely changes program.
//
// What makes it fast compared with a plain interpreter: the bytecode is re-encoded on the
// host for the launch's T into 32-bit words whose operands are byte offsets of slot rows
// (slot * T * 4), operand lists 16-byte aligned, so a consumer reads four operand offsets
// with one shared-memory vector load and each operand costs one address add and one load
// (3-input XORs via LOP3); the per-tile header written by the producer gives the program
// index and output block pointers without a dependent global load.
//
// Shared memory: [0,128) barriers | S tile headers | code32 (cap words) | S slot regions of
// nslots x T x 4 bytes.  The slot assignment is the compiler's (build_bytecode: max-live
// slots under the DFS schedule): constants are TMA'd into their slots, each
// variable is written once to its slot and read by its users, goals are stored to HBM when
// computed.
#include <cuda_runtime.h>

#include <algorithm>

#include "xslp_api.h"

namespace xslp {

void count_launch();  // device.cu

// ---- host: bytecode (u16, build_bytecode) -> micro-op code for consumer width T ---------
// A branch-light format: every micro-op XORs exactly four slot rows into the accumulator
// (short operand lists are padded with the zero row `nslots`), so the consumer loop has no
// data-dependent trip counts.  Layout (32-bit words):
//   [0] nloads [1] nmops [2] total words [3] nslots (without the zero row)
//   loads: nloads x (constant index, slot byte offset), padded to a multiple of 8 words
//   micro-ops: 8 words each = 4 operand byte offsets (slot * T * 4),
//              flags (1 = reset acc first, 2 = store acc to the dst slot, 4 = store acc to
//              goal), dst slot byte offset, goal index, 0.
// An instruction of arity a becomes ceil(a/4) micro-ops (reset on the first, stores on the
// last); an instruction with several goals adds operand-free micro-ops, one per extra goal.
std::vector<uint32_t> build_code32(const std::vector<uint16_t> &code, int T) {
  const int nl = code[0], ni = code[1], nslots = code[3];
  const uint32_t row = (uint32_t)T * 4, zero = (uint32_t)nslots * row;
  std::vector<uint32_t> out = {(uint32_t)nl, 0, 0, (uint32_t)nslots};
  for (int i = 0; i < nl; ++i) {
    out.push_back(code[4 + 2 * i]);
    out.push_back(code[5 + 2 * i] * row);
  }
  while (out.size() % 8) out.push_back(0);
  uint32_t nm = 0;
  auto mop = [&](const uint32_t o[4], uint32_t flags, uint32_t dst, uint32_t goal) {
    out.insert(out.end(), {o[0], o[1], o[2], o[3], flags, dst, goal, 0u});
    ++nm;
  };
  size_t pc = 4 + 2 * (size_t)nl;
  for (int k = 0; k < ni; ++k) {
    const int hdr = code[pc++];
    const int arity = hdr & 1023, ng = (hdr >> 10) & 15;
    const bool hasdst = hdr & 0x8000;
    const uint32_t dst = hasdst ? code[pc++] * row : 0;
    std::vector<uint32_t> goals;
    for (int g = 0; g < ng; ++g) goals.push_back(code[pc++]);
    pc += pc & 1;
    std::vector<uint32_t> ops;
    for (int q = 0; q < arity; ++q) ops.push_back(code[pc++] * row);
    pc += pc & 1;
    const int chunks = std::max(1, (arity + 3) / 4);
    for (int c = 0; c < chunks; ++c) {
      uint32_t o[4];
      for (int u = 0; u < 4; ++u) o[u] = 4 * c + u < arity ? ops[4 * c + u] : zero;
      uint32_t flags = c == 0 ? 1u : 0u;
      uint32_t goal = 0;
      if (c == chunks - 1) {
        if (hasdst) flags |= 2;
        if (!goals.empty()) { flags |= 4; goal = goals[0]; }
      }
      mop(o, flags, dst, goal);
    }
    const uint32_t z[4] = {zero, zero, zero, zero};
    for (size_t g = 1; g < goals.size(); ++g) mop(z, 4, 0, goals[g]);
  }
  out[1] = nm;
  out[2] = (uint32_t)out.size();
  return out;
}

struct InterpArgs {
  const uint32_t *code;          // code32 pool
  const int64_t *prog_off;       // word offset of each program's code32 in the pool
  const int32_t *prog_of_stripe; // nullable: program 0 for every stripe
  const int32_t *ids;            // nullable: tile stripe = ids[entry]
  const uint8_t *const *in_tbl;
  uint8_t *const *out_tbl;
  uint64_t strip;
  uint32_t words, tps, ntiles;
  int32_t n_in, n_out, S, code_cap, region;  // region = nslots * T * 4 bytes
};

__device__ __forceinline__ uint32_t sm_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
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

constexpr int kHdr = 16 + 8 * 32;  // per-stage tile header: stripe, prog, pad, up to 32 output ptrs

__global__ void __launch_bounds__(1024) xslp_interp_pipe(InterpArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t T = blockDim.x - 32, tid = threadIdx.x;
  const int S = a.S;
  const uint32_t base = sm_addr(sm);
  const uint32_t hdr0 = base + 128;                               // S headers
  uint32_t *code = reinterpret_cast<uint32_t *>(sm + 128 + S * kHdr);
  const uint32_t regions = base + 128 + S * kHdr + a.code_cap * 4;
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(base + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(base + 64 + 8 * k), "r"(T / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // contiguous tile run of this CTA
  const uint32_t chunk = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const uint32_t t0 = blockIdx.x * chunk, t1 = min(a.ntiles, t0 + chunk);
  if (tid >= T) {  // ---------------- producer (one lane)
    if (tid != T) return;
    for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
      const uint32_t st = it % S, ph = (it / S) & 1;
      const uint32_t entry = tile / a.tps, tw = tile % a.tps;
      const uint32_t stripe = a.ids ? (uint32_t)a.ids[entry] : entry;
      const int prog = a.prog_of_stripe ? a.prog_of_stripe[stripe] : 0;
      const uint32_t *pc = a.code + a.prog_off[prog];
      const uint8_t *const *in = a.in_tbl + (size_t)stripe * a.n_in;
      uint8_t *const *out = a.out_tbl + (size_t)stripe * a.n_out;
      if (it >= (uint32_t)S)
        while (!try_wait(base + 64 + 8 * st, ph ^ 1)) {
        }
      const uint32_t h = hdr0 + st * kHdr;
      sts(h, stripe);
      sts(h + 4, (uint32_t)prog);
      for (int i = 0; i < a.n_out; ++i) {
        const uint64_t p = (uint64_t)out[i];
        asm volatile("st.shared.u64 [%0], %1;" ::"r"(h + 16 + 8 * i), "l"(p) : "memory");
      }
      const uint32_t nb = min(T, a.words - tw * T) * 4;
      const uint32_t nl = pc[0];
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(base + 8 * st),
                   "r"(nb * nl) : "memory");
      const uint32_t reg = regions + st * a.region;
      const size_t toff = (size_t)tw * T * 4;
      for (uint32_t i = 0; i < nl; ++i) {
        const uint32_t c = pc[4 + 2 * i], off = pc[5 + 2 * i];
        const uint8_t *src = in[c >> 3] + (c & 7) * a.strip + toff;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(reg + off), "l"(src), "r"(nb), "r"(base + 8 * st) : "memory");
      }
    }
    return;
  }
  // ---------------- consumers
  int cur = -1;
  const uint32_t lane = tid & 31;
  for (uint32_t tile = t0, it = 0; tile < t1; ++tile, ++it) {
    const uint32_t st = it % S, ph = (it / S) & 1;
    while (!try_wait(base + 8 * st, ph)) {
    }
    const uint32_t h = hdr0 + st * kHdr;
    const int prog = (int)lds(h + 4);
    if (prog != cur) {  // (re)load the program's code32 (rare: tiles are program-sorted)
      asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
      const uint32_t *g = a.code + a.prog_off[prog];
      const uint32_t nw = g[2];
      for (uint32_t i = tid; i < nw / 4; i += T)
        reinterpret_cast<uint4 *>(code)[i] = reinterpret_cast<const uint4 *>(g)[i];
      const uint32_t zrow = g[3];   // from global: the smem copy is not complete yet
      for (int k = 0; k < S; ++k)   // the zero row (slot nslots) of every region
        sts(regions + k * a.region + zrow * T * 4 + tid * 4, 0u);
      asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
      cur = prog;
    }
    const uint32_t tw = tile % a.tps;
    const uint32_t w = tw * T + tid;
    if (w < a.words) {
      const uint32_t R = regions + st * a.region + tid * 4;
      const uint64_t off = (uint64_t)w * 4;
      const uint32_t nl = code[0], nm = code[1];
      const uint4 *mp = reinterpret_cast<const uint4 *>(code + ((4 + 2 * nl + 7) & ~7u));
      uint32_t acc = 0;
#pragma unroll 2
      for (uint32_t m = 0; m < nm; ++m) {
        const uint4 o = mp[2 * m], f = mp[2 * m + 1];
        acc = (f.x & 1) ? 0u : acc;
        acc = xor3(acc, lds(R + o.x), lds(R + o.y));
        acc = xor3(acc, lds(R + o.z), lds(R + o.w));
        // predicated stores (no divergent branch): variable slot, goal strip
        asm volatile(
            "{\n .reg .pred p, q;\n .reg .b32 t;\n .reg .b64 g, a;\n"
            " and.b32 t, %0, 2;\n setp.ne.u32 p, t, 0;\n @p st.shared.u32 [%1], %2;\n"
            " and.b32 t, %0, 4;\n setp.ne.u32 q, t, 0;\n"
            " @q ld.shared.u64 g, [%3];\n @q mad.wide.u32 a, %4, %5, %6;\n @q add.s64 a, a, g;\n"
            " @q st.global.cs.u32 [a], %2;\n}\n"
            ::"r"(f.x), "r"(R + f.y), "r"(acc), "r"(h + 16 + 8 * (f.z >> 3)), "r"(f.z & 7),
            "r"((uint32_t)a.strip), "l"(off)
            : "memory");
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(base + 64 + 8 * st) : "memory");
  }
}

// ---- host launch -----------------------------------------------------------------------
struct Code32Pool {
  uint32_t *code = nullptr;
  int64_t *off = nullptr;
  int cap = 0;  // max words of one program
};
static std::mutex g_c32_mu;
static std::map<std::tuple<int, int, std::vector<const Program *>>, Code32Pool> g_c32;

static Code32Pool code32_pool(const Program *const *progs, int np, int T, int dev) {
  std::vector<const Program *> key(progs, progs + np);
  std::lock_guard<std::mutex> g(g_c32_mu);
  auto it = g_c32.find({dev, T, key});
  if (it != g_c32.end()) return it->second;
  std::vector<uint32_t> all;
  std::vector<int64_t> off;
  int cap = 0;
  for (int i = 0; i < np; ++i) {
    auto c = build_code32(progs[i]->code, T);
    off.push_back((int64_t)all.size());
    cap = std::max(cap, (int)c.size());
    all.insert(all.end(), c.begin(), c.end());
  }
  Code32Pool P;
  P.cap = cap;
  CUDA_OK(cudaMalloc(&P.code, all.size() * 4));
  CUDA_OK(cudaMemcpy(P.code, all.data(), all.size() * 4, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMalloc(&P.off, off.size() * 8));
  CUDA_OK(cudaMemcpy(P.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  g_c32[{dev, T, key}] = P;
  return P;
}

// Programs are freed by their owners; a pool must not outlive a member program (a later
// program allocated at the same address would otherwise find it).  Called by ~Program.
void drop_code32_of(const Program *p) {
  std::lock_guard<std::mutex> g(g_c32_mu);
  for (auto it = g_c32.begin(); it != g_c32.end();) {
    const auto &progs = std::get<2>(it->first);
    if (std::find(progs.begin(), progs.end(), p) != progs.end()) {
      int cur = -1;
      const bool have = cudaGetDevice(&cur) == cudaSuccess;
      cudaSetDevice(std::get<0>(it->first));
      cudaFree(it->second.code);
      cudaFree(it->second.off);
      if (have) cudaSetDevice(cur);
      it = g_c32.erase(it);
    } else {
      ++it;
    }
  }
}

static size_t interp_pipe_smem(int S, int cap, int nslots, int T) {
  return 128 + (size_t)S * kHdr + (size_t)cap * 4 + (size_t)S * nslots * T * 4;
}

// Launch the pipelined interpreter; false if it does not apply (then the caller uses the
// one-tile interpreter): needs pointer tables, strip % 16 == 0 (TMA), <= 32 output blocks.
struct InterpPlan {
  int T = 0, S = 2, nslots = 0, cap = 0;
  size_t smem = 0;
  int grid_per_sm = 1;
  Code32Pool pool;
};

// Everything a launch needs that is not capturable in a CUDA graph (pool allocation and upload,
// the function attribute, the occupancy query), done once per (programs, T, device).
static bool interp_pipe_plan(const Program *const *progs, int np, size_t B, int want_T,
                             InterpPlan &out) {
  const uint64_t strip = B / 8;
  if (strip % 16 || progs[0]->n_goals / 8 > 32) return false;
  int nslots = 1, maxcode = 8;
  for (int i = 0; i < np; ++i) {
    nslots = std::max(nslots, progs[i]->nslots);
    maxcode = std::max(maxcode, (int)progs[i]->code.size());
  }
  nslots += 1;  // + the zero row
  const int S = 2;
  int T = std::min(992, std::max(32, want_T / 32 * 32));
  // micro-op code is about 4x the u16 code (8 words per <= 4 operands)
  while (T >= 32 && interp_pipe_smem(S, 5 * maxcode + 64, nslots, T) > 227 * 1024) T -= 32;
  if (T < 32) return false;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  Code32Pool pool = code32_pool(progs, np, T, dev);
  const int cap = (pool.cap + 31) / 32 * 32;
  const size_t smem = interp_pipe_smem(S, cap, nslots, T);
  if (smem > 227 * 1024) return false;
  static std::mutex m;
  static std::map<int, bool> attr;
  static std::map<std::tuple<int, int, size_t>, int> occ;
  int per = 1;
  {
    std::lock_guard<std::mutex> g(m);
    if (!attr[dev]) {
      CUDA_OK(cudaFuncSetAttribute(xslp_interp_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr[dev] = true;
    }
    auto key = std::make_tuple(dev, T, smem);
    auto it = occ.find(key);
    if (it == occ.end()) {
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, xslp_interp_pipe, T + 32, smem));
      occ[key] = std::max(1, per);
    }
    per = occ[key];
  }
  out.T = T;
  out.S = S;
  out.nslots = nslots;
  out.cap = cap;
  out.smem = smem;
  out.grid_per_sm = per;
  out.pool = pool;
  return true;
}

bool interp_pipe_prepare(const Program *p, size_t B) {
  const Program *ps[1] = {p};
  InterpPlan plan;
  return interp_pipe_plan(ps, 1, B, p->opts.threads, plan);
}

bool interp_pipe_launch(const Program *const *progs, int np, const int32_t *d_pos,
                        const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                        int nstripes, size_t B, cudaStream_t st, int want_T) {
  if (!in || !out || nstripes <= 0) return false;
  InterpPlan plan;
  if (!interp_pipe_plan(progs, np, B, want_T, plan)) return false;
  const int T = plan.T;
  const uint64_t strip = B / 8;
  InterpArgs a{};
  a.code = plan.pool.code;
  a.prog_off = plan.pool.off;
  a.prog_of_stripe = d_pos;
  a.ids = d_ids;
  a.in_tbl = in;
  a.out_tbl = out;
  a.strip = strip;
  a.words = (uint32_t)(strip / 4);
  a.tps = (a.words + T - 1) / T;
  if ((uint64_t)a.tps * nstripes > 0xffffffffull) throw Error(XSLP_EINVAL, "too many tiles");
  a.ntiles = a.tps * (uint32_t)nstripes;
  a.n_in = progs[0]->n_const / 8;
  a.n_out = progs[0]->n_goals / 8;
  a.S = plan.S;
  a.code_cap = plan.cap;
  a.region = plan.nslots * T * 4;
  int dev = 0, sms = 148;
  CUDA_OK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<uint64_t>(a.ntiles, (uint64_t)sms * plan.grid_per_sm);
  xslp_interp_pipe<<<grid, T + 32, plan.smem, st>>>(a);
  CUDA_OK(cudaGetLastError());
  count_launch();
  return true;
}

}  // namespace xslp
