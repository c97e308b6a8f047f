// Device side of libxslp: the generic SLP interpreter kernel, the seeded fill kernel,
// loading of the JIT-compiled straight-line kernels, and the C-ABI launch entry
// points (xslp_encode / decode / *_batch / decode_batch_multi / encode_host).
//
// Hot path: H8 load strips -> H9 execute the scheduled MultiSLP -> H10 store goals
// -> H11 grid over (stripe x tile); the paper's blocked loop
// "for i in 0..len/B { v1[i] = xor(...) ... }" ([Peb]) becomes one
// thread per word position, registers (straight-line) or shared-memory slots
// (interpreter) standing in for the paper's L1-resident blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "xslp_api.h"

namespace xslp {

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches++; }
bool interp_pipe_launch(const Program *const *progs, int np, const int32_t *d_pos,
                        const int32_t *d_ids, const uint8_t *const *in, uint8_t *const *out,
                        int nstripes, size_t B, cudaStream_t st, int want_T);  // interp.cu


// ---------------------------------------------------------------------------------
// Interpreter kernel (A29: "run optimized SLPs line-by-line ... in the interpreter
// style").  One thread = one 32-bit word position of every strip of one
// stripe.  Slot s of the thread lives at smem[s * blockDim.x + tid] (bank-conflict
// free); bytecode format in compiler.cpp build_bytecode().  Each CTA reads its own
// program, so one launch can run a different program per stripe (cfg3).
struct OnePtrs {
  const uint8_t *p[128];
};

__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared memory: [0,128) mbarrier | code (code_cap u16 words) | slot rows [nslots][T] u32.
// Constants reach their slot rows by TMA bulk copies (one per used constant, issued by
// thread 0, completion counted on one mbarrier) when `tma` is set (strip % 16 == 0),
// otherwise by batched per-thread streaming loads.  The bytecode is staged with
// coalesced 16-byte copies.
__global__ void __launch_bounds__(1024) xslp_interp_kernel(
    const uint16_t *__restrict__ code_pool, const int64_t *__restrict__ prog_off,
    const int32_t *__restrict__ prog_of_stripe, const uint8_t *const *__restrict__ in_tbl,
    uint8_t *const *__restrict__ out_tbl, int n_in, int n_out, uint64_t strip, uint32_t words,
    uint32_t stripe_base, int code_cap, int tma, OnePtrs one) {
  extern __shared__ __align__(128) uint8_t smraw[];
  const uint32_t T = blockDim.x, tid = threadIdx.x;
  const uint32_t tile0 = blockIdx.x * T;
  const uint32_t w = tile0 + tid;
  const uint32_t s = blockIdx.y + stripe_base;
  const int prog = prog_of_stripe ? prog_of_stripe[s] : 0;
  const uint16_t *gcode = code_pool + prog_off[prog];
  uint16_t *code = reinterpret_cast<uint16_t *>(smraw + 128);
  uint32_t *rows = reinterpret_cast<uint32_t *>(smraw + 128 + (size_t)code_cap * 2);
  const uint32_t mbar = smem_u32(smraw);
  const uint8_t *const *in;
  uint8_t *const *out;
  if (in_tbl) {
    in = in_tbl + (size_t)s * n_in;
    out = out_tbl + (size_t)s * n_out;
  } else {
    in = one.p;
    out = (uint8_t *const *)(one.p + n_in);
  }
  // stage the bytecode (total words is a multiple of 8)
  const int total = __ldg(gcode + 2);
  for (int i = tid; i < total / 8; i += T)
    reinterpret_cast<uint4 *>(code)[i] = __ldg(reinterpret_cast<const uint4 *>(gcode) + i);
  if (tma && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nl = code[0];
  const uint32_t ntile = min(T, words - tile0);
  if (tma) {
    if (tid == 0) {
      const uint32_t bytes = ntile * 4;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar),
                   "r"(bytes * nl) : "memory");
      for (int i = 0; i < nl; ++i) {
        const int c = code[4 + 2 * i], slot = code[5 + 2 * i];
        const uint8_t *src = in[c >> 3] + (c & 7) * strip + (size_t)tile0 * 4;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(smem_u32(rows + (size_t)slot * T)), "l"(src), "r"(bytes), "r"(mbar) : "memory");
      }
    }
    asm volatile(
        "{\n .reg .pred p;\n XSLP_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra XSLP_WAIT_%=;\n}\n" ::"r"(mbar) : "memory");
    if (w >= words) return;
  } else {
    if (w >= words) return;
    const size_t off = (size_t)w * 4;
    int i = 0;
    for (; i + 16 <= nl; i += 16) {  // 16 independent loads in flight per thread
      uint32_t v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int c = code[4 + 2 * (i + u)];
        v[u] = ld_stream((const uint32_t *)(in[c >> 3] + (c & 7) * strip + off));
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) rows[code[5 + 2 * (i + u)] * T + tid] = v[u];
    }
    for (; i < nl; ++i) {
      const int c = code[4 + 2 * i];
      rows[code[5 + 2 * i] * T + tid] = ld_stream((const uint32_t *)(in[c >> 3] + (c & 7) * strip + off));
    }
  }
  const size_t off = (size_t)w * 4;
  uint32_t *my = rows + tid;
  const uint32_t *code32 = reinterpret_cast<const uint32_t *>(code);
  int pc = 4 + 2 * nl;
  const int ni = code[1];
  for (int k = 0; k < ni; ++k) {
    const int hdr = code[pc++];
    const int arity = hdr & 1023, ng = (hdr >> 10) & 15;
    const int dst = (hdr & 0x8000) ? code[pc++] : -1;
    const int gp = pc;
    pc += ng;
    pc += pc & 1;
    uint32_t acc = 0;
    const uint32_t *ops = code32 + (pc >> 1);
    const int npairs = arity >> 1;
#pragma unroll 4
    for (int q = 0; q < npairs; ++q) {
      const uint32_t w2 = ops[q];
      acc ^= my[(w2 & 0xffff) * T] ^ my[(w2 >> 16) * T];
    }
    if (arity & 1) acc ^= my[code[pc + arity - 1] * T];
    pc += arity + (arity & 1);
    if (dst >= 0) my[dst * T] = acc;
    for (int g = 0; g < ng; ++g) {
      const int gi = code[gp + g];
      __stcs((uint32_t *)(out[gi >> 3] + (gi & 7) * strip + off), acc);
    }
  }
}

// Seeded synthetic bytes (same counter-based generator as synth/__init__.py).
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void xslp_fill_kernel(uint64_t *buf, uint64_t wpb, int nblocks, uint64_t total,
                                 uint64_t seed, int64_t stripe0) {
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t w = idx % wpb, blk = idx / wpb;
    const uint64_t s = blk / nblocks + (uint64_t)stripe0, j = blk % nblocks;
    const uint64_t base = seed * 0x9E3779B97F4A7C15ull + ((s * 64 + j) << 40);
    buf[idx] = splitmix64(base + w);
  }
}

// ---------------------------------------------------------------------------------
// Per-program device state.
struct Program::Dev {
  uint16_t *d_code = nullptr;
  int64_t *d_off = nullptr;
};

struct JitLib {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t batch = nullptr, one = nullptr, tma = nullptr, pipe = nullptr, pipe_one = nullptr;
  std::map<int, int> smem_set;       // device -> max dynamic smem configured for `tma`
  std::map<int, int> smem_set_pipe;  // same for `pipe`
  std::map<int, int> pipe_occ;       // device -> resident pipe CTAs per SM (at smem_set_pipe)
  std::map<int, int> smem_set_one;   // same two for `pipe_one`
  std::map<int, int> one_occ;
};

// Libraries are context independent (cudaLibraryLoadData); keyed by program serial.
static std::mutex g_mu;
static std::map<const Program *, std::pair<JitLib, JitLib>> g_libs;

static void load_lib(const std::vector<char> &cubin, JitLib &L) {
  if (cubin.empty() || L.lib) return;
  CUDA_OK(cudaLibraryLoadData(&L.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  CUDA_OK(cudaLibraryGetKernel(&L.batch, L.lib, "xslp_sl_batch"));
  CUDA_OK(cudaLibraryGetKernel(&L.one, L.lib, "xslp_sl_one"));
  // the byte layout has no TMA variants
  if (cudaLibraryGetKernel(&L.tma, L.lib, "xslp_sl_tma") != cudaSuccess) L.tma = nullptr;
  if (cudaLibraryGetKernel(&L.pipe, L.lib, "xslp_sl_pipe") != cudaSuccess) L.pipe = nullptr;
  // single-stripe pipeline (strip layout without phases or consumer groups)
  if (cudaLibraryGetKernel(&L.pipe_one, L.lib, "xslp_sl_pipe_one") != cudaSuccess) L.pipe_one = nullptr;
  cudaGetLastError();
}

static std::pair<JitLib, JitLib> libs_of(const Program *p) {
  std::lock_guard<std::mutex> g(g_mu);
  auto &e = g_libs[p];
  load_lib(p->cubin_generic, e.first);
  load_lib(p->cubin_baked, e.second);
  return e;
}

static int current_device() {
  int d = -1;
  CUDA_OK(cudaGetDevice(&d));
  return d;
}

static std::shared_ptr<Program::Dev> dev_of(const Program *p) {
  const int d = current_device();
  std::lock_guard<std::mutex> g(p->mu);
  auto &e = p->dev[d];
  if (!e) {
    auto D = std::make_shared<Program::Dev>();
    CUDA_OK(cudaMalloc(&D->d_code, p->code.size() * 2));
    CUDA_OK(cudaMemcpy(D->d_code, p->code.data(), p->code.size() * 2, cudaMemcpyHostToDevice));
    int64_t z = 0;
    CUDA_OK(cudaMalloc(&D->d_off, 8));
    CUDA_OK(cudaMemcpy(D->d_off, &z, 8, cudaMemcpyHostToDevice));
    e = D;
  }
  return e;
}

static void drop_pools_of(const Program *p);  // below: pools that contain p's bytecode

void drop_code32_of(const Program *p);  // interp.cu
void drop_lanes_of(const Program *p);   // interp_lanes.cu
void drop_tmem_of(const Program *p);    // interp_tmem.cu

Program::~Program() {
  {
    // kernels of this program (its JIT library, its code pools) may still be in flight on any
    // device (e.g. an LRU eviction in a codec while another thread's decode runs): wait for
    // them before unloading / freeing anything (destruction is rare; launches are async)
    bool used;
    {
      std::lock_guard<std::mutex> g(g_mu);
      used = g_libs.count(this) != 0;
    }
    used = used || !dev.empty();
    int ndev = 0, cur = -1;
    if (used && cudaGetDeviceCount(&ndev) == cudaSuccess && cudaGetDevice(&cur) == cudaSuccess) {
      for (int d = 0; d < ndev; ++d) {
        cudaSetDevice(d);
        cudaDeviceSynchronize();
      }
      cudaSetDevice(cur);
    }
  }
  drop_pools_of(this);  // a later program at the same address must not find this one's pool
  drop_code32_of(this);
  drop_lanes_of(this);
  drop_tmem_of(this);
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_libs.find(this);
    if (it != g_libs.end()) {
      if (it->second.first.lib) cudaLibraryUnload(it->second.first.lib);
      if (it->second.second.lib) cudaLibraryUnload(it->second.second.lib);
      g_libs.erase(it);
    }
  }
  int cur = -1;
  bool have = cudaGetDevice(&cur) == cudaSuccess;
  for (auto &kv : dev) {
    if (!kv.second) continue;
    cudaSetDevice(kv.first);
    cudaFree(kv.second->d_code);
    cudaFree(kv.second->d_off);
  }
  if (have) cudaSetDevice(cur);
}

// ---------------------------------------------------------------------------------
static void check_geometry(const Program *p, size_t block_bytes) {
  if (block_bytes % 32)
    throw Error(XSLP_EINVAL, "block_bytes must be a multiple of 32 (strip = whole 32-bit words)");
  if (p->n_const % 8 || p->n_goals % 8)
    throw Error(XSLP_EINVAL, "program does not act on whole blocks");
  if (block_bytes / 8 / 4 > 0xffffffffull) throw Error(XSLP_EINVAL, "block too large");
}

static size_t interp_smem(int nslots, int code_cap, int T) {
  return 128 + (size_t)code_cap * 2 + (size_t)nslots * T * 4;
}

// code words rounded to 64 (128-byte alignment of the slot rows)
static int code_cap_of(const Program *const *progs, int np) {
  size_t m = 8;
  for (int i = 0; i < np; ++i) m = std::max(m, progs[i]->code.size());
  return (int)((m + 63) / 64 * 64);
}

static int interp_threads(const Program *const *progs, int np, int want) {
  int nslots = 1;
  for (int i = 0; i < np; ++i) nslots = std::max(nslots, progs[i]->nslots);
  const int cap = code_cap_of(progs, np);
  int T = want;
  while (T >= 32 && interp_smem(nslots, cap, T) > 227 * 1024) T -= 32;
  if (T < 32) throw Error(XSLP_EINVAL, "program too large for the interpreter's shared memory");
  return T;
}

static void set_smem_attr() {
  static std::mutex m;
  static std::map<int, bool> done;
  int d = current_device();
  std::lock_guard<std::mutex> g(m);
  if (done[d]) return;
  CUDA_OK(cudaFuncSetAttribute(xslp_interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024));
  done[d] = true;
}

// Launch the interpreter over `nstripes` stripes (tables) or one stripe (one != null).
static void launch_interp(const uint16_t *code_pool, const int64_t *offs, const int32_t *pos,
                          int np_threads_T, const Program *p0, int nslots_max, int code_cap,
                          const uint8_t *const *in_tbl, uint8_t *const *out_tbl, int nstripes,
                          size_t block_bytes, cudaStream_t st, const OnePtrs *one) {
  set_smem_attr();
  const uint64_t strip = block_bytes / 8;
  const uint32_t words = (uint32_t)(strip / 4);
  const int T = np_threads_T;
  const size_t smem = interp_smem(nslots_max, code_cap, T);
  const int tma = (strip % 16 == 0) && in_tbl != nullptr;
  OnePtrs op{};
  if (one) op = *one;
  for (int base = 0; base < nstripes; base += 65535) {
    dim3 grid((words + T - 1) / T, std::min(65535, nstripes - base));
    xslp_interp_kernel<<<grid, T, smem, st>>>(code_pool, offs, pos, in_tbl, out_tbl,
                                              p0->n_const / 8, p0->n_goals / 8, strip, words,
                                              (uint32_t)base, code_cap, tma, op);
    CUDA_OK(cudaGetLastError());
    g_launches++;
  }
}

static bool can_straight(const Program *p, size_t block_bytes, bool &baked) {
  const int L = p->opts.lane_words;
  const uint64_t strip = block_bytes / 8;
  baked = !p->cubin_baked.empty() && (int64_t)strip == p->baked_strip;
  if (p->cubin_generic.empty() && !baked) return false;
  return strip % (4 * L) == 0;
}

// AUTO: the persistent TMA pipeline when its stages fit in shared memory and there are
// enough tiles to keep every SM busy (measured fastest: profiles/r01_*), otherwise the
// register-resident LDG kernel.
static int auto_kernel(const Program *p, size_t block_bytes, int nstripes) {
  if (p->opts.layout == XSLP_LAYOUT_BYTE) {  // 32-byte chunks staged once, read once
    const int T = p->opts.threads;
    const size_t smem = 128 + (size_t)p->opts.stages * p->stage_used_const * 4 * T;
    const uint64_t tiles = (block_bytes / 32 + T - 1) / T * (uint64_t)nstripes;
    if (smem > 227 * 1024 || p->opts.stages < 2 || tiles < 4 * 148 || T > 992)
      return XSLP_KERNEL_STRAIGHT;
    return XSLP_KERNEL_PIPE;
  }
  const uint64_t strip = block_bytes / 8;
  const int T = p->opts.threads, L = p->opts.lane_words;
  if (strip % 16 || p->opts.threads * std::max<int>(1, (int)p->groups.size()) > 992) return XSLP_KERNEL_STRAIGHT;
  const size_t smem = 128 + (size_t)p->opts.stages * p->stage_used_const * 4 * L * T;
  const uint64_t tiles = (strip / (4 * L) + T - 1) / T * (uint64_t)nstripes;
  if (smem > 227 * 1024 || p->opts.stages < 2 || tiles < 4 * 148) return XSLP_KERNEL_STRAIGHT;
  // shared-memory bytes per data byte of the pipeline (one 4-byte read per constant read
  // the emitted code issues under the reuse window, 32n data bytes per word position): above
  // ~6 the pipeline was smem-bound (uncompressed programs without the reuse window,
  // profiles/r01_cfg4_sweep.md) and the register-resident kernel wins
  if (p->const_reads * 4.0 / (4.0 * p->n_const) > 6.0) return XSLP_KERNEL_STRAIGHT;
  return XSLP_KERNEL_PIPE;
}

// PIPE CTA size: `groups` consumer groups of `threads` threads plus one producer warp
static int pipe_block(const Program *p) {
  return p->opts.threads * (p->groups.empty() ? 1 : (int)p->groups.size()) + 32;
}

static void apply_batch(const Program *p, const uint8_t *const *d_in, uint8_t *const *d_out,
                        const int32_t *d_ids, int nstripes, size_t block_bytes,
                        cudaStream_t st) {
  check_geometry(p, block_bytes);
  if (nstripes < 0) throw Error(XSLP_EINVAL, "nstripes < 0");
  if (!d_in || !d_out) throw Error(XSLP_EINVAL, "null pointer table");
  if (nstripes == 0 || block_bytes == 0) return;
  bool baked = false;
  int kind = p->opts.kernel;
  bool straight = kind != XSLP_KERNEL_INTERP && can_straight(p, block_bytes, baked);
  if (kind == XSLP_KERNEL_AUTO && straight) kind = auto_kernel(p, block_bytes, nstripes);
  if ((kind == XSLP_KERNEL_STRAIGHT || kind == XSLP_KERNEL_TMA || kind == XSLP_KERNEL_PIPE) &&
      !straight)
    throw Error(XSLP_EINVAL, "straight-line kernel unavailable for this block size / program");
  if (straight && kind == XSLP_KERNEL_PIPE) {
    const int T = p->opts.threads, L = p->opts.lane_words;
    uint64_t strip = block_bytes / 8;
    const bool bytel = p->opts.layout == XSLP_LAYOUT_BYTE;
    if (!bytel && strip % 16) throw Error(XSLP_EINVAL, "TMA staging needs block_bytes % 128 == 0");
    // byte layout: a "word" is a thread's 32-byte chunk of every block
    uint32_t words = bytel ? (uint32_t)(block_bytes / 32) : (uint32_t)(strip / (4 * L));
    uint32_t tps = (words + T - 1) / T;
    if ((uint64_t)tps * (uint64_t)nstripes > 0xffffffffull) throw Error(XSLP_EINVAL, "too many tiles");
    uint32_t ntiles = tps * (uint32_t)nstripes;
    const size_t smem = 128 + (size_t)p->opts.stages * p->stage_used_const * 4 * L * T;
    if (smem > 227 * 1024) throw Error(XSLP_EINVAL, "pipeline stages do not fit in shared memory");
    cudaKernel_t k;
    int grid;
    {
      libs_of(p);
      std::lock_guard<std::mutex> g(g_mu);
      JitLib &J = baked ? g_libs[p].second : g_libs[p].first;
      k = J.pipe;
      const int d = current_device();
      if (J.smem_set_pipe[d] < (int)smem) {
        CUDA_OK(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, d));
        J.smem_set_pipe[d] = (int)smem;
      }
      int sms = 148, per = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
      auto it = J.pipe_occ.find(d);
      if (it != J.pipe_occ.end()) {
        per = it->second;
      } else {
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)k, pipe_block(p), smem));
        J.pipe_occ[d] = per;
      }
      grid = (int)std::min<uint64_t>(ntiles, (uint64_t)sms * std::max(1, per));
    }
    void *args[] = {(void *)&d_in, (void *)&d_out, (void *)&d_ids, &strip, &words, &tps, &ntiles};
    CUDA_OK(cudaLaunchKernel((const void *)k, dim3(grid), dim3(pipe_block(p)), args, smem, st));
    g_launches++;
    return;
  }
  if (straight) {
    const bool tma = kind == XSLP_KERNEL_TMA;
    const int T = p->opts.threads;
    uint64_t strip = block_bytes / 8;
    if (tma && strip % 16)
      throw Error(XSLP_EINVAL, "TMA staging needs block_bytes % 128 == 0");
    uint32_t words = (uint32_t)(strip / (4 * p->opts.lane_words));
    size_t smem = 0;
    cudaKernel_t k;
    {
      libs_of(p);
      std::lock_guard<std::mutex> g(g_mu);
      JitLib &L = baked ? g_libs[p].second : g_libs[p].first;
      k = tma ? L.tma : L.batch;
      if (tma) {
        smem = 128 + (size_t)p->n_used_const * 4 * p->opts.lane_words * T;
        if (smem > 227 * 1024) throw Error(XSLP_EINVAL, "TMA tile does not fit in shared memory; use fewer threads");
        const int d = current_device();
        if (L.smem_set[d] < (int)smem) {
          CUDA_OK(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, d));
          L.smem_set[d] = (int)smem;
        }
      }
    }
    for (int base = 0; base < nstripes; base += 65535) {
      uint32_t b = (uint32_t)base;
      void *args[] = {(void *)&d_in, (void *)&d_out, (void *)&d_ids, &strip, &words, &b};
      dim3 grid((words + T - 1) / T, std::min(65535, nstripes - base));
      CUDA_OK(cudaLaunchKernel((const void *)k, grid, dim3(T), args, smem, st));
      g_launches++;
    }
    return;
  }
  {  // the pipelined interpreter (interp.cu) when it applies, else the one-tile interpreter
    const Program *ps1[1] = {p};
    if (interp_pipe_launch(ps1, 1, nullptr, d_ids, d_in, d_out, nstripes, block_bytes, st,
                           p->opts.threads))
      return;
  }
  if (d_ids) throw Error(XSLP_EINVAL, "stripe id lists need the straight-line kernel");
  auto D = dev_of(p);
  const Program *ps[1] = {p};
  const int T = interp_threads(ps, 1, p->opts.threads);
  launch_interp(D->d_code, D->d_off, nullptr, T, p, p->nslots, code_cap_of(ps, 1), d_in, d_out,
                nstripes, block_bytes, st, nullptr);
}

static void apply_one(const Program *p, const uint8_t *const *in, uint8_t *const *out,
                      size_t block_bytes, cudaStream_t st) {
  check_geometry(p, block_bytes);
  if (!in || !out) throw Error(XSLP_EINVAL, "null block pointer array");
  const int n_in = p->n_const / 8, n_out = p->n_goals / 8;
  if (n_in + n_out > 128) throw Error(XSLP_EINVAL, "too many blocks");
  OnePtrs one{};
  const uintptr_t am = p->opts.layout == XSLP_LAYOUT_BYTE ? 31 : 15;
  for (int j = 0; j < n_in; ++j) {
    if (!in[j] || ((uintptr_t)in[j] & am)) throw Error(XSLP_EINVAL, "input block pointer null or misaligned");
    one.p[j] = in[j];
  }
  for (int i = 0; i < n_out; ++i) {
    if (!out[i] || ((uintptr_t)out[i] & am)) throw Error(XSLP_EINVAL, "output block pointer null or misaligned");
    one.p[n_in + i] = out[i];
  }
  if (block_bytes == 0) return;
  bool baked = false;
  const int kind = p->opts.kernel;
  bool straight = kind != XSLP_KERNEL_INTERP && can_straight(p, block_bytes, baked);
  if (kind == XSLP_KERNEL_STRAIGHT && !straight)
    throw Error(XSLP_EINVAL, "straight-line kernel unavailable for this block size / program");
  if (straight && kind == XSLP_KERNEL_PIPE && p->opts.layout == XSLP_LAYOUT_STRIP &&
      p->groups.empty() && p->phases.empty()) {
    // kernel = PIPE: one stripe through the persistent TMA pipeline with the block pointers
    // passed by value (xslp_sl_pipe_one), no pointer table upload.  AUTO keeps the
    // register-resident kernel for single stripes: on one stripe of 16-107 MiB blocks the two
    // measure the same (4.2-4.35 TB/s, profiles/r01_s2_codec.md) and the LDG form wins for the
    // codec's copy-goal programs
    const int T = p->opts.threads, L = p->opts.lane_words;
    uint64_t strip = block_bytes / 8;
    const size_t smem = 128 + (size_t)p->opts.stages * p->stage_used_const * 4 * L * T;
    cudaKernel_t k = nullptr;
    int grid = 0;
    uint32_t words = (uint32_t)(strip / (4 * L)), tps = (words + T - 1) / T, ntiles = tps;
    if (strip % 16 == 0 && smem <= 227 * 1024) {
      libs_of(p);
      std::lock_guard<std::mutex> g(g_mu);
      JitLib &J = baked ? g_libs[p].second : g_libs[p].first;
      k = J.pipe_one;
      if (k) {
        const int d = current_device();
        if (J.smem_set_one[d] < (int)smem) {
          CUDA_OK(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, d));
          J.smem_set_one[d] = (int)smem;
          J.one_occ.erase(d);
        }
        int sms = 148, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        auto it = J.one_occ.find(d);
        if (it != J.one_occ.end()) {
          per = it->second;
        } else {
          CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)k, pipe_block(p), smem));
          J.one_occ[d] = per;
        }
        grid = (int)std::min<uint64_t>(ntiles, (uint64_t)sms * std::max(1, per));
      }
    }
    if (k) {
      const int32_t *no_ids = nullptr;
      void *args[] = {&one, (void *)&no_ids, &strip, &words, &tps, &ntiles};
      CUDA_OK(cudaLaunchKernel((const void *)k, dim3(grid), dim3(pipe_block(p)), args, smem, st));
      g_launches++;
      return;
    }
    // otherwise (phases, consumer groups, misaligned strips): the register-resident kernel
  }
  if (straight) {
    auto libs = libs_of(p);
    const JitLib &L = baked ? libs.second : libs.first;
    const int T = p->opts.threads;
    uint64_t strip = block_bytes / 8;
    uint32_t words = (uint32_t)(strip / (4 * p->opts.lane_words));
    void *args[] = {&one, &strip, &words};
    CUDA_OK(cudaLaunchKernel((const void *)L.one, dim3((words + T - 1) / T), dim3(T), args, 0, st));
    g_launches++;
    return;
  }
  auto D = dev_of(p);
  const Program *ps[1] = {p};
  const int T = interp_threads(ps, 1, p->opts.threads);
  launch_interp(D->d_code, D->d_off, nullptr, T, p, p->nslots, code_cap_of(ps, 1), nullptr, nullptr,
                1, block_bytes, st, &one);
}

// Pools of several programs' bytecode for one heterogeneous launch, cached by the
// programs' identities per device.
struct Pool {
  uint16_t *code = nullptr;
  int64_t *off = nullptr;
};
static std::map<std::pair<int, std::vector<const Program *>>, Pool> g_pools;

static Pool pool_of(const Program *const *progs, int np) {
  const int d = current_device();
  std::vector<const Program *> key(progs, progs + np);
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_pools.find({d, key});
  if (it != g_pools.end()) return it->second;
  std::vector<uint16_t> all;
  std::vector<int64_t> off;
  for (int i = 0; i < np; ++i) {
    off.push_back((int64_t)all.size());
    all.insert(all.end(), progs[i]->code.begin(), progs[i]->code.end());
  }
  Pool P;
  CUDA_OK(cudaMalloc(&P.code, all.size() * 2));
  CUDA_OK(cudaMemcpy(P.code, all.data(), all.size() * 2, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMalloc(&P.off, off.size() * 8));
  CUDA_OK(cudaMemcpy(P.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
  g_pools[{d, key}] = P;
  return P;
}

static void drop_pools_of(const Program *p) {
  std::lock_guard<std::mutex> g(g_mu);
  for (auto it = g_pools.begin(); it != g_pools.end();) {
    const auto &progs = it->first.second;
    if (std::find(progs.begin(), progs.end(), p) != progs.end()) {
      int cur = -1;
      const bool have = cudaGetDevice(&cur) == cudaSuccess;
      cudaSetDevice(it->first.first);
      cudaFree(it->second.code);
      cudaFree(it->second.off);
      if (have) cudaSetDevice(cur);
      it = g_pools.erase(it);
    } else {
      ++it;
    }
  }
}

// ---------------------------------------------------------------------------------
// Grouped heterogeneous decode: stripes sorted by program on the host; each program's
// straight-line kernel runs over its own stripe-id list.  The launches fan out over a
// per-device pool of internal streams (fork / join with events on the caller's stream)
// so the small per-pattern kernels overlap on the GPU.
struct StreamPool {
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t fork = nullptr;
};
static std::map<int, StreamPool> g_pools_st;
static std::mutex g_st_mu;

static void grouped(const Program *const *progs, int np, const int32_t *d_ids,
                    const int32_t *off, const uint8_t *const *d_in, uint8_t *const *d_out,
                    size_t B, cudaStream_t user, int nstreams) {
  if (!progs || np <= 0 || !off || !d_ids) throw Error(XSLP_EINVAL, "bad grouped arguments");
  for (int i = 0; i < np; ++i) {
    if (!progs[i]) throw Error(XSLP_EINVAL, "null program");
    if (progs[i]->n_const != progs[0]->n_const || progs[i]->n_goals != progs[0]->n_goals)
      throw Error(XSLP_EINVAL, "programs disagree on constants/goals");
    if (off[i + 1] < off[i]) throw Error(XSLP_EINVAL, "group offsets must be non-decreasing");
  }
  if (off[0] < 0) throw Error(XSLP_EINVAL, "negative group offset");
  nstreams = std::max(1, std::min(nstreams, 32));
  const int d = current_device();
  std::lock_guard<std::mutex> g(g_st_mu);
  StreamPool &P = g_pools_st[d];
  while ((int)P.st.size() < nstreams) {
    cudaStream_t s;
    cudaEvent_t e;
    CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P.st.push_back(s);
    P.ev.push_back(e);
  }
  if (!P.fork) CUDA_OK(cudaEventCreateWithFlags(&P.fork, cudaEventDisableTiming));
  CUDA_OK(cudaEventRecord(P.fork, user));
  for (int k = 0; k < nstreams; ++k) CUDA_OK(cudaStreamWaitEvent(P.st[k], P.fork, 0));
  for (int i = 0; i < np; ++i) {
    const int cnt = off[i + 1] - off[i];
    if (cnt == 0) continue;
    apply_batch(progs[i], d_in, d_out, d_ids + off[i], cnt, B, P.st[i % nstreams]);
  }
  for (int k = 0; k < nstreams; ++k) {
    CUDA_OK(cudaEventRecord(P.ev[k], P.st[k]));
    CUDA_OK(cudaStreamWaitEvent(user, P.ev[k], 0));
  }
}

// ---------------------------------------------------------------------------------
// Host-buffer path: chunks of stripes staged through two device buffer sets on two
// internal streams so the H2D copy of chunk c+1 overlaps the kernel and D2H of chunk c.
struct HostWs {
  size_t cap_in = 0, cap_out = 0;
  uint8_t *din[2] = {nullptr, nullptr}, *dout[2] = {nullptr, nullptr};
  const uint8_t **tin[2] = {nullptr, nullptr};
  uint8_t **tout[2] = {nullptr, nullptr};
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t ev = nullptr;
  int n_in = -1, n_out = -1, chunk = -1;
  size_t B = 0;
};
static std::map<int, HostWs> g_ws;
static std::mutex g_ws_mu;  // separate from g_mu: host_apply calls apply_batch (which takes g_mu)

static void host_apply(const Program *p, const uint8_t *h_in, uint8_t *h_out, int nstripes,
                       size_t B, cudaStream_t user) {
  check_geometry(p, B);
  if (nstripes < 0) throw Error(XSLP_EINVAL, "nstripes < 0");
  if (!h_in || !h_out) throw Error(XSLP_EINVAL, "null host buffer");
  if (nstripes == 0 || B == 0) return;
  const int d = current_device();
  const int n_in = p->n_const / 8, n_out = p->n_goals / 8;
  const size_t target = (size_t)256 << 20;
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>(nstripes, target / (n_in * B)));
  std::lock_guard<std::mutex> g(g_ws_mu);
  HostWs &w = g_ws[d];
  if (!w.st[0]) {
    CUDA_OK(cudaStreamCreateWithFlags(&w.st[0], cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&w.st[1], cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&w.ev, cudaEventDisableTiming));
  }
  const size_t need_in = (size_t)chunk * n_in * B, need_out = (size_t)chunk * n_out * B;
  if (need_in > w.cap_in || need_out > w.cap_out) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(w.din[b]);
      cudaFree(w.dout[b]);
      CUDA_OK(cudaMalloc(&w.din[b], need_in));
      CUDA_OK(cudaMalloc(&w.dout[b], need_out));
    }
    w.cap_in = need_in;
    w.cap_out = need_out;
    w.n_in = -1;
  }
  if (w.n_in != n_in || w.n_out != n_out || w.chunk != chunk || w.B != B) {
    for (int b = 0; b < 2; ++b) {
      cudaFree(w.tin[b]);
      cudaFree(w.tout[b]);
      std::vector<const uint8_t *> ti((size_t)chunk * n_in);
      std::vector<uint8_t *> to((size_t)chunk * n_out);
      for (size_t i = 0; i < ti.size(); ++i) ti[i] = w.din[b] + i * B;
      for (size_t i = 0; i < to.size(); ++i) to[i] = w.dout[b] + i * B;
      CUDA_OK(cudaMalloc(&w.tin[b], ti.size() * 8));
      CUDA_OK(cudaMalloc(&w.tout[b], to.size() * 8));
      CUDA_OK(cudaMemcpy(w.tin[b], ti.data(), ti.size() * 8, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(w.tout[b], to.data(), to.size() * 8, cudaMemcpyHostToDevice));
    }
    w.n_in = n_in;
    w.n_out = n_out;
    w.chunk = chunk;
    w.B = B;
  }
  CUDA_OK(cudaEventRecord(w.ev, user));
  CUDA_OK(cudaStreamWaitEvent(w.st[0], w.ev, 0));
  CUDA_OK(cudaStreamWaitEvent(w.st[1], w.ev, 0));
  int c = 0;
  for (int s0 = 0; s0 < nstripes; s0 += chunk, ++c) {
    const int b = c & 1;
    const int ns = std::min(chunk, nstripes - s0);
    CUDA_OK(cudaMemcpyAsync(w.din[b], h_in + (size_t)s0 * n_in * B, (size_t)ns * n_in * B,
                            cudaMemcpyHostToDevice, w.st[b]));
    apply_batch(p, w.tin[b], w.tout[b], nullptr, ns, B, w.st[b]);
    CUDA_OK(cudaMemcpyAsync(h_out + (size_t)s0 * n_out * B, w.dout[b], (size_t)ns * n_out * B,
                            cudaMemcpyDeviceToHost, w.st[b]));
  }
  CUDA_OK(cudaStreamSynchronize(w.st[0]));
  CUDA_OK(cudaStreamSynchronize(w.st[1]));
}

}  // namespace xslp

// =====================================================================================
// C ABI (device entry points)
using namespace xslp;


static const Program *P(const xslp_program *p) {
  if (!p) throw Error(XSLP_EINVAL, "null program");
  return reinterpret_cast<const Program *>(p);
}

// Load everything a launch of `prog` may need on the current device (JIT libraries,
// shared-memory attributes, pipeline occupancy, interpreter bytecode) so later launches do
// no allocation or synchronous copy and can be captured into a CUDA graph.
namespace xslp {
bool interp_pipe_prepare(const Program *p, size_t B);  // interp.cu
}

extern "C" int xslp_prepare(const xslp_program *prog, size_t block_bytes) {
  API_BEGIN
  const Program *p = P(prog);
  dev_of(p);  // interpreter bytecode
  if (block_bytes && block_bytes % 32 == 0)
    interp_pipe_prepare(p, block_bytes);  // the pipelined interpreter's code pool
  set_smem_attr();
  libs_of(p);
  if (block_bytes && block_bytes % 32 == 0) {
    const int T = p->opts.threads, L = p->opts.lane_words;
    const size_t smem_pipe = 128 + (size_t)p->opts.stages * p->stage_used_const * 4 * L * T;
    const size_t smem_tma = 128 + (size_t)p->n_used_const * 4 * L * T;
    const int d = current_device();
    std::lock_guard<std::mutex> g(g_mu);
    for (JitLib *J : {&g_libs[p].first, &g_libs[p].second}) {
      if (J->pipe && smem_pipe <= 227 * 1024 && J->smem_set_pipe[d] < (int)smem_pipe) {
        CUDA_OK(cudaKernelSetAttributeForDevice(J->pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem_pipe, d));
        J->smem_set_pipe[d] = (int)smem_pipe;
        int per = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)J->pipe, pipe_block(p), smem_pipe));
        J->pipe_occ[d] = per;
      }
      if (J->pipe_one && smem_pipe <= 227 * 1024 && J->smem_set_one[d] < (int)smem_pipe) {
        CUDA_OK(cudaKernelSetAttributeForDevice(J->pipe_one, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem_pipe, d));
        J->smem_set_one[d] = (int)smem_pipe;
        int per = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void *)J->pipe_one, pipe_block(p),
                                                              smem_pipe));
        J->one_occ[d] = per;
      }
      if (J->tma && smem_tma <= 227 * 1024 && J->smem_set[d] < (int)smem_tma) {
        CUDA_OK(cudaKernelSetAttributeForDevice(J->tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem_tma, d));
        J->smem_set[d] = (int)smem_tma;
      }
    }
  }
  API_END
}

extern "C" int xslp_encode(const xslp_program *prog, const uint8_t *const *in_blocks,
                           uint8_t *const *out_blocks, size_t block_bytes, void *stream) {
  API_BEGIN
  apply_one(P(prog), in_blocks, out_blocks, block_bytes, (cudaStream_t)stream);
  API_END
}

extern "C" int xslp_decode(const xslp_program *prog, const uint8_t *const *in_blocks,
                           uint8_t *const *out_blocks, size_t block_bytes, void *stream) {
  return xslp_encode(prog, in_blocks, out_blocks, block_bytes, stream);
}

extern "C" int xslp_encode_batch(const xslp_program *prog, const uint8_t *const *d_in_tbl,
                                 uint8_t *const *d_out_tbl, int nstripes, size_t block_bytes,
                                 void *stream) {
  API_BEGIN
  apply_batch(P(prog), d_in_tbl, d_out_tbl, nullptr, nstripes, block_bytes, (cudaStream_t)stream);
  API_END
}

extern "C" int xslp_decode_batch_multi(const xslp_program *const *progs, int nprogs,
                                       const int32_t *d_prog_of_stripe,
                                       const uint8_t *const *d_in_tbl, uint8_t *const *d_out_tbl,
                                       int nstripes, size_t block_bytes, void *stream) {
  API_BEGIN
  if (!progs || nprogs <= 0) throw Error(XSLP_EINVAL, "no programs");
  std::vector<const Program *> ps;
  for (int i = 0; i < nprogs; ++i) ps.push_back(P(progs[i]));
  for (auto q : ps)
    if (q->n_const != ps[0]->n_const || q->n_goals != ps[0]->n_goals)
      throw Error(XSLP_EINVAL, "programs disagree on constants/goals");
  if (nprogs == 1) {
    apply_batch(ps[0], d_in_tbl, d_out_tbl, nullptr, nstripes, block_bytes, (cudaStream_t)stream);
  } else {
    check_geometry(ps[0], block_bytes);
    if (!d_prog_of_stripe || !d_in_tbl || !d_out_tbl) throw Error(XSLP_EINVAL, "null table");
    if (nstripes < 0) throw Error(XSLP_EINVAL, "nstripes < 0");
    if (nstripes == 0 || block_bytes == 0) return XSLP_OK;
    if (interp_pipe_launch(ps.data(), nprogs, d_prog_of_stripe, nullptr, d_in_tbl, d_out_tbl,
                           nstripes, block_bytes, (cudaStream_t)stream, ps[0]->opts.threads))
      return XSLP_OK;
    Pool pool = pool_of(ps.data(), nprogs);
    int nsl = 1;
    for (auto q : ps) nsl = std::max(nsl, q->nslots);
    const int T = interp_threads(ps.data(), nprogs, ps[0]->opts.threads);
    launch_interp(pool.code, pool.off, d_prog_of_stripe, T, ps[0], nsl,
                  code_cap_of(ps.data(), nprogs), d_in_tbl, d_out_tbl, nstripes, block_bytes,
                  (cudaStream_t)stream, nullptr);
  }
  API_END
}

extern "C" int xslp_decode_batch_grouped(const xslp_program *const *progs, int nprogs,
                                         const int32_t *d_stripe_ids, const int32_t *group_offsets,
                                         const uint8_t *const *d_in_tbl, uint8_t *const *d_out_tbl,
                                         size_t block_bytes, int nstreams, void *stream) {
  API_BEGIN
  if (!progs || nprogs <= 0) throw Error(XSLP_EINVAL, "no programs");
  std::vector<const Program *> ps;
  for (int i = 0; i < nprogs; ++i) ps.push_back(P(progs[i]));
  if (!d_in_tbl || !d_out_tbl) throw Error(XSLP_EINVAL, "null table");
  check_geometry(ps[0], block_bytes);
  if (block_bytes == 0) return XSLP_OK;
  grouped(ps.data(), nprogs, d_stripe_ids, group_offsets, d_in_tbl, d_out_tbl, block_bytes,
          (cudaStream_t)stream, nstreams);
  API_END
}

extern "C" int xslp_encode_host(const xslp_program *prog, const uint8_t *h_in, uint8_t *h_out,
                                int nstripes, size_t block_bytes, void *stream) {
  API_BEGIN
  host_apply(P(prog), h_in, h_out, nstripes, block_bytes, (cudaStream_t)stream);
  API_END
}

extern "C" int xslp_fill_random(uint8_t *d_buf, int nstripes, int nblocks, size_t block_bytes,
                                uint64_t seed, int64_t stripe0, void *stream) {
  API_BEGIN
  if (!d_buf || nstripes < 0 || nblocks < 0 || block_bytes % 8 || ((uintptr_t)d_buf & 7))
    throw Error(XSLP_EINVAL, "bad fill arguments");
  // the counter key ((s*64 + j) << 40) + i is distinct only for j < 64, s < 2^18, i < 2^40
  if (nblocks > 64 || stripe0 < 0 || stripe0 + (int64_t)nstripes > (int64_t(1) << 18) ||
      block_bytes / 8 >= (uint64_t(1) << 40))
    throw Error(XSLP_EINVAL, "fill key range: need nblocks <= 64 and stripes < 2^18");
  const uint64_t wpb = block_bytes / 8;
  const uint64_t total = wpb * (uint64_t)nblocks * (uint64_t)nstripes;
  if (total == 0) return XSLP_OK;
  int dev = current_device(), sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (total + 255) / 256;
  const int grid = (int)std::min<uint64_t>(want, (uint64_t)sms * 16);
  xslp_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((uint64_t *)d_buf, wpb, nblocks, total,
                                                          seed, stripe0);
  CUDA_OK(cudaGetLastError());
  g_launches++;
  API_END
}

extern "C" int64_t xslp_launch_count(void) { return g_launches.load(); }
