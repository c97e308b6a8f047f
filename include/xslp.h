/*
 * xslp.h -- C ABI of libxslp: XOR straight-line-program (SLP_xor) erasure coding on B200.
 *
 * What it computes (arXiv 2108.02692, Uezato SC'21; "P:n" = line n of the paper
 * text, section tags as in DESIGN.md):
 *   RS(n,p) over GF(2^8) (polynomial x^8+x^4+x^3+x^2+1) is lowered to a
 *   GF(2) bitmatrix V~ ([Intro]) and lifted to an SLP_xor whose
 *   constants are the 8n input strips and whose goals are the 8p parity (or 8e
 *   recovered) strips ([Appr]).  The host compiler shrinks it with
 *   RePair / XorRePair ([SLP]), XOR fusion ([Fus]) and the
 *   DFS pebble-game schedule ([Peb]); the device executes it over
 *   byte arrays with hand-written sm_100a kernels.
 *
 * Strip layout: a block of B bytes is 8 contiguous strips of B/8
 * bytes; constant c_{8j+k} is strip k of input block j, goal g_{8i+r} is strip r
 * of output block i.  Bitmatrix entry (8i+r, 8j+k) = bit r of (G_ij * 2^k)
 * (LSB-first byte<->bit-vector map, reading R3).
 *
 * Conventions for every call
 *   - Return value: XSLP_OK (0) or a negative XSLP_E* code.  Calls never abort;
 *     the message of the last failure on the calling thread is xslp_last_error().
 *   - Host pointers are plain C arrays owned by the caller and only read/written
 *     during the call.  Device pointers are owned by the caller; the library
 *     never frees them.  Device calls are asynchronous on the given stream (a
 *     cudaStream_t passed as void*; NULL = legacy default stream) and use the
 *     calling thread's current CUDA device.
 *   - Device buffers: every block pointer 16-byte aligned; outputs must not
 *     alias inputs; block_bytes must be a multiple of 32 (so a strip is a whole
 *     number of 32-bit words).  block_bytes == 0 or nstripes == 0 is a no-op.
 *   - Bitmatrices are row-major, one byte (0 or 1) per bit.
 *   - There is no CPU fallback: a device call on a machine without a usable CUDA
 *     device fails with XSLP_ECUDA.
 */
#ifndef XSLP_H
#define XSLP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XSLP_OK 0
#define XSLP_EINVAL (-1)         /* null / out-of-range / misaligned / non-divisible argument */
#define XSLP_ESINGULAR (-2)      /* singular GF(2^8) matrix */
#define XSLP_EUNRECOVERABLE (-3) /* more than p erasures */
#define XSLP_ECUDA (-4)          /* CUDA runtime error, or no device */
#define XSLP_ENOMEM (-5)         /* host or device allocation failed */
#define XSLP_ECOMPILE (-6)       /* PTX -> sm_100a compilation failed */

/* Coding-matrix families (readings R1, R2). */
#define XSLP_RS_ISAL 0    /* [I_n; R], R[i][j] = (2^i)^j: reproduces the paper's counts */
#define XSLP_RS_SYSVAND 1 /* [I_n; M V^-1], the text's reduced Vandermonde */
#define XSLP_CAUCHY 2     /* [I_n; R], R[i][j] = inv((n+i) xor j) (BASELINE cfg1) */

#define XSLP_COMPRESS_NONE 0      /* the lifted SLP of P:599-629 ("Base") */
#define XSLP_COMPRESS_REPAIR 1    /* RePair */
#define XSLP_COMPRESS_XORREPAIR 2 /* XorRePair = RePair + Rebuild */

#define XSLP_SCHED_NONE 0 /* keep creation order */
#define XSLP_SCHED_DFS 1  /* DFS post-order + pebble reuse */
#define XSLP_SCHED_GREEDY 2 /* bottom-up greedy with cache capacity greedy_capacity */

#define XSLP_LAYOUT_STRIP 0 /* a block is 8 contiguous strips; the paper's layout */
#define XSLP_LAYOUT_BYTE 1  /* a block is plain bytes; outputs equal textbook byte-wise RS
                                via in-register bit-plane transposes; block_bytes % 32
                               == 0, block pointers 32-byte aligned; straight-line (LDG) or PIPE
                               kernel */

#define XSLP_KERNEL_AUTO 0     /* batched calls: PIPE when its stages fit and there are >= 4 tiles per
                                  SM (and, strip layout, the program reads <= ~6 shared-memory
                                  bytes per data byte), else STRAIGHT; interpreter when nothing
                                  was compiled */
#define XSLP_KERNEL_STRAIGHT 1 /* the JIT-compiled straight-line specialisation */
#define XSLP_KERNEL_INTERP 2   /* the generic SLP interpreter kernel */
#define XSLP_KERNEL_TMA 3      /* straight-line kernel with TMA (cp.async.bulk) staging of the
                                  constant strips in shared memory; needs block_bytes % 128 == 0 */
#define XSLP_KERNEL_PIPE 4     /* persistent warp-specialised variant: a producer warp streams
                                  tiles by TMA through `stages` shared-memory stages (mbarrier
                                  full/empty ring) while `threads` consumer threads compute;
                                  needs block_bytes % 128 == 0 */

/* xslp_opts.interp: organisation of the batched interpreter (XSLP_KERNEL_INTERP) */
#define XSLP_INTERP_LANES 0 /* the 32 lanes of a warp run 32 independent SLP instructions
                               (a round) over the same 16 bytes of every strip, 128-bit shared
                               loads; max(16, threads / 32) consumer warps per CTA */
#define XSLP_INTERP_PAIRS 1 /* every thread owns lane_words words; micro-ops of four operands run
                               warp-uniformly in software-pipelined pairs; threads consumers */
#define XSLP_INTERP_TMEM 2  /* default: every thread owns 2 words (1 when the TMEM slots or the
                               shared-memory stages do not fit; the lane interpreter when neither);
                               SLP variables live in tensor memory (tcgen05.ld/st, one TMEM lane
                               per thread), constants in shared memory; 128 consumer threads */

typedef struct xslp_opts {
  int32_t compress;        /* XSLP_COMPRESS_*; default XORREPAIR */
  int32_t fuse;            /* 1 = XOR fusion; default 1 */
  int32_t schedule;        /* XSLP_SCHED_*; default DFS */
  int32_t specialise;      /* 1 = emit PTX and compile the straight-line kernel now; default 1 */
  int32_t lane_words;      /* 32-bit words per thread per strip in the straight-line kernel: 1, 2 or 4; default 1 */
  int32_t threads;         /* CTA size of the kernels (32..1024, multiple of 32); default 128 */
  int64_t block_bytes_hint;/* if > 0, bake strip = hint/8 into the straight-line kernel's addressing */
  int32_t kernel;          /* XSLP_KERNEL_* used by xslp_encode/decode(_batch); default AUTO */
  int32_t goal_order;      /* DFS root order: 0 = by the term order of the goal nodes, 1 = goal index */
  int32_t min_blocks;      /* if > 0, ask ptxas for this many resident CTAs per SM (.minnctapersm) */
  int32_t stages;          /* shared-memory stages of the PIPE kernel (1..8); default 2 */
  int32_t greedy_capacity; /* cache capacity c (blocks) of XSLP_SCHED_GREEDY */
  int32_t layout;          /* XSLP_LAYOUT_*; default STRIP */
  int32_t groups;          /* PIPE kernel consumer groups (1..4; default 1): the goals are split
                              into `groups` sets (contiguous, balanced by instruction count) and
                              each set's sub-program (the instructions its goals reach) runs on
                              its own `threads` consumer threads over the same shared-memory
                              stage, so a wide program keeps more warps issuing per SM */
  int32_t phases;          /* PIPE input phases (0 = auto, the default: ceil(n/10) for n > 10 input
                              blocks, else 1; or 1..8): the input blocks are cut into
                              `phases` contiguous ranges, each compiled as its own program over all
                              goals; a tile is streamed one range at a time and the goal partials
                              are XORed in registers, so a stage holds one range's strips (wide
                              codes such as RS(20,4) keep more consumer threads per SM).  Not
                              combinable with groups > 1. */
  int32_t reuse;           /* constant register reuse window of the TMA-staged kernels (PIPE, TMA,
                              fused multi-program / syndrome): a constant read from shared memory
                              within the last `reuse` instructions keeps its register instead of
                              a fresh read; 0 = auto (the default: 64 for single-program kernels
                              and the fused M^-1 multi-program kernels, which run one CTA per
                              SM, 16 for the syndrome-form kernels, which keep two CTAs per SM),
                              -1 = a fresh shared-memory read at every use, or 1..4096 */
  int32_t interp;          /* XSLP_INTERP_*: batched interpreter organisation; default TMEM */
} xslp_opts;

typedef struct xslp_stats {
  int32_t n_const;    /* constants (input strips) = columns of the bitmatrix */
  int32_t n_goals;    /* goals (output strips) = rows of the bitmatrix */
  int64_t xor_count;  /* #xor = sum(arity - 1) over instructions */
  int64_t mem_count;  /* #M = sum(arity + 1) */
  int32_t n_instr;    /* instructions */
  int32_t nvar;       /* NVar of the program as dumped (pebbles after DFS) */
  int32_t maxlive;    /* max live 32-bit values per lane under eager goal stores (interpreter slots) */
  int32_t n_copy_goals; /* goals equal to one constant (identity rows) */
  int32_t n_zero_goals; /* goals equal to the empty set (all-zero rows) */
  int32_t regs;       /* registers per thread of the straight-line kernel (0 if not compiled) */
  int32_t spill_bytes;/* local-memory spill stores of the straight-line kernel */
  int32_t regs_tma;   /* registers per thread of the TMA-staged straight-line kernel */
  int32_t spill_bytes_tma; /* its spill stores */
  int32_t regs_pipe;  /* registers per thread of the persistent TMA pipeline kernel */
  int32_t spill_bytes_pipe; /* its spill stores */
  double compile_ms;  /* host compile time of xslp_compile (SLP passes + PTX -> cubin) */
  int64_t group_xor;  /* PIPE consumer groups / input phases: XORs executed per word position
                         summed over the groups or phases, including the phases' accumulation
                         XORs (>= xor_count in practice); 0 if neither is used */
  int64_t smem_reads; /* shared-memory reads of constants per word position that the
                         TMA-staged kernels issue under opts.reuse (single program, no phases):
                         #constant operand uses with reuse off, down to n_const */
} xslp_stats;

typedef struct xslp_program xslp_program; /* opaque, immutable after compile, thread-safe to share */

/* Fill opts with the defaults listed above. */
void xslp_default_opts(xslp_opts *opts);

/* ---- host helpers: matrices -------------------------------- */

/* gf_out: (n+p) x n bytes, row-major; 1 <= n, 0 <= p, n+p <= 255. */
int xslp_coding_matrix(int n, int p, int kind, uint8_t *gf_out);

/* bits_out: (8p) x (8n), the lowering x~ of the parity rows of gf ((n+p) x n). */
int xslp_encode_bitmatrix(const uint8_t *gf, int n, int p, uint8_t *bits_out);

/* Decode bitmatrix for the erased block indices erased[0..ne) (0-based, any order,
 * 1 <= ne <= p).  Survivors are the first n non-erased indices ascending; goals are
 * the erased blocks in ascending index: a data block e is row e of M^-1, a parity
 * block e is G[e] M^-1 (reading R4).
 * bits_out: (8ne) x (8n); survivors_out: n ints.  Errors: XSLP_EUNRECOVERABLE if
 * ne > p, XSLP_EINVAL for bad/duplicate indices, XSLP_ESINGULAR if M is singular. */
int xslp_decode_bitmatrix(const uint8_t *gf, int n, int p, const int32_t *erased, int ne,
                          uint8_t *bits_out, int32_t *survivors_out);

/* Decode bitmatrix over an explicit survivor set: survivors[0..n) are n distinct non-erased
 * block indices in the order the decode program will read them (its input block j is block
 * survivors[j]).  Same goal rows as xslp_decode_bitmatrix (reading R4) with M =
 * the survivors' rows; any n survivors of an MDS code work.  Used by the
 * cross-GPU decode to read as many survivors as possible from local memory.  bits_out:
 * (8ne) x (8n).  Errors: XSLP_EUNRECOVERABLE if ne > p; XSLP_EINVAL for bad, duplicate or
 * erased survivor indices; XSLP_ESINGULAR if M is singular. */
int xslp_decode_bitmatrix_from(const uint8_t *gf, int n, int p, const int32_t *erased, int ne,
                               const int32_t *survivors, uint8_t *bits_out);

/* Syndrome-form decode (a GPU restructuring of P:526-530, csrc/syndrome.cpp): with the
 * parity-check matrix H = [R | I_p] of the systematic code, s = H c' over the codeword whose
 * erased blocks are replaced by zero blocks equals H_E c_E, and c_E = H_E[J]^-1 s_J for e rows J
 * of H with H_E[J] invertible.  syn_bits (may be NULL): (8p) x (8(n+p)), the lowering of H;
 * solve_bits (may be NULL): (8ne) x (8p), the erased blocks (ascending) as XORs of the
 * syndrome words.  gf must be systematic ([I_n; R]).  Errors as xslp_decode_bitmatrix. */
int xslp_syndrome_bitmatrices(const uint8_t *gf, int n, int p, const int32_t *erased, int ne,
                              uint8_t *syn_bits, uint8_t *solve_bits);

/* ---- compile (host, untimed) ------------------------------------------------------- */

/* bits: out_rows x in_cols (in_cols a multiple of 8, out_rows a multiple of 8, in_cols <= 512).
 * opts may be NULL (defaults).  *out receives a new program (free with xslp_free). */
int xslp_compile(const uint8_t *bits, int out_rows, int in_cols, const xslp_opts *opts,
                 xslp_program **out);

/* Compile an SLP given in the text format (below) instead of a bitmatrix.  With
 * compress = NONE its instruction structure is kept and only fused/scheduled;
 * otherwise its goal sets are recomputed and compressed.  n_const = number of
 * constants c0..c{n_const-1} (any positive count; the device path additionally
 * needs a multiple of 8). */
int xslp_compile_text(const char *text, int n_const, const xslp_opts *opts, xslp_program **out);

/* The program's metrics (xslp_stats above: #xor, #M, NVar, registers of the JIT kernels, ...)
 * into *stats (caller-owned).  XSLP_EINVAL on NULL arguments. */
int xslp_program_stats(const xslp_program *prog, xslp_stats *stats);

/* Text of the program.  form 0: the scheduled MultiSLP with the paper's pebble
 * names and a final "return" line; form 1: the interpreter's slot program
 * (initial "s<k> = c<j>" loads, slot instructions, "out <g> = ..." stores);
 * form 2: the straight-line kernel's PTX; form 3: the pipelined interpreter's paired micro-op
 * code (stage-0 variant) for T = opts.threads, L = opts.lane_words, S = opts.stages, as decimal
 * 32-bit words (layout in csrc/interp.cu emit_variant); form 4: the lane-parallel interpreter's
 * code (csrc/interp_lanes.cu); forms 5 / 6 / 7: the TMEM interpreter's batch schedule, its device
 * code, and its two-stream device code (XSLP_EINVAL if the program has no goal-half streams),
 * as decimal words with one word per thread (layouts in csrc/interp_tmem.cu emit_code,
 * emit_device, emit_streams).  Forms 0/1 format: one statement per line,
 * "<var> = <term> ^ <term> ...", "out <g> = <term>", "return <term> ...", terms
 * c<j> (constant), 0 (empty set) or a variable name; statements are sequential.
 * Writes at most cap bytes including the NUL; returns the full length needed
 * (excluding the NUL), or a negative error. */
int64_t xslp_program_dump(const xslp_program *prog, int form, char *buf, size_t cap);

/* Cache measures of the program as dumped (form 0) on the paper's abstract LRU cache
 * (P:1007-1091): *ccap = CCap, the least capacity (in blocks) with no reload;
 * *iocost = IOcost(prog, capacity) = loads + evictions.  Either output may be NULL
 * (capacity is ignored when iocost is NULL).  Host-side analysis; not on the device path. */
int xslp_program_cache(const xslp_program *prog, int capacity, int64_t *iocost, int32_t *ccap);

/* Release a program and every device resource cached for it (JIT libraries, bytecode and
 * micro-op pools).  The caller must not free a program while launches using it are queued on
 * a stream it has not synchronised.  NULL is a no-op. */
void xslp_free(xslp_program *prog);

/* ---- device application (timed hot path) ---------------------------------------- */

/* Load the program's device state on the current device (JIT kernels, shared-memory
 * attributes, occupancy, interpreter bytecode) for block size block_bytes (0 = skip the
 * size-dependent part).  After it, launches of this program on this device allocate and
 * synchronise nothing, so they can be captured into CUDA graphs (the host-buffer form
 * xslp_encode_host is synchronous and cannot be captured). */
int xslp_prepare(const xslp_program *prog, size_t block_bytes);

/* One stripe: in_blocks[0..n) and out_blocks[0..m) are HOST arrays of DEVICE
 * pointers (n = n_const/8 input blocks, m = n_goals/8 output blocks).  For
 * encode, inputs are the data blocks and outputs the parity blocks; for decode,
 * inputs are the survivors in survivors_out order and outputs the erased blocks
 * in ascending index.  xslp_encode and xslp_decode are the same operation. */
int xslp_encode(const xslp_program *prog, const uint8_t *const *in_blocks,
                uint8_t *const *out_blocks, size_t block_bytes, void *stream);
int xslp_decode(const xslp_program *prog, const uint8_t *const *in_blocks,
                uint8_t *const *out_blocks, size_t block_bytes, void *stream);

/* Many stripes, one program: d_in_tbl / d_out_tbl are DEVICE arrays of device
 * pointers, [nstripes][n] and [nstripes][m] row-major. */
int xslp_encode_batch(const xslp_program *prog, const uint8_t *const *d_in_tbl,
                      uint8_t *const *d_out_tbl, int nstripes, size_t block_bytes, void *stream);

/* Many stripes, a program per stripe (heterogeneous erasure patterns):
 * progs[0..nprogs) share n_const and n_goals; d_prog_of_stripe is a DEVICE
 * int32 array [nstripes] of indices into progs.  Runs the interpreter kernel
 * in one launch (nprogs == 1 behaves like xslp_encode_batch). */
int xslp_decode_batch_multi(const xslp_program *const *progs, int nprogs,
                            const int32_t *d_prog_of_stripe, const uint8_t *const *d_in_tbl,
                            uint8_t *const *d_out_tbl, int nstripes, size_t block_bytes,
                            void *stream);

/* Many stripes, a program per stripe, grouped: the stripes of program i are
 * d_stripe_ids[group_offsets[i] .. group_offsets[i+1]) (a DEVICE int32 array of stripe
 * indices into d_in_tbl / d_out_tbl); group_offsets is a HOST array of nprogs+1
 * non-decreasing offsets.  Each program's straight-line (or TMA) kernel runs over its
 * own stripes; launches fan out over `nstreams` internal streams that fork from and
 * join back into `stream`.  Programs must share n_const and n_goals. */
int xslp_decode_batch_grouped(const xslp_program *const *progs, int nprogs,
                              const int32_t *d_stripe_ids, const int32_t *group_offsets,
                              const uint8_t *const *d_in_tbl, uint8_t *const *d_out_tbl,
                              size_t block_bytes, int nstreams, void *stream);

/* Heterogeneous decode in few launches: the programs (same n_const and n_goals; typically one
 * per erasure pattern) are fused into persistent multi-program pipeline kernels.  A kernel's
 * producer warp streams the union of its programs' constant strips through `opts->stages`
 * shared-memory stages by TMA; each consumer warp reads its stripe's program index and jumps
 * to that program's straight-line code (a branch table), so a kernel serves many erasure
 * patterns.  Programs are packed per_module (<= 0: 20) to a module; modules compile in
 * parallel host threads.  opts: threads (consumer threads, <= 992), stages (2..8),
 * lane_words, block_bytes_hint (> 0: bake that block size in; launches must then use it),
 * phases (input phases as for the PIPE kernel; 0 = ceil(n/10) for codes wider than 10 blocks:
 * each program is recompiled per input-block range and a tile is streamed range by range).
 * The programs must stay alive while the multi is used.  Free with xslp_multi_free. */
typedef struct xslp_multi xslp_multi;
int xslp_multi_create(const xslp_program *const *progs, int nprogs, int per_module,
                      const xslp_opts *opts, xslp_multi **out);
/* d_prog_of_stripe: DEVICE int32 [stripes] program index (into the create-time progs) of each
 * stripe; d_stripe_ids / group_offsets: the stripes of program i are d_stripe_ids[
 * group_offsets[i] .. group_offsets[i+1]) (DEVICE ids, HOST offsets, as in
 * xslp_decode_batch_grouped, which must agree with d_prog_of_stripe).  One launch per module
 * that has stripes; consecutive modules alternate between two internal streams forked from
 * and joined back into `stream` (capturable in a CUDA graph).  block_bytes % 128 == 0.
 * Tables as in xslp_encode_batch.  group_offsets must hold nprogs + 1 non-decreasing entries
 * (XSLP_EINVAL otherwise; the library reads exactly that many).  A d_prog_of_stripe entry
 * outside the module that owns the stripe makes that launch trap (a CUDA error reported at
 * the next synchronisation) rather than branch outside the module's code. */
int xslp_multi_decode(const xslp_multi *multi, const int32_t *d_prog_of_stripe,
                      const int32_t *d_stripe_ids, const int32_t *group_offsets,
                      const uint8_t *const *d_in_tbl, uint8_t *const *d_out_tbl,
                      size_t block_bytes, void *stream);
/* Heterogeneous decode in syndrome form (see xslp_syndrome_bitmatrices): one shared syndrome
 * program over all n+p blocks of a stripe (compiled once, streamed in opts->phases input
 * phases; 0 = ceil((n+p)/10)) followed by the stripe's pattern's small solve program, fused
 * in the multi-program kernels; the result is a multi usable with xslp_multi_decode,
 * xslp_multi_info and xslp_multi_free.  patterns: npat x ne erased block indices (each row any
 * order, the outputs are the erased blocks ascending).  For xslp_multi_decode, d_in_tbl is
 * [stripes][n+p]: every block of the stripe, the ERASED ones pointing at a zero block of
 * block_bytes (any readable all-zero device buffer); d_out_tbl is [stripes][ne].  Same bytes
 * as the M^-1 decode (the solution is unique).  gf must be systematic.  Patterns are packed
 * per_module (<= 0: 16) to a module. */
int xslp_syndrome_create(const uint8_t *gf, int n, int p, const int32_t *patterns, int npat, int ne,
                         int per_module, const xslp_opts *opts, xslp_multi **out);
/* modules, max registers / spill bytes per thread over the modules, host compile time. */
int xslp_multi_info(const xslp_multi *multi, int32_t *modules, int32_t *regs, int32_t *spill_bytes,
                    double *compile_ms);
void xslp_multi_free(xslp_multi *multi);

/* Comparison path, the paper's approach (1): byte-layout RS as MM over GF(2^8)
 * with table-driven field multiplication (ISA-L splits bytes into nibbles for PSHUFB; here
 * each byte is split into bit groups [0,3), [3,6), [6,8) looked up in 8-entry tables by PRMT).
 * coef: HOST [m][n] GF(2^8) coefficients (1 <= n <= 64, 1 <= m <= 8); output block i of
 * each stripe = sum_j coef[i][j] * input block j, byte by byte -- the same bytes
 * as an XSLP_LAYOUT_BYTE program of those rows.  Tables as in xslp_encode_batch; block
 * pointers 16-byte aligned, block_bytes % 16 == 0. */
int xslp_gf_table_apply(const uint8_t *coef, int n, int m, const uint8_t *const *d_in_tbl,
                        uint8_t *const *d_out_tbl, int nstripes, size_t block_bytes, void *stream);

/* End-to-end form with HOST buffers: h_in = [nstripes][n][block_bytes] and
 * h_out = [nstripes][m][block_bytes], contiguous (ideally pinned) host memory.
 * Stages chunks of stripes through device memory owned by the program's
 * per-device workspace, overlapping host->device copies, the kernel and
 * device->host copies; synchronous (returns when h_out is written). */
int xslp_encode_host(const xslp_program *prog, const uint8_t *h_in, uint8_t *h_out,
                     int nstripes, size_t block_bytes, void *stream);

/* Seeded synthetic input on the device (same counter-based generator as the
 * repo's synth module; no coding arithmetic): d_buf = [nstripes][nblocks][block_bytes],
 * block j of global stripe s word i = splitmix64(seed*0x9E3779B97F4A7C15 +
 * ((s*64 + j) << 40) + i), s = stripe0 + local index.  block_bytes % 8 == 0.
 * XSLP_EINVAL unless nblocks <= 64 and 0 <= stripe0, stripe0 + nstripes <= 2^18 (the range
 * in which the counter keys of distinct words are distinct). */
int xslp_fill_random(uint8_t *d_buf, int nstripes, int nblocks, size_t block_bytes,
                     uint64_t seed, int64_t stripe0, void *stream);

/* ---- peer memory: cross-GPU decode over NVLink ---------------- */

/* A decode whose survivor blocks live on other GPUs of the box reads them in place: the
 * owning process exports its block storage, the decoding process maps it, and the pointer
 * tables of xslp_encode_batch / xslp_decode_batch_grouped name the mapped (peer) addresses,
 * so the kernel's strip loads travel over NVLink 5 / NVSwitch and feed the XORs directly
 * (no staging copy).  The library never synchronises with other processes: the caller
 * orders the owner's writes before the reads (e.g. a host barrier after a device sync) and
 * keeps the exported memory alive until every mapping is closed. */
#define XSLP_PEER_HANDLE_BYTES 128

/* handle_out (XSLP_PEER_HANDLE_BYTES host bytes): a process-portable handle of the device
 * allocation containing d_ptr (cudaIpcGetMemHandle of its base) plus d_ptr's offset in it.
 * d_ptr must come from cudaMalloc (not VMM / expandable segments).  Errors: XSLP_EINVAL for a
 * non-device pointer, XSLP_ECUDA from the runtime. */
int xslp_peer_export(const void *d_ptr, uint8_t *handle_out);

/* Map a handle from xslp_peer_export on the current device; *d_ptr_out = the exported
 * pointer as seen from here.  Another process's allocation is opened once (IPC, peer access
 * enabled lazily) and reference-counted; a handle exported by this same process returns the
 * original pointer (peer access from the current device to the exporter's device enabled).
 * Errors: XSLP_EINVAL for a malformed handle, XSLP_ECUDA when the runtime refuses. */
int xslp_peer_open(const uint8_t *handle, void **d_ptr_out);

/* Release one xslp_peer_open of d_ptr (the IPC mapping is closed with its last release).
 * XSLP_EINVAL if d_ptr was not returned by xslp_peer_open. */
int xslp_peer_close(void *d_ptr);

/* Enable direct access from the current device to peer_device (idempotent); for one process
 * driving several GPUs.  XSLP_ECUDA if the pair has no P2P path. */
int xslp_peer_enable(int peer_device);

/* ---- codec front end ------------------------------------------ */

/* RS(n,p) over arbitrary-length device data.  Data of len bytes is zero-padded to n*B,
 * B = xslp_codec_block_bytes(len) (a multiple of 128, >= 128); shard j < n is bytes
 * [jB, (j+1)B) of the padded data, shard n+i is parity block i.  Device shard buffers are
 * one contiguous (n+p) x B array, 16-byte aligned, owned by the caller.  The codec owns
 * the encode program and an LRU memo (cache_entries, default 1024 when <= 0) of decode
 * programs per erasure pattern; it is safe to use from several threads.  kind / opts as
 * in xslp_coding_matrix / xslp_compile (block_bytes_hint is ignored).  n + p <= 64. */
typedef struct xslp_codec xslp_codec;
int xslp_codec_create(int n, int p, int kind, const xslp_opts *opts, int cache_entries,
                      xslp_codec **out);
void xslp_codec_free(xslp_codec *codec);   /* also frees its memoised programs; NULL is a no-op */
/* Block (shard) size B for len bytes of data: ceil(len / n) rounded up to a multiple of 128,
 * at least 128; negative (XSLP_EINVAL) for len < 0. */
int64_t xslp_codec_block_bytes(const xslp_codec *codec, int64_t len);
/* d_data: len device bytes -> d_shards: (n+p) x B (data copied + padded, parity computed; with
 * d_data 16-byte aligned in one pass that reads each data block once and writes its data shard
 * and the parity). */
int xslp_codec_encode(const xslp_codec *codec, const uint8_t *d_data, int64_t len, uint8_t *d_shards,
                      void *stream);
/* Rebuild the erased shards (any order, <= p) in place from the survivors. */
int xslp_codec_reconstruct(const xslp_codec *codec, uint8_t *d_shards, const int32_t *erased, int ne,
                           int64_t len, void *stream);
/* Write the original len bytes to d_data_out (16-byte aligned: one pass that reads the
 * survivors and writes the data blocks, surviving ones copied and lost ones solved; otherwise
 * rebuild in place and copy out).  Lost shards that hold the data's tail may be rebuilt in
 * place in d_shards. */
int xslp_codec_decode(const xslp_codec *codec, uint8_t *d_shards, const int32_t *erased, int ne,
                      int64_t len, uint8_t *d_data_out, void *stream);
/* The memoised program for an erasure pattern (ne == 0: the encode program); owned by the codec
 * and valid until xslp_codec_free (a program handed out here is never freed by LRU eviction). */
int xslp_codec_program(const xslp_codec *codec, const int32_t *erased, int ne,
                       const xslp_program **out);
int xslp_codec_cached(const xslp_codec *codec);   /* erasure patterns with a memoised decode program */

/* 32-byte shard header (SPEC wire format): "XSLP", version 1, n, p, shard index,
 * original length (u64 LE), block size (u32 LE), 12 reserved zero bytes. */
int xslp_shard_header(uint8_t *out32, int n, int p, int shard, uint64_t original_length,
                      uint32_t block_bytes);
int xslp_shard_header_parse(const uint8_t *in32, int32_t *n, int32_t *p, int32_t *shard,
                            uint64_t *original_length, uint32_t *block_bytes);

/* Number of kernels this library launched on the calling process so far. */
int64_t xslp_launch_count(void);

const char *xslp_last_error(void);
const char *xslp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* XSLP_H */
