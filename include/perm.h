/* perm.h -- C ABI of libperm: B200-native sparse matrix permanent.
 *
 * Method: the Gray-code-ordered Nijenhuis-Wilf / Ryser permanent sweep of
 * Elbek & Kaya, arXiv 2501.15126 ("P:n" = /root/reference/PAPER.md line n):
 *   Alg. 1 SparsePerman, chunked per Sec. II-A,
 *   Theorem 1 / Lemma 1 aligned power-of-two chunks,
 *   Alg. 3 PermanentOrdering, Alg. 4 Partitioning,
 *   matrix-specific generated kernels (Listings 2-5).
 *
 * Conventions for every entry point:
 *   - extern "C", plain host pointers and sizes; no torch/CUDA types in the
 *     signatures (streams and device buffers are passed as void*).
 *   - Return value: perm_status (0 = PERM_OK) unless stated otherwise; on
 *     failure perm_last_error() gives a message (thread-local, valid until the
 *     next libperm call on the same thread).
 *   - Inputs are COPIED: callers may free their arrays on return.
 *   - A plan is used by one host thread at a time; different plans are
 *     independent.  There is NO CPU fallback: without a usable sm_100 device,
 *     device-touching calls fail with PERM_ECUDA.
 */
#ifndef PERM_H_
#define PERM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct perm_plan_s *perm_plan_t; /* opaque; owned by libperm */

/* Sparse input layout (Sec. II).
 * PERM_CCS: ptr = cptrs[n+1], idx = rids[nnz], val = cvals[nnz] (column-major)
 * PERM_CRS: ptr = rptrs[n+1], idx = cids[nnz], val = rvals[nnz] (row-major)
 * nnz = ptr[n].  Requirements (else PERM_EINVAL): ptr[0] = 0, ptr nondecreasing,
 * indices in [0,n) strictly increasing inside each column (row), values finite
 * and nonzero (the paper's formats store no zeros). */
typedef enum { PERM_CCS = 0, PERM_CRS = 1 } perm_format;

/* Column/row ordering (perm(PAQ) = perm(A)). */
typedef enum {
  PERM_ORDER_NONE = 0,      /* input order */
  PERM_ORDER_DEGREE = 1,    /* ascending column degree, Sec. VI-B */
  PERM_ORDER_PERMANENT = 2, /* Alg. 3 PermanentOrdering */
  PERM_ORDER_AUTO = 3       /* the one with the lowest planned FP64 work W_plan */
} perm_ordering;

typedef enum {
  PERM_OK = 0,
  PERM_EINVAL = 1,  /* malformed input or argument */
  PERM_ERANGE = 2,  /* n outside [1,64], or INT01 result may exceed int128 */
  PERM_ENOMEM = 3,  /* host or device allocation failed */
  PERM_ECUDA = 4,   /* CUDA runtime error / no sm_100 device */
  PERM_ENVRTC = 5,  /* NVRTC compilation failed */
  PERM_ENCCL = 6,   /* NCCL unavailable or a collective failed */
  PERM_ESPILL = 7   /* generated kernel spills to local memory (register budget) */
} perm_status;

/* Kernel family (codegen mode). */
typedef enum {
  PERM_MODE_AUTO = 0,   /* INT01 for 0/1 inputs whose result provably fits int128, else REG */
  PERM_MODE_REG = 1,    /* FP64, x of every in-chunk row in registers (Sec. III) */
  PERM_MODE_HYBRID = 2, /* FP64, rows first flipped by columns >= c (Alg. 4) live in a
                           per-thread memory tier (Sec. V; B200: shared memory) */
  PERM_MODE_INT01 = 3,  /* exact: 2x in int32, products/sums mod 2^128 (0/1 inputs) */
  PERM_MODE_COMPLEX = 4 /* reported by perm_plan_get_info for perm_plan_complex plans
                           (complex FP64 sweep; not a valid request mode) */
} perm_mode;

/* Options; a zero-initialised struct means "all defaults". */
typedef struct {
  int mode;              /* perm_mode */
  int device;            /* CUDA device ordinal the plan binds to (cudaSetDevice) */
  void *cuda_stream;     /* cudaStream_t to launch on; NULL = plan-owned stream */
  int chunk_log2;        /* B: each lane sweeps aligned chunks of 2^B Gray steps
                            (Lemma 1).  0 = auto */
  int block_log2;        /* U: 2^U Gray steps unrolled per generated block. 0 = auto */
  int task_chunks;       /* M: chunks per lane per warp-task (power of two). 0 = auto */
  double gr_ratio;       /* Alg. 4 GRratio. 0 = 16 */
  int hybrid_c;          /* HYBRID: register/tier split column c; 0 = Alg. 4's c */
  int threads_per_block; /* 0 = auto (128) */
  int no_device;         /* 1 = plan + codegen + NVRTC only; never touch a GPU
                            (for CPU-side inspection; compute calls then fail) */
  int factor_cols;       /* K, closed-form summed columns (DESIGN.md "Factored
                            columns"): 0 = auto (the K with the lowest planned
                            work), -1 = off (plain Alg. 1 sweep), k > 0 = at most k */
  int min_blocks;        /* __launch_bounds__ min blocks per SM (register cap);
                            0 = auto from the planner's register estimate */
  int zero_skip;         /* INT01 zero tracking: 0 = on, -1 = off */
  int autotune;          /* 0 = with a device, time the compiled candidates on a
                            strided sample of their task range and keep a clearly
                            (>4 %) faster one over the model's pick; -1 = off
                            (the model's pick: deterministic across processes) */
  int rank, world;       /* multi-GPU: perm_compute / _ex / _async sweep
                            shard `rank` of `world` (power of two) and all-gather the
                            partials over nccl_comm; world 0 or 1 = one GPU */
  int reseed_log2;       /* R: x is re-seeded exactly from x0 at least every 2^R swept
                            steps (Sec. II-A seeding; bounds FP64 drift, SURVEY
                            8(c)).  Every chunk is seeded exactly, so this caps the
                            chunk: B <= R.  0 = auto (B) */
  int reserved0;
  void *nccl_comm;       /* ncclComm_t over the `world` ranks (perm_comm_init, or the
                            caller's from the same libnccl.so.2 instance); borrowed */
  const char *cache_dir; /* on-disk plan cache directory (plan files named by a hash of
                            matrix + options + library build); NULL = $PERM_CACHE_DIR,
                            unset = no disk cache.  Read at perm_plan time only */
} perm_opts;

/* Result of a computation. */
typedef struct {
  double value;          /* perm(A) (or, for a shard, the UNSCALED partial sum) */
  uint64_t exact_lo;     /* INT01: value as two's-complement int128 (lo, hi);  */
  uint64_t exact_hi;     /*        for a shard: unscaled T' partial mod 2^128  */
  int exact_valid;       /* 1 if exact_lo/hi hold an exact integer result */
  int world, rank;       /* shard geometry of this result */
  uint64_t products;     /* product terms evaluated (2^(n-1) for a full run) */
  double sweep_ms;       /* device time of the sweep kernel (CUDA events) */
  double reduce_ms;      /* device time of the deterministic reduction */
  double value_im;       /* complex plans: imaginary part of `value` (else 0) */
  uint64_t steps;        /* Gray steps of Alg. 1 this result covers (= products) */
  double seconds;        /* device seconds of sweep + reduction (+ fold / collective) */
  double w_plan;         /* the plan's FP64 (INT01: integer) ops per Gray step */
  int k, c;              /* Alg. 4 partition of the base ordering */
  int b;                 /* B, chunk log2 (Lemma 1) */
  int mode;              /* perm_mode of the kernel that ran */
  int K;                 /* eliminated columns (DESIGN 3.6) */
  int reserved_r;
} perm_result;

/* Plan inspection (all indices refer to the ORDERED matrix unless noted). */
typedef struct {
  int n, nnz;
  int mode, ordering;     /* resolved perm_mode / perm_ordering */
  int singular;           /* 1: structural rank < n, perm = 0, no launch */
  int struct_rank;
  int k, c;               /* Alg. 4 partition (B200 register model) */
  int B, U;               /* chunk and unrolled-block log2 */
  int M;                  /* chunks per lane per warp-task */
  int K;                  /* factored leading columns: pairwise row-disjoint ordered
                             columns 0..K-1 summed in closed form; the sweep runs
                             over h-space = states of columns K..n-2 (2^(n-1-K)) */
  int swept_order;        /* 0: swept columns in base order; 1: sorted by flip cost;
                             2 / 3 (INT01): zero-aware placement of zero-prone rows
                             on lane-uniform bits >= B+5 (3: also on [U, B)) */
  uint64_t tasks;         /* warp-tasks over the whole h-range (power of two);
                             task t covers h in [t*L, (t+1)*L), L = 32*M*2^B, i.e.
                             Gray steps g in [t*L*2^K, (t+1)*L*2^K); its partial
                             times (-1)^K equals the Alg. 1 partial sum there */
  int reg_rows;           /* rows of x held in registers */
  int tier_rows;          /* HYBRID rows in the per-thread tier */
  int seed_rows;          /* rows untouched by columns < B: folded into one
                             per-chunk constant at seed time */
  int levels;             /* nonempty product-cache levels */
  double w_plan;          /* FP64 ops (DADD/DMUL/DFMA) per Gray step of the
                             generated code, incl. amortised seeding */
  double w_alg1;          /* FP64 ops per step of Alg. 1 as written */
  int block, grid, blocks_per_sm, sms;
  int regs_per_thread, local_bytes;
  int smem_bytes;         /* dynamic shared memory per block: loop-carried values the
                             unrolled block body never references (per-thread slots) */
  double plan_ms;         /* wall time of perm_plan (all phases below + device setup) */
  double codegen_ms;      /* wall: ordering + elimination searches + candidate codegen */
  double nvrtc_ms;        /* wall: concurrent NVRTC compiles of the kept candidates */
  int cubin_cached;       /* 1 if the cubin came from the in-process cache */
  int plan_cached;        /* 1 if ordering/codegen/NVRTC came from the in-process
                             planner cache (same CCS content and options) */
  int row_perm[64];       /* ordered row i = original row row_perm[i] */
  int col_perm[64];       /* ordered column j = original column col_perm[j] */
  double autotune_ms;     /* wall: on-device timing of the compiled candidates */
  double nvrtc_cpu_ms;    /* sum of the individual NVRTC compile times (> nvrtc_ms when
                             candidates compile concurrently) */
  int disk_cached;        /* 1 if the planning output came from the on-disk plan cache
                             or from perm_plan_import */
  int candidates_compiled;
} perm_plan_info;

/* ---- plan / compute / free (north-star surface) ------------------------ */

/* Validate, rank-check, order, partition, generate and JIT-compile (NVRTC,
 * sm_100a) a matrix-specific kernel, load it on the device and allocate the
 * per-task partial buffer.  n in [1,64].  *out receives the plan. */
int perm_plan(int n, perm_format fmt, const int32_t *ptr, const int32_t *idx,
              const double *val, perm_ordering ord, perm_plan_t *out);
int perm_plan_ex(int n, perm_format fmt, const int32_t *ptr, const int32_t *idx,
                 const double *val, perm_ordering ord, const perm_opts *opts,
                 perm_plan_t *out);

/* Complex matrices (boson-sampling unitaries): as perm_plan_ex
 * but val_re_im holds 2*nnz doubles, (re, im) per nonzero in idx order; a
 * nonzero is any pair other than (0, 0).  Modes AUTO/REG (complex FP64 sweep,
 * info.mode = PERM_MODE_COMPLEX); results carry value + i*value_im; partials
 * are 16 bytes (re, im). */
int perm_plan_complex(int n, perm_format fmt, const int32_t *ptr, const int32_t *idx,
                      const double *val_re_im, perm_ordering ord, const perm_opts *opts,
                      perm_plan_t *out);

/* perm(A).  One GPU (opts.world <= 1): the whole Gray range.  Multi-GPU
 * (opts.world > 1, opts.nccl_comm set): this rank sweeps shard opts.rank, the
 * partials are all-gathered over NCCL on the plan's stream and folded in rank
 * order -- every rank returns the same bits as a one-GPU run.  NaN on error
 * (see perm_last_error).  Synchronises the plan's stream. */
double perm_compute(perm_plan_t p);
int perm_compute_ex(perm_plan_t p, perm_result *r);

/* Asynchronous perm_compute on the plan's stream: writes perm(A) (8 bytes FP64,
 * 16 bytes complex (re, im) or INT01 int128) to the DEVICE pointer d_out; no
 * host synchronisation (sweep -> tree -> [all-gather] -> fold, all enqueued). */
int perm_compute_async(perm_plan_t p, void *d_out);

/* SURVEY 8(b) surface: UNSCALED partial of shard `rank` of `world` to host
 * memory -- 1 double (FP64; INT01: the exact T' partial rounded to double, use
 * perm_compute_shard for the exact bits), 2 doubles (re, im) for complex plans. */
int perm_compute_partial(perm_plan_t p, int rank, int world, double *partial);

/* Shard `rank` of `world` (world a power of two; Sec. 8(e) Gray-range
 * sharding): r->value = UNSCALED partial sum over this shard's contiguous,
 * power-of-two-aligned Gray range (INT01: exact_lo/hi = T' partial).  Folding
 * the world partials with perm_fold reproduces perm_compute bit for bit. */
int perm_compute_shard(perm_plan_t p, int rank, int world, perm_result *r);

/* Device-side shard: writes the unscaled partial (8 bytes FP64 / 16 bytes
 * INT01 as lo,hi) to the DEVICE pointer d_partial on the plan's stream,
 * without synchronising (for a following NCCL all-gather). */
int perm_compute_shard_async(perm_plan_t p, int rank, int world, void *d_partial);

/* Fixed-order pairwise fold of `world` unscaled partials followed by the
 * Alg. 1 line-23 scale 4(n mod 2)-2.  Host version: partials given as
 * perm_result[world] from perm_compute_shard.  Device version: d_partials is a
 * device array of world entries (8 or 16 bytes each); result (8 or 16 bytes,
 * INT01: perm as int128) written to the device pointer d_out, asynchronously. */
int perm_fold(perm_plan_t p, const perm_result *shards, int world, perm_result *out);
int perm_fold_async(perm_plan_t p, const void *d_partials, int world, void *d_out);

/* Size in bytes of one partial / result for this plan (8 FP64, 16 INT01). */
int perm_partial_bytes(perm_plan_t p);

/* Shard geometry (host only, works for no_device plans): warp-tasks
 * [*first_task, *first_task + *ntasks) and the Gray-step range
 * [*g_begin, *g_end) of Alg. 1 that shard `rank` of `world` covers.  The
 * shards of a world partition [0, 2^(n-1)) into contiguous aligned ranges. */
int perm_shard_range(perm_plan_t p, int rank, int world, uint64_t *first_task, uint64_t *ntasks,
                     uint64_t *g_begin, uint64_t *g_end);

/* Host reference of perm_fold for FP64 plans (no device): fixed-order
 * pairwise fold of `world` unscaled partials times the scale
 * 2(-1)^(n-1)(-1)^K.  NaN on error.  Same arithmetic as the fold kernel. */
double perm_fold_host(perm_plan_t p, const double *partials, int world);

/* Copy the per-warp-task partial sums of the LAST shard/compute call to host
 * memory (double[ntask] for FP64; 2*uint64 per task for INT01).  Task t covers
 * the Gray range [ (t0+t) * L, (t0+t+1) * L ) with L = 32 * M * 2^B and t0 the
 * shard's first task.  *count receives the number of tasks copied. */
int perm_debug_task_partials(perm_plan_t p, void *host, uint64_t cap, uint64_t *count,
                             uint64_t *first_task);

/* Device durations of the last sweep launch and its reduction, from CUDA
 * events the plan records on its launching stream around each launch
 * (waits for those events).  0 when the last call launched nothing. */
int perm_last_timing(perm_plan_t p, double *sweep_ms, double *reduce_ms);

int perm_plan_get_info(perm_plan_t p, perm_plan_info *info);
/* NUL-terminated generated CUDA source of the plan's kernel (owned by plan). */
const char *perm_plan_source(perm_plan_t p);
/* Copy the sm_100a cubin; *size in: capacity, out: bytes needed/copied. */
int perm_plan_cubin(perm_plan_t p, void *buf, size_t *size);

void perm_free(perm_plan_t p); /* NULL-safe */

/* ---- plan transport: on-disk cache and rank-0 broadcast ----------------
 * perm_plan_export serialises a plan's planning output (validated matrix,
 * orderings, kernel spec and source, sm_100a cubin, info) to buf; *size in:
 * capacity, out: bytes needed/copied (call with buf = NULL to size).
 * perm_plan_import builds a plan from such a blob (from the same libperm build;
 * PERM_EINVAL otherwise) without re-planning: no search, no NVRTC -- the device
 * part (module load, buffers) follows `opts` (device, stream, rank/world/comm,
 * no_device).  Multi-GPU runs plan on rank 0 and broadcast the blob so every
 * rank runs the same kernel bits. */
int perm_plan_export(perm_plan_t p, void *buf, size_t *size);
int perm_plan_import(const void *blob, size_t size, const perm_opts *opts, perm_plan_t *out);

/* ---- NCCL communicator owned by libperm (dlopen'd libnccl.so.2) ---------
 * Rank 0 calls perm_comm_unique_id, ships the 128 bytes to every rank (e.g.
 * over torch.distributed), each rank calls perm_comm_init (collective: all
 * ranks must call it) and passes the comm as perm_opts.nccl_comm. */
int perm_comm_unique_id(void *id128);
int perm_comm_init(int world, int rank, const void *id128, int device, void **comm);
int perm_comm_destroy(void *comm);

/* Measured FP64 lane-op throughput of `device` (DFMA chains at full occupancy;
 * one DADD/DMUL/DFMA thread-instruction = one op): the roofline denominator of
 * the sweep.  *ms = best kernel time. */
int perm_probe_fp64_peak(int device, double *lane_ops_per_s, double *ms);

const char *perm_last_error(void);
const char *perm_version(void);

/* ---- host planner entry points (exposed for parity tests) -------------- */

/* Structural rank (maximum bipartite matching, Hopcroft-Karp).
 * Returns the rank, or -1 on invalid input. */
int perm_structural_rank(int n, perm_format fmt, const int32_t *ptr, const int32_t *idx,
                         const double *val);

/* Row/column ordering of the matrix: row_perm[i] / col_perm[j] = original index
 * at ordered position i / j (Alg. 3 / degree sort / identity). */
int perm_order(int n, perm_format fmt, const int32_t *ptr, const int32_t *idx,
               const double *val, perm_ordering ord, int32_t *row_perm, int32_t *col_perm);

/* Alg. 4 Partitioning on an ORDERED matrix given in CCS, with
 * CalculateNoThreads modelled for `sms` SMs of 65536 registers, 2048 threads,
 * 255 registers per thread, 32 overhead registers. */
int perm_partition(int n, const int32_t *cptrs, const int32_t *rids, double gr_ratio,
                   int sms, int *k, int *c);

/* Alg. 2 GenerateLaunchParameters, reference planner: writes up to
 * cap triples (start, delta, end) to out[3*i..]; returns the count or -1. */
int perm_alg2_launch_parameters(uint64_t tau, int n, uint64_t *out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* PERM_H_ */
