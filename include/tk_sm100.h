/*
 * tk_sm100.h -- C ABI of the B200 (sm_100a) flexible GEMM library (libtk_sm100.so).
 *
 * This is the drop-in boundary for the reference package's GEMM path
 * (reference = /root/reference/pkg, "tilekit"):
 *
 *   tk_gemm          replaces kernel.gemm_execute / api.matmul
 *                    (pkg/src/tilekit/kernel.py:253-330, pkg/src/tilekit/api.py:37-40):
 *                    one resolved KernelConfig, lowered by the host planner to a
 *                    TkGemmPlan, executed as one stream-ordered device launch.
 *   tk_gemm_ex_raw   replaces api.gemm_ex_raw / GEMM_EX_CFUNC
 *                    (pkg/src/tilekit/api.py:317-373): identical parameter list and
 *                    status convention (0 ok, 1 configuration error); pointers may be
 *                    host or device memory; synchronous like the reference.
 *   tk_gemm_ex_raw_async  same on device pointers, ordered on a caller stream.
 *
 * No CUDA or torch types appear in the signatures: streams are passed as void*
 * (a cudaStream_t / CUstream value, NULL = legacy default stream).
 * Every matrix is addressed through a TkLayout "digit" map: logical index i of
 * a dimension is decomposed fastest-first into digits d_t = (i / prod(ext[<t])) % ext[t]
 * and the element offset is sum_t d_t * stride[t] (+ the second plane for pair types).
 */
#ifndef TK_SM100_H
#define TK_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TK_ABI_VERSION 2
#define TK_MAX_DIGITS 5   /* digits per logical dimension: StridedPermutation up to rank 5 */
#define TK_MAX_TOPS 8

/* storage / accumulation scalars */
enum TkScalar { TK_F16 = 0, TK_BF16 = 1, TK_F32 = 2, TK_F64 = 3 };
/* operators (reference operators.py:98-188) */
enum TkOperator { TK_OP_REAL = 0, TK_OP_COMPLEX = 1, TK_OP_DUAL = 2 };
/* layout kinds (reference layouts.py: ColMajor/RowMajor/Padded/StridedPermutation are
 * STRIDED digit maps; Diagonal; Zero) */
enum TkLayoutKind { TK_LAYOUT_STRIDED = 0, TK_LAYOUT_DIAGONAL = 1, TK_LAYOUT_ZERO = 2 };
/* pair element storage (reference layouts.py:314-394) */
enum TkPairMode { TK_PAIR_NONE = 0, TK_PAIR_INTERLEAVED = 1, TK_PAIR_SPLIT = 2 };
/* element-wise transform ops (reference components.py:52-94) */
enum TkTransformOp { TK_T_SCALE = 1, TK_T_ADD = 2, TK_T_RELU = 3 };
/* predicates (reference components.py:171-191) */
enum TkPredicate { TK_PRED_ALWAYS = 0, TK_PRED_DIAGONAL = 1, TK_PRED_MASK = 2 };
/* execution lanes */
enum TkLane { TK_LANE_AUTO = 0, TK_LANE_TCGEN05 = 1, TK_LANE_SIMT = 2 };
/* status codes: 0 and 1 follow the reference gemm_ex_raw convention */
enum TkStatus { TK_OK = 0, TK_ERR_CONFIG = 1, TK_ERR_CUDA = 2 };
/* gemm_ex_raw type tags: 0-5 as the reference (api.py:318-326), 6-11 new */
enum TkTag {
  TK_TAG_F32 = 0, TK_TAG_F64 = 1, TK_TAG_C64 = 2, TK_TAG_C128 = 3,
  TK_TAG_DUAL32 = 4, TK_TAG_DUAL64 = 5,
  TK_TAG_F16F32 = 6,     /* A,B float16; C float32 */
  TK_TAG_BF16F32 = 7,    /* A,B bfloat16; C float32 */
  TK_TAG_C32C64 = 8,     /* A,B interleaved complex-half; C complex64 */
  TK_TAG_CBF16C64 = 9,   /* A,B interleaved complex-bf16; C complex64 */
  TK_TAG_DUAL16F32 = 10, /* A,B interleaved dual-half; C dual32 */
  TK_TAG_DUALBF16F32 = 11
};

typedef struct TkLayout {
  int32_t kind;                 /* TkLayoutKind */
  int32_t pair;                 /* TkPairMode */
  int32_t scalar;               /* TkScalar of the backing buffer */
  int32_t reserved;
  int32_t ndigits[2];           /* digits per logical dimension (1..TK_MAX_DIGITS) */
  int64_t ext[2][TK_MAX_DIGITS];
  int64_t stride[2][TK_MAX_DIGITS]; /* in elements (a pair counts as one element) */
  int64_t plane_stride;         /* SPLIT: element offset of the second plane */
  int64_t size;                 /* physical_size() in scalars */
} TkLayout;

typedef struct TkTransform {
  int32_t n;                    /* number of ops, applied left to right */
  int32_t op[TK_MAX_TOPS];      /* TkTransformOp */
  int32_t promote[TK_MAX_TOPS]; /* 1: evaluate in f64 then round to the stream type */
  double re[TK_MAX_TOPS];       /* constant (real part) */
  double im[TK_MAX_TOPS];       /* constant (imaginary part, complex streams) */
} TkTransform;

typedef struct TkGemmPlan {
  int32_t abi_version;          /* TK_ABI_VERSION */
  int32_t op;                   /* TkOperator */
  int32_t compute;              /* accumulator scalar: TK_F32 or TK_F64 */
  int32_t lane;                 /* TkLane requested */
  int64_t m, n, k;
  int64_t op_k;                 /* operator K (chunking of complex/dual products) */
  int64_t block[3];             /* logical block tile (bm, bn, bk) */
  TkLayout a, b, c, d;
  TkTransform t_a, t_b, t_c, t_r2s, t_s2g; /* the five streams, kernel.py:153-157 */
  int32_t bias_axis;            /* 0 none, 1 bias[j] (axis n), 2 bias[i] (axis m) */
  int32_t bias_scalar;          /* TkScalar of the bias vector */
  int32_t predicate;            /* TkPredicate */
  int32_t reserved;
} TkGemmPlan;

/* ABI version compiled into the library. */
int tk_abi_version(void);

/* Lane that tk_gemm would use for this plan (TK_LANE_TCGEN05 / TK_LANE_SIMT), or -1
 * with tk_last_error() set when the plan is invalid. */
int tk_plan_lane(const TkGemmPlan* plan);

/* Device workspace (bytes) tk_gemm needs for this plan (de-interleave planes, gathered
 * GETT operands, transformed operand planes of g2s_a / g2s_b programs, split-K partials and
 * their counters).  Caller allocates it. */
int64_t tk_workspace_bytes(const TkGemmPlan* plan);

/* Execute one GEMM (replaces kernel.gemm_execute, kernel.py:253-330).
 * a,b,c,d,bias,kmask are device pointers; d may alias c (gemm_ex is in place,
 * api.py:161).  kmask: row-major [num_blocks(M/bm * N/bn, column-major block rank)]
 * x [K/bk] bytes, only read when plan->predicate == TK_PRED_MASK.
 * Returns TK_OK, TK_ERR_CONFIG (nothing written) or TK_ERR_CUDA. */
int tk_gemm(const TkGemmPlan* plan, const void* a, const void* b, const void* c, void* d,
            const void* bias, const uint8_t* kmask, void* workspace, int64_t workspace_bytes,
            void* stream);

/* BLAS-like entry with the reference's exact parameter list (api.py:335-357).
 * Column-major as stored: A is m x k (k x m when trans_a), B is k x n (n x k when
 * trans_b), C is m x n and updated in place.  Host or device pointers. Synchronous. */
int tk_gemm_ex_raw(int type_tag, int trans_a, int trans_b, long long m, long long n,
                   long long k, double alpha_re, double alpha_im, void* a, void* b,
                   double beta_re, double beta_im, void* c);

/* Same, device pointers only, enqueued on `stream` (no host synchronisation). */
int tk_gemm_ex_raw_async(int type_tag, int trans_a, int trans_b, long long m, long long n,
                         long long k, double alpha_re, double alpha_im, const void* a,
                         const void* b, double beta_re, double beta_im, void* c, void* stream);

/* tk_gemm plus a fused all-gather of D (north star: C sharded by column slabs, "an optional
 * all-gather of C over NVLink"): peer_d[q] points at this rank's slab position inside peer q's
 * full-D buffer (mapped with tk_ipc_open).  When the streamed-epilogue CTA-pair kernel runs,
 * every D tile is TMA-stored to the local slab and to all peers from the same shared-memory box
 * (the transfer overlaps the remaining tiles' math); otherwise the slab is copied to the peers
 * after the GEMM on `stream`.  Real operator, dense column-major D, at most 7 peers.  The caller
 * synchronises the ranks (stream sync + barrier) before reading the gathered D. */
int tk_gemm_peers(const TkGemmPlan* plan, const void* a, const void* b, const void* c, void* d,
                  const void* bias, const uint8_t* kmask, void* workspace,
                  int64_t workspace_bytes, void* stream, void* const* peer_d, int npeers);

/* How the last tk_gemm_peers delivered the slab: 1 = epilogue stores to peers, 2 = copies. */
int tk_last_peer_mode(void);

/* CUDA IPC helpers for the peer buffers (one process per GPU).  The handle names the whole
 * allocation; *offset_out is dev_ptr's byte offset in it (add it to tk_ipc_open's pointer). */
int tk_ipc_handle(void* dev_ptr, void* handle_out64, int64_t* offset_out);
int tk_ipc_open(const void* handle64, void** dev_ptr_out);
int tk_ipc_close(void* dev_ptr);

/* Number of device kernels the last successful tk_gemm / tk_gemm_ex_raw launched. */
int tk_last_launch_count(void);

/* Message of the last failure in this thread ("" if none). */
const char* tk_last_error(void);

/* ---- introspection and tuning (no reference counterpart) --------------------------------- */

/* What the last tk_gemm / tk_gemm_ex_raw call on this thread launched: the main kernel's
 * on-chip plan (the reference's allocation audit, kernel.py:74-95, logs its per-worker scratch;
 * here the per-CTA shared-memory stages, C ring and TMEM accumulator columns are the analogue).
 * Sizes in bytes unless noted. */
typedef struct TkPlanInfo {
  char kernel[32];          /* "pair", "pair_cembed", "pair_ops", "ksplit", "single", "stream", "quad", "diag_stream", "simt" */
  int32_t lane;             /* TkLane of the launch, -1 before any */
  int32_t op;               /* TkOperator */
  int32_t tile_m, tile_n;   /* output tile per cluster (or CTA) */
  int32_t tile_k;           /* K per pipeline stage */
  int32_t mma_n, nsub;      /* instruction N, MMAs sharing one A stage */
  int32_t mmas_per_k16;     /* tcgen05.mma per K=16 step (real 1, complex 4, dual 3, split-precision 3) */
  int32_t cluster;          /* CTAs per cluster */
  int32_t stages, stage_bytes;
  int32_t cring_bytes;      /* streamed-C ring (per CTA) */
  int32_t smem_bytes;       /* dynamic shared memory per CTA */
  int32_t tmem_cols;        /* TMEM columns allocated per CTA (x 128 lanes x 4 bytes) */
  int32_t grid_ctas;
  int32_t tiles, units;     /* output tiles; schedule units (tiles + split-K parts) */
  int32_t sk_parts, sk_tiles, sk_tma;
  int32_t serpentine, group_m, pdl, c_stream, d_tma;
  int32_t launches;         /* device kernels of the call (prep passes included) */
  int32_t overlap_kb;       /* pair kernel, 256 x 512 tiles: lo-only / hi-only k-blocks per tile end */
  int64_t workspace_bytes;
} TkPlanInfo;

/* Copy the plan of the last call on this thread into *out. */
int tk_last_plan_info(TkPlanInfo* out);

/* Tuning knobs (the TK_* names of DESIGN.md), read from the environment once when the library
 * is first used.  tk_tune_set overrides one (value NULL or "" restores its default); it returns
 * TK_ERR_CONFIG for an unknown name or malformed value.  tk_tune_reset re-reads the environment.
 * tk_tune_get returns the current value or INT32_MIN when unset. */
int tk_tune_set(const char* name, const char* value);
int tk_tune_reset(void);
int tk_tune_get(const char* name);

/* ---- diagnostics (no reference counterpart; used by bench.py and tools/) ---------------- */

/* Effective SM clock (MHz) of CTA 0 over the last CTA-pair GEMM launch: clock64 ticks over
 * %globaltimer ns, read after the launch completed.  NVML reports the boost clock while a
 * tensor-core GEMM runs power/current-limited; this is the clock the kernel actually saw. */
double tk_debug_pair_mhz(void);

/* globaltimer stamps (us after entry) of the CTA selected by TK_DBG_CTA in the last pair-kernel
 * launch: entry, prologue, first stage full, last MMA issued, last accumulator full, epilogue
 * done, stores drained, exit, then four epilogue-internal stamps (16 doubles; -1 if unset). */
int tk_debug_pair_ts(double* out16);

/* Launch a 1-CTA sleeper on `stream` for `us` microseconds that measures the SM clock while
 * other work runs; read the result with tk_debug_clock_probe_mhz() after synchronising. */
int tk_debug_clock_probe(double us, void* stream);
double tk_debug_clock_probe_mhz(void);

#ifdef __cplusplus
}
#endif

#endif /* TK_SM100_H */
