// tk_api.cu -- the C ABI of libtk_sm100.so (declared in include/tk_sm100.h).
//
// Plan validation -> lane selection -> (prep kernels) -> one persistent tcgen05 launch, or the
// bit-exact CUDA-core lane.  There is no host compute path: every GEMM runs on the device.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <climits>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tk_sm100.h"
#include "tk_prep.cuh"
#include "tk_simt.cuh"
#include "tk_tc_gemm.cuh"
#include "tk_tc_gemm2.cuh"
#include "tk_tc_gemm4.cuh"
#include "tk_tc_gemm2c.cuh"
#include "tk_tc_gemm_ks.cuh"

static_assert(tk::MAX_DIGITS == TK_MAX_DIGITS, "device digit maps match the C ABI");

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
// fused all-gather request of the current tk_gemm_peers call: D slab pointers inside each
// peer's full-D buffer, and how the last call delivered them (1 epilogue stores, 2 copies)
thread_local void* const* g_peer_d = nullptr;
thread_local int g_npeer = 0;
thread_local int g_peer_mode = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define TK_CUDA(call)                                                                 \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(TK_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));       \
  } while (0)

// ------------------------------------------------------------------ tuning knobs
// Every dispatch choice with a tunable default reads this table.  It is filled once from the
// TK_* environment when the library is first used and changes only through tk_tune_set /
// tk_tune_reset (tests, tools/): no launch path calls getenv.  Knobs that change results
// (skipping loads, MMAs, C or the epilogue) exist only in diagnostic builds (-DTK_DIAG).
enum Knob {
  K_TC_KERNEL, K_PAIR_BNI, K_PAIR_NSUB, K_SERPENTINE, K_GROUP_M, K_SPLITK, K_SPLITK_MINKB,
  K_SPLITK_S, K_SK_TMA, K_PDL, K_MN3D, K_PAIR_CSTREAM, K_PAIR_DTMA, K_C_PF, K_C_PF_SPREAD,
  K_NSUB2_CSL, K_STAGGER, K_PAIR_GRID, K_PAIR_DEEPC, K_PAIROPS_BN, K_DIAG_STREAM, K_D_TMA,
  K_L2_PROMO, K_POLICY_AB, K_POL_A, K_POL_B, K_PAIR_CLUSTERS, K_EX_SLABS, K_VERBOSE,
  K_NSUB2_OVERLAP, K_PAIR_KPS, K_CPLX_EMBED, K_POL_C, K_POL_D, K_SIMT_TILED, K_GATHER, K_KSPLIT,
  K_KSPLIT_KPS, K_KSPLIT_NT, K_KSPLIT_BNI,
  K_DBG_C_ZERO, K_DBG_SKIP_EPI, K_DBG_NO_LOAD, K_DBG_NO_MMA, K_DBG_CTA, K_COUNT
};
constexpr int K_FIRST_DIAG = K_DBG_C_ZERO;
const char* const kKnobNames[K_COUNT] = {
  "TK_TC_KERNEL", "TK_PAIR_BNI", "TK_PAIR_NSUB", "TK_SERPENTINE", "TK_GROUP_M", "TK_SPLITK",
  "TK_SPLITK_MINKB", "TK_SPLITK_S", "TK_SK_TMA", "TK_PDL", "TK_MN3D", "TK_PAIR_CSTREAM",
  "TK_PAIR_DTMA", "TK_C_PF", "TK_C_PF_SPREAD", "TK_NSUB2_CSL", "TK_STAGGER", "TK_PAIR_GRID",
  "TK_PAIR_DEEPC", "TK_PAIROPS_BN", "TK_DIAG_STREAM", "TK_D_TMA", "TK_L2_PROMO", "TK_POLICY_AB",
  "TK_POL_A", "TK_POL_B", "TK_PAIR_CLUSTERS", "TK_EX_SLABS", "TK_VERBOSE", "TK_NSUB2_OVERLAP",
  "TK_PAIR_KPS", "TK_CPLX_EMBED", "TK_POL_C", "TK_POL_D", "TK_SIMT_TILED", "TK_GATHER", "TK_KSPLIT",
  "TK_KSPLIT_KPS", "TK_KSPLIT_NT", "TK_KSPLIT_BNI", "TK_DBG_C_ZERO", "TK_DBG_SKIP_EPI", "TK_DBG_NO_LOAD", "TK_DBG_NO_MMA", "TK_DBG_CTA"};
#ifdef TK_DIAG
constexpr int K_ENABLED = K_COUNT;
#else
constexpr int K_ENABLED = K_FIRST_DIAG;
#endif
constexpr int KNOB_UNSET = INT32_MIN;

struct KnobTable {
  std::atomic<int> v[K_COUNT];
};

// TK_TC_KERNEL takes a kernel name; every other knob an integer
int parse_knob(int id, const char* s, int* out) {
  if (!s || !*s) { *out = KNOB_UNSET; return TK_OK; }
  if (id == K_TC_KERNEL) {
    static const char* names[] = {"auto", "single", "pair", "stream", "quad", "diagstream"};
    for (int i = 0; i < 6; ++i)
      if (!strcmp(s, names[i])) { *out = i; return TK_OK; }
    return fail(TK_ERR_CONFIG, "TK_TC_KERNEL: unknown kernel '%s'", s);
  }
  char* end = nullptr;
  const long v = strtol(s, &end, 10);
  if (end == s || *end) return fail(TK_ERR_CONFIG, "%s: integer expected, got '%s'", kKnobNames[id], s);
  *out = int(v);
  return TK_OK;
}

void knobs_from_env(KnobTable& t) {
  for (int i = 0; i < K_COUNT; ++i) {
    int v = KNOB_UNSET;
    if (i < K_ENABLED && parse_knob(i, getenv(kKnobNames[i]), &v) != TK_OK) v = KNOB_UNSET;
    t.v[i].store(v, std::memory_order_relaxed);
  }
  g_err.clear();
}

KnobTable& knob_table() {
  static KnobTable t;
  static std::once_flag once;
  std::call_once(once, [] { knobs_from_env(t); });
  return t;
}

// value of a knob, or `def` when it is not set
inline int knob(Knob id, int def) {
  const int v = knob_table().v[id].load(std::memory_order_relaxed);
  return v == KNOB_UNSET ? def : v;
}
inline bool knob_set(Knob id) { return knob_table().v[id].load(std::memory_order_relaxed) != KNOB_UNSET; }

// what the last launch ran (tk_last_plan_info)
thread_local TkPlanInfo g_info;

void info_reset() {
  memset(&g_info, 0, sizeof(g_info));
  g_info.lane = -1;
}
void info_kernel(const char* name) {
  snprintf(g_info.kernel, sizeof(g_info.kernel), "%s", name);
  g_info.tile_k = strcmp(name, "simt") && strcmp(name, "diag_stream") ? 64 : 0;  // tk::TC_BK
}

// ------------------------------------------------------------------ plan checks
int64_t scalar_bytes(int s) { return s == TK_F16 || s == TK_BF16 ? 2 : s == TK_F32 ? 4 : 8; }
bool is_half(int s) { return s == TK_F16 || s == TK_BF16; }

int64_t dim_extent(const TkLayout& L, int d) {
  int64_t e = 1;
  for (int t = 0; t < L.ndigits[d]; ++t) e *= L.ext[d][t];
  return e;
}

int check_layout(const TkLayout& L, const char* name, int64_t r, int64_t c) {
  if (L.kind < 0 || L.kind > 2) return fail(TK_ERR_CONFIG, "layout %s: bad kind %d", name, L.kind);
  if (L.scalar < 0 || L.scalar > 3) return fail(TK_ERR_CONFIG, "layout %s: bad scalar", name);
  if (L.kind == TK_LAYOUT_ZERO) return TK_OK;
  for (int d = 0; d < 2; ++d)
    if (L.ndigits[d] < 1 || L.ndigits[d] > TK_MAX_DIGITS)
      return fail(TK_ERR_CONFIG, "layout %s: bad digit count", name);
  if (L.kind == TK_LAYOUT_DIAGONAL) {
    if (r != c) return fail(TK_ERR_CONFIG, "layout %s: Diagonal needs a square matrix", name);
    if (L.size < r) return fail(TK_ERR_CONFIG, "layout %s: diagonal buffer too small", name);
    return TK_OK;
  }
  if (dim_extent(L, 0) != r || dim_extent(L, 1) != c)
    return fail(TK_ERR_CONFIG, "layout %s: extents (%lld, %lld) != expected (%lld, %lld)", name,
                (long long)dim_extent(L, 0), (long long)dim_extent(L, 1), (long long)r, (long long)c);
  // largest reachable element offset must lie inside the buffer
  int64_t maxoff = 0;
  for (int d = 0; d < 2; ++d)
    for (int t = 0; t < L.ndigits[d]; ++t) {
      if (L.stride[d][t] < 0) return fail(TK_ERR_CONFIG, "layout %s: negative stride", name);
      maxoff += (L.ext[d][t] - 1) * L.stride[d][t];
    }
  int64_t need = maxoff + 1;
  if (L.pair == TK_PAIR_INTERLEAVED) need = 2 * need;
  else if (L.pair == TK_PAIR_SPLIT) need = L.plane_stride + need;
  if (need > L.size) return fail(TK_ERR_CONFIG, "layout %s: addresses beyond physical size", name);
  return TK_OK;
}

int check_transform(const TkTransform& t, const char* name) {
  if (t.n < 0 || t.n > TK_MAX_TOPS) return fail(TK_ERR_CONFIG, "transform %s: bad length", name);
  for (int i = 0; i < t.n; ++i)
    if (t.op[i] < TK_T_SCALE || t.op[i] > TK_T_RELU)
      return fail(TK_ERR_CONFIG, "transform %s: bad op %d", name, t.op[i]);
  return TK_OK;
}

int check_plan(const TkGemmPlan* p) {
  if (!p) return fail(TK_ERR_CONFIG, "null plan");
  if (p->abi_version != TK_ABI_VERSION)
    return fail(TK_ERR_CONFIG, "plan ABI version %d != library %d", p->abi_version, TK_ABI_VERSION);
  if (p->m < 1 || p->n < 1 || p->k < 1) return fail(TK_ERR_CONFIG, "GEMM extents must be >= 1");
  if (p->op < TK_OP_REAL || p->op > TK_OP_DUAL) return fail(TK_ERR_CONFIG, "bad operator");
  if (p->compute != TK_F32 && p->compute != TK_F64)
    return fail(TK_ERR_CONFIG, "accumulator must be f32 or f64");
  for (int d = 0; d < 3; ++d)
    if (p->block[d] < 1) return fail(TK_ERR_CONFIG, "block tile must be positive");
  if (p->m % p->block[0] || p->n % p->block[1] || p->k % p->block[2])
    return fail(TK_ERR_CONFIG, "block tile must divide GEMM shape");
  if (p->op_k < 1 || p->block[2] % p->op_k) return fail(TK_ERR_CONFIG, "operator K must divide block K");
  int rc;
  if ((rc = check_layout(p->a, "A", p->m, p->k))) return rc;
  if ((rc = check_layout(p->b, "B", p->k, p->n))) return rc;
  if ((rc = check_layout(p->c, "C", p->m, p->n))) return rc;
  if ((rc = check_layout(p->d, "D", p->m, p->n))) return rc;
  if (p->d.kind != TK_LAYOUT_STRIDED) return fail(TK_ERR_CONFIG, "D must be a strided layout");
  if (p->b.kind == TK_LAYOUT_DIAGONAL) return fail(TK_ERR_CONFIG, "Diagonal B is not supported");
  const bool pair = p->op != TK_OP_REAL;
  const TkLayout* ls[4] = {&p->a, &p->b, &p->c, &p->d};
  for (const TkLayout* L : ls)
    if (L->kind == TK_LAYOUT_STRIDED && (L->pair != TK_PAIR_NONE) != pair)
      return fail(TK_ERR_CONFIG, "pair layouts must match the operator");
  if (pair && p->a.kind == TK_LAYOUT_DIAGONAL)
    return fail(TK_ERR_CONFIG, "Diagonal A needs the real operator");
  if ((rc = check_transform(p->t_a, "g2s_a")) || (rc = check_transform(p->t_b, "g2s_b")) ||
      (rc = check_transform(p->t_c, "g2s_c")) || (rc = check_transform(p->t_r2s, "r2s_d")) ||
      (rc = check_transform(p->t_s2g, "s2g_d")))
    return rc;
  if (pair) {
    const TkTransform* ts[5] = {&p->t_a, &p->t_b, &p->t_c, &p->t_r2s, &p->t_s2g};
    for (const TkTransform* t : ts)
      for (int i = 0; i < t->n; ++i) {
        if (t->op[i] == TK_T_RELU) return fail(TK_ERR_CONFIG, "relu is undefined on pair elements");
        if (p->op == TK_OP_DUAL && t->op[i] == TK_T_ADD)
          return fail(TK_ERR_CONFIG, "add_constant is undefined on dual elements");
      }
    if (p->bias_axis) return fail(TK_ERR_CONFIG, "bias epilogue needs the real operator");
  }
  if (p->bias_axis < 0 || p->bias_axis > 2) return fail(TK_ERR_CONFIG, "bad bias axis");
  if (p->predicate < 0 || p->predicate > 2) return fail(TK_ERR_CONFIG, "bad predicate");
  const bool a64 = p->a.scalar == TK_F64;
  if (p->compute == TK_F32 && a64) return fail(TK_ERR_CONFIG, "f64 storage needs f64 accumulation");
  return TK_OK;
}

// ------------------------------------------------------------------ lane selection
// A load transform whose result is always representable in the operand's own half type
// (relu, scale by +-1, add 0): the transform pass writes one plane and the ordinary real
// kernels run on it.  Any other program needs the hi + lo split (OP_SPLIT kernels).
bool half_exact(const TkTransform& t) {
  for (int i = 0; i < t.n; ++i) {
    if (t.op[i] == TK_T_RELU) continue;
    if (t.op[i] == TK_T_SCALE && (t.re[i] == 1.0 || t.re[i] == -1.0)) continue;
    if (t.op[i] == TK_T_ADD && t.re[i] == 0.0) continue;
    return false;
  }
  return true;
}

// strided operand the tensor cores can take straight from TMA: one digit per dimension,
// one unit-stride dimension, 16-byte aligned pitch.
bool tma_operand(const TkLayout& L, int& mn_major_dim0, int64_t& pitch) {
  if (L.kind != TK_LAYOUT_STRIDED || L.ndigits[0] != 1 || L.ndigits[1] != 1) return false;
  const int64_t s0 = L.stride[0][0], s1 = L.stride[1][0];
  if (s0 == 1 && (s1 * 2) % 16 == 0 && s1 >= L.ext[0][0]) { mn_major_dim0 = 1; pitch = s1; }
  else if (s1 == 1 && (s0 * 2) % 16 == 0 && s0 >= L.ext[1][0]) { mn_major_dim0 = 0; pitch = s0; }
  else return false;
  if (L.pair == TK_PAIR_SPLIT && (L.plane_stride * 2) % 16 != 0) return false;
  if (L.pair == TK_PAIR_INTERLEAVED) {  // de-interleaved into dense planes: must be a bijection
    const int64_t vol = L.ext[0][0] * L.ext[1][0];
    if (pitch != (mn_major_dim0 ? L.ext[0][0] : L.ext[1][0])) return false;
    if (2 * vol > L.size) return false;
  }
  return true;
}

// ---- complex embedding (tc_gemm_pair_kernel<..., EMB>): an interleaved complex GEMM run as
// the real GEMM D^ = A~ B^ + C^ over the interleaved buffers read as real matrices (2M x N,
// 2K x N; A~ built on chip from A^ = A as a 2M x K real matrix).  Taken when every operand is a
// dense column-major interleaved pair buffer TMA can read, the epilogue is real-separable
// (empty or real-scale transforms, no bias, no predicate) and the shape fills CTA-pair tiles.
bool cplx_col(const TkLayout& L, int64_t& ld) {
  if (L.kind != TK_LAYOUT_STRIDED || L.pair != TK_PAIR_INTERLEAVED || L.ndigits[0] != 1 || L.ndigits[1] != 1)
    return false;
  if (L.stride[0][0] != 1 || L.stride[1][0] < L.ext[0][0]) return false;
  ld = L.stride[1][0];
  return true;
}
bool real_scale_only(const TkTransform& t) {
  for (int i = 0; i < t.n; ++i)
    if (t.op[i] != TK_T_SCALE || t.im[i] != 0.0) return false;
  return true;
}
bool embed_ok(const TkGemmPlan* p) {
  if (p->op != TK_OP_COMPLEX || p->compute != TK_F32 || !is_half(p->a.scalar)) return false;
  if (p->t_a.n || p->t_b.n || p->bias_axis || p->predicate != TK_PRED_ALWAYS) return false;
  if (!real_scale_only(p->t_c) || !real_scale_only(p->t_r2s) || !real_scale_only(p->t_s2g)) return false;
  int64_t lda, ldb, ldc = 0, ldd;
  if (!cplx_col(p->a, lda) || !cplx_col(p->b, ldb) || !cplx_col(p->d, ldd)) return false;
  if (p->c.kind != TK_LAYOUT_ZERO && !cplx_col(p->c, ldc)) return false;
  // 16-byte TMA pitches (2*ld halves for A^ / B^, 2*ld floats for C^ / D^), 64-row A^ chunks,
  // and enough of a problem for the CTA-pair tiles (2M >= 256 rows, > 4 block-K steps of 2K)
  if ((lda * 4) % 16 || (ldb * 4) % 16 || (ldc * 8) % 16 || (ldd * 8) % 16) return false;
  if (p->m % 32 || p->m < 128 || p->k <= 128) return false;
  if (2 * p->m >= (1ll << 31) || 2 * p->k >= (1ll << 31)) return false;
  return knob(K_CPLX_EMBED, 1) != 0;
}
void real_col(TkLayout& L, int64_t rows, int64_t cols, int64_t ld) {
  const int scalar = L.scalar, kind = L.kind;
  memset(&L, 0, sizeof(L));
  L.kind = kind;
  L.scalar = scalar;
  if (kind == TK_LAYOUT_ZERO) return;
  L.ndigits[0] = L.ndigits[1] = 1;
  L.ext[0][0] = rows;
  L.ext[1][0] = cols;
  L.stride[0][0] = 1;
  L.stride[1][0] = ld;
  L.size = ld * (cols - 1) + rows;
}
// The real plan of the embedding: M' = 2M, K' = 2K; A describes A^ (2M x K, the kernel's
// staging source), B^ / C^ / D^ the interleaved buffers as real column-major matrices.
void embed_plan(const TkGemmPlan* p, TkGemmPlan* out) {
  *out = *p;
  out->op = TK_OP_REAL;
  out->m = 2 * p->m;
  out->k = 2 * p->k;
  real_col(out->a, 2 * p->m, p->k, 2 * p->a.stride[1][0]);
  real_col(out->b, 2 * p->k, p->n, 2 * p->b.stride[1][0]);
  if (p->c.kind != TK_LAYOUT_ZERO) real_col(out->c, 2 * p->m, p->n, 2 * p->c.stride[1][0]);
  real_col(out->d, 2 * p->m, p->n, 2 * p->d.stride[1][0]);
}

// ---- digit-mapped operands read in place (GETT / tensor contractions on the CTA-pair kernel):
// a half operand with <= 2 digits per GEMM dimension whose fastest digit is contiguous becomes a
// 5-D TMA map -- MN-major {64, K0, MN0/64, MN1, K1} or K-major {64, MN0, MN1, K0/64, K1} -- whose
// box lands in shared memory exactly as the dense operand's tile would, so no pack pass runs.
// Needs the contiguous digit's run to hold whole CTA blocks: MN0 % 128 == 0 (a 128-row A half,
// 64 / 128 B columns) and, with two K digits, K0 % 64 == 0.
CUtensorMapL2promotion l2_promo();
PFN_cuTensorMapEncodeTiled_v12000 get_encode();
struct Gather {
  int g = 0;                          // 1 MN-major, 2 K-major
  int64_t e0 = 1, s0 = 0, e1 = 1, s1 = 0;  // MN digits (extent, stride in elements)
  int64_t f0 = 1, t0 = 0, f1 = 1, t1 = 0;  // K digits
};
bool gather_layout(const TkLayout& L, int role, Gather& gl) {
  if (L.kind != TK_LAYOUT_STRIDED || L.pair || !is_half(L.scalar) || !knob(K_GATHER, 1)) return false;
  const int dm = role == 0 ? 0 : 1, dk = 1 - dm;
  if (L.ndigits[dm] > 2 || L.ndigits[dk] > 2) return false;
  Gather g;
  g.e0 = L.ext[dm][0]; g.s0 = L.stride[dm][0];
  if (L.ndigits[dm] == 2) { g.e1 = L.ext[dm][1]; g.s1 = L.stride[dm][1]; }
  g.f0 = L.ext[dk][0]; g.t0 = L.stride[dk][0];
  if (L.ndigits[dk] == 2) { g.f1 = L.ext[dk][1]; g.t1 = L.stride[dk][1]; }
  auto ok16 = [](int64_t st) { return st > 0 && (st * 2) % 16 == 0 && st * 2 < (int64_t(1) << 40); };
  if (g.s0 == 1) {
    g.g = 1;
    if (g.e0 % 128 || !ok16(g.t0) || (g.e1 > 1 && !ok16(g.s1)) || (g.f1 > 1 && (!ok16(g.t1) || g.f0 % 64))) return false;
  } else if (g.t0 == 1) {
    // (the contiguous K digit is cut into 64-element chunks: they must tile it exactly, since a
    // chunk past its end would read the next MN row instead of zero-filling)
    g.g = 2;
    if (!ok16(g.s0) || g.f0 % 64 || (g.e1 > 1 && (!ok16(g.s1) || g.e0 % 128)) || (g.f1 > 1 && !ok16(g.t1)))
      return false;
  } else {
    return false;
  }
  if (g.e0 >= (int64_t(1) << 31) || g.f0 >= (int64_t(1) << 31)) return false;
  gl = g;
  return true;
}
// the 5-D map of a gathered operand; box_mn = the CTA's rows (A: 128) or columns (B: BNI/2)
int make_map_gather(CUtensorMap* map, const void* base, int scalar, const Gather& g, uint32_t box_mn) {
  auto enc = get_encode();
  if (!enc) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[5];
  cuuint64_t strides[4];
  cuuint32_t box[5];
  const cuuint64_t unit = 16;  // stride of an extent-1 dimension (never stepped)
  if (g.g == 1) {
    dims[0] = 64; dims[1] = g.f0; dims[2] = g.e0 / 64; dims[3] = g.e1; dims[4] = g.f1;
    strides[0] = g.t0 * 2; strides[1] = 128; strides[2] = g.e1 > 1 ? g.s1 * 2 : unit;
    strides[3] = g.f1 > 1 ? g.t1 * 2 : unit;
    box[0] = 64; box[1] = 64; box[2] = box_mn / 64; box[3] = 1; box[4] = 1;
  } else {
    dims[0] = 64; dims[1] = g.e0; dims[2] = g.e1; dims[3] = g.f0 / 64; dims[4] = g.f1;
    strides[0] = g.s0 * 2; strides[1] = g.e1 > 1 ? g.s1 * 2 : unit; strides[2] = 128;
    strides[3] = g.f1 > 1 ? g.t1 * 2 : unit;
    box[0] = 64; box[1] = box_mn; box[2] = 1; box[3] = 1; box[4] = 1;
  }
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(map, scalar == TK_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, l2_promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled (5-D gather) failed (%d)", int(r));
  return TK_OK;
}

// The plan runs on the CTA-pair kernel with plain operands (so a digit-mapped operand may be
// gathered by the TMA instead of packed): the dispatch in run_tc takes the pair path for it.
bool gather_path(const TkGemmPlan* p) {
  const int ov = knob(K_TC_KERNEL, 0);
  return p->op == TK_OP_REAL && !p->t_a.n && !p->t_b.n && p->a.kind == TK_LAYOUT_STRIDED &&
         p->predicate == TK_PRED_ALWAYS && p->m > 128 && (p->k + 63) / 64 > 4 && (ov == 0 || ov == 2);
}
// tensor contraction: A with its two M digits swapped (m' = m1 + e1*m0, see permuted_plan)
TkLayout swapped_a(const TkLayout& A0) {
  TkLayout A = A0;
  std::swap(A.ext[0][0], A.ext[0][1]);
  std::swap(A.stride[0][0], A.stride[0][1]);
  return A;
}
// B's shared-memory major-ness on the pair kernel: MN-major when N is contiguous (dense or
// gathered); a packed B is K-major
bool b_mn_major(const TkLayout& b) {
  int mn;
  int64_t pitch;
  if (tma_operand(b, mn, pitch)) return !mn;
  Gather g;
  return gather_layout(b, 1, g) && g.g == 1;
}

// A half-precision strided operand the TMA cannot read directly (multi-digit permutations,
// non-unit innermost strides, non-bijective interleaved pairs) is gathered once into a dense
// column-major workspace by pack_half_kernel and then takes the normal tensor-core path.
bool pack_needed(const TkLayout& L) {
  int mn;
  int64_t pitch;
  return L.kind == TK_LAYOUT_STRIDED && is_half(L.scalar) && !tma_operand(L, mn, pitch);
}

// rewrite a layout as the dense column-major rows x cols operand pack_half_kernel produces
void dense_operand(TkLayout& L, int64_t rows, int64_t cols) {
  const int pair = L.pair ? TK_PAIR_SPLIT : 0;
  const int scalar = L.scalar;
  memset(&L, 0, sizeof(L));
  L.kind = TK_LAYOUT_STRIDED;
  L.pair = pair;
  L.scalar = scalar;
  L.ndigits[0] = L.ndigits[1] = 1;
  L.ext[0][0] = rows;
  L.ext[1][0] = cols;
  L.stride[0][0] = 1;
  L.stride[1][0] = rows;
  L.plane_stride = pair ? rows * cols : 0;
  L.size = rows * cols * (pair ? 2 : 1);
}

// GETT-as-GEMM (tensor contraction, reference api.py:259-290): A's M index has two digits
// (e0, s0), (e1, s1) and D's M digits are the same extents with the order swapped into a
// dense run (t1 == 1, t0 == e1).  Rewrite to a plain column-major GEMM over m' = m1 + e1*m0:
// A is permuted once into a dense M' x K workspace (pack_half_kernel), D (and C) become
// column-major with the N stride as leading dimension.
bool permuted_plan(const TkGemmPlan* p, TkGemmPlan* out) {
  const TkLayout& A = p->a;
  const TkLayout& D = p->d;
  if (A.kind != TK_LAYOUT_STRIDED || A.pair || A.ndigits[0] != 2 || A.ndigits[1] != 1) return false;
  if (D.kind != TK_LAYOUT_STRIDED || D.pair || D.ndigits[0] != 2 || D.ndigits[1] != 1) return false;
  const int64_t e0 = A.ext[0][0], e1 = A.ext[0][1];
  if (D.ext[0][0] != e0 || D.ext[0][1] != e1 || D.stride[0][1] != 1 || D.stride[0][0] != e1) return false;
  if (p->c.kind != TK_LAYOUT_ZERO &&
      (p->c.kind != TK_LAYOUT_STRIDED || p->c.pair || p->c.ndigits[0] != 2 || p->c.ndigits[1] != 1 ||
       p->c.ext[0][0] != e0 || p->c.ext[0][1] != e1 || p->c.stride[0][1] != 1 || p->c.stride[0][0] != e1))
    return false;
  if (p->bias_axis == 2 || p->predicate != TK_PRED_ALWAYS || !is_half(A.scalar) || p->k > 65535)
    return false;
  if (out) {
    *out = *p;
    auto dense_cm = [](TkLayout& L, int64_t rows, int64_t cols, int64_t ld) {
      memset(L.ext, 0, sizeof(L.ext));
      memset(L.stride, 0, sizeof(L.stride));
      L.ndigits[0] = L.ndigits[1] = 1;
      L.ext[0][0] = rows; L.stride[0][0] = 1;
      L.ext[1][0] = cols; L.stride[1][0] = ld;
    };
    dense_cm(out->a, p->m, p->k, p->m);
    out->a.size = p->m * p->k;
    dense_cm(out->d, p->m, p->n, D.stride[1][0]);
    if (p->c.kind == TK_LAYOUT_STRIDED) dense_cm(out->c, p->m, p->n, p->c.stride[1][0]);
  }
  return true;
}

// A block predicate the tensor-core lane evaluates itself: a host-evaluated mask, or the diagonal
// rule over a dense A (a Diagonal A layout instead restricts the k range in its own kernels).
bool pred_on_tc(const TkGemmPlan* p) {
  return p->predicate == TK_PRED_MASK || (p->predicate == TK_PRED_DIAGONAL && p->a.kind != TK_LAYOUT_DIAGONAL);
}

// Instruction N of the CTA-pair kernel for a predicated plan: every 256 x BNI tile must lie in one
// reference block (bm % 256, bn % BNI) and each K=16 MMA step in one block-K chunk (bk % 16);
// 0 when no tile shape fits (the exact lane then runs the predicate).
int pred_bni(const TkGemmPlan* p, std::string* why = nullptr) {
  auto no = [&](const char* w) { if (why) *why = w; return 0; };
  if (p->op != TK_OP_REAL || p->t_a.n || p->t_b.n) return no("block predicates on the tensor cores: real operator, no A/B transforms");
  if (p->block[2] % 16) return no("block predicate with bk % 16 != 0 (an MMA step would straddle two block-K chunks)");
  if (p->block[0] % 256) return no("block predicate with bm % 256 != 0 (a 256-row pair tile would straddle blocks)");
  if (p->m <= 128 || (p->k + 63) / 64 <= 4) return no("block predicate on a shape below the CTA-pair kernel");
  int mn = 1;
  int64_t pitch;
  const bool b_mn = tma_operand(p->b, mn, pitch) ? !mn : false;  // a gathered B is K-major
  for (int bni : {256, 128, 64})
    if (p->block[1] % bni == 0 && !(bni == 64 && b_mn)) return bni;
  return no("block predicate with bn not a multiple of the pair tile width");
}

bool tc_lane_ok(const TkGemmPlan* p, std::string& why) {
  TkGemmPlan rewritten;
  if (permuted_plan(p, &rewritten)) return tc_lane_ok(&rewritten, why);
  auto no = [&](const char* w) { why = w; return false; };
  if (p->compute != TK_F32) return no("tcgen05 lane accumulates in f32 only");
  if (!is_half(p->a.scalar) || p->b.scalar != p->a.scalar) return no("A/B must be f16 or bf16");
  if (p->b.kind != TK_LAYOUT_STRIDED) return no("B must be strided");
  int mn;
  int64_t pitch;
  if (p->a.kind == TK_LAYOUT_DIAGONAL) {
    if (p->op != TK_OP_REAL || p->t_a.n) return no("Diagonal A only with real op, identity g2s_a");
  } else if (p->a.kind != TK_LAYOUT_STRIDED) {
    return no("A layout is neither strided nor diagonal");
  } else if (!tma_operand(p->a, mn, pitch) && (p->m * p->k * 2 * 2 > (int64_t(1) << 40))) {
    return no("A too large to pack");
  }
  if (p->c.kind != TK_LAYOUT_ZERO && p->c.scalar != TK_F32) return no("C must be f32");
  if (p->d.scalar != TK_F32) return no("D must be f32");
  if (p->c.kind == TK_LAYOUT_DIAGONAL) return no("Diagonal C unsupported on tcgen05 lane");
  if (p->op != TK_OP_REAL && (p->t_a.n || p->t_b.n)) return no("pair operands need identity g2s");
  // transformed operands go through the transform pass: fp16 splits into hi + lo planes; bf16
  // would need three planes for the reference's f32 transform result, so only exact programs
  if (p->a.scalar == TK_BF16 && !(half_exact(p->t_a) && half_exact(p->t_b)))
    return no("bf16 operand transforms beyond relu / scale(+-1) run on the exact lane");
  if (pred_on_tc(p) && !pred_bni(p, &why)) return false;
  if (p->bias_axis && p->bias_scalar != TK_F32) return no("bias must be f32");
  if (p->m >= (1ll << 31) || p->n >= (1ll << 31) || p->k >= (1ll << 31)) return no("extent >= 2^31");
  return true;
}

int choose_lane(const TkGemmPlan* p, std::string* why_out = nullptr) {
  std::string why;
  const bool tc = tc_lane_ok(p, why);
  if (why_out) *why_out = why;
  if (p->lane == TK_LANE_TCGEN05 && !tc) return -1;
  if (p->lane == TK_LANE_SIMT) return TK_LANE_SIMT;
  return tc ? TK_LANE_TCGEN05 : TK_LANE_SIMT;
}

// ------------------------------------------------------------------ workspace plan
struct Workspace {
  int64_t a_planes = -1, b_planes = -1, a_perm = -1, a_pack = -1, b_pack = -1, splitk = -1,
          a_tx = -1, b_tx = -1, tx_flags = -1, kbits = -1, total = 0;
  bool tx_split = false;  // transformed operands carry hi + lo planes (OP_SPLIT)
};

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

struct SplitPlan;
SplitPlan split_plan(int64_t tiles, int clusters, int kb_total, int bnp);
int choose_pair_bni(int64_t m, int64_t n, bool b_mn_major, int clusters);
int pair_clusters();
int tc_kernel_override();
int64_t split_ws_bytes(int64_t m, int64_t n, int64_t k, const TkLayout& b);

Workspace plan_workspace(const TkGemmPlan* p0, int lane) {
  Workspace w;
  if (lane != TK_LANE_TCGEN05) return w;
  TkGemmPlan rewritten;
  const TkGemmPlan* p = p0;
  Gather gl;
  if (permuted_plan(p0, &rewritten)) {
    if (gather_path(&rewritten) && gather_layout(swapped_a(p0->a), 0, gl)) {
      rewritten.a = swapped_a(p0->a);  // read in place by a 5-D TMA map
    } else {
      w.a_perm = w.total;
      w.total += align256(p0->m * p0->k * 2);
    }
    p = &rewritten;
  }
  TkGemmPlan packed = *p;
  const bool gp = gather_path(p);
  if (pack_needed(p->a) && !(gp && gather_layout(p->a, 0, gl))) {
    w.a_pack = w.total;
    w.total += align256(p->m * p->k * 2 * (p->a.pair ? 2 : 1));
    dense_operand(packed.a, p->m, p->k);
  }
  if (pack_needed(p->b) && !(gp && gather_layout(p->b, 1, gl))) {
    w.b_pack = w.total;
    w.total += align256(p->k * p->n * 2 * (p->b.pair ? 2 : 1));
    dense_operand(packed.b, p->k, p->n);
  }
  p = &packed;
  if (embed_ok(p0)) return w;  // complex embedding: interleaved operands are read in place
  if (p->a.kind == TK_LAYOUT_STRIDED && p->a.pair == TK_PAIR_INTERLEAVED) {
    w.a_planes = w.total;
    w.total += align256(p->m * p->k * 2 * 2);
  }
  if (p->b.pair == TK_PAIR_INTERLEAVED) {
    w.b_planes = w.total;
    w.total += align256(p->k * p->n * 2 * 2);
  }
  // load transforms (g2s_a / g2s_b): transformed operand planes, hi (+ lo), and the lo flags
  if (p->op == TK_OP_REAL && (p->t_a.n || p->t_b.n)) {
    w.tx_split = !(half_exact(p->t_a) && half_exact(p->t_b));
    const int planes = w.tx_split ? 2 : 1;
    if (p->t_a.n) { w.a_tx = w.total; w.total += align256(p->m * p->k * 2 * planes); }
    if (p->t_b.n) { w.b_tx = w.total; w.total += align256(p->k * p->n * 2 * planes); }
    w.tx_flags = w.total;
    w.total += 256;
  }
  if (pred_on_tc(p)) {  // per-tile MMA-step bits of the block predicate (expand_kbits_kernel)
    const int bni = pred_bni(p);
    const int64_t tiles = ((p->m + 255) / 256) * ((p->n + bni - 1) / bni);
    w.kbits = w.total;
    w.total += align256(tiles * (((p->k + 15) / 16 + 31) / 32) * 4);
  } else if (p->op == TK_OP_REAL && !w.tx_split && p->a.kind != TK_LAYOUT_DIAGONAL) {  // split-K partials (pair kernel)
    const int64_t sb = split_ws_bytes(p->m, p->n, p->k, p->b);
    if (sb > 0) { w.splitk = w.total; w.total += align256(sb); }
  }
  return w;
}

// ------------------------------------------------------------------ TMA
// TK_L2_PROMO=0|64|128|256 (tuning knob; default 256B L2 sector promotion for TMA loads)
CUtensorMapL2promotion l2_promo() {
  const int v = knob(K_L2_PROMO, 256);
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
       : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
       : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

int make_map_2d(CUtensorMap* map, const void* base, int scalar, uint64_t inner, uint64_t outer,
                uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, bool swizzle = true) {
  auto enc = get_encode();
  if (!enc) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const bool f32 = scalar == TK_F32;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                     : scalar == TK_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                        : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (f32 || !swizzle) ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   l2_promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return TK_OK;
}

// MN-major operand as {64 (MN inner), K, MN/64}: one TMA box {64, 64, atoms} fills `atoms`
// consecutive 128B-swizzled 64x64 atoms (8 KB apart) -- the same smem image as `atoms` 2-D boxes.
int make_map_mn3d(CUtensorMap* map, const void* base, int scalar, uint64_t mn, uint64_t k,
                  uint64_t pitch_elems, uint32_t atoms) {
  auto enc = get_encode();
  if (!enc) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, k, (mn + 63) / 64};
  cuuint64_t strides[2] = {pitch_elems * 2, 128};
  cuuint32_t box[3] = {64, 64, atoms};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, scalar == TK_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                   3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, l2_promo(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d)", int(r));
  return TK_OK;
}

tk::DigitMap to_map(const TkLayout& L) {
  tk::DigitMap m{};
  for (int d = 0; d < 2; ++d) {
    m.nd[d] = L.kind == TK_LAYOUT_STRIDED ? L.ndigits[d] : 1;
    for (int t = 0; t < TK_MAX_DIGITS; ++t) {
      m.e[d][t] = t < L.ndigits[d] ? L.ext[d][t] : 1;
      m.s[d][t] = t < L.ndigits[d] ? L.stride[d][t] : 0;
    }
  }
  return m;
}

tk::EpiProg to_prog(const TkTransform& t) {
  tk::EpiProg g{};
  g.n = t.n;
  for (int i = 0; i < t.n; ++i) {
    g.op[i] = t.op[i];
    g.promote[i] = t.promote[i];
    g.fre[i] = float(t.re[i]);
    g.fim[i] = float(t.im[i]);
    g.dre[i] = t.re[i];
    g.dim[i] = t.im[i];
  }
  return g;
}

// Per-device caches (SM count, raised shared-memory limits, co-resident cluster counts) are
// indexed by the current device: a process may drive several GPUs.
constexpr int TK_MAX_DEV = 64;
int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < TK_MAX_DEV ? dev : 0;
}

int sm_count() {
  static int cache[TK_MAX_DEV] = {};
  const int dev = cur_dev();
  int n = cache[dev];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
  }
  return n;
}

template <int OP, bool DENSE, int CSTREAM = 0>
int launch_tc_variant(const tk::TcParams& prm, cudaStream_t s) {
  using S = tk::TcSmem<OP, CSTREAM>;
  static bool attr[TK_MAX_DEV] = {};
  const int dev = cur_dev();
  if (!attr[dev]) {
    TK_CUDA(cudaFuncSetAttribute(tk::tc_gemm_kernel<OP, DENSE, CSTREAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL));
    attr[dev] = true;
  }
  const int grid = std::min(prm.num_tiles, sm_count());
  tk::tc_gemm_kernel<OP, DENSE, CSTREAM><<<grid, tk::TC_THREADS, S::TOTAL, s>>>(prm);
  TK_CUDA(cudaGetLastError());
  ++g_launches;
  info_kernel(CSTREAM ? "stream" : "single");
  g_info.tile_m = tk::TC_BM;
  g_info.tile_n = tk::TcCfg<OP>::BN;
  g_info.mma_n = tk::TcCfg<OP>::BN;
  g_info.nsub = 1;
  g_info.mmas_per_k16 = OP == tk::OP_REAL ? 1 : OP == tk::OP_COMPLEX ? 4 : 3;
  g_info.cluster = 1;
  g_info.stages = S::STAGES;
  g_info.stage_bytes = S::STAGE_BYTES;
  g_info.cring_bytes = S::CRING_BYTES;
  g_info.smem_bytes = S::TOTAL;
  g_info.tmem_cols = tk::TcCfg<OP>::TMEM_COLS;
  g_info.grid_ctas = grid;
  g_info.tiles = g_info.units = prm.num_tiles;
  g_info.sk_parts = 1;
  g_info.group_m = prm.group_m;
  g_info.c_stream = CSTREAM ? 1 : 0;
  g_info.d_tma = prm.d_tma;
  return TK_OK;
}

template <bool DENSE, bool CSTREAM = false, int NSUB = 1, int BNI = 256, int CSL = tk::TC2S_CSLOTS, int KPS = 1,
          bool EMB = false>
int launch_tc_pair(const tk::TcParams& prm, cudaStream_t s) {
  constexpr int SMEM = tk::Tc2Plan<NSUB, CSTREAM, BNI, CSL, KPS, EMB>::SMEM;
  constexpr int THREADS = tk::Tc2Plan<NSUB, CSTREAM, BNI, CSL, KPS, EMB>::THREADS;
  auto kern = tk::tc_gemm_pair_kernel<DENSE, CSTREAM, NSUB, BNI, CSL, KPS, EMB>;
  static bool attr[TK_MAX_DEV] = {};
  static int max_clusters_dev[TK_MAX_DEV] = {};
  const int dev = cur_dev();
  if (!attr[dev]) {
    TK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    attr[dev] = true;
  }
  int& max_clusters = max_clusters_dev[dev];
  if (!max_clusters) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (sm_count() / 2));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters <= 0) {
      cudaGetLastError();
      max_clusters = sm_count() / 2;
    }
    if (knob(K_VERBOSE, 0)) fprintf(stderr, "tk: pair kernel max active clusters %d\n", max_clusters);
  }
  tk::TcParams run = prm;
  if (run.sk_parts > 1 && max_clusters != pair_clusters()) {  // split parts must all be co-resident
    run.num_units = run.sk_first = run.num_tiles;
    run.sk_parts = 1;
    run.sk_tma = 0;
  }
  const bool eg = knob_set(K_PAIR_GRID);
  if (run.nar_units > 0 && (max_clusters != pair_clusters() || eg)) {  // staggered lists assume P
    run.num_units = run.num_tiles;
    run.nar_units = 0;
  }
  int clusters = std::min(run.num_units, max_clusters);
  if (eg) clusters = std::max(1, std::min(clusters, knob(K_PAIR_GRID, clusters)));
  // every split unit must be the LAST unit of its cluster (units c, c+P, ...: sk_first a
  // multiple of the cluster count, at most one split unit per cluster) -- the epilogue's C-ring
  // bookkeeping (smask in tc_gemm_pair_kernel) relies on it; any other schedule runs unsplit
  if (run.sk_parts > 1 && (run.sk_first % clusters != 0 || run.num_units - run.sk_first > clusters)) {
    run.num_units = run.sk_first = run.num_tiles;
    run.sk_parts = 1;
    run.sk_tma = 0;
    clusters = std::min(run.num_units, clusters);
  }
  const int grid = 2 * clusters;
  // programmatic dependent launch: the next GEMM in the stream may be scheduled while this one
  // drains; its CTAs run their prologue (barriers, TMEM, tensor-map prefetch) and then wait in
  // griddepcontrol.wait until this grid has completed and its writes are visible
  const bool pdl = knob(K_PDL, 1) != 0;
  // not after the split-K flag memset: a programmatic launch may start before a preceding
  // memset node completes, and the flags must be zero before any part counts in
  run.pdl = (pdl && run.sk_parts == 1) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = run.pdl ? 1 : 0;
  TK_CUDA(cudaLaunchKernelEx(&cfg, kern, run));
  ++g_launches;
  using PL = tk::Tc2Plan<NSUB, CSTREAM, BNI, CSL, KPS, EMB>;
  info_kernel(EMB ? "pair_cembed" : "pair");
  g_info.tile_m = 256;
  g_info.tile_k = 64 * KPS;
  g_info.tile_n = PL::BNP;
  g_info.mma_n = BNI;
  g_info.nsub = NSUB;
  g_info.mmas_per_k16 = NSUB;
  g_info.cluster = 2;
  g_info.stages = PL::STAGES;
  g_info.stage_bytes = PL::STAGE_BYTES;
  g_info.cring_bytes = PL::CRING_BYTES;
  g_info.smem_bytes = SMEM;
  g_info.tmem_cols = PL::TMEM_COLS;
  g_info.grid_ctas = grid;
  g_info.tiles = run.num_tiles;
  g_info.units = run.num_units;
  g_info.sk_parts = run.sk_parts;
  g_info.sk_tiles = run.sk_parts > 1 ? (run.num_units - run.sk_first) / run.sk_parts : 0;
  g_info.sk_tma = run.sk_tma;
  g_info.serpentine = run.serp;
  g_info.group_m = run.group_m;
  g_info.pdl = run.pdl;
  g_info.c_stream = CSTREAM ? 1 : 0;
  g_info.d_tma = run.d_tma;
  g_info.overlap_kb = NSUB == 2 ? run.ovl_kb : 0;
  return TK_OK;
}

// instantiate the pair kernel for the chosen instruction N
template <bool DENSE, bool CSTREAM>
int launch_tc_pair_bni(const tk::TcParams& prm, int bni, cudaStream_t s) {
  // narrow tiles: two K-blocks per ring stage (halves the barrier round trips per operand byte)
  // unless a block predicate needs per-K-block MMA bits
  // (4 K-blocks per stage measured +1 % at 1024^3 and -20 % at 1536^3, where only one stage fits)
  const bool kps2 = !prm.kbits && knob(K_PAIR_KPS, 2) == 2;
  if (bni == 64) return kps2 ? launch_tc_pair<DENSE, CSTREAM, 1, 64, tk::TC2S_CSLOTS, 2>(prm, s)
                             : launch_tc_pair<DENSE, CSTREAM, 1, 64>(prm, s);
  if (bni == 128) return kps2 ? launch_tc_pair<DENSE, CSTREAM, 1, 128, tk::TC2S_CSLOTS, 2>(prm, s)
                              : launch_tc_pair<DENSE, CSTREAM, 1, 128>(prm, s);
  // single wave, 256-wide tiles: a 4-slot C ring holds each warp's whole C block
  if (CSTREAM && prm.num_units <= pair_clusters() && knob(K_PAIR_DEEPC, 1))
    return launch_tc_pair<DENSE, CSTREAM, 1, 256, 4>(prm, s);
  return launch_tc_pair<DENSE, CSTREAM, 1, 256>(prm, s);
}

// On-chip split-K (tk_tc_gemm_ks.cuh): clusters of 4*NT CTAs, two CTA pairs per 256 x 128 tile,
// one K half each, reduced through distributed shared memory; NT = 2 puts two N-adjacent tiles
// in one 8-CTA cluster that multicasts the shared A atoms.  Single wave only: every cluster owns
// its tile(s), so there may not be more of them than co-resident clusters.
template <int BNI, int KPS, int NT>
int ksplit_max_clusters() {
  using PL = tk::KsPlan<BNI, KPS>;
  static int cache[TK_MAX_DEV] = {};
  const int dev = cur_dev();
  int& mc = cache[dev];
  if (!mc) {
    auto kern = tk::tc_gemm_ksplit_kernel<BNI, KPS, NT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM) != cudaSuccess) {
      cudaGetLastError();
      return mc = -1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * NT * (sm_count() / (4 * NT)));
    cfg.blockDim = dim3(tk::TC_THREADS);
    cfg.dynamicSmemBytes = PL::SMEM;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 4 * NT;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc <= 0) {
      cudaGetLastError();
      mc = -1;
    }
    if (knob(K_VERBOSE, 0))
      fprintf(stderr, "tk: k-split kernel (256x%d tiles, %d-CTA clusters) max active clusters %d\n", BNI, 4 * NT, mc);
  }
  return mc;
}
// one K-block per stage: measured faster than two here (1024^3 8.0 vs 8.4 us, 1024^2 x 8192
// 21.3 vs 24.4 us) -- unlike the whole-K narrow tiles, whose stage count is not the limit
int ksplit_kps() { return knob(K_KSPLIT_KPS, 1) == 2 ? 2 : 1; }
// k-split variants: 1 = 256 x 128 tiles, 4-CTA clusters; 2 = the same, two tiles per 8-CTA
// cluster with multicast A; 3 = 256 x 256 tiles, 4-CTA clusters
int ksplit_clusters(int variant) {
  const bool k1 = ksplit_kps() == 1;
  switch (variant) {
    case 1: return k1 ? ksplit_max_clusters<128, 1, 1>() : ksplit_max_clusters<128, 2, 1>();
    case 2: return k1 ? ksplit_max_clusters<128, 1, 2>() : ksplit_max_clusters<128, 2, 2>();
    default: return k1 ? ksplit_max_clusters<256, 1, 1>() : ksplit_max_clusters<256, 2, 1>();
  }
}

template <int BNI, int KPS, int NT>
int launch_tc_ksplit(const tk::TcParams& prm, cudaStream_t s) {
  using PL = tk::KsPlan<BNI, KPS>;
  tk::TcParams run = prm;
  run.pdl = knob(K_PDL, 1) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(4 * NT * run.num_tiles);
  cfg.blockDim = dim3(tk::TC_THREADS);
  cfg.dynamicSmemBytes = PL::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = run.pdl ? 1 : 0;
  TK_CUDA(cudaLaunchKernelEx(&cfg, tk::tc_gemm_ksplit_kernel<BNI, KPS, NT>, run));
  ++g_launches;
  info_kernel("ksplit");
  g_info.tile_m = 256;
  g_info.tile_k = 64 * KPS;
  g_info.tile_n = BNI * NT;
  g_info.mma_n = BNI;
  g_info.nsub = 1;
  g_info.mmas_per_k16 = 1;
  g_info.cluster = 4 * NT;
  g_info.stages = PL::STAGES;
  g_info.stage_bytes = PL::STAGE_BYTES;
  g_info.cring_bytes = PL::CRING_BYTES;
  g_info.smem_bytes = PL::SMEM;
  g_info.tmem_cols = PL::TMEM_COLS;
  g_info.grid_ctas = 4 * NT * run.num_tiles;
  g_info.tiles = g_info.units = run.num_tiles * NT;
  g_info.sk_parts = 2;
  g_info.sk_tiles = run.num_tiles * NT;
  g_info.group_m = run.group_m;
  g_info.pdl = run.pdl;
  g_info.c_stream = 1;
  g_info.d_tma = 1;
  return TK_OK;
}
int launch_tc_ksplit_any(const tk::TcParams& prm, int variant, cudaStream_t s) {
  const bool k1 = ksplit_kps() == 1;
  switch (variant) {
    case 1: return k1 ? launch_tc_ksplit<128, 1, 1>(prm, s) : launch_tc_ksplit<128, 2, 1>(prm, s);
    case 2: return k1 ? launch_tc_ksplit<128, 1, 2>(prm, s) : launch_tc_ksplit<128, 2, 2>(prm, s);
    default: return k1 ? launch_tc_ksplit<256, 1, 1>(prm, s) : launch_tc_ksplit<256, 2, 1>(prm, s);
  }
}

// Use the on-chip split-K kernel?  TK_KSPLIT: 0 never, 1 auto (default), 2 whenever legal.
// Auto compares the per-k-block ingest model of choose_pair_bni: whole-K pair tiles (waves x
// KB x t(bni)) against half-K tiles (KB/2 x t(tile width) + the reduce-scatter).  Returns the
// variant (ksplit_clusters), or 0 for the pair kernel: 256 x 128 tiles when they all fit the
// co-resident 4-CTA clusters, else 256 x 256 tiles when those fit; TK_KSPLIT_NT=2 asks for
// 8-CTA clusters, TK_KSPLIT_BNI=256 for the wide tiles.
int ksplit_choice(int64_t m, int64_t n, int kb_total, int pair_bni, int clusters) {
  const int mode = knob(K_KSPLIT, 1);
  if (mode == 0 || kb_total < 4) return 0;
  // (auto leaves pinned pair-kernel configurations -- TK_TC_KERNEL / TK_PAIR_BNI -- alone)
  if (mode == 1 && (tc_kernel_override() != 0 || knob_set(K_PAIR_BNI))) return 0;
  const int64_t tiles = ((m + 255) / 256) * ((n + 127) / 128);
  const int64_t tiles2 = ((m + 255) / 256) * ((n + 255) / 256);
  const int want_nt = knob(K_KSPLIT_NT, 0), want_bni = knob(K_KSPLIT_BNI, 0);
  int v = 0;
  if (want_nt == 2) {
    const int mc = ksplit_clusters(2);
    if (mc > 0 && tiles2 <= mc) v = 2;
  } else if (want_bni != 256) {
    const int mc = ksplit_clusters(1);
    if (mc > 0 && tiles <= mc) v = 1;
  }
  if (!v && want_nt != 2 && want_bni != 128) {
    const int mc = ksplit_clusters(3);
    if (mc > 0 && tiles2 <= mc) v = 3;
  }
  if (!v || mode == 2) return v;
  auto per_kb = [](int bni) { return std::max(2.0 * bni, (16384.0 + 64.0 * bni) / 60.0); };
  const int64_t ptiles = ((m + 255) / 256) * ((n + pair_bni - 1) / pair_bni);
  const double t_pair = double((ptiles + clusters - 1) / clusters) * kb_total * per_kb(pair_bni);
  const double t_ks = 0.5 * kb_total * per_kb(v == 3 ? 256 : 128) + (v == 3 ? 800.0 : 500.0);
  return t_ks < t_pair ? v : 0;
}

// Split-K of a poorly filled last wave: with T tiles over P clusters, W = T / P full waves and
// R = T % P left over, the R tiles are cut into S K-parts (S <= 4, R*S <= P, >= 64 k-blocks per
// part) when the last wave would otherwise leave at least half of the clusters idle.
struct SplitPlan {
  int first = 0, parts = 1, tiles = 0;
  int64_t ws_bytes = 0;
};
SplitPlan split_plan(int64_t tiles, int clusters, int kb_total, int bnp) {
  SplitPlan sp;
  sp.first = int(tiles);
  if (!knob(K_SPLITK, 1)) return sp;
  const int64_t r = tiles % clusters;
  if (r == 0 || r > clusters / 2) return sp;
  // >= 64 block-K steps per part: below that the partial hand-off costs what the wave gains
  // (measured: 4096^3 -2 %, 4096x4096x16384 +6.5 %, 1536x4096x16384 +13 %)
  const int min_kb = std::max(1, knob(K_SPLITK_MINKB, 64));
  int parts = int(std::min<int64_t>(std::min<int64_t>(4, clusters / r), kb_total / min_kb));
  if (knob_set(K_SPLITK_S)) parts = std::max(1, std::min(parts, knob(K_SPLITK_S, parts)));
  if (parts < 2) return sp;
  sp.first = int(tiles - r);
  sp.parts = parts;
  sp.tiles = int(r);
  sp.ws_bytes = r * (parts - 1) * 2 * 128 * int64_t(bnp) * 4 + 256 + align256(r * 4);
  return sp;
}

int64_t split_ws_bytes(int64_t m, int64_t n, int64_t k, const TkLayout& b) {
  const bool b_mn = b_mn_major(b);
  const int bni = choose_pair_bni(m, n, b_mn, pair_clusters());
  const int64_t tiles = ((m + 255) / 256) * ((n + bni - 1) / bni);
  return split_plan(tiles, pair_clusters(), int((k + 63) / 64), bni).ws_bytes;
}

// Pair-tile width for the real operator: the instruction N (256 / 128 / 64) minimising
// waves x per-tile time (per k-block, per SM: MMA 2*BNI clocks vs operand ingest of
// (16 KB + 64*BNI B) at ~60 B/clock); 64 needs K-major B (64-column MN-major atoms).
int choose_pair_bni(int64_t m, int64_t n, bool b_mn_major, int clusters) {
  if (knob_set(K_PAIR_BNI)) {
    const int v = knob(K_PAIR_BNI, 256);
    if (v == 64 || v == 128 || v == 256) return (v == 64 && b_mn_major) ? 128 : v;
  }
  int best = 256;
  double best_t = 1e300;
  for (int bni : {256, 128, 64}) {
    if (bni == 64 && b_mn_major) continue;
    const int64_t tiles = ((m + 255) / 256) * ((n + bni - 1) / bni);
    const int64_t waves = (tiles + clusters - 1) / clusters;
    const double per_kb = std::max(2.0 * bni, (16384.0 + 64.0 * bni) / 60.0);
    const double t = double(waves) * per_kb;
    if (t < best_t * 0.97) { best_t = t; best = bni; }
  }
  return best;
}

int pair_clusters() {
  const int c = sm_count() / 2;
  return knob_set(K_PAIR_CLUSTERS) ? std::max(1, knob(K_PAIR_CLUSTERS, c)) : c;
}

template <bool DENSE>
int launch_tc_quad(const tk::TcParams& prm, cudaStream_t s) {
  static bool attr[TK_MAX_DEV] = {};
  static int max_clusters_dev[TK_MAX_DEV] = {};
  const int dev = cur_dev();
  if (!attr[dev]) {
    TK_CUDA(cudaFuncSetAttribute(tk::tc_gemm_quad_kernel<DENSE>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, tk::TC2_SMEM));
    attr[dev] = true;
  }
  int& max_clusters = max_clusters_dev[dev];
  if (!max_clusters) {  // 4-CTA clusters do not tile every GPC: ask how many are co-resident
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * (sm_count() / 4));
    cfg.blockDim = dim3(tk::TC_THREADS);
    cfg.dynamicSmemBytes = tk::TC2_SMEM;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 4;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, tk::tc_gemm_quad_kernel<DENSE>, &cfg) != cudaSuccess ||
        max_clusters <= 0) {
      cudaGetLastError();
      max_clusters = sm_count() / 4;
    }
    if (knob(K_VERBOSE, 0)) fprintf(stderr, "tk: quad kernel max active clusters %d\n", max_clusters);
  }
  const int grid = 4 * std::min(prm.num_tiles, max_clusters);
  tk::tc_gemm_quad_kernel<DENSE><<<grid, tk::TC_THREADS, tk::TC2_SMEM, s>>>(prm);
  TK_CUDA(cudaGetLastError());
  ++g_launches;
  info_kernel("quad");
  g_info.tile_m = 512;
  g_info.tile_n = tk::TC2_BN;
  g_info.mma_n = tk::TC2_BN;
  g_info.nsub = 1;
  g_info.mmas_per_k16 = 1;
  g_info.cluster = 4;
  g_info.stages = tk::TC2_STAGES;
  g_info.stage_bytes = tk::TC2_STAGE_BYTES;
  g_info.smem_bytes = tk::TC2_SMEM;
  g_info.tmem_cols = 512;
  g_info.grid_ctas = grid;
  g_info.tiles = g_info.units = prm.num_tiles;
  g_info.sk_parts = 1;
  g_info.group_m = prm.group_m;
  return TK_OK;
}

// TK_TC_KERNEL=quad|pair|single forces the CTA-pair / single-CTA tcgen05 kernel (tests, tuning)
int tc_kernel_override() {
  return knob(K_TC_KERNEL, 0);  // parse_knob: auto 0, single 1, pair 2, stream 3, quad 4, diagstream 5
}

template <int OP>
int launch_tc(const tk::TcParams& prm, bool dense, cudaStream_t s) {
  return dense ? launch_tc_variant<OP, true>(prm, s) : launch_tc_variant<OP, false>(prm, s);
}

// Fold a transform program into relu?(x * mul + add) (complex mul/add for pair streams);
// false when a relu is followed by further ops (then the generic epilogue runs it as is).
bool decode_affine(const TkTransform& t, bool pair, float mul[2], float add[2], int32_t& relu) {
  std::complex<double> m(1.0, 0.0), a(0.0, 0.0);
  relu = 0;
  for (int i = 0; i < t.n; ++i) {
    if (relu) return false;
    const std::complex<double> c(t.re[i], pair ? t.im[i] : 0.0);
    if (t.op[i] == TK_T_SCALE) { m *= c; a *= c; }
    else if (t.op[i] == TK_T_ADD) a += c;
    else if (t.op[i] == TK_T_RELU && !pair) relu = 1;
    else return false;
  }
  mul[0] = float(m.real()); mul[1] = float(m.imag());
  add[0] = float(a.real()); add[1] = float(a.imag());
  return true;
}

// column-major dense element map (one digit per dimension, unit row stride)
bool colmajor_dense(const TkLayout& L, int64_t& ld) {
  if (L.kind != TK_LAYOUT_STRIDED || L.ndigits[0] != 1 || L.ndigits[1] != 1 || L.stride[0][0] != 1)
    return false;
  ld = L.stride[1][0];
  return true;
}

// Gather one half operand (any digit map, both planes of a pair) into a dense column-major
// rows x cols workspace with pack_half_kernel.  Digits chained in both the source and the
// destination (e.g. a GETT index that stays adjacent to its neighbour) are merged first, so a
// permutation of two blocks becomes one wide 2-D transpose instead of many narrow ones.
int launch_pack(const TkLayout& L, const void* src, uint16_t* dst, int64_t rows, int64_t cols, cudaStream_t s) {
  tk::PackDesc pd;
  memset(&pd, 0, sizeof(pd));
  int64_t q = 1;
  for (int d = 0; d < 2; ++d) {
    if (d == 1) q = rows;
    for (int t = 0; t < L.ndigits[d]; ++t) {
      pd.ext[pd.n] = L.ext[d][t];
      pd.ss[pd.n] = L.stride[d][t];
      pd.ds[pd.n] = q;
      q *= L.ext[d][t];
      ++pd.n;
    }
  }
  // merge digit j into i when j continues i in both tensors
  for (bool again = true; again;) {
    again = false;
    for (int i = 0; i < pd.n && !again; ++i)
      for (int j = 0; j < pd.n && !again; ++j)
        if (i != j && pd.ss[j] == pd.ss[i] * pd.ext[i] && pd.ds[j] == pd.ds[i] * pd.ext[i]) {
          pd.ext[i] *= pd.ext[j];
          for (int t = j; t + 1 < pd.n; ++t) {
            pd.ext[t] = pd.ext[t + 1];
            pd.ss[t] = pd.ss[t + 1];
            pd.ds[t] = pd.ds[t + 1];
          }
          --pd.n;
          again = true;
        }
  }
  for (int t = 0; t < pd.n; ++t)
    if (pd.ss[t] < pd.ss[pd.fs] || (pd.ss[t] == pd.ss[pd.fs] && pd.ext[t] > pd.ext[pd.fs])) pd.fs = t;
  pd.fd = 0;  // first row digit: destination stride 1
  if (pd.fd == pd.fs) {
    pd.fd = -1;
    for (int t = 0; t < pd.n; ++t)
      if (t != pd.fs && (pd.fd < 0 || pd.ds[t] < pd.ds[pd.fd])) pd.fd = t;
    if (pd.fd < 0) {  // single digit: pad with a unit digit
      pd.ext[pd.n] = 1;
      pd.ss[pd.n] = pd.ds[pd.n] = 0;
      pd.fd = pd.n++;
    }
  }
  // 16-byte vectors: unit stride along the vector digit, extents and every other stride
  // multiples of 8 elements, 16-byte aligned base (interleaved pairs read scalar-wise)
  auto all8 = [&](const int64_t* st, int skip) {
    for (int t = 0; t < pd.n; ++t)
      if (t != skip && (st[t] % 8) != 0) return false;
    return true;
  };
  const int64_t pl_off = L.pair == TK_PAIR_SPLIT ? L.plane_stride : 0;
  pd.vec_rd = L.pair != TK_PAIR_INTERLEAVED && pd.ss[pd.fs] == 1 && pd.ext[pd.fs] % 8 == 0 &&
              all8(pd.ss, pd.fs) && pl_off % 8 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  pd.wr_x = pd.ds[pd.fs] < pd.ds[pd.fd];
  const int wd = pd.wr_x ? pd.fs : pd.fd;
  pd.vec_wr = pd.ds[wd] == 1 && pd.ext[wd] % 8 == 0 && all8(pd.ds, wd) &&
              (rows * cols) % 8 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  pd.tiles_s = (pd.ext[pd.fs] + 63) / 64;
  pd.tiles_d = (pd.ext[pd.fd] + 63) / 64;
  pd.outer = 1;
  for (int t = 0; t < pd.n; ++t)
    if (t != pd.fs && t != pd.fd) pd.outer *= pd.ext[t];
  const int64_t blocks = pd.tiles_s * pd.tiles_d * pd.outer;
  const unsigned grid = unsigned(std::min<int64_t>(blocks, 64 * sm_count()));
  for (int pl = 0; pl < (L.pair ? 2 : 1); ++pl) {
    tk::pack_half_kernel<<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(src), dst + pl * rows * cols, pd,
                                              L.pair, L.plane_stride, pl);
    TK_CUDA(cudaGetLastError());
    ++g_launches;
  }
  return TK_OK;
}

int run_tc(const TkGemmPlan* p0, const void* a, const void* b, const void* c, void* d, const void* bias,
           const uint8_t* kmask, uint8_t* ws, const Workspace& w, cudaStream_t s) {
  TkGemmPlan rewritten;
  const TkGemmPlan* p = p0;
  // complex embedding: from here on a real plan (M' = 2M, K' = 2K); A^ streams into the
  // kernel's staging ring and the transform warps build A~ on chip
  TkGemmPlan embedded;
  const bool emb = embed_ok(p0);
  if (emb) {
    embed_plan(p0, &embedded);
    p = p0 = &embedded;
  }
  if (permuted_plan(p0, &rewritten)) {
    // A's two M digits swapped (m' = m1 + e1*m0): gathered into a dense M' x K workspace, or
    // (no a_perm workspace) read in place by the pair kernel's 5-D TMA map
    const TkLayout A = swapped_a(p0->a);
    if (w.a_perm >= 0) {
      uint16_t* at = reinterpret_cast<uint16_t*>(ws + w.a_perm);
      int rc0 = launch_pack(A, a, at, p0->m, p0->k, s);
      if (rc0) return rc0;
      a = at;
    } else {
      rewritten.a = A;
    }
    p = &rewritten;
  }
  TkGemmPlan packed;
  if (w.a_pack >= 0 || w.b_pack >= 0) {
    packed = *p;
    int rc;
    if (w.a_pack >= 0) {
      uint16_t* dst = reinterpret_cast<uint16_t*>(ws + w.a_pack);
      if ((rc = launch_pack(p->a, a, dst, p->m, p->k, s))) return rc;
      dense_operand(packed.a, p->m, p->k);
      a = dst;
    }
    if (w.b_pack >= 0) {
      uint16_t* dst = reinterpret_cast<uint16_t*>(ws + w.b_pack);
      if ((rc = launch_pack(p->b, b, dst, p->k, p->n, s))) return rc;
      dense_operand(packed.b, p->k, p->n);
      b = dst;
    }
    p = &packed;
  }
  // ---- load transforms (g2s_a / g2s_b, reference kernel.py:406-418): one pass per transformed
  // operand writes t(x) as an fp16 hi plane (+ lo plane: OP_SPLIT) in the operand's orientation
  TkGemmPlan txp;
  if (w.tx_flags >= 0) {
    txp = *p;
    int32_t* flags = reinterpret_cast<int32_t*>(ws + w.tx_flags);
    TK_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), s));
    auto run_tx = [&](const TkLayout& L, const TkTransform& t, const void*& ptr, TkLayout& out,
                      int64_t rows, int64_t cols, int64_t off, int32_t* flag) -> int {
      int mn;  // 1: dim 0 contiguous
      int64_t pitch;
      tma_operand(L, mn, pitch);
      const int64_t fast = mn ? rows : cols, slow = mn ? cols : rows, vol = rows * cols;
      __half* hi = reinterpret_cast<__half*>(ws + off);
      const unsigned grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((vol / 8 + 255) / 256, 8 * sm_count())));
      if (w.tx_split)
        tk::transform_split_kernel<true><<<grid, 256, 0, s>>>(static_cast<const __half*>(ptr), hi, hi + vol,
                                                              fast, slow, pitch, to_prog(t), flag);
      else
        tk::transform_split_kernel<false><<<grid, 256, 0, s>>>(static_cast<const __half*>(ptr), hi, hi + vol,
                                                               fast, slow, pitch, to_prog(t), flag);
      TK_CUDA(cudaGetLastError());
      ++g_launches;
      dense_operand(out, rows, cols);
      if (!mn) {  // keep the source orientation (K-major A / N-major B stay so)
        out.stride[0][0] = cols;
        out.stride[1][0] = 1;
      }
      out.pair = w.tx_split ? TK_PAIR_SPLIT : TK_PAIR_NONE;
      out.plane_stride = w.tx_split ? vol : 0;
      out.size = vol * (w.tx_split ? 2 : 1);
      ptr = hi;
      return TK_OK;
    };
    int rc;
    if (p->t_a.n && (rc = run_tx(p->a, p->t_a, a, txp.a, p->m, p->k, w.a_tx, flags))) return rc;
    if (p->t_b.n && (rc = run_tx(p->b, p->t_b, b, txp.b, p->k, p->n, w.b_tx, flags + 1))) return rc;
    if (w.tx_split) {  // an untransformed operand: its "lo plane" is never read (flag stays 0)
      if (!p->t_a.n) { txp.a.pair = TK_PAIR_SPLIT; txp.a.plane_stride = 0; }
      if (!p->t_b.n) { txp.b.pair = TK_PAIR_SPLIT; txp.b.plane_stride = 0; }
    }
    txp.t_a.n = txp.t_b.n = 0;
    p = &txp;
  }
  tk::TcParams prm;
  memset(&prm, 0, sizeof(prm));
  // kernel operator: the plan's, or OP_SPLIT for hi + lo transformed operands (a real GEMM)
  const int kop = w.tx_split ? int(tk::OP_SPLIT) : p->op;
  const int op = kop;
  if (w.tx_flags >= 0) prm.split_flags = reinterpret_cast<const int32_t*>(ws + w.tx_flags);
  const int planes = op == TK_OP_REAL ? 1 : 2;
  const int BN = op == TK_OP_REAL ? tk::TcCfg<tk::OP_REAL>::BN : tk::TcCfg<tk::OP_COMPLEX>::BN;
  prm.m = int(p->m);
  prm.n = int(p->n);
  prm.k = int(p->k);
  prm.ab_fmt = p->a.scalar == TK_BF16 ? 1 : 0;
  const int64_t ha = 2;  // bytes per half scalar

  // ---- A operand
  const void* a_pl[2] = {a, nullptr};
  const void* a_plane0 = a;
  const void* b_plane0 = b;
  const void* planes_a[2] = {a, nullptr};
  const void* planes_b[2] = {b, nullptr};
  if (emb) {
    // A^ (2M x K halves, pitch 2*lda) in 128-row x 32-k boxes, unswizzled, for the staging ring
    prm.a_mn = 1;
    prm.a_embed = 1;
    int rc = make_map_2d(&prm.ta[0], a, p->a.scalar, p->m, p->k / 2, p->a.stride[1][0], 128, 32,
                         /*swizzle=*/false);
    if (rc) return rc;
  } else if (p->a.kind == TK_LAYOUT_DIAGONAL) {
    prm.diag_a = 1;
    prm.diag = a;
  } else if (Gather ga; !pack_needed(p->a) ? false : gather_layout(p->a, 0, ga)) {
    // digit-mapped A read in place (5-D TMA map built with the pair kernel's box below)
    prm.a_g = ga.g;
    prm.a_mn = ga.g == 1;
    prm.ga_e0 = int(ga.e0);
    prm.ga_f0 = int(ga.f0);
    if (int rc = make_map_gather(&prm.ta[0], a, p->a.scalar, ga, 128)) return rc;
  } else {
    int mn;
    int64_t pitch;
    tma_operand(p->a, mn, pitch);
    prm.a_mn = mn;
    if (p->a.pair == TK_PAIR_SPLIT) {
      a_pl[1] = static_cast<const uint8_t*>(a) + p->a.plane_stride * ha;
    } else if (p->a.pair == TK_PAIR_INTERLEAVED) {
      const int64_t vol = p->m * p->k;
      uint16_t* p0 = reinterpret_cast<uint16_t*>(ws + w.a_planes);
      tk::deinterleave_kernel<<<std::min<int64_t>((vol + 1023) / 1024, 4 * sm_count()), 256, 0, s>>>(
          static_cast<const uint32_t*>(a), p0, p0 + vol, vol);
      TK_CUDA(cudaGetLastError());
      ++g_launches;
      a_pl[0] = p0;
      a_pl[1] = p0 + vol;
    }
    a_plane0 = a_pl[0];
    planes_a[0] = a_pl[0];
    planes_a[1] = a_pl[1];
    for (int pl = 0; pl < planes; ++pl) {
      int rc = mn ? make_map_2d(&prm.ta[pl], a_pl[pl], p->a.scalar, p->m, p->k, pitch, 64, 64)
                  : make_map_2d(&prm.ta[pl], a_pl[pl], p->a.scalar, p->k, p->m, pitch, 64, 128);
      if (rc) return rc;
    }
  }
  // ---- B operand
  Gather gb;
  if (pack_needed(p->b) && gather_layout(p->b, 1, gb)) {
    // digit-mapped B read in place (the map, whose box depends on the pair tile, is built there)
    prm.b_g = gb.g;
    prm.b_mn = gb.g == 1;
    prm.gb_e0 = int(gb.e0);
    prm.gb_f0 = int(gb.f0);
  } else {
    int mn_k;  // 1: dim0 (K) contiguous -> K-major smem; 0: N contiguous -> MN-major
    int64_t pitch;
    tma_operand(p->b, mn_k, pitch);
    prm.b_mn = mn_k ? 0 : 1;
    const void* b_pl[2] = {b, nullptr};
    if (p->b.pair == TK_PAIR_SPLIT) {
      b_pl[1] = static_cast<const uint8_t*>(b) + p->b.plane_stride * ha;
    } else if (p->b.pair == TK_PAIR_INTERLEAVED) {
      const int64_t vol = p->k * p->n;
      uint16_t* p0 = reinterpret_cast<uint16_t*>(ws + w.b_planes);
      tk::deinterleave_kernel<<<std::min<int64_t>((vol + 1023) / 1024, 4 * sm_count()), 256, 0, s>>>(
          static_cast<const uint32_t*>(b), p0, p0 + vol, vol);
      TK_CUDA(cudaGetLastError());
      ++g_launches;
      b_pl[0] = p0;
      b_pl[1] = p0 + vol;
    }
    b_plane0 = b_pl[0];
    planes_b[0] = b_pl[0];
    planes_b[1] = b_pl[1];
    for (int pl = 0; pl < planes; ++pl) {
      int rc = mn_k ? make_map_2d(&prm.tb[pl], b_pl[pl], p->b.scalar, p->k, p->n, pitch, 64, BN)
                    : make_map_2d(&prm.tb[pl], b_pl[pl], p->b.scalar, p->n, p->k, pitch, 64, 64);
      if (rc) return rc;
    }
  }
  // ---- epilogue
  prm.c_zero = p->c.kind == TK_LAYOUT_ZERO;
  prm.c_zero |= knob(K_DBG_C_ZERO, 0) ? 1 : 0;  // diagnostic builds only: skip C
  prm.c_pair = p->c.pair;
  prm.d_pair = p->d.pair;
  prm.c_ptr = c;
  prm.d_ptr = d;
  prm.c_map = to_map(p->c);
  prm.d_map = to_map(p->d);
  prm.c_plane = p->c.plane_stride;
  prm.d_plane = p->d.plane_stride;
  prm.bias_axis = p->bias_axis;
  prm.bias = static_cast<const float*>(bias);
  prm.t_c = to_prog(p->t_c);
  prm.t_r2s = to_prog(p->t_r2s);
  prm.t_s2g = to_prog(p->t_s2g);
  // ---- schedule
  prm.num_mb = int((p->m + tk::TC_BM - 1) / tk::TC_BM);
  prm.num_nb = int((p->n + BN - 1) / BN);
  prm.num_tiles = prm.num_mb * prm.num_nb;
  prm.kb_total = int((p->k + tk::TC_BK - 1) / tk::TC_BK);
  prm.num_units = prm.num_tiles;  // pair kernel schedule: whole tiles unless split below
  prm.sk_first = prm.num_tiles;
  prm.sk_parts = 1;
  // grouped raster: 16 M-blocks per group keeps the group's A panel L2-resident while B
  // streams (8192^3: DRAM reads 1.18 -> 1.12 GB, +2 %; 4 / 32 are worse)
  prm.group_m = 16;
  prm.group_m = std::max(1, knob(K_GROUP_M, prm.group_m));
  // result-changing diagnostics (TK_DIAG builds only; the table never holds them otherwise)
  prm.dbg_skip_epi = knob(K_DBG_SKIP_EPI, 0) | (knob(K_DBG_NO_LOAD, 0) ? 2 : 0) | (knob(K_DBG_NO_MMA, 0) ? 4 : 0);
  prm.dbg_cta = -1;  // timestamp probes off unless a CTA is selected (tools/ts_probe.py)
  prm.dbg_cta = knob(K_DBG_CTA, -1);
  // serpentine K order on the pair kernel: DRAM reads 1.43 -> 1.29 GB at 8192^3, ~+1 %
  prm.serp = 1;
  prm.serp = knob(K_SERPENTINE, prm.serp);
  prm.pol_ab = 1;  // A/B panels are re-read by neighbouring tiles: keep them in L2
  prm.pol_ab = knob(K_POLICY_AB, prm.pol_ab);
  prm.pol_a = prm.pol_b = prm.pol_ab ? 1 : 0;
  prm.pol_a = knob(K_POL_A, prm.pol_a);
  prm.pol_b = knob(K_POL_B, prm.pol_b);
  prm.pol_c = knob(K_POL_C, 0);  // streamed C loads / D stores: no L2 hint unless tuned
  prm.pol_d = knob(K_POL_D, 0);
  const bool pair = op == TK_OP_COMPLEX || op == TK_OP_DUAL;  // pair-valued epilogue
  // real operator: C/D rows may follow any digit map (GETT outputs whose M indices are not
  // one contiguous run) as long as columns are one strided digit -- the register epilogue
  // then adds a per-thread row offset instead of i (rows stay coalesced inside a run)
  auto rowmapped = [&](const TkLayout& L, int64_t& ld, int32_t& flag) {
    if (colmajor_dense(L, ld)) return true;
    if (pair || L.kind != TK_LAYOUT_STRIDED || L.ndigits[1] != 1) return false;
    ld = L.stride[1][0];
    flag = 1;
    return true;
  };
  bool dense = rowmapped(p->d, prm.ldd, prm.d_rmap) &&
               (p->c.kind == TK_LAYOUT_ZERO || rowmapped(p->c, prm.ldc, prm.c_rmap)) &&
               decode_affine(p->t_c, pair, prm.c_mul, prm.c_add, prm.c_relu) &&
               decode_affine(p->t_r2s, pair, prm.r_mul, prm.r_add, prm.r_relu) &&
               decode_affine(p->t_s2g, pair, prm.s_mul, prm.s_add, prm.s_relu);
  prm.c_ident = p->t_c.n == 0;
  prm.r_ident = p->t_r2s.n == 0;
  prm.s_ident = p->t_s2g.n == 0;
  // HBM-bound shapes (diagonal A, K <= 4 block-K steps): C streamed through TMA by a loader warp
  const int ov = tc_kernel_override();
  // the CTA pair takes every real-operator shape with more than 4 block-K steps and at least
  // 256 rows (narrower pair tiles keep small problems spread over the SMs)
  const bool pair_ok = !prm.diag_a && prm.kb_total > 4 && p->m > 128;
  // streamed-C single-CTA kernel: HBM-bound shapes, and single-wave dense shapes too small
  // for the CTA pair (C prefetched by the loader warp while the mainloop runs)
  const bool single_wave = prm.num_tiles <= sm_count();
  const bool rmapped = prm.c_rmap || prm.d_rmap;
  // diagonal A: an HBM stream, run as one (vectorised) elementwise pass, not on the tensor cores
  if (op == TK_OP_REAL && prm.diag_a && dense && !rmapped && prm.b_mn == 0 &&
      (ov == 0 || ov == 5)) {
    if (knob(K_DIAG_STREAM, 1)) {
      int mnk;
      int64_t ldb;
      tma_operand(p->b, mnk, ldb);
      auto al = [](const void* q, int bytes) { return (reinterpret_cast<uintptr_t>(q) % bytes) == 0; };
      tk::TcParams ps = prm;
      ps.vec_ok = ldb % 4 == 0 && prm.ldd % 4 == 0 && (prm.c_zero || (prm.ldc % 4 == 0 && al(c, 16))) &&
                  al(b, 8) && al(prm.diag, 8) && al(d, 16);
      const int64_t rows4 = (p->m + 3) / 4;
      const dim3 grid(unsigned(std::min<int64_t>((rows4 + 255) / 256, 1024)),
                      unsigned(std::min<int64_t>(p->n, 16384)));
      if (prm.ab_fmt == 0)
        tk::diag_stream_kernel<__half><<<grid, 256, 0, s>>>(ps, static_cast<const __half*>(b), ldb);
      else
        tk::diag_stream_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(ps, static_cast<const __nv_bfloat16*>(b), ldb);
      TK_CUDA(cudaGetLastError());
      ++g_launches;
      info_kernel("diag_stream");
      g_info.grid_ctas = int(grid.x * grid.y);
      return TK_OK;
    }
  }
  const bool pred_tc = w.kbits >= 0;  // block predicate: the CTA-pair kernel evaluates it
  if (op == TK_OP_REAL && dense && !rmapped && !pred_tc && !emb &&
      (ov == 3 || (ov == 0 && (prm.diag_a || prm.kb_total <= 4 || (single_wave && !pair_ok))))) {
    const bool cs = prm.c_zero || ((prm.ldc * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0);
    if (cs) {
      tk::TcParams ps = prm;
      int rc;
      if (!prm.c_zero && (rc = make_map_2d(&ps.tcmap, c, TK_F32, p->m, p->n, prm.ldc, 32, 32))) return rc;
      ps.d_tma = (prm.ldd * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0;
      ps.d_tma = ps.d_tma && knob(K_D_TMA, 1);
      if (ps.d_tma && (rc = make_map_2d(&ps.tdmap, d, TK_F32, p->m, p->n, prm.ldd, 32, 32))) return rc;
      const bool hbm = prm.diag_a || prm.kb_total <= 4;
      return hbm ? launch_tc_variant<tk::OP_REAL, true, 1>(ps, s) : launch_tc_variant<tk::OP_REAL, true, 2>(ps, s);
    }
  }
  if (op == TK_OP_REAL && !prm.diag_a) {
    // CTA pair (256x256 tiles) once there are enough pair tiles to cover the SMs
    if (ov == 4 && !pred_tc && !emb) {
      tk::TcParams pp = prm;
      pp.num_mb = int((p->m + 511) / 512);
      pp.num_nb = int((p->n + tk::TC2_BN - 1) / tk::TC2_BN);
      pp.num_tiles = pp.num_mb * pp.num_nb;
      int mn;
      int64_t pitch;
      int rc;
      tma_operand(p->b, mn, pitch);  // 64x64 B sub-boxes for both majors
      if (mn && (rc = make_map_2d(&pp.tb[0], b_plane0, p->b.scalar, p->k, p->n, pitch, 64, 64))) return rc;
      return dense ? launch_tc_quad<true>(pp, s) : launch_tc_quad<false>(pp, s);
    }
    if (ov == 2 || (ov == 0 && pair_ok) || pred_tc || emb) {
      tk::TcParams pp = prm;
      // 256 x 512 pair tiles (two MMAs share each A tile: 25 % fewer L2->SM bytes per flop, so
      // more flops per joule under the power cap) once K is long enough to amortise their
      // exposed single-accumulator drain and there are >= 4 waves of them; measured:
      // 8192^3 +1 %, 16384^3 +13 % (burst) / +22 % (sustained), 6144^3 -3 % (so not there)
      const int64_t tiles2 = ((p->m + 255) / 256) * ((p->n + 511) / 512);
      int nsub = (p->k >= 8192 && tiles2 >= 4 * int64_t(pair_clusters())) ? 2 : 1;
      if (knob_set(K_PAIR_NSUB)) nsub = knob(K_PAIR_NSUB, 1) == 2 ? 2 : 1;
      if (pred_tc) nsub = 1;
      int mn;
      int64_t pitch;
      int rc;
      tma_operand(p->b, mn, pitch);
      int bni = pred_tc ? pred_bni(p) : (nsub == 2 || emb) ? 256
                      : choose_pair_bni(p->m, p->n, /*b_mn_major=*/prm.b_g ? prm.b_mn != 0 : !mn, pair_clusters());
      // on-chip split-K of single-wave shapes (256 x 128 tiles, K halves on two CTA pairs)
      const int ks_v = (nsub == 1 && !pred_tc && !emb && !prm.a_g && !prm.b_g && dense && !rmapped)
                           ? ksplit_choice(p->m, p->n, pp.kb_total, bni, pair_clusters()) : 0;
      const bool ks = ks_v > 0;
      if (ks) bni = ks_v == 3 ? 256 : 128;
      pp.num_mb = int((p->m + 255) / 256);
      pp.num_nb = int((p->n + bni * nsub - 1) / (bni * nsub));
      pp.num_tiles = pp.num_mb * pp.num_nb;
      pp.num_units = pp.sk_first = pp.num_tiles;
      pp.sk_parts = 1;
      pp.nar_units = 0;
      if (pred_tc) {  // block predicate -> per-tile MMA-step bits, before the GEMM on the stream
        pp.kwords = int(((p->k + 15) / 16 + 31) / 32);
        pp.kbits = reinterpret_cast<const uint32_t*>(ws + w.kbits);
        const int64_t words = int64_t(pp.num_tiles) * pp.kwords;
        tk::expand_kbits_kernel<<<unsigned((words + 255) / 256), 256, 0, s>>>(
            const_cast<uint32_t*>(pp.kbits), pp.num_tiles, pp.kwords, pp.num_mb, pp.num_nb, pp.group_m, bni,
            p->m, p->k, p->block[0], p->block[1], p->block[2], kmask, p->predicate == TK_PRED_DIAGONAL ? 1 : 2);
        TK_CUDA(cudaGetLastError());
        ++g_launches;
      }
      if (nsub == 2) {  // staggered schedule (unit_at in tk_tc_gemm2.cuh): clusters [0, S)
        // split one wide tile into a leading and a trailing half; balanced when T mod P >= S.
        // Opt-in: bitwise equal, but measured 3-6 % slower (8192^3, 16384^3, 8192x16384x8192)
        // -- under the power cap the overlapped drains raise average power and lower clocks.
        const int P = pair_clusters(), S = P / 2;
        if (knob(K_STAGGER, 0) && pp.num_tiles >= 2 * P && !emb) {
          pp.nar_units = S;
          pp.num_units = pp.num_tiles + S;  // (>= P: the grid is all P clusters)
        }
        // drain overlap (nsub2_step in tk_tc_gemm2.cuh): 16 lo-only + 16 hi-only k-block steps
        // at each tile boundary hide the half-accumulator drains under MMAs
        pp.ovl_kb = (pp.nar_units || emb) ? 0 : std::max(0, std::min(knob(K_NSUB2_OVERLAP, 16), pp.kb_total / 4));
      }
      if (nsub == 1 && dense && w.splitk >= 0 && !knob_set(K_PAIR_GRID) && !ks) {
        const SplitPlan sp = split_plan(pp.num_tiles, pair_clusters(), pp.kb_total, bni);
        if (sp.parts > 1 && sp.ws_bytes <= split_ws_bytes(p->m, p->n, p->k, p->b)) {
          pp.sk_first = sp.first;
          pp.sk_parts = sp.parts;
          pp.num_units = sp.first + sp.tiles * sp.parts;
          pp.sk_ws = reinterpret_cast<float*>(ws + w.splitk);
          pp.sk_flags = reinterpret_cast<int32_t*>(ws + w.splitk + (sp.ws_bytes - align256(sp.tiles * 4)));
          TK_CUDA(cudaMemsetAsync(pp.sk_flags, 0, sp.tiles * 4, s));
        }
      }
      // per-CTA halves: A box 128 rows / B box bni/2 columns
      pp.mn3d = 0;
      const bool use3d = knob(K_MN3D, 1) != 0;
      if (!emb && !prm.a_g) {  // (embedding: ta[0] is the A^ staging map; gathered A: the 5-D map)
        tma_operand(p->a, mn, pitch);
        // MN-major A (M % 64 == 0 so atoms never straddle the M edge): one 3-D box per stage
        if (mn && use3d && p->m % 64 == 0) {
          if ((rc = make_map_mn3d(&pp.ta[0], a_plane0, p->a.scalar, p->m, p->k, pitch, 2))) return rc;
          pp.mn3d |= 1;
        }
        if (!mn && (rc = make_map_2d(&pp.ta[0], a_plane0, p->a.scalar, p->k, p->m, pitch, 64, 128))) return rc;
      }
      if (prm.b_g) {  // digit-mapped B: 5-D map, this CTA's bni/2 columns per box
        Gather gbx;
        gather_layout(p->b, 1, gbx);
        if ((rc = make_map_gather(&pp.tb[0], b_plane0, p->b.scalar, gbx, uint32_t(bni / 2)))) return rc;
      } else if (tma_operand(p->b, mn, pitch), mn) {
        if ((rc = make_map_2d(&pp.tb[0], b_plane0, p->b.scalar, p->k, p->n, pitch, 64, bni / 2))) return rc;
      } else if (use3d && p->n % 64 == 0) {
        if ((rc = make_map_mn3d(&pp.tb[0], b_plane0, p->b.scalar, p->n, p->k, pitch, bni / 128))) return rc;
        pp.mn3d |= 2;
      }
      if (knob(K_VERBOSE, 0)) fprintf(stderr, "tk: pair kernel bni %d nsub %d tiles %d\n", bni, nsub, pp.num_tiles);
      // streamed C/D epilogue (TMA ring + bulk stores) when C/D are TMA-compatible
      bool cs = dense && !rmapped && (prm.c_zero || ((prm.ldc * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0)) &&
                (prm.ldd * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0;
      cs = cs && knob(K_PAIR_CSTREAM, 1);
      if (cs) {
        if (!prm.c_zero && (rc = make_map_2d(&pp.tcmap, c, TK_F32, p->m, p->n, prm.ldc, 32, 32))) return rc;
        if ((rc = make_map_2d(&pp.tdmap, d, TK_F32, p->m, p->n, prm.ldd, 32, 32))) return rc;
        pp.d_tma = 1;
        pp.npeer = 0;
        if (g_npeer > 0 && g_npeer <= 7) {
          for (int q = 0; q < g_npeer; ++q)
            if ((rc = make_map_2d(&pp.tdpeer[q], g_peer_d[q], TK_F32, p->m, p->n, prm.ldd, 32, 32))) return rc;
          pp.npeer = g_npeer;
          g_peer_mode = 1;
        }
        if (!pp.npeer) pp.d_tma = knob(K_PAIR_DTMA, 1);
        pp.c_pf_kb = knob(K_C_PF, 0);  // L2 prefetch of the next drain's C: measured neutral-to-negative
        pp.c_pf_spread = knob(K_C_PF_SPREAD, 0);
        pp.c_pf_kb = std::min(pp.c_pf_kb, pp.kb_total);
        // split-K partials as TMA boxes through the C ring (written from the ring by the K-parts,
        // loaded into it by the last part's C loader) instead of per-thread stores and loads
        pp.sk_tma = 0;
        if (pp.sk_parts > 1 && !prm.c_zero && pp.d_tma) {
          if (knob(K_SK_TMA, 1)) {
            const int64_t cols = int64_t(pp.num_units - pp.sk_first) / pp.sk_parts * (pp.sk_parts - 1) * 2 * bni;
            if ((rc = make_map_2d(&pp.tskmap, pp.sk_ws, TK_F32, 128, cols, 128, 32, 32))) return rc;
            pp.sk_tma = 1;
          }
        }
        if (emb)
          return nsub == 2 ? launch_tc_pair<true, true, 2, 256, tk::TC2S_CSLOTS, 1, true>(pp, s)
                           : launch_tc_pair<true, true, 1, 256, tk::TC2S_CSLOTS, 1, true>(pp, s);
        if (nsub == 2) {
          const int csl = knob(K_NSUB2_CSL, 2);  // C-ring slots per warp (tuning)
          if (csl == 3) return launch_tc_pair<true, true, 2, 256, 3>(pp, s);
          if (csl == 4) return launch_tc_pair<true, true, 2, 256, 4>(pp, s);
          return launch_tc_pair<true, true, 2>(pp, s);
        }
        if (ks && !pp.npeer) {
          tk::TcParams kp = pp;
          if (ks_v == 2) {  // tile pairs; A in 64-row atoms (each CTA multicasts one)
            kp.num_nb = int((p->n + 255) / 256);
            kp.num_tiles = kp.num_mb * kp.num_nb;
            tma_operand(p->a, mn, pitch);
            if ((rc = mn ? make_map_2d(&kp.ta[0], a_plane0, p->a.scalar, p->m, p->k, pitch, 64, 64)
                         : make_map_2d(&kp.ta[0], a_plane0, p->a.scalar, p->k, p->m, pitch, 64, 64)))
              return rc;
          }
          return launch_tc_ksplit_any(kp, ks_v, s);
        }
        return launch_tc_pair_bni<true, true>(pp, bni, s);
      }
      if (emb)  // (C / D not TMA-aligned: register epilogue)
        return nsub == 2 ? launch_tc_pair<true, false, 2, 256, tk::TC2S_CSLOTS, 1, true>(pp, s)
                         : launch_tc_pair<true, false, 1, 256, tk::TC2S_CSLOTS, 1, true>(pp, s);
      if (nsub == 2) return dense ? launch_tc_pair<true, false, 2>(pp, s) : launch_tc_pair<false, false, 2>(pp, s);
      return dense ? launch_tc_pair_bni<true, false>(pp, bni, s) : launch_tc_pair_bni<false, false>(pp, bni, s);
    }
  }
  if (op != TK_OP_REAL) {
    // complex / dual on a CTA pair once there are enough 256x128 pair tiles
    const int64_t pair_tiles = ((p->m + 255) / 256) * ((p->n + tk::TC2C_BN - 1) / tk::TC2C_BN);
    if (ov == 2 || (ov == 0 && pair_tiles >= sm_count() / 2 && prm.kb_total > 4)) {
      tk::TcParams pp = prm;
      // two A planes per tile: 8 M-blocks per group keep the panel L2-resident (16: -4 %)
      pp.group_m = std::max(1, knob(K_GROUP_M, 8));
      // 256-wide pair tiles (N=256 MMAs: 96 instead of 128 B/clk of shared-memory operand
      // reads) when there are >= 4 waves of them to amortise the single accumulator's drain
      const int64_t tiles256 = ((p->m + 255) / 256) * ((p->n + 255) / 256);
      int bn = tiles256 >= 4 * int64_t(pair_clusters()) ? 256 : 128;
      if (knob_set(K_PAIROPS_BN)) bn = knob(K_PAIROPS_BN, 128) == 256 ? 256 : 128;
      pp.num_mb = int((p->m + 255) / 256);
      pp.num_nb = int((p->n + bn - 1) / bn);
      pp.num_tiles = pp.num_mb * pp.num_nb;
      int mn;
      int64_t pitch;
      int rc;
      tma_operand(p->a, mn, pitch);
      pp.mn3d = 0;
      if (p->a.pair == TK_PAIR_INTERLEAVED) pitch = mn ? p->m : p->k;  // de-interleaved planes
      if (mn && p->m % 64 == 0) {
        for (int pl = 0; pl < 2; ++pl)
          if ((rc = make_map_mn3d(&pp.ta[pl], planes_a[pl], p->a.scalar, p->m, p->k, pitch, 2))) return rc;
        pp.mn3d |= 1;
      }
      tma_operand(p->b, mn, pitch);
      if (p->b.pair == TK_PAIR_INTERLEAVED) pitch = mn ? p->k : p->n;
      if (mn)  // K-major B: this CTA's bn/2-column half per box
        for (int pl = 0; pl < 2; ++pl)
          if ((rc = make_map_2d(&pp.tb[pl], planes_b[pl], p->b.scalar, p->k, p->n, pitch, 64, bn / 2))) return rc;
      static bool attr_dev[TK_MAX_DEV][3][2][2] = {};  // [device][complex, dual, split][dense][bn 256]
      auto& attr = attr_dev[cur_dev()];
      const int oi = op == TK_OP_COMPLEX ? 0 : op == TK_OP_DUAL ? 1 : 2;
      const int smem_bytes = bn == 256 ? tk::Tc2cPlan<256>::SMEM : tk::Tc2cPlan<128>::SMEM;
      auto launch = [&](auto kern) -> int {
        if (!attr[oi][dense][bn == 256]) {
          TK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
          attr[oi][dense][bn == 256] = true;
        }
        const int grid = 2 * std::min(pp.num_tiles, sm_count() / 2);
        tk::TcParams run = pp;
        run.pdl = knob(K_PDL, 1) ? 1 : 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(tk::TC_THREADS);
        cfg.dynamicSmemBytes = smem_bytes;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = run.pdl ? 1 : 0;
        TK_CUDA(cudaLaunchKernelEx(&cfg, kern, run));
        ++g_launches;
        info_kernel("pair_ops");
        g_info.tile_m = 256;
        g_info.tile_n = bn;
        g_info.mma_n = bn;
        g_info.nsub = 1;
        g_info.mmas_per_k16 = op == TK_OP_COMPLEX ? 4 : 3;  // dual / split: 3 (split: at most)
        g_info.cluster = 2;
        g_info.stages = bn == 256 ? tk::Tc2cPlan<256>::STAGES : tk::Tc2cPlan<128>::STAGES;
        g_info.stage_bytes = bn == 256 ? tk::Tc2cPlan<256>::STAGE_BYTES : tk::Tc2cPlan<128>::STAGE_BYTES;
        g_info.smem_bytes = smem_bytes;
        g_info.tmem_cols = 512;
        g_info.grid_ctas = grid;
        g_info.tiles = g_info.units = run.num_tiles;
        g_info.sk_parts = 1;
        g_info.serpentine = run.serp;
        g_info.group_m = run.group_m;
        g_info.pdl = run.pdl;
        return TK_OK;
      };
      if (bn == 256) {
        if (op == TK_OP_COMPLEX)
          return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_COMPLEX, true, 256>)
                       : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_COMPLEX, false, 256>);
        if (op == tk::OP_SPLIT)
          return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_SPLIT, true, 256>)
                       : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_SPLIT, false, 256>);
        return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_DUAL, true, 256>)
                     : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_DUAL, false, 256>);
      }
      if (op == TK_OP_COMPLEX)
        return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_COMPLEX, true>)
                     : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_COMPLEX, false>);
      if (op == tk::OP_SPLIT)
        return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_SPLIT, true>)
                     : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_SPLIT, false>);
      return dense ? launch(tk::tc_gemm_pair_ops_kernel<tk::OP_DUAL, true>)
                   : launch(tk::tc_gemm_pair_ops_kernel<tk::OP_DUAL, false>);
    }
  }
  switch (op) {
    case TK_OP_REAL: return launch_tc<tk::OP_REAL>(prm, dense, s);
    case TK_OP_COMPLEX: return launch_tc<tk::OP_COMPLEX>(prm, dense, s);
    case tk::OP_SPLIT: return launch_tc<tk::OP_SPLIT>(prm, dense, s);
    default: return launch_tc<tk::OP_DUAL>(prm, dense, s);
  }
}

tk::SimtLayout to_simt(const TkLayout& L, const void* ptr) {
  tk::SimtLayout s{};
  s.kind = L.kind;
  s.pair = L.pair;
  s.scalar = L.scalar;
  s.map = to_map(L);
  s.plane = L.plane_stride;
  s.ptr = ptr;
  return s;
}

template <int OP, typename T, typename Acc>
int launch_simt(const tk::SimtParams& sp, cudaStream_t s) {
  if (OP == tk::OP_REAL && sp.predicate == 0 && knob(K_SIMT_TILED, 1)) {  // 128 x 128 smem tiles
    const dim3 grid(unsigned((sp.m + tk::ST_BM - 1) / tk::ST_BM), unsigned((sp.n + tk::ST_BN - 1) / tk::ST_BN));
    if (grid.y <= 65535) {
      const int want = sizeof(T) == 4 ? tk::S_F32 : tk::S_F64;
      auto plain = [&](const tk::SimtLayout& L) {
        return L.kind == tk::L_STRIDED && L.pair == 0 && L.scalar == want && L.map.nd[0] == 1 && L.map.nd[1] == 1;
      };
      if (plain(sp.a) && plain(sp.b) && sp.t_a.n == 0 && sp.t_b.n == 0)
        tk::simt_tiled_kernel<T, Acc, true><<<grid, tk::ST_THREADS, 0, s>>>(sp);
      else
        tk::simt_tiled_kernel<T, Acc><<<grid, tk::ST_THREADS, 0, s>>>(sp);
      TK_CUDA(cudaGetLastError());
      ++g_launches;
      info_kernel("simt");
      g_info.tile_m = tk::ST_BM;
      g_info.tile_n = tk::ST_BN;
      g_info.tile_k = sizeof(T) == 8 ? tk::ST_BK / 2 : tk::ST_BK;
      g_info.grid_ctas = int(grid.x * grid.y);
      return TK_OK;
    }
  }
  const int64_t total = sp.m * sp.n;
  const int threads = 128;
  tk::simt_gemm_kernel<OP, T, Acc><<<int((total + threads - 1) / threads), threads, 0, s>>>(sp);
  TK_CUDA(cudaGetLastError());
  ++g_launches;
  info_kernel("simt");
  g_info.tile_m = g_info.tile_n = 1;
  g_info.grid_ctas = int((total + threads - 1) / threads);
  return TK_OK;
}

template <int OP>
int dispatch_simt(const TkGemmPlan* p, const tk::SimtParams& sp, cudaStream_t s) {
  const bool t64 = p->a.scalar == TK_F64 || p->b.scalar == TK_F64;
  if (t64) return launch_simt<OP, double, double>(sp, s);
  if (p->compute == TK_F64) return launch_simt<OP, float, double>(sp, s);
  return launch_simt<OP, float, float>(sp, s);
}

int run_simt(const TkGemmPlan* p, const void* a, const void* b, const void* c, void* d, const void* bias,
             const uint8_t* kmask, cudaStream_t s) {
  tk::SimtParams sp;
  memset(&sp, 0, sizeof(sp));
  sp.m = p->m;
  sp.n = p->n;
  sp.k = p->k;
  sp.op_k = p->op_k;
  sp.bm = p->block[0];
  sp.bn = p->block[1];
  sp.bk = p->block[2];
  sp.predicate = p->predicate;
  sp.bias_axis = p->bias_axis;
  sp.bias_scalar = p->bias_scalar;
  sp.kmask = kmask;
  sp.bias = bias;
  sp.a = to_simt(p->a, a);
  sp.b = to_simt(p->b, b);
  sp.c = to_simt(p->c, c);
  sp.d = to_simt(p->d, d);
  sp.t_a = to_prog(p->t_a);
  sp.t_b = to_prog(p->t_b);
  sp.t_c = to_prog(p->t_c);
  sp.t_r2s = to_prog(p->t_r2s);
  sp.t_s2g = to_prog(p->t_s2g);
  switch (p->op) {
    case TK_OP_REAL: return dispatch_simt<tk::OP_REAL>(p, sp, s);
    case TK_OP_COMPLEX: return dispatch_simt<tk::OP_COMPLEX>(p, sp, s);
    default: return dispatch_simt<tk::OP_DUAL>(p, sp, s);
  }
}

bool aligned16(const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; }

}  // namespace

// ====================================================================== C ABI
namespace {
// Canonical digit maps: unit digits dropped, and adjacent digits whose strides chain
// (stride[t+1] == stride[t] * ext[t]) merged into one -- the same element map
// (d0*s0 + d1*s0*e0 == (d0 + e0*d1)*s0), but many GETT operands become plain strided
// matrices the TMA reads directly instead of needing a gather pass.
void normalize_layout(TkLayout& L) {
  if (L.kind != TK_LAYOUT_STRIDED) return;
  for (int d = 0; d < 2; ++d) {
    int64_t e[TK_MAX_DIGITS], st[TK_MAX_DIGITS];
    int n = 0;
    for (int t = 0; t < L.ndigits[d]; ++t) {
      if (L.ext[d][t] == 1 && L.ndigits[d] > 1) continue;
      if (n > 0 && L.stride[d][t] == st[n - 1] * e[n - 1]) {
        e[n - 1] *= L.ext[d][t];
        continue;
      }
      e[n] = L.ext[d][t];
      st[n] = L.stride[d][t];
      ++n;
    }
    if (n == 0) { e[0] = 1; st[0] = 1; n = 1; }
    for (int t = 0; t < TK_MAX_DIGITS; ++t) {
      L.ext[d][t] = t < n ? e[t] : 0;
      L.stride[d][t] = t < n ? st[t] : 0;
    }
    L.ndigits[d] = n;
  }
}

const TkGemmPlan* normalized(const TkGemmPlan* p, TkGemmPlan& out) {
  out = *p;
  normalize_layout(out.a);
  normalize_layout(out.b);
  normalize_layout(out.c);
  normalize_layout(out.d);
  return &out;
}
}  // namespace

extern "C" {

int tk_abi_version(void) { return TK_ABI_VERSION; }

const char* tk_last_error(void) { return g_err.c_str(); }

int tk_last_launch_count(void) { return g_launches; }

namespace {
__global__ void clock_probe_kernel(unsigned long long ns, unsigned long long* out) {
  unsigned long long t0, t1, c0 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < ns);
  out[0] = clock64() - c0;
  out[1] = t1 - t0;
}
unsigned long long* g_probe_buf = nullptr;
}  // namespace

// tuning aids (not part of the ABI header).  tk_debug_clock_probe launches one 32-thread CTA
// that sleeps for `us` microseconds on `stream` and records SM clock ticks vs globaltimer;
// tk_debug_clock_probe_mhz() reads the result (after a synchronize): the SM clock seen while
// other work (e.g. a library GEMM) ran concurrently.
int tk_debug_clock_probe(double us, void* stream) {
  if (!g_probe_buf && cudaMalloc(&g_probe_buf, 16) != cudaSuccess) return 2;
  clock_probe_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>((unsigned long long)(us * 1e3), g_probe_buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
double tk_debug_clock_probe_mhz(void) {
  unsigned long long v[2] = {0, 0};
  if (!g_probe_buf || cudaMemcpy(v, g_probe_buf, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess || !v[1])
    return 0.0;
  return double(v[0]) * 1e3 / double(v[1]);
}

// tuning aid: the 8 globaltimer stamps of CTA 0 of the last pair-kernel launch, relative to entry (us)
int tk_debug_pair_ts(double* out) {
  unsigned long long v[16];
  if (cudaMemcpyFromSymbol(v, tk::g_dbg_ts, sizeof(v)) != cudaSuccess) return 2;
  for (int i = 0; i < 16; ++i) out[i] = v[i] >= v[0] ? double(v[i] - v[0]) * 1e-3 : -1.0;
  // (k-split kernel: slot 15 = the previous launch's exit, signed, relative to this entry)
  if (v[15]) out[15] = double(int64_t(v[15] - v[0])) * 1e-3;
  return 0;
}

// tuning aid (not part of the ABI header): effective SM MHz of CTA 0 over the last
// pair-kernel launch (clock64 ticks / globaltimer ns), after a device synchronize.
double tk_debug_pair_mhz(void) {
  unsigned long long v[2] = {0, 0};
  if (cudaMemcpyFromSymbol(v, tk::g_dbg_clk, sizeof(v)) != cudaSuccess || !v[1]) return 0.0;
  return double(v[0]) * 1e3 / double(v[1]);
}

int tk_plan_lane(const TkGemmPlan* plan0) {
  if (check_plan(plan0)) return -1;
  TkGemmPlan norm;
  const TkGemmPlan* plan = normalized(plan0, norm);
  std::string why;
  int lane = choose_lane(plan, &why);
  if (lane < 0) {
    fail(TK_ERR_CONFIG, "tcgen05 lane requested but not applicable: %s", why.c_str());
    return -1;
  }
  return lane;
}

int64_t tk_workspace_bytes(const TkGemmPlan* plan0) {
  if (check_plan(plan0)) return -1;
  TkGemmPlan norm;
  const TkGemmPlan* plan = normalized(plan0, norm);
  int lane = choose_lane(plan);
  if (lane < 0) return -1;
  return plan_workspace(plan, lane).total;
}

int tk_gemm(const TkGemmPlan* plan0, const void* a, const void* b, const void* c, void* d, const void* bias,
            const uint8_t* kmask, void* workspace, int64_t workspace_bytes, void* stream) {
  g_err.clear();
  g_launches = 0;
  info_reset();
  int rc = check_plan(plan0);
  if (rc) return rc;
  TkGemmPlan norm;
  const TkGemmPlan* plan = normalized(plan0, norm);
  std::string why;
  int lane = choose_lane(plan, &why);
  if (lane < 0) return fail(TK_ERR_CONFIG, "tcgen05 lane requested but not applicable: %s", why.c_str());
  if (plan->bias_axis && !bias) return fail(TK_ERR_CONFIG, "bias epilogue without a bias vector");
  if (plan->predicate == TK_PRED_MASK && !kmask) return fail(TK_ERR_CONFIG, "mask predicate without a mask");
  if (lane == TK_LANE_TCGEN05) {
    const bool ok = (plan->a.kind != TK_LAYOUT_STRIDED || aligned16(a)) && aligned16(b);
    if (!ok) {
      if (plan->lane == TK_LANE_TCGEN05) return fail(TK_ERR_CONFIG, "operands not 16-byte aligned");
      lane = TK_LANE_SIMT;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (lane == TK_LANE_TCGEN05) {
    Workspace w = plan_workspace(plan, lane);
    if (w.total > 0 && (!workspace || workspace_bytes < w.total))
      return fail(TK_ERR_CONFIG, "workspace of %lld bytes required", (long long)w.total);
    rc = run_tc(plan, a, b, c, d, bias, kmask, static_cast<uint8_t*>(workspace), w, s);
    g_info.workspace_bytes = w.total;
  } else {
    rc = run_simt(plan, a, b, c, d, bias, kmask, s);
  }
  g_info.lane = lane;
  g_info.op = plan->op;
  g_info.launches = g_launches;
  return rc;
}

int tk_last_plan_info(TkPlanInfo* out) {
  if (!out) return fail(TK_ERR_CONFIG, "null output");
  *out = g_info;
  return TK_OK;
}

int tk_tune_set(const char* name, const char* value) {
  if (!name) return fail(TK_ERR_CONFIG, "null knob name");
  for (int i = 0; i < K_ENABLED; ++i)
    if (!strcmp(name, kKnobNames[i])) {
      int v;
      if (int rc = parse_knob(i, value, &v)) return rc;
      knob_table().v[i].store(v, std::memory_order_relaxed);
      return TK_OK;
    }
  return fail(TK_ERR_CONFIG, "unknown tuning knob '%s'%s", name,
              strncmp(name, "TK_DBG_", 7) ? "" : " (diagnostic knobs need a -DTK_DIAG build)");
}

int tk_tune_reset(void) {
  knobs_from_env(knob_table());
  return TK_OK;
}

int tk_tune_get(const char* name) {
  for (int i = 0; name && i < K_ENABLED; ++i)
    if (!strcmp(name, kKnobNames[i])) return knob_table().v[i].load(std::memory_order_relaxed);
  return KNOB_UNSET;
}

int tk_gemm_peers(const TkGemmPlan* plan, const void* a, const void* b, const void* c, void* d,
                  const void* bias, const uint8_t* kmask, void* workspace, int64_t workspace_bytes,
                  void* stream, void* const* peer_d, int npeers) {
  if (npeers < 0 || npeers > 7 || (npeers && !peer_d))
    return fail(TK_ERR_CONFIG, "between 0 and 7 peer D slabs expected");
  if (npeers && (plan->op != TK_OP_REAL || plan->d.kind != TK_LAYOUT_STRIDED || plan->d.pair ||
                 plan->d.ndigits[0] != 1 || plan->d.ndigits[1] != 1 || plan->d.stride[0][0] != 1 ||
                 plan->d.stride[1][0] != plan->m))
    return fail(TK_ERR_CONFIG, "a fused all-gather needs a real, dense column-major D slab");
  g_peer_d = peer_d;
  g_npeer = npeers;
  g_peer_mode = 0;
  int rc = tk_gemm(plan, a, b, c, d, bias, kmask, workspace, workspace_bytes, stream);
  g_peer_d = nullptr;
  g_npeer = 0;
  if (rc || !npeers || g_peer_mode == 1) return rc;
  // the chosen kernel has no streamed epilogue: deliver the slab with peer copies instead
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int q = 0; q < npeers; ++q)
    TK_CUDA(cudaMemcpyAsync(peer_d[q], d, size_t(plan->m) * size_t(plan->n) * 4, cudaMemcpyDefault, s));
  g_peer_mode = 2;
  return TK_OK;
}

int tk_last_peer_mode(void) { return g_peer_mode; }

// CUDA IPC for the peer buffers of a fused all-gather (one process per GPU): the 64-byte handle
// of a device allocation, and mapping / unmapping a peer's allocation into this process.
// The handle names the whole allocation (a caching allocator hands out sub-ranges of larger
// cudaMalloc blocks), so the byte offset of dev_ptr inside it is returned too.
int tk_ipc_handle(void* dev_ptr, void* handle_out64, int64_t* offset_out) {
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, dev_ptr) != cudaSuccess) {
    const char* m = cudaGetErrorString(cudaGetLastError());
    return fail(TK_ERR_CUDA, "cudaIpcGetMemHandle: %s", m);
  }
  using GetAttr = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static GetAttr get_attr = nullptr;
  if (!get_attr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(TK_ERR_CUDA, "cuPointerGetAttribute unavailable");
    get_attr = reinterpret_cast<GetAttr>(fn);
  }
  CUdeviceptr start = 0;
  if (get_attr(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, reinterpret_cast<CUdeviceptr>(dev_ptr)) !=
      CUDA_SUCCESS)
    return fail(TK_ERR_CUDA, "allocation range of an IPC buffer");
  memcpy(handle_out64, &h, sizeof(h));
  *offset_out = int64_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - start);
  return TK_OK;
}
int tk_ipc_open(const void* handle64, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  if (cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    const char* m = cudaGetErrorString(cudaGetLastError());
    return fail(TK_ERR_CUDA, "cudaIpcOpenMemHandle: %s", m);
  }
  return TK_OK;
}
int tk_ipc_close(void* dev_ptr) {
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? TK_OK : fail(TK_ERR_CUDA, "cudaIpcCloseMemHandle");
}

}  // extern "C"

// ====================================================================== gemm_ex_raw
namespace {

void set_dense(TkLayout& L, int scalar, int pair, int64_t rows, int64_t cols, bool row_major) {
  memset(&L, 0, sizeof(L));
  L.kind = TK_LAYOUT_STRIDED;
  L.pair = pair;
  L.scalar = scalar;
  L.ndigits[0] = L.ndigits[1] = 1;
  L.ext[0][0] = rows;
  L.ext[1][0] = cols;
  L.stride[0][0] = row_major ? cols : 1;
  L.stride[1][0] = row_major ? 1 : rows;
  L.plane_stride = pair == TK_PAIR_SPLIT ? rows * cols : 0;
  L.size = rows * cols * (pair ? 2 : 1);
}

void set_scale(TkTransform& t, double re, double im) {
  memset(&t, 0, sizeof(t));
  t.n = 1;
  t.op[0] = TK_T_SCALE;
  t.re[0] = re;
  t.im[0] = im;
}

struct TagInfo {
  int ab_scalar, c_scalar, op, compute;
};

bool tag_info(int tag, TagInfo& ti) {
  switch (tag) {
    case TK_TAG_F32: ti = {TK_F32, TK_F32, TK_OP_REAL, TK_F32}; return true;
    case TK_TAG_F64: ti = {TK_F64, TK_F64, TK_OP_REAL, TK_F64}; return true;
    case TK_TAG_C64: ti = {TK_F32, TK_F32, TK_OP_COMPLEX, TK_F32}; return true;
    case TK_TAG_C128: ti = {TK_F64, TK_F64, TK_OP_COMPLEX, TK_F64}; return true;
    case TK_TAG_DUAL32: ti = {TK_F32, TK_F32, TK_OP_DUAL, TK_F32}; return true;
    case TK_TAG_DUAL64: ti = {TK_F64, TK_F64, TK_OP_DUAL, TK_F64}; return true;
    case TK_TAG_F16F32: ti = {TK_F16, TK_F32, TK_OP_REAL, TK_F32}; return true;
    case TK_TAG_BF16F32: ti = {TK_BF16, TK_F32, TK_OP_REAL, TK_F32}; return true;
    case TK_TAG_C32C64: ti = {TK_F16, TK_F32, TK_OP_COMPLEX, TK_F32}; return true;
    case TK_TAG_CBF16C64: ti = {TK_BF16, TK_F32, TK_OP_COMPLEX, TK_F32}; return true;
    case TK_TAG_DUAL16F32: ti = {TK_F16, TK_F32, TK_OP_DUAL, TK_F32}; return true;
    case TK_TAG_DUALBF16F32: ti = {TK_BF16, TK_F32, TK_OP_DUAL, TK_F32}; return true;
    default: return false;
  }
}

// The reference's block-tile heuristic (components.py:196-240) at the default operator
// shape (8,8,8) and 64 KiB budget: gemm_ex_raw reports status 1 exactly when it finds none.
bool reference_block_tile(int64_t m, int64_t n, int64_t k, int64_t shared_scalar_bytes, int pair,
                          int64_t block[3]) {
  const int64_t op = 8, budget = 64 * 1024;
  if (k % op) return false;
  int64_t best_area = -1;
  bool best_square = false;
  for (int64_t bn = 1; bn <= n; bn <<= 1) {
    if (bn % op || n % bn) continue;
    for (int64_t bm : {bn, 2 * bn}) {
      if (bm > m || bm % op || m % bm) continue;
      const int64_t foot = (bm * op + op * bn) * (pair ? 2 : 1) * shared_scalar_bytes;
      if (foot > budget) continue;
      const bool square = bm == bn;
      if (bm * bn > best_area || (bm * bn == best_area && square && !best_square)) {
        best_area = bm * bn;
        best_square = square;
        block[0] = bm;
        block[1] = bn;
        block[2] = op;
      }
    }
  }
  return best_area > 0;
}

int build_ex_plan(TkGemmPlan& p, int tag, int ta, int tb, long long m, long long n, long long k,
                  double are, double aim, double bre, double bim) {
  TagInfo ti;
  if (!tag_info(tag, ti)) return fail(TK_ERR_CONFIG, "unknown type tag %d", tag);
  if (m < 1 || n < 1 || k < 1) return fail(TK_ERR_CONFIG, "extents must be >= 1");
  memset(&p, 0, sizeof(p));
  p.abi_version = TK_ABI_VERSION;
  p.op = ti.op;
  p.compute = ti.compute;
  p.lane = TK_LANE_AUTO;
  p.m = m;
  p.n = n;
  p.k = k;
  p.op_k = 8;
  const int pair = ti.op == TK_OP_REAL ? TK_PAIR_NONE : TK_PAIR_INTERLEAVED;
  if (!reference_block_tile(m, n, k, scalar_bytes(ti.ab_scalar), pair, p.block))
    return fail(TK_ERR_CONFIG, "no feasible block tile (reference heuristic) for (%lld, %lld, %lld)",
                m, n, k);
  const bool cplx = ti.op == TK_OP_COMPLEX;
  if (!cplx) { aim = 0.0; bim = 0.0; }
  const std::complex<double> alpha(are, aim), beta(bre, bim);
  set_dense(p.c, ti.c_scalar, pair, m, n, false);
  p.d = p.c;
  if (alpha == 0.0) {
    memset(&p.a, 0, sizeof(p.a));
    p.a.kind = TK_LAYOUT_ZERO;
    p.a.scalar = ti.ab_scalar;
    p.b = p.a;
    set_scale(p.t_c, beta.real(), beta.imag());
  } else {
    set_dense(p.a, ti.ab_scalar, pair, m, k, ta != 0);
    set_dense(p.b, ti.ab_scalar, pair, k, n, tb != 0);
    const std::complex<double> q = beta / alpha;
    if (q != 1.0) set_scale(p.t_c, q.real(), q.imag());
    if (alpha != 1.0) set_scale(p.t_r2s, alpha.real(), alpha.imag());
  }
  return TK_OK;
}

int64_t elems_of(const TkLayout& L) { return L.kind == TK_LAYOUT_ZERO ? 0 : L.size; }

}  // namespace

extern "C" int tk_gemm_ex_raw_async(int tag, int ta, int tb, long long m, long long n, long long k,
                                    double are, double aim, const void* a, const void* b, double bre,
                                    double bim, void* c, void* stream) {
  g_err.clear();
  TkGemmPlan p;
  int rc = build_ex_plan(p, tag, ta, tb, m, n, k, are, aim, bre, bim);
  if (rc) return rc;
  int lane = choose_lane(&p);
  Workspace w = plan_workspace(&p, lane);
  void* ws = nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (w.total) TK_CUDA(cudaMallocAsync(&ws, w.total, s));
  rc = tk_gemm(&p, a, b, c, c, nullptr, nullptr, ws, w.total, stream);
  if (ws) cudaFreeAsync(ws, s);
  return rc;
}

namespace {

struct ExStreams {
  cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
  cudaMemPool_t pool = nullptr;  // private: staging memory stays cached between calls
  bool ok = false;
};

// Per device: three streams and a private stream-ordered pool for the staging buffers (the
// device's default pool, which the host application may use too, is left untouched).
ExStreams& ex_streams() {
  static ExStreams st_dev[TK_MAX_DEV];
  static std::once_flag once[TK_MAX_DEV];
  const int dev = cur_dev();
  ExStreams& st = st_dev[dev];
  std::call_once(once[dev], [&st, dev] {
    st.ok = cudaStreamCreateWithFlags(&st.in, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&st.comp, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&st.out, cudaStreamNonBlocking) == cudaSuccess;
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (st.ok && cudaMemPoolCreate(&st.pool, &props) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(st.pool, cudaMemPoolAttrReleaseThreshold, &thr);
    } else {
      st.ok = false;
    }
  });
  return st;
}

// Host-buffer gemm_ex: H2D of column slabs of B and C, the slab GEMMs and the D2H of finished
// slabs run on three streams, so both PCIe directions and the tensor cores overlap.  Column
// slabs of column-major B (not transposed) and C are contiguous sub-buffers.
int ex_pipelined(int tag, int ta, long long m, long long n, long long k, double are, double aim,
                 const void* a, const void* b, double bre, double bim, void* c, int64_t esz_ab,
                 int64_t esz_c, int pairf) {
  ExStreams& st = ex_streams();
  if (!st.ok) return fail(TK_ERR_CUDA, "stream creation failed");
  const int64_t sa = m * k * esz_ab * pairf, sb = k * n * esz_ab * pairf, sc = m * n * esz_c * pairf;
  void *da = nullptr, *db = nullptr, *dc = nullptr;
  TK_CUDA(cudaMallocFromPoolAsync(&da, sa, st.pool, st.in));
  TK_CUDA(cudaMallocFromPoolAsync(&db, sb, st.pool, st.in));
  TK_CUDA(cudaMallocFromPoolAsync(&dc, sc, st.pool, st.in));
  TK_CUDA(cudaMemcpyAsync(da, a, sa, cudaMemcpyHostToDevice, st.in));
  const int max_slabs = std::max(1, knob(K_EX_SLABS, 8));
  int slabs = int(std::max<long long>(1, std::min<long long>(max_slabs, n / 1024)));
  const long long w = ((n / slabs + 255) / 256) * 256;
  slabs = int((n + w - 1) / w);
  int rc = TK_OK;
  int launches = 0;
  std::vector<cudaEvent_t> ev_in(slabs), ev_done(slabs);
  for (int i = 0; i < slabs; ++i) {
    cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming);
  }
  for (int i = 0; i < slabs && rc == TK_OK; ++i) {
    const long long j0 = i * w, cols = std::min<long long>(w, n - j0);
    const int64_t ob = j0 * k * esz_ab * pairf, oc = j0 * m * esz_c * pairf;
    const int64_t nb = cols * k * esz_ab * pairf, nc = cols * m * esz_c * pairf;
    if (cudaMemcpyAsync(static_cast<char*>(db) + ob, static_cast<const char*>(b) + ob, nb,
                        cudaMemcpyHostToDevice, st.in) != cudaSuccess ||
        cudaMemcpyAsync(static_cast<char*>(dc) + oc, static_cast<char*>(c) + oc, nc,
                        cudaMemcpyHostToDevice, st.in) != cudaSuccess) {
      rc = fail(TK_ERR_CUDA, "host-to-device copy failed");
      break;
    }
    cudaEventRecord(ev_in[i], st.in);
    cudaStreamWaitEvent(st.comp, ev_in[i], 0);
    rc = tk_gemm_ex_raw_async(tag, ta, 0, m, cols, k, are, aim, da, static_cast<char*>(db) + ob,
                              bre, bim, static_cast<char*>(dc) + oc, st.comp);
    launches += g_launches;
    cudaEventRecord(ev_done[i], st.comp);
    cudaStreamWaitEvent(st.out, ev_done[i], 0);
    if (rc == TK_OK && cudaMemcpyAsync(static_cast<char*>(c) + oc, static_cast<char*>(dc) + oc, nc,
                                       cudaMemcpyDeviceToHost, st.out) != cudaSuccess)
      rc = fail(TK_ERR_CUDA, "device-to-host copy failed");
  }
  cudaStreamSynchronize(st.in);
  cudaStreamSynchronize(st.comp);
  cudaStreamSynchronize(st.out);
  cudaFreeAsync(da, st.out);
  cudaFreeAsync(db, st.out);
  cudaFreeAsync(dc, st.out);
  cudaStreamSynchronize(st.out);
  for (int i = 0; i < slabs; ++i) {
    cudaEventDestroy(ev_in[i]);
    cudaEventDestroy(ev_done[i]);
  }
  g_launches = launches;
  g_info.launches = launches;
  if (rc == TK_OK) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TK_ERR_CUDA, "pipelined gemm_ex: %s", cudaGetErrorString(e));
  }
  return rc;
}

}  // namespace

extern "C" int tk_gemm_ex_raw(int tag, int ta, int tb, long long m, long long n, long long k,
                              double are, double aim, void* a, void* b, double bre, double bim, void* c) {
  g_err.clear();
  TkGemmPlan p;
  int rc = build_ex_plan(p, tag, ta, tb, m, n, k, are, aim, bre, bim);
  if (rc) return rc;
  // host pointers (the reference's numpy buffers) are staged through device memory
  auto on_device = [](const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
  };
  const int64_t sa = elems_of(p.a) * scalar_bytes(p.a.scalar);
  const int64_t sb = elems_of(p.b) * scalar_bytes(p.b.scalar);
  const int64_t sc = p.c.size * scalar_bytes(p.c.scalar);
  const bool dev = on_device(c) && (sa == 0 || on_device(a)) && (sb == 0 || on_device(b));
  if (dev) {
    rc = tk_gemm_ex_raw_async(tag, ta, tb, m, n, k, are, aim, a, b, bre, bim, c, nullptr);
    if (rc) return rc;
    TK_CUDA(cudaDeviceSynchronize());
    return TK_OK;
  }
  // large problems: overlap the host<->device traffic with the slab GEMMs
  if (!tb && p.a.kind != TK_LAYOUT_ZERO && m * n * k >= (1ll << 30)) {
    TagInfo ti;
    tag_info(tag, ti);
    return ex_pipelined(tag, ta, m, n, k, are, aim, a, b, bre, bim, c, scalar_bytes(ti.ab_scalar),
                        scalar_bytes(ti.c_scalar), ti.op == TK_OP_REAL ? 1 : 2);
  }
  void *da = nullptr, *db = nullptr, *dc = nullptr;
  auto cleanup = [&] {
    if (da) cudaFree(da);
    if (db) cudaFree(db);
    if (dc) cudaFree(dc);
  };
  if ((sa && cudaMalloc(&da, sa) != cudaSuccess) || (sb && cudaMalloc(&db, sb) != cudaSuccess) ||
      cudaMalloc(&dc, sc) != cudaSuccess) {
    cleanup();
    return fail(TK_ERR_CUDA, "device allocation failed");
  }
  if ((sa && cudaMemcpy(da, a, sa, cudaMemcpyHostToDevice) != cudaSuccess) ||
      (sb && cudaMemcpy(db, b, sb, cudaMemcpyHostToDevice) != cudaSuccess) ||
      cudaMemcpy(dc, c, sc, cudaMemcpyHostToDevice) != cudaSuccess) {
    cleanup();
    return fail(TK_ERR_CUDA, "host-to-device copy failed");
  }
  rc = tk_gemm_ex_raw_async(tag, ta, tb, m, n, k, are, aim, da, db, bre, bim, dc, nullptr);
  if (rc == TK_OK && cudaMemcpy(c, dc, sc, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(TK_ERR_CUDA, "device-to-host copy failed");
  cleanup();
  return rc;
}
