// C ABI of the FlashInside engine: workspace planning and the width sweeps
// that sequence the sm_100a kernels (fi_kernels.cuh, fi_gemm.cuh).
//
// Forward  (inside_flash, inside.py:274-340, batched over sentences):
//   K1 W = exp([L|R]) once per call            -> k_prep_weights
//   width 1: x†, E1 = exp(unary - x†)          -> k_prep_width1
//            [a1|b1] = x† + log(E1 W_NP^T)     -> tcgen05 GEMM, EPI_FWD
//   w = 2..l: split contraction -> o, x†, E    -> k_split_fwd (cluster/DSMEM)
//            [aw|bw] = x† + log(Ew W_NN^T)     -> tcgen05 GEMM, EPI_FWD
// Backward (inside_backward + _projection_backward, inside.py:375-447):
//   seed lq at each top span, d_root           -> k_seed_bwd
//   m = l-1..1: G_m (gather split backward)    -> k_gather_bwd
//            lq_m = log|G_m W| - x†            -> tcgen05 GEMM, EPI_DGRAD
//            (m = 1: dunary = E1 * (G_1 W_NP)) -> tcgen05 GEMM, EPI_DUNARY
//   dW = G^T E over all spans, d{L,R} = W*dW   -> tcgen05 GEMM, EPI_WGRAD
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <type_traits>
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cudaTypedefs.h>

#include "../../include/flashinside.h"
#ifndef FI_FP32_CHUNK
#define FI_FP32_CHUNK 16  // fp32 mode: K-iterations per round-to-nearest accumulation chunk
                          // (8 / 16 / 32 measured: worst config-2 error 2.0e-6 / 2.5e-6 /
                          // 1.1e-5 of the 1e-4 bound, 54.3 / 52.9 / 52.6 ms at config 3)
#endif
#include "fi_gemm.cuh"
#include "fi_kernels.cuh"
#include "fi_decode.cuh"
#include "fi_param.cuh"

using namespace fi;

namespace {

thread_local char g_err[512] = "";
// Process-wide count of kernels this library enqueued (autograd runs the
// backward on its own thread, so nothing here is thread-local).
std::atomic<long long> g_launches{0};
// > 0 while this thread times GEMM tile candidates (see tuned_choice): those
// launches are neither counted nor recorded by the profiler.
thread_local int g_tuning = 0;

// ---------------------------------------------------------------- profiler
// Optional per-kernel-class CUDA-event timing (bench.py roofline): when
// enabled, every launch is bracketed by two events on its own stream.
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};
std::atomic<bool> g_prof_on{false};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {  // caller holds g_prof_mu
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

thread_local int g_prof_class = -1;  // >= 0: class of this thread's GEMM launches
struct ProfClassScope {  // the parameterisation's GEMMs count as FI_PROF_PARAM
  int saved;
  explicit ProfClassScope(int c) : saved(g_prof_class) { g_prof_class = c; }
  ~ProfClassScope() { g_prof_class = saved; }
};
struct ProfScope {
  cudaStream_t st;
  ProfRec rec;
  bool on;
  ProfScope(int cls, cudaStream_t s) : st(s), on(g_prof_on.load() && g_tuning == 0) {
    if (!on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    rec.cls = cls;
    rec.a = prof_event();
    rec.b = prof_event();
    cudaEventRecord(rec.a, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(rec.b, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(rec);
  }
};

int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define FI_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(FI_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                               \
  } while (0)

#define FI_TRY(expr)           \
  do {                         \
    int r_ = (expr);           \
    if (r_ != FI_OK) return r_; \
  } while (0)

// split-K partial tiles: ksplit x split tiles <= the CTA slots, so at most
// one (256 x 256 or 128 x 256) fp32 tile per slot
constexpr long long kKPartFloats = 160LL * 256 * 256;
constexpr int kKPartSems = 256;  // split-K tile counters (in-kernel reduction), after the partials

// ------------------------------------------------------------------ layout
struct Decomp {
  int clusters, threads, v, cols_per_cta, stages;
};

struct Plan {
  int N, P, B, l, Np, Pp, esz;
  Decomp dsplit, dgather;
  long long rows;
  size_t wnn, wnp, e1, eall, gall, a, b, o, lq, lqs, x, top, topz, wsum, flag, lens, kpart, total;
  // element offsets of the lo planes of the GEMM operands (fp32 mode only)
  long long wnn_lo, wnp_lo, e1_lo, eall_lo, gall_lo;
  bool store_o, tf32, split, half_chart;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// An exact column decomposition of a Np-wide row: c CTAs x `threads`
// consumers (a multiple of 32, <= 256) x v in {1, 2, 4} groups of 4 columns,
// c * threads * 4 * v == Np.  Returns false if this c admits none.
bool decomp_for(int Np, int c, Decomp* d) {
  if (c < 1 || c > 8 || Np % c) return false;
  const int cols = Np / c;
  for (int v : {1, 2, 4}) {
    if (cols % (4 * v)) continue;
    const int threads = cols / (4 * v);
    if (threads % 32 == 0 && threads <= 256) {
      d->clusters = c;
      d->threads = threads;
      d->v = v;
      d->cols_per_cta = cols;
      return true;
    }
  }
  return false;
}

// The valid decomposition whose CTA count is closest to `c` (the FI_*
// override first, if valid).
int make_decomp(int Np, int c, const char* env_c, const char* env_s, int stages, Decomp* d) {
  const int want = env_int(env_c, 0);
  bool ok = want > 0 && decomp_for(Np, want, d);
  for (int delta = 0; !ok && delta < 8; ++delta)
    ok = decomp_for(Np, c + delta, d) || decomp_for(Np, c - delta, d);
  if (!ok)
    return set_err(FI_ERR_UNSUPPORTED, "no column decomposition for Np=%d (C near %d)", Np, c);
  const int st = env_int(env_s, stages);
  d->stages = st < 2 ? 2 : (st > 16 ? 16 : st);
  return FI_OK;
}

int make_plan(const fi_shape* s, Plan* p) {
  if (!s) return set_err(FI_ERR_ARG, "null shape");
  if (s->n_nt < 1 || s->n_pt < 1 || s->batch < 1)
    return set_err(FI_ERR_ARG, "n_nt, n_pt and batch must be >= 1 (got %d, %d, %d)", s->n_nt,
                   s->n_pt, s->batch);
  if (s->max_len < 2)
    return set_err(FI_ERR_ARG, "need sentences of length >= 2, got max_len %d", s->max_len);
  if (s->gemm_dtype != FI_GEMM_BF16 && s->gemm_dtype != FI_GEMM_TF32 &&
      s->gemm_dtype != FI_GEMM_FP32)
    return set_err(FI_ERR_ARG, "unknown gemm_dtype %d", s->gemm_dtype);
  if (s->chart_dtype != FI_CHART_AUTO && s->chart_dtype != FI_CHART_F32 &&
      s->chart_dtype != FI_CHART_F16)
    return set_err(FI_ERR_ARG, "unknown chart_dtype %d", s->chart_dtype);
  if (s->n_nt > 16384 || s->n_pt > 16384)
    return set_err(FI_ERR_UNSUPPORTED, "symbol counts above 16384 are not supported");
  if (s->max_len > 1024)  // per-span term tables live in shared memory
    return set_err(FI_ERR_UNSUPPORTED, "sentences longer than 1024 tokens are not supported");
  p->N = s->n_nt;
  p->P = s->n_pt;
  p->B = s->batch;
  p->l = s->max_len;
  // padded symbol count: multiple of 256 / 512 / 1024 / 2048 so the bandwidth
  // kernels always find an exact column decomposition (make_decomp)
  p->Np = static_cast<int>(
      align_up(p->N, p->N <= 1024 ? 256 : p->N <= 4096 ? 512 : p->N <= 8192 ? 1024 : 2048));
  p->Pp = static_cast<int>(align_up(p->P, 256));
  p->tf32 = s->gemm_dtype == FI_GEMM_TF32;
  p->split = s->gemm_dtype == FI_GEMM_FP32;
  p->esz = p->tf32 ? 4 : 2;
  p->half_chart = s->chart_dtype == FI_CHART_F16 ||
                  (s->chart_dtype == FI_CHART_AUTO && s->gemm_dtype != FI_GEMM_FP32);
  const int planes = p->split ? 2 : 1;
  p->store_o = s->store_chart != 0;
  // column decomposition of a span row for the bandwidth kernels: C CTAs
  // (a thread-block cluster for the split contraction's row max), each
  // `threads` consumer threads x V 4-column groups.  C is sized by the bytes
  // a CTA streams per term: ~8 KB per a/b row chunk in the split contraction,
  // ~4 KB per sibling chunk in the gather (measured on B200 at N = 4096:
  // fp32 chart split C = 2 / gather C = 4, fp16 chart split C = 1 / gather
  // C = 2).  FI_CLUSTER / FI_GCLUSTER / FI_STAGES / FI_GSTAGES override.
  const int cesz = p->half_chart ? 2 : 4;
  auto pick_c = [&](int bytes) {  // target CTAs per row; make_decomp finds the nearest exact one
    int c = p->Np * cesz / bytes;
    return c < 1 ? 1 : (c > 8 ? 8 : c);
  };
  FI_TRY(make_decomp(p->Np, pick_c(8192), "FI_CLUSTER", "FI_STAGES", 4, &p->dsplit));
  FI_TRY(make_decomp(p->Np, pick_c(4096), "FI_GCLUSTER", "FI_GSTAGES", 6, &p->dgather));
  p->rows = rowbase(p->l, p->B, p->l) + p->B;
  const long long rows = p->rows;
  if (static_cast<long long>(p->B) * p->l > 65535 || rows > (1LL << 30))
    return set_err(FI_ERR_UNSUPPORTED, "batch x length above 65535 spans per width");
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 1024);
    return o;
  };
  auto plane = [&](long long elems, long long* lo) {
    *lo = p->split ? elems : 0;
    return take(static_cast<size_t>(elems) * p->esz * planes);
  };
  p->wnn = plane(2LL * p->Np * p->Np, &p->wnn_lo);
  p->wnp = plane(2LL * p->Np * p->Pp, &p->wnp_lo);
  p->e1 = plane(1LL * p->B * p->l * p->Pp, &p->e1_lo);
  p->eall = plane(rows * p->Np, &p->eall_lo);
  p->gall = plane(2LL * rows * p->Np, &p->gall_lo);
  const size_t ab_esz = p->half_chart ? 2 : 4;
  p->a = take(ab_esz * rows * p->Np);
  p->b = take(ab_esz * rows * p->Np);
  p->o = p->store_o ? take(4ull * rows * p->Np) : static_cast<size_t>(-1);
  p->lq = take(ab_esz * rows * p->Np);  // fp16 |q| in the half chart, else fp32 LQ^
  p->lqs = p->half_chart ? take(4ull * rows * (p->Np / 32)) : static_cast<size_t>(-1);
  p->x = take(8ull * rows);  // fp64 row shifts
  p->top = take(4ull * p->B * p->Np);
  p->topz = take(4ull * p->B);
  p->wsum = take(16);
  p->flag = take(256);
  p->lens = take(4ull * p->B);  // sanitized lengths (k_check_lengths)
  // split-K partial tiles + counters, one region per concurrent stream (dual sweep)
  p->kpart = take(2 * (4ull * kKPartFloats + 4ull * kKPartSems));
  p->total = off;
  return FI_OK;
}

template <typename P>
P* at(void* ws, size_t off) {
  return reinterpret_cast<P*>(static_cast<uint8_t*>(ws) + off);
}

// ------------------------------------------------------------ TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int load_encode() {
  if (g_encode) return FI_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return set_err(FI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return FI_OK;
}

struct Operand {
  const void* ptr;
  long long inner;  // contiguous extent (elements)
  long long outer;  // rows
  long long ld;     // row stride (elements)
  bool mn_major;
  long long lo;     // element offset of the lo plane (fp32 mode), else 0
};

template <typename T>
int encode(CUtensorMap* m, const Operand& op, int box_inner, int box_outer) {
  // tf32 MN-major tiles must land in the 32B-atom swizzle the UMMA expects
  const CUtensorMapSwizzle sw = (sizeof(T) == 4 && op.mn_major)
                                    ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                    : CU_TENSOR_MAP_SWIZZLE_128B;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(op.inner), static_cast<cuuint64_t>(op.outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(op.ld * sizeof(T))};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapDataType dt =
      sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(op.ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(FI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld",
                   static_cast<int>(r), op.inner, op.outer);
  return FI_OK;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev);
  return cached[dev] > 0 ? cached[dev] : 148;
}

// Hot-path launches go through cudaLaunchKernelEx with programmatic
// dependent launch (PDL): a kernel may be scheduled while its predecessor
// is still finishing, runs its prologue (barrier init, TMEM alloc, tensor
// map prefetch), then blocks in griddepcontrol.wait until the predecessor's
// writes are visible.  Persistent kernels trigger their dependents right
// after their own wait (so the chain stays transitive); grid-stride ones
// never trigger early.  FI_PDL=0 disables the attribute.
bool use_pdl() {
  static const int v = env_int("FI_PDL", 1);
  return v != 0;
}

template <typename K, typename... Args>
int launch_ex(K kern, int cluster, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (use_pdl()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  FI_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
  if (g_tuning == 0) ++g_launches;
  return FI_OK;
}

template <typename K, typename... Args>
int launch_cluster(K kern, int cluster, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                   Args... args) {
  return launch_ex(kern, cluster, grid, block, smem, st, args...);
}

// Split-K partial tiles of the GEMMs enqueued by this thread (a workspace
// region set by the ABI entry points; thread-local, so calls on different
// threads / streams never share it).  Null: no split-K.
struct KPartScratch {
  float* ptr = nullptr;
  size_t floats = 0;
  int* sem = nullptr;  // kKPartSems zeroed tile counters (each split-K launch leaves them zero)
  float* region[2] = {nullptr, nullptr};  // per-stream regions (dual sweep: one per half)
};
thread_local KPartScratch g_kpart;
constexpr long long kKPartRegion = kKPartFloats + kKPartSems;  // floats per region
struct KPartScope {
  KPartScratch saved;
  int err = FI_OK;
  // p: `regions` x (kKPartFloats partial floats + the counters, zeroed here)
  KPartScope(float* p, cudaStream_t st, int regions) : saved(g_kpart) {
    for (int k = 0; k < 2; ++k) g_kpart.region[k] = p + (k < regions ? k : 0) * kKPartRegion;
    select(0);
    for (int k = 0; k < regions && err == FI_OK; ++k)
      if (cudaMemsetAsync(p + k * kKPartRegion + kKPartFloats, 0, sizeof(int) * kKPartSems, st) !=
          cudaSuccess)
        err = set_err(FI_ERR_CUDA, "split-K counter reset: %s",
                      cudaGetErrorString(cudaGetLastError()));
  }
  static void select(int k) {
    g_kpart.ptr = g_kpart.region[k];
    g_kpart.floats = static_cast<size_t>(kKPartFloats);
    g_kpart.sem = reinterpret_cast<int*>(g_kpart.region[k] + kKPartFloats);
  }
  ~KPartScope() { g_kpart = saved; }
};
struct KPartSelect {  // launches of one half of a dual sweep use that half's region
  float* saved;
  explicit KPartSelect(int k) : saved(g_kpart.ptr) { KPartScope::select(k); }
  ~KPartSelect() {
    g_kpart.ptr = saved;
    g_kpart.sem = reinterpret_cast<int*>(saved + kKPartFloats);
  }
};

// GEMM smem ring depth for launches enqueued by this thread: 0 = the deepest
// ring that fits (one CTA per SM); the dual-stream sweep (see forward_impl)
// caps it so a bandwidth-kernel CTA can share each SM with a GEMM CTA.
thread_local int g_gemm_stages = 0;
constexpr int kGemmSmemMax = 227 * 1024;  // opt-in dynamic shared memory per CTA
constexpr int kGemmStagesMax = 12;        // barrier block (256 B) holds 2 x 12 + 4 mbarriers

// Co-resident clusters of `cl` CTAs of `kern` (one per SM-group), cached per
// kernel and device: the persistent grid of a multicast-cluster GEMM.
template <typename K>
int max_clusters(K kern, int cl, int threads, size_t smem) {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (cache[dev & 63]) return cache[dev & 63];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * 64);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cl;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = num_sms() / cl;
  }
  cache[dev & 63] = n;
  return n;
}

// TR: A and B are the kernel's operands (A = the weight table, B = the chart
// rows), M / N the kernel's dims; `a_row0` is then the chart rows' offset.
template <typename T, int BN, bool AMN, bool BMN, int EPI, bool SPLIT, int CHUNK, bool PAIR,
          bool MC = false, bool TR = false>
int launch_gemm(const Operand& A, const Operand& B, int M, int N, int K, int a_row0,
                const GemmEpi& ep, cudaStream_t st, int bn, int ksplit, int tail,
                bool streamk = false) {
  using Cf = GemmCfg<T, BN>;
  constexpr int NCTA = PAIR ? 2 : 1;
  constexpr int CL = MC ? 4 : NCTA;
  CUtensorMap ta, tb, ta2, tb2;
  // MC: each CTA loads (and multicasts) half of its 128 A rows
  const int abi = AMN ? Cf::ATOM : Cf::BK, abo = AMN ? Cf::BK : (MC ? Cf::BM / 2 : Cf::BM);
  const int bbi = BMN ? Cf::ATOM : Cf::BK, bbo = BMN ? Cf::BK : bn / NCTA;
  FI_TRY(encode<T>(&ta, A, abi, abo));
  FI_TRY(encode<T>(&tb, B, bbi, bbo));
  if (SPLIT) {
    Operand a2 = A, b2 = B;
    a2.ptr = static_cast<const T*>(A.ptr) + A.lo;
    b2.ptr = static_cast<const T*>(B.ptr) + B.lo;
    FI_TRY(encode<T>(&ta2, a2, abi, abo));
    FI_TRY(encode<T>(&tb2, b2, bbi, bbo));
  } else {
    ta2 = ta;
    tb2 = tb;
  }
  GemmShape sh;
  sh.M = M;
  sh.N = N;
  sh.K = K;
  sh.a_row0 = TR ? 0 : a_row0;
  sh.b_row0 = TR ? a_row0 : 0;
  sh.bn = bn;
  // ring depth: as many (A + this CTA's share of B) stages as fit in 227 KB
  // (a pair CTA stages half the N tile, so pairs run deeper rings)
  sh.b_stage = bn / NCTA * 128 * (SPLIT ? 2 : 1);  // SPLIT: hi and lo tiles per stage
  const int stage_bytes = Cf::A_BYTES * (SPLIT ? 2 : 1) + sh.b_stage;
  constexpr int kTransBytes = TR ? 4 * 32 * 33 * 4 : 0;  // epilogue transpose tiles
  int max_stages = (kGemmSmemMax - 1024 - 256 - kTransBytes) / stage_bytes;
  max_stages = max_stages > kGemmStagesMax ? kGemmStagesMax : max_stages;
  static const int env_stages = env_int("FI_GEMM_STAGES", 0);  // A/B experiments
  const int cap = g_gemm_stages > 1 ? g_gemm_stages : env_stages;
  sh.stages = (cap > 1 && cap < max_stages) ? cap : max_stages;
  const size_t smem_bytes = static_cast<size_t>(sh.stages) * stage_bytes + 1024 + 256 + kTransBytes;

  sh.num_m = (M + Cf::BM * NCTA - 1) / (Cf::BM * NCTA);
  sh.num_n = (N + bn - 1) / bn;
  sh.num_k = (K + Cf::BK - 1) / Cf::BK;
  const int tiles = sh.num_m * (MC ? (sh.num_n + 1) / 2 : sh.num_n);  // MC: cluster tiles
  if (MC) ksplit = 1;  // split-K partials are indexed per pair tile
  sh.ksplit = 1;
  sh.part = nullptr;
  sh.sem = nullptr;
  sh.tile_begin = 0;
  sh.tile_end = 0;
  sh.sk = 0;
  sh.sk_first = 0;

  // persistent: one CTA (pair, cluster) per SM (pair, group of 4 SMs)
  const int nslots = num_sms() / NCTA;
  if (streamk && !MC && !TR && CHUNK == 0 && g_kpart.ptr && g_kpart.sem && tail > 0 &&
      tail == tiles % nslots && tail <= kKPartSems &&
      sh.stages * stage_bytes >= Cf::BM * (bn + 4) * 4 &&  // the finalizer's staging tile
      static_cast<size_t>(2) * nslots * Cf::BM * NCTA * bn <= g_kpart.floats) {
    // one launch: whole waves, then the last `tail` tiles' K iterations in
    // equal runs over every slot, reduced in-kernel (see GemmShape::sk)
    sh.sk = nslots;
    sh.sk_first = tiles - tail;
    sh.part = g_kpart.ptr;
    sh.sem = g_kpart.sem;
  }
  if (streamk) {
    tail = 0;
    ksplit = 1;
  }
  const long long tsplit = tail > 0 ? tail : tiles;
  if (ksplit > 1 && g_kpart.ptr &&
      static_cast<size_t>(ksplit) * tsplit * Cf::BM * NCTA * bn <= g_kpart.floats) {
    sh.ksplit = ksplit;
    sh.part = g_kpart.ptr;
    // FI_GEMM_INKERNEL_RED=1: every unit of a split tile is resident at once
    // (units <= slots), so the tile's CTAs can reduce the partials themselves
    // (no fixup launch).  Their wait needs every unit of the launch to get an
    // SM; split launches of two streams running at once could each hold SMs
    // the other needs, so it is opt-in (measured: no faster than the fixup
    // kernel at config 3, 14.35-14.48 vs 14.41-14.64 ms).
    static const int inkernel = env_int("FI_GEMM_INKERNEL_RED", 0);
    if (inkernel && !TR && CHUNK == 0 && g_kpart.sem && tsplit <= kKPartSems) sh.sem = g_kpart.sem;
  } else {
    tail = 0;  // no split-K available: whole tiles only
  }
  auto kern = k_gemm<T, BN, AMN, BMN, EPI, SPLIT, CHUNK, PAIR, MC, TR>;
  static bool attr_done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    FI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kGemmSmemMax));
    attr_done[dev & 63] = true;
  }
  // persistent: one CTA (pair, cluster) per SM (pair, group of 4 SMs)
  const int slots = MC ? max_clusters(kern, CL, gemm_threads<CHUNK>(), smem_bytes)
                       : num_sms() / NCTA;
  static const int log_slots = env_int("FI_GEMM_LOG", 0);
  if (log_slots && MC) fprintf(stderr, "[fi gemm] multicast clusters: %d co-resident\n", slots);
  if (log_slots && PAIR && !MC)
    fprintf(stderr, "[fi gemm] pair clusters: %d co-resident (smem %zu)\n",
            max_clusters(kern, 2, gemm_threads<CHUNK>(), smem_bytes), smem_bytes);
  ProfScope prof(g_prof_class >= 0 ? g_prof_class
                 : EPI == EPI_FWD || EPI == EPI_FWD_H ? FI_PROF_GEMM_FWD
                 : EPI == EPI_WGRAD ? FI_PROF_GEMM_WGRAD
                 : EPI == EPI_STORE ? FI_PROF_PREP : FI_PROF_GEMM_DGRAD, st);  // DGRAD(_H), DUNARY
  auto go = [&](const GemmShape& g) -> int {
    // (stream-K: exactly one CTA per slot -- the runs are cut per slot)
    const int units = g.sk > 0 ? g.sk
                               : ((g.tile_end > 0 ? g.tile_end : tiles) - g.tile_begin) * g.ksplit;
    const int grid = (units < slots ? units : slots) * CL;
    if (grid <= 0) return FI_OK;
    if constexpr (PAIR) {
      FI_TRY(launch_cluster(kern, CL, dim3(grid), dim3(gemm_threads<CHUNK>()), smem_bytes, st, ta,
                            tb, ta2, tb2, g, ep));
    } else {
      FI_TRY(launch_ex(kern, 1, dim3(grid), dim3(gemm_threads<CHUNK>()), smem_bytes, st, ta, tb,
                       ta2, tb2, g, ep));
    }
    FI_CUDA(cudaGetLastError());
    return FI_OK;
  };
  if (sh.ksplit > 1 && tail > 0 && tail < tiles) {  // whole waves first, then the K-split tail
    GemmShape head = sh;
    head.ksplit = 1;
    head.part = nullptr;
    head.sem = nullptr;
    head.tile_end = tiles - tail;
    FI_TRY(go(head));
    sh.tile_begin = tiles - tail;
  }
  FI_TRY(go(sh));
  if (TR && sh.ksplit > 1) {  // transposed partial tiles: sum, transpose, epilogue
    const int tile_rows = Cf::BM * NCTA;
    const long long blocks = static_cast<long long>(tiles - sh.tile_begin) * (tile_rows / 32);
    const size_t fsm = sizeof(float) * 32 * (bn + 1);
    FI_TRY(launch_ex(k_gemm_fixup_tr<EPI>, 1, dim3(static_cast<unsigned>(blocks)), dim3(256), fsm,
                     st, static_cast<const float*>(sh.part), sh.ksplit, M, N, sh.num_m,
                     tile_rows, bn, sh.tile_begin, tiles, ep));
    FI_CUDA(cudaGetLastError());
  } else if (sh.ksplit > 1 && !sh.sem) {  // sum the partials in order and run the epilogue
    const int tile_rows = Cf::BM * NCTA;
    const long long blocks = static_cast<long long>(tiles - sh.tile_begin) * (tile_rows / kFixRows);
    const size_t fsm = sizeof(float) * kFixRows * (bn / 32) * 36;  // <= 18 KB
    FI_TRY(launch_ex(k_gemm_fixup<EPI>, 1, dim3(static_cast<unsigned>(blocks)), dim3(256), fsm,
                     st, static_cast<const float*>(sh.part), sh.ksplit, M, N, sh.num_m,
                     tile_rows, bn, sh.tile_begin, tiles, ep));
    FI_CUDA(cudaGetLastError());
  }
  return FI_OK;
}

// Tile shape per launch from a cost model in microseconds: a wave of
// persistent tiles costs k_iters x 0.55 us x t(bn) with
//   single CTA  T = ceil(M/128) ceil(N/bn) tiles over 148 slots, t = 0.77 + 0.23 bn/256
//   CTA pair    T = ceil(M/256) ceil(N/bn) tiles over  74 slots, t = 0.965 t_single
//               (bn <= 256), 0.965 (1 + 0.476 (bn - 256) / 256) above, plus a
//               serial epilogue per wave (the single-buffered accumulator)
// fitted to B200 measurements (scripts/experiments/gemm_bn_sweep.py,
// scripts/gemm_vs_cublas.py; whole waves, long K): a k-iteration has a
// large fixed part (the per-SM shared-memory fill of A and B), so narrow N
// tiles are nearly as expensive as wide ones, and a pair tile (two SMs, 256
// rows) costs 3.5% less per row than two single tiles.  The N tile is free
// in steps of 32 (K-major B) or of one 128-B atom per CTA (MN-major B) so
// tile counts can land on whole waves; split-K options (whole GEMM, or only
// the partial last wave) add their partial-tile traffic and reduction.
// FI_GEMM_PAIR / FI_GEMM_BN / FI_GEMM_KSPLIT / FI_GEMM_NOTAIL force choices
// for A/B runs; FI_GEMM_LOG=1 prints them.
int gemm_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

struct GemmChoice {
  int bn;
  bool pair;
  int ksplit;
  int tail;  // > 0: whole waves, then the last `tail` tiles split ksplit ways over K
  bool sk = false;  // the `tail` tiles are run stream-K over every slot (ksplit 1)
  bool tr = false;  // transposed output (weight table on the MMA's M side; see k_gemm TR)
};

double gemm_t_single(int bn) { return 0.77 + 0.23 * bn / 256.0; }
// Per pair k-iteration.  Above 256 the pair tile issues two MMAs per K step
// and stages 48 KB per CTA instead of 32 KB: measured 1.476x the 256 time
// for 2x the work at bn = 512 (a 256-wide tile is bound by the per-SM
// L2->shared fill rate, ~70 GB/s, not by the tensor core).
double gemm_t_pair(int bn) {
  return bn > 256 ? 0.965 * (1.0 + 0.476 * (bn - 256) / 256.0) : 0.965 * gemm_t_single(bn);
}
// Tiles above 256 fill TMEM with one accumulator, so the epilogue is not
// overlapped with the next tile's main loop: its cost per wave (model units).
double gemm_epi_serial(int bn) { return bn > 256 ? 6.0 * bn / 512.0 : 0.0; }

struct GemmCand {
  double cost;
  GemmChoice c;
};

GemmChoice choose_gemm(long long M, int N, int k_iters, int bn_max, int bn_max_pair,
                       int step_single, int step_pair, bool allow_ksplit,
                       std::vector<GemmCand>* all = nullptr) {
  static const int force_pair = gemm_env("FI_GEMM_PAIR", -1);
  static const int force_bn = gemm_env("FI_GEMM_BN", 0);
  static const int force_ks = gemm_env("FI_GEMM_KSPLIT", 0);  // 1: never split K
  static const int no_tail = gemm_env("FI_GEMM_NOTAIL", 0);
  GemmChoice best{0, false, 1, 0};
  double best_cost = 1e300;  // microseconds
  const double us_per_kiter = 0.55;  // one 128 x 256 bf16 k-iteration on one SM (measured)
  // split-K reduction cost: partials at ~3 TB/s plus a fixed 12 us for the
  // fixup kernel (8 us with FI_GEMM_INKERNEL_RED=1; its split tails: a
  // handshake plus each CTA's own partial rows at the per-SM fill rate,
  // ~60 GB/s: 2 x 128 x bn x 4 B).  Measured at config 3: 256 x 512 tails
  // for the dgrad at M >= 2368 (-10..-25 us each) and the wgrad (-0.18 ms);
  // 256 x 512 whole-tile splits at small M measured slower (kept to N tiles
  // <= 256 there).
  static const bool inkernel_red = gemm_env("FI_GEMM_INKERNEL_RED", 0) != 0;
  // k_gemm_fixup: fixed cost (launch + ramp, us) and partial-read rate (GB/s)
  static const double fix_us = gemm_env("FI_GEMM_FIXUP_US", 12);
  static const double fix_gbs = gemm_env("FI_GEMM_FIXUP_GBS", 3000);
  for (int pair = 0; pair < 2; ++pair) {
    if (force_pair >= 0 && pair != force_pair) continue;
    const int step = pair ? step_pair : step_single;
    const int slots = num_sms() / (pair ? 2 : 1);
    const int tile_rows = pair ? 256 : 128;
    const long long mt = (M + tile_rows - 1) / tile_rows;
    const int bmax = pair ? bn_max_pair : bn_max;
    for (int bn = bmax / step * step; bn >= 64 && bn >= step; bn -= step) {
      if (bn > 256 && bn % 64) continue;  // two sub-tiles: 256 + a multiple of 64
      if (force_bn && bn != force_bn) continue;
      const long long T = mt * ((N + bn - 1) / bn);
      const double t = us_per_kiter * (pair ? gemm_t_pair(bn) : gemm_t_single(bn));
      // split-K over `units` tiles of which `r` are split: feasibility and fixup cost
      auto ks_ok = [&](long long r, int ks, bool tail_split) {
        return allow_ksplit && force_ks != 1 && (tail_split || bn <= 256) &&
               r * ks <= slots && k_iters / ks >= 4 &&
               static_cast<double>(ks) * r * tile_rows * bn <= static_cast<double>(g_kpart.floats);
      };
      auto fixup_us = [&](long long r, int ks) {  // whole-tile split
        return (inkernel_red ? 8.0 : fix_us) +
               2.0 * ks * static_cast<double>(r) * tile_rows * bn * 4.0 / (fix_gbs * 1e3);
      };
      auto tail_red_us = [&](long long r, int ks) {
        if (inkernel_red) return 3.0 + 2.0 * 128 * bn * 4.0 / 60.0e3;
        return fix_us + 2.0 * ks * static_cast<double>(r) * tile_rows * bn * 4.0 / (fix_gbs * 1e3);
      };
      auto consider = [&](double cost, int ks, int tail, bool sk = false) {
        if (all) all->push_back({cost, {bn, pair != 0, ks, tail, sk}});
        if (cost < best_cost * 0.995) {
          best_cost = cost;
          best = {bn, pair != 0, ks, tail, sk};
        }
      };
      // whole tiles, optionally all split over K (small M: fewer tiles than slots)
      const bool forced = force_ks > 1 && ks_ok(T, force_ks, false);
      for (int ks = 1; ks <= 8; ++ks) {
        if (ks > 1 && !ks_ok(T, ks, false)) break;
        if (forced && ks != force_ks) continue;
        double cost = static_cast<double>((T * ks + slots - 1) / slots) *
                      (((k_iters + ks - 1) / ks) * t + gemm_epi_serial(bn));
        if (ks > 1) cost += fixup_us(T, ks);
        consider(cost, ks, 0);
      }
      // whole waves, then the partial last wave split over K (no tail gap)
      const long long r = T % slots;
      if (!no_tail && T > slots && r > 0 && force_ks != 1) {
        for (int ks = 2; ks <= 8; ++ks) {
          if (!ks_ok(r, ks, true)) break;
          // (+3 us: the tail is a second launch)
          const double cost = static_cast<double>(T / slots) * (k_iters * t + gemm_epi_serial(bn)) +
                              static_cast<double>((k_iters + ks - 1) / ks) * t +
                              gemm_epi_serial(bn) + tail_red_us(r, ks) + 3.0;
          consider(cost, ks, static_cast<int>(r));
        }
      }
      // stream-K (one launch): whole waves, then the K iterations of the last
      // r tiles (all T tiles below one wave) cut into equal runs over every
      // slot; a tile's segments are summed in-kernel by the one that ends it.
      // Kept to r >= slots / 12 (<= 13 segments per tile), partials that fit,
      // and the double-buffered tiles (bn <= 256: the finalizer waits while
      // holding its accumulator).
      // FI_GEMM_STREAMK: 0 (default) never, 1 a candidate (cost model / tuner), 2 whenever it fits
      static const int sk_env = gemm_env("FI_GEMM_STREAMK", 0);
      if (sk_env != 0 && !no_tail && force_ks != 1 && allow_ksplit && r > 0 && r * 12 >= slots &&
          bn <= 256 && r <= kKPartSems &&
          2.0 * slots * tile_rows * bn <= static_cast<double>(g_kpart.floats)) {
        const double per = static_cast<double>(r) * k_iters / slots;
        const double segs = static_cast<double>(r + slots);
        const double cost = static_cast<double>(T / slots) * (k_iters * t + gemm_epi_serial(bn)) +
                            (per + 2.0) * t + gemm_epi_serial(bn) + 2.0 +
                            2.0 * segs * tile_rows * bn * 4.0 / (fix_gbs * 1e3);
        consider(sk_env == 2 ? cost * 0.01 : cost, 1, static_cast<int>(r), true);
      }
    }
  }
  return best;
}

// ------------------------------------------------------ measured tile choice
// The cost model above ranks tile shapes from whole-wave fits; per shape its
// pick is within ~10% of the best, but which alternative wins (pair 256 x 512
// with a split tail, 256 x 256 double-buffered, a narrower N tile on whole
// waves ...) depends on the epilogue and on the box.  FI_GEMM_TUNE=1 (the
// default) times the model's cheapest candidates (cost within 1.6x of the
// best, at most 10) on the caller's stream the first time a (kernel, M, N, K)
// is launched eagerly, and keeps the fastest for the life of the process.
// Launches inside a CUDA-graph capture use the stored pick (or the model's
// when the shape was never run eagerly).  Every GEMM epilogue is a pure
// function of its operands, so re-running a launch while timing it is
// harmless.  A forced tile (FI_GEMM_PAIR / BN / KSPLIT) disables tuning.
bool same_choice(const GemmChoice& a, const GemmChoice& b) {
  return a.bn == b.bn && a.pair == b.pair && a.ksplit == b.ksplit && a.tail == b.tail &&
         a.sk == b.sk && a.tr == b.tr;
}

struct TuneKey {
  int dev, sig;
  long long M;
  int N, K;
  bool operator<(const TuneKey& o) const {
    return std::tie(dev, sig, M, N, K) < std::tie(o.dev, o.sig, o.M, o.N, o.K);
  }
};
std::mutex g_tune_mu;
std::map<TuneKey, GemmChoice> g_tuned;

bool gemm_tune_on() {
  static const bool on = env_int("FI_GEMM_TUNE", 1) != 0 && !getenv("FI_GEMM_PAIR") &&
                         !getenv("FI_GEMM_BN") && !getenv("FI_GEMM_KSPLIT");
  return on;
}

struct TuningScope {
  TuningScope() { ++g_tuning; }
  ~TuningScope() { --g_tuning; }
};

// candidates timed per shape: model cost within kTuneSpan x the cheapest, at most kTuneMax
static const double kTuneSpan = env_int("FI_GEMM_TUNE_SPAN_PCT", 160) / 100.0;
static const int kTuneMax = env_int("FI_GEMM_TUNE_MAX", 10);

template <typename L>
int tuned_choice(const TuneKey& key, GemmChoice model, std::vector<GemmCand> cands,
                 cudaStream_t st, L&& launch, GemmChoice* out) {
  *out = model;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    auto it = g_tuned.find(key);
    if (it != g_tuned.end()) {
      *out = it->second;
      return FI_OK;
    }
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {  // e.g. the legacy stream while another
    cudaGetLastError();                                  // stream captures: do not time
    return FI_OK;
  }
  if (cs != cudaStreamCaptureStatusNone) return FI_OK;  // never time inside a capture
  // distinct candidates, cheapest first; the model's pick leads
  std::stable_sort(cands.begin(), cands.end(),
                   [](const GemmCand& a, const GemmCand& b) { return a.cost < b.cost; });
  // distinct candidates, at most two per tile shape (bn, pair, transposed):
  // the split-K variants of one shape differ little, other shapes may win
  std::vector<GemmChoice> list{model};
  const double limit = (cands.empty() ? 0.0 : cands.front().cost) * kTuneSpan;
  for (const GemmCand& g : cands) {
    if (static_cast<int>(list.size()) >= kTuneMax || g.cost > limit) break;
    bool dup = false;
    int same_shape = 0;
    for (const GemmChoice& c : list) {
      dup = dup || same_choice(c, g.c);
      same_shape += c.bn == g.c.bn && c.pair == g.c.pair && c.tr == g.c.tr;
    }
    if (!dup && same_shape < 2) list.push_back(g.c);
  }
  GemmChoice best = model;
  if (list.size() > 1) {
    TuningScope mute;
    cudaEvent_t e0, e1;
    FI_CUDA(cudaEventCreate(&e0));
    FI_CUDA(cudaEventCreate(&e1));
    // two interleaved passes (each candidate: 3 timed launches per pass, the
    // faster pass counts), so clock drift and one-off noise do not decide
    std::vector<float> t(list.size(), 1e30f);
    int rc = FI_OK;
    for (int pass = 0; pass < 2 && rc == FI_OK; ++pass) {
      for (size_t i = 0; i < list.size() && rc == FI_OK; ++i) {
        if (pass == 0) {
          rc = launch(list[i]);  // warm (TMA descriptors, first-touch)
          if (rc != FI_OK) break;
        }
        cudaEventRecord(e0, st);
        for (int r = 0; r < 3 && rc == FI_OK; ++r) rc = launch(list[i]);
        cudaEventRecord(e1, st);
        if (rc != FI_OK || cudaEventSynchronize(e1) != cudaSuccess) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        t[i] = ms < t[i] ? ms : t[i];
      }
    }
    static const int log_tune = env_int("FI_GEMM_LOG", 0);
    size_t bi = 0;
    for (size_t i = 0; i < list.size(); ++i) {
      if (log_tune >= 2)
        fprintf(stderr, "[fi tune] sig=%d M=%lld N=%d K=%d  bn=%d pair=%d ks=%d tail=%d%s: %.1f us\n",
                key.sig, key.M, key.N, key.K, list[i].bn, static_cast<int>(list[i].pair),
                list[i].ksplit, list[i].tail, list[i].sk ? " sk" : list[i].tr ? " tr" : "",
                t[i] * 1e3f / 3.f);
      if (t[i] < t[bi]) bi = i;
    }
    // an alternative has to beat the model's pick by 2% to replace it
    if (bi != 0 && t[bi] < 0.98f * t[0]) best = list[bi];
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc != FI_OK) return rc;
    FI_CUDA(cudaGetLastError());
  }
  std::lock_guard<std::mutex> lk(g_tune_mu);
  g_tuned[key] = best;
  *out = best;
  return FI_OK;
}

template <typename T, bool AMN, bool BMN, int EPI, bool SPLIT>
int run_gemm_s(const Operand& A, const Operand& B, int M, int N, int K, int a_row0,
               const GemmEpi& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0) return FI_OK;
  if (N % 64) return set_err(FI_ERR_ARG, "GEMM N=%d must be a multiple of 64", N);
  constexpr int BK = 128 / static_cast<int>(sizeof(T));
  constexpr int ATOM = 128 / static_cast<int>(sizeof(T));
  // SPLIT: a K block stages 2x the operand bytes for 3 MMAs (cost-model units)
  const int k_iters = (SPLIT ? 2 : 1) * ((K + BK - 1) / BK);
  // fp32 mode: chunked round-to-nearest accumulation (8 K-iterations per
  // TMEM chunk) to bound the tensor-core truncation bias; N tile <= 128.
  // pair tiles up to 256 x 512 for bf16 (two N = 256 MMAs per K step; the
  // accumulator then fills TMEM, single-buffered)
  constexpr int kBnMax = SPLIT ? 128 : (sizeof(T) == 2 ? 512 : 256);
  constexpr int kBnSingle = kBnMax > 256 ? 256 : kBnMax;
  constexpr int kChunk = SPLIT ? FI_FP32_CHUNK : 0;
  // MN-major B is staged in whole 128-B atoms per CTA
  const int step1 = BMN ? (ATOM > 32 ? ATOM : 32) : 32;
  const int step2 = BMN ? 2 * ATOM : 32;
  static const int log_choice = env_int("FI_GEMM_LOG", 0);
  // Transposed output (TR, see k_gemm): the weight table on the MMA's M side
  // and the chart rows as the N tile, where it applies (bf16 operands,
  // K-major chart rows, not the weight gradients).  FI_GEMM_TRANS=1 forces
  // it, 0 never uses it; by default its tiles are tuner candidates.
  static const int use_tr = env_int("FI_GEMM_TRANS", -1);
  constexpr bool kTrOk = !AMN && !SPLIT && kChunk == 0 && sizeof(T) == 2 && EPI != EPI_WGRAD;
  if constexpr (kTrOk) {
    if (use_tr == 1) {
      const GemmChoice t = choose_gemm(N, M, k_iters, kBnSingle, kBnSingle, 32, 32, true);
      if (log_choice)
        fprintf(stderr, "[fi gemm] EPI=%d M=%d N=%d K=%d -> TR bn=%d pair=%d ksplit=%d tail=%d\n",
                EPI, M, N, K, t.bn, static_cast<int>(t.pair), t.ksplit, t.tail);
      if (t.bn == 0) return set_err(FI_ERR_ARG, "no transposed GEMM tile for M=%d", M);
      if (t.pair)
        return launch_gemm<T, kBnSingle, BMN, false, EPI, SPLIT, kChunk, true, false, true>(
            B, A, N, M, K, a_row0, ep, st, t.bn, t.ksplit, t.tail);
      return launch_gemm<T, kBnSingle, BMN, false, EPI, SPLIT, kChunk, false, false, true>(
          B, A, N, M, K, a_row0, ep, st, t.bn, t.ksplit, t.tail);
    }
  }
  std::vector<GemmCand> cands;
  const bool tune = gemm_tune_on();
  // (fp32 mode: split-K partials are the chunked round-to-nearest sums)
  GemmChoice c = choose_gemm(M, N, k_iters, kBnSingle, kBnMax, step1, step2, true,
                             tune ? &cands : nullptr);
  if (c.bn == 0) return set_err(FI_ERR_ARG, "no GEMM tile for N=%d (FI_GEMM_BN?)", N);
  if constexpr (kTrOk) {
    if (tune && use_tr < 0) {  // the transposed tiles compete in the measured choice
      std::vector<GemmCand> tc;
      choose_gemm(N, M, k_iters, kBnSingle, kBnSingle, 32, 32, true, &tc);
      for (GemmCand& x : tc) {
        if (x.c.sk) continue;
        x.c.tr = true;
        cands.push_back(x);
      }
    }
  }
  auto launch = [&](const GemmChoice& ch) -> int {
    if constexpr (kTrOk) {
      if (ch.tr) {
        if (ch.pair)
          return launch_gemm<T, kBnSingle, BMN, false, EPI, SPLIT, kChunk, true, false, true>(
              B, A, N, M, K, a_row0, ep, st, ch.bn, ch.ksplit, ch.tail);
        return launch_gemm<T, kBnSingle, BMN, false, EPI, SPLIT, kChunk, false, false, true>(
            B, A, N, M, K, a_row0, ep, st, ch.bn, ch.ksplit, ch.tail);
      }
    }
    if (ch.pair) {
      if (ch.bn > kBnSingle)  // 256 x 512-class pair tiles: two MMAs per K step
        return launch_gemm<T, kBnMax, AMN, BMN, EPI, SPLIT, kChunk, true>(
            A, B, M, N, K, a_row0, ep, st, ch.bn, ch.ksplit, ch.tail, ch.sk);
      return launch_gemm<T, kBnSingle, AMN, BMN, EPI, SPLIT, kChunk, true>(
          A, B, M, N, K, a_row0, ep, st, ch.bn, ch.ksplit, ch.tail, ch.sk);
    }
    return launch_gemm<T, kBnSingle, AMN, BMN, EPI, SPLIT, kChunk, false>(
        A, B, M, N, K, a_row0, ep, st, ch.bn, ch.ksplit, ch.tail, ch.sk);
  };
  const GemmChoice model = c;
  if (tune) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int sig = (((EPI * 8 + static_cast<int>(sizeof(T))) * 2 + AMN) * 2 + BMN) * 2 + SPLIT;
    FI_TRY(tuned_choice(TuneKey{dev, sig, M, N, K}, model, std::move(cands), st, launch, &c));
  }
  if (log_choice)
    fprintf(stderr, "[fi gemm] EPI=%d M=%d N=%d K=%d -> bn=%d pair=%d ksplit=%d tail=%d%s%s%s\n",
            EPI, M, N, K, c.bn, static_cast<int>(c.pair), c.ksplit, c.tail,
            c.sk ? " stream-K" : "", c.tr ? " transposed" : "",
            same_choice(c, model) ? "" : " (measured; model picked another)");
  // FI_GEMM_MC=1: pair tiles of N <= 256 run as multicast clusters of two
  // pairs (A rows shared, adjacent N tiles; see k_gemm) when eligible
  static const int use_mc = env_int("FI_GEMM_MC", 0);
  if constexpr (!AMN && !SPLIT && kChunk == 0) {
    if (use_mc && !c.tr && c.pair && c.bn <= kBnSingle && c.ksplit == 1 && c.tail == 0)
      return launch_gemm<T, kBnSingle, AMN, BMN, EPI, SPLIT, kChunk, true, true>(
          A, B, M, N, K, a_row0, ep, st, c.bn, 1, 0);
  }
  return launch(c);
}

// Dispatch on the split (fp32 / bf16x3) mode; tf32 operands are never split.
template <typename T, bool AMN, bool BMN, int EPI>
int run_gemm(const Operand& A, const Operand& B, int M, int N, int K, int a_row0,
             const GemmEpi& ep, cudaStream_t st) {
  if constexpr (sizeof(T) == 2) {
    if (A.lo || B.lo) return run_gemm_s<T, AMN, BMN, EPI, true>(A, B, M, N, K, a_row0, ep, st);
  }
  return run_gemm_s<T, AMN, BMN, EPI, false>(A, B, M, N, K, a_row0, ep, st);
}

template <int V>
using VC = std::integral_constant<int, V>;
template <typename F>
int dispatch_v(int v, F&& f) {
  switch (v) {
    case 1: return f(VC<1>{});
    case 2: return f(VC<2>{});
    case 4: return f(VC<4>{});
    case 8: return f(VC<8>{});
  }
  return set_err(FI_ERR_UNSUPPORTED, "columns per thread %d", v);
}

template <typename K>
int set_smem(K kern, size_t bytes) {
  FI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(bytes < 49152 ? 49152 : bytes)));
  return FI_OK;
}


int check_ptrs(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (!p) return set_err(FI_ERR_ARG, "null pointer argument");
  return FI_OK;
}

// ------------------------------------------------------ dual-stream sweep
// The width sweep is a chain of dependent launches, alternating a tensor-bound
// GEMM and an HBM-bound split / gather kernel.  Sentences are independent, so
// the batch is cut in two halves run on two streams, the second one launch
// behind the first: while one half's GEMM runs, the other half's bandwidth
// kernel streams HBM on the same SMs (the GEMM ring is capped at
// FI_DUAL_GEMM_STAGES so a bandwidth CTA fits beside it).  FI_DUAL=0 runs the
// whole batch on the caller's stream (the default: measured 15.4 vs 14.6 ms at
// config 3 -- the co-resident kernels contend more than they overlap).
struct AuxStream {
  cudaStream_t s[64] = {};
};
cudaStream_t aux_stream(int& err) {
  static AuxStream a;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!a.s[dev & 63]) {
    if (cudaStreamCreateWithFlags(&a.s[dev & 63], cudaStreamNonBlocking) != cudaSuccess) {
      err = 1;
      return nullptr;
    }
  }
  return a.s[dev & 63];
}

// Record on `from`, make `to` wait; the event is released once enqueued.
int stream_wait(cudaStream_t to, cudaStream_t from) {
  cudaEvent_t e;
  FI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FI_CUDA(cudaEventRecord(e, from));
  FI_CUDA(cudaStreamWaitEvent(to, e, 0));
  FI_CUDA(cudaEventDestroy(e));
  return FI_OK;
}

struct Halves {
  int n = 1;
  int b0[2] = {0, 0}, nb[2] = {0, 0};
  cudaStream_t st[2] = {nullptr, nullptr};
};

// FI_DUAL_ROWS = R > 0: launches of at most R rows (the narrow end of each
// sweep: wide spans in the forward, wide children first in the backward)
// run as two half-batch chains on two streams, so one half's bandwidth
// kernel overlaps the other half's GEMM where neither fills the GPU alone.
// (FI_DUAL = 1: every width, measured slower -- contention.)
long long dual_rows() {
  static const long long r = env_int("FI_DUAL", 0) ? (1LL << 40) : env_int("FI_DUAL_ROWS", 0);
  return r;
}

int make_halves(const Plan& p, cudaStream_t st, Halves* h) {
  h->st[0] = st;
  h->b0[0] = 0;
  h->nb[0] = p.B;
  h->n = 1;
  if (dual_rows() <= 0 || p.B < 2) return FI_OK;
  int err = 0;
  cudaStream_t s2 = aux_stream(err);
  if (err || !s2) return set_err(FI_ERR_CUDA, "cannot create the auxiliary stream");
  h->n = 2;
  h->st[1] = s2;
  h->nb[0] = p.B / 2;
  h->b0[1] = p.B / 2;
  h->nb[1] = p.B - p.B / 2;
  return FI_OK;  // the caller makes the second stream wait when its dual phase starts
}
bool dual_width(const Halves& h, const Plan& p, int w) {
  return h.n > 1 && static_cast<long long>(p.B) * (p.l - w + 1) <= dual_rows();
}

struct GemmStagesScope {  // cap the GEMM ring for this thread's launches
  int saved;
  explicit GemmStagesScope(int s) : saved(g_gemm_stages) { g_gemm_stages = s; }
  ~GemmStagesScope() { g_gemm_stages = saved; }
};
int dual_gemm_stages(const Halves& h) {
  static const int s = env_int("FI_DUAL_GEMM_STAGES", 3);
  return h.n > 1 ? s : 0;
}

// ------------------------------------------------------------------ forward
template <typename T, typename CT>
int forward_impl(const Plan& p, const float* L, const float* R, const float* root,
                 const float* unary, const int* lengths, float* logZ, void* ws,
                 cudaStream_t st) {
  constexpr int kEpiFwd = sizeof(CT) == 2 ? EPI_FWD_H : EPI_FWD;
  T* wnn = at<T>(ws, p.wnn);
  T* wnp = at<T>(ws, p.wnp);
  T* e1 = at<T>(ws, p.e1);
  T* eall = at<T>(ws, p.eall);
  float* A = at<float>(ws, p.a);   // CT storage; GemmEpi / SplitArgs carry it untyped
  float* Bc = at<float>(ws, p.b);
  float* O = p.store_o ? at<float>(ws, p.o) : nullptr;
  double* X = at<double>(ws, p.x);
  float* TOP = at<float>(ws, p.top);
  float* TOPZ = at<float>(ws, p.topz);

  float* wsum = at<float>(ws, p.wsum);
  int* flag = at<int>(ws, p.flag);
  {  // length guard first: every later kernel reads the sanitized copy
    ProfScope prof(FI_PROF_PREP, st);
    FI_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
    k_check_lengths<<<(p.B + 255) / 256, 256, 0, st>>>(lengths, at<int>(ws, p.lens), logZ, flag,
                                                        p.B, p.l);
    FI_CUDA(cudaGetLastError());
    lengths = at<int>(ws, p.lens);
  }
  {  // K1: exp of the child tables, once per call
    ProfScope prof(FI_PROF_PREP, st);
    FI_CUDA(cudaMemsetAsync(wsum, 0, 16, st));
    const int vec = (p.N % 4 == 0 && p.P % 4 == 0 && reinterpret_cast<uintptr_t>(L) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(R) % 16 == 0) ? 1 : 0;
    FI_TRY(launch_ex(k_prep_weights<T>, 1, dim3(2 * p.Np), dim3(256), 0, st, L, R, wnn, wnp, wsum,
                     p.N, p.P, p.Np, p.Pp, p.wnn_lo, p.wnp_lo, vec));
    FI_CUDA(cudaGetLastError());
  }
  {
  ProfScope prof(FI_PROF_PREP, st);
  const int vec1 = p.P % 4 == 0 && (reinterpret_cast<uintptr_t>(unary) & 15) == 0;
  FI_TRY(launch_ex(k_prep_width1<T>, 1, dim3(p.B * p.l), dim3(256), 0, st, unary, lengths, e1, X,
                   p.l, p.P, p.Pp, p.e1_lo, vec1));
  FI_CUDA(cudaGetLastError());
  }

  const Operand opWnn{wnn, p.Np, 2LL * p.Np, p.Np, false, p.wnn_lo};
  const Operand opWnp{wnp, p.Pp, 2LL * p.Np, p.Pp, false, p.wnp_lo};
  const Operand opE1{e1, p.Pp, static_cast<long long>(p.B) * p.l, p.Pp, false, p.e1_lo};
  const Operand opEall{eall, p.Np, p.rows, p.Np, false, p.eall_lo};

  // projection GEMM of width w for sentences [b0, b0 + nb)
  auto gemm = [&](int w, int b0, int nb, cudaStream_t s) -> int {
    GemmEpi ep = {};
    ep.X = X;
    ep.outA = A;
    ep.outB = Bc;
    ep.Np = p.Np;
    if (w == 1) {
      ep.M = nb * p.l;
      ep.row0 = static_cast<long long>(b0) * p.l;
      return run_gemm<T, false, false, kEpiFwd>(opE1, opWnp, ep.M, 2 * p.Np, p.Pp,
                                                 static_cast<int>(ep.row0), ep, s);
    }
    const int n_w = p.l - w + 1;
    ep.M = nb * n_w;
    ep.row0 = rowbase(w, p.B, p.l) + static_cast<long long>(b0) * n_w;
    return run_gemm<T, false, false, kEpiFwd>(opEall, opWnn, ep.M, 2 * p.Np, p.Np,
                                               static_cast<int>(ep.row0), ep, s);
  };
  // split contraction of width w for sentences [b0, b0 + nb)
  auto split = [&](int w, int b0, int nb, cudaStream_t s) -> int {
    const int n_w = p.l - w + 1;
    SplitArgs sa;
    sa.A = A;
    sa.Bc = Bc;
    sa.O = O;
    sa.E = w < p.l ? static_cast<void*>(eall) : nullptr;
    sa.e_lo = p.eall_lo;
    sa.X = X;
    sa.wsum = wsum;
    sa.TOP = TOP;
    sa.TOPZ = TOPZ;
    sa.logZ = logZ;
    sa.root = root;
    sa.lengths = lengths;
    sa.B = p.B;
    sa.lmax = p.l;
    sa.N = p.N;
    sa.Np = p.Np;
    sa.w = w;
    sa.b0 = b0;
    sa.nb = nb;
    const Decomp& dc = p.dsplit;
    sa.cols_per_cta = dc.cols_per_cta;
    ProfScope prof(FI_PROF_SPLIT, s);
    static const int pers = env_int("FI_SPLIT_PERS", 1);
    // persistent kernel unless the width has about one row per slot or fewer
    // (the widest spans: there the one-shot kernel's launch ramp is cheaper;
    // measured at |N| = 4096, l = 40: widths 34..40, -30 us per step)
    bool use_pers = pers && p.Np <= 8192;
    if (use_pers) {
      // persistent one-CTA-per-row kernel: ~72 KB of ring per CTA (2-3 CTAs/SM)
      // one CTA per row: Np = 4 * cons * V with cons <= 256 a multiple of 32
      int V = 1;
      while (V < 8 && (p.Np / (4 * V) > 256 || (p.Np / (4 * V)) % 32)) V *= 2;
      const int cons = p.Np / (4 * V);
      if (4 * cons * V != p.Np || cons % 32 || cons > 256)
        return set_err(FI_ERR_UNSUPPORTED, "no one-CTA row decomposition for Np=%d", p.Np);
      const size_t stage_bytes = 2ull * p.Np * sizeof(CT);
      static const int env_st = env_int("FI_PSTAGES", 0);
      int stages = env_st ? env_st : static_cast<int>(73728 / stage_bytes);
      stages = stages < 2 ? 2 : (stages > 8 ? 8 : stages);
      static const int nprod = env_int("FI_NPROD", 4);
      const size_t smem = static_cast<size_t>(stages) * (stage_bytes + 16 + sizeof(StageHdr)) +
                          8ull * p.l + 64;
      const int nrows = nb * n_w;
      FI_TRY(dispatch_v(V, [&](auto vc) {
        constexpr int VV = decltype(vc)::value;
        auto kern = k_split_fwd_pers<T, CT, VV>;
        FI_TRY(set_smem(kern, smem));
        int occ = 0;
        FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 + cons, smem));
        occ = occ < 1 ? 1 : occ;
        if (pers < 2 && static_cast<long long>(nrows) * 20 <= static_cast<long long>(occ) * num_sms() * 21) {
          use_pers = false;  // FI_SPLIT_PERS=2 forces the persistent kernel
          return FI_OK;
        }
        // every CTA gets the same number of rows (no partial last round)
        static const int balance = env_int("FI_SPLIT_BALANCE", 0);  // measured slightly slower
        const int slots = occ * num_sms();
        int grid = nrows < slots ? nrows : slots;
        if (balance) {
          const int per = (nrows + slots - 1) / slots;
          grid = (nrows + per - 1) / per;
        }
        FI_TRY(launch_ex(kern, 1, dim3(grid), dim3(32 + cons), smem, s, sa, stages, nprod));
        FI_CUDA(cudaGetLastError());
        return FI_OK;
      }));
      if (use_pers) return FI_OK;
    }
    // one-shot kernel (the widest spans: few rows, many terms each): with
    // fewer rows than half the SMs, cut each row into more column chunks (a
    // cluster per row, <= 8 CTAs) toward ~3 CTAs per SM, the ring deepened
    // to keep ~24 KB per CTA in flight.  (With more rows it measured slower:
    // widths 35-36 at |N| = 4096, B = 64 went 47 -> 57 us at 2 CTAs per row.)
    Decomp dcl = dc;
    static const int wide = env_int("FI_SPLIT_WIDE", 1);
    const long long nrows_w = static_cast<long long>(nb) * n_w;
    if (wide && !getenv("FI_CLUSTER") && 2 * nrows_w < num_sms()) {
      const long long want = (3LL * num_sms() + nrows_w - 1) / nrows_w;
      for (int c = static_cast<int>(want < 8 ? want : 8); c > dc.clusters; --c) {
        Decomp t;
        if (decomp_for(p.Np, c, &t)) {
          t.stages = static_cast<int>(24576 / (2 * t.cols_per_cta * sizeof(CT)));
          t.stages = t.stages < dc.stages ? dc.stages : (t.stages > 16 ? 16 : t.stages);
          dcl = t;
          break;
        }
      }
    }
    sa.cols_per_cta = dcl.cols_per_cta;
    const int stages = dcl.stages;
    const size_t smem = align128(sizeof(SplitTerm) * (w - 1)) +
                        static_cast<size_t>(stages) * (2 * dcl.cols_per_cta * sizeof(CT) + 16);
    const dim3 grid(dcl.clusters, nb * n_w);
    const dim3 block(32 + dcl.threads);
    return dispatch_v(dcl.v, [&](auto vc) {
      constexpr int V = decltype(vc)::value;
      if constexpr (V > 4) {
        return set_err(FI_ERR_UNSUPPORTED, "split decomposition V=%d", V);
      } else {
        FI_TRY(set_smem(k_split_fwd_bulk<T, CT, V>, smem));
        return launch_cluster(k_split_fwd_bulk<T, CT, V>, dcl.clusters, grid, block, smem, s, sa,
                              stages);
      }
    });
  };

  Halves h;
  FI_TRY(make_halves(p, st, &h));
  FI_TRY(gemm(1, 0, p.B, st));
  bool dual = false;  // from the first narrow width on, two half-batch chains
  for (int w = 2; w <= p.l; ++w) {
    if (!dual && dual_width(h, p, w)) {
      FI_TRY(stream_wait(h.st[1], st));
      dual = true;
    }
    if (!dual) {
      FI_TRY(split(w, 0, p.B, st));
      if (w < p.l) FI_TRY(gemm(w, 0, p.B, st));
      continue;
    }
    GemmStagesScope gs(dual_gemm_stages(h));
    for (int k = 0; k < 2; ++k) {
      KPartSelect kp(k);
      FI_TRY(split(w, h.b0[k], h.nb[k], h.st[k]));
      if (w < p.l) FI_TRY(gemm(w, h.b0[k], h.nb[k], h.st[k]));
    }
  }
  if (dual) FI_TRY(stream_wait(st, h.st[1]));  // join: the caller's stream sees all
  return FI_OK;
}

// ----------------------------------------------------------------- backward
template <typename T, typename CT>
int backward_impl(const Plan& p, const float* L, const float* R, const float* root,
                  const float* unary, const int* lengths, const float* logZ, const float* g,
                  float* dL, float* dR, float* droot, float* dunary, void* ws, cudaStream_t st,
                  cudaEvent_t dl_ready = nullptr) {
  T* wnn = at<T>(ws, p.wnn);
  T* wnp = at<T>(ws, p.wnp);
  T* eall = at<T>(ws, p.eall);
  T* e1 = at<T>(ws, p.e1);
  T* gall = at<T>(ws, p.gall);
  float* A = at<float>(ws, p.a);
  float* Bc = at<float>(ws, p.b);
  float* LQ = at<float>(ws, p.lq);  // CT-typed storage (see make_plan)
  float* LQS = p.half_chart ? at<float>(ws, p.lqs) : nullptr;
  double* X = at<double>(ws, p.x);
  float* TOP = at<float>(ws, p.top);
  float* TOPZ = at<float>(ws, p.topz);
  int* flag = at<int>(ws, p.flag);

  FI_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  k_check_lengths<<<(p.B + 255) / 256, 256, 0, st>>>(lengths, at<int>(ws, p.lens), nullptr, flag,
                                                      p.B, p.l);
  FI_CUDA(cudaGetLastError());
  lengths = at<int>(ws, p.lens);
  {
  ProfScope prof(FI_PROF_SEED, st);
  (void)logZ;  // the fp64-consistent log2 Z - x† (TOPZ) is used instead
  FI_TRY(launch_ex(k_seed_bwd<sizeof(CT) == 2>, 1, dim3((p.Np + 255) / 256, p.B), dim3(256), 0, st,
                   root, static_cast<const float*>(TOP), static_cast<const float*>(TOPZ), g,
                   lengths, static_cast<void*>(LQ), LQS, droot, flag, p.B, p.l, p.N, p.Np));
  FI_CUDA(cudaGetLastError());
  }

  const Operand opWnnMN{wnn, p.Np, 2LL * p.Np, p.Np, true, p.wnn_lo};  // K = 2Np, N = Np
  const Operand opWnpMN{wnp, p.Pp, 2LL * p.Np, p.Pp, true, p.wnp_lo};
  const Operand opGall{gall, 2LL * p.Np, p.rows, 2LL * p.Np, false, p.gall_lo};

  // gather-form split backward of child width m for sentences [b0, b0 + nb)
  auto gather = [&](int m, int b0, int nb, cudaStream_t s) -> int {
    const int n_m = p.l - m + 1;
    GatherArgs ga;
    ga.A = A;
    ga.Bc = Bc;
    ga.LQ = LQ;
    ga.LQS = LQS;
    ga.X = X;
    ga.G = gall;
    ga.g_lo = p.gall_lo;
    ga.lengths = lengths;
    ga.g = g;
    ga.B = p.B;
    ga.lmax = p.l;
    ga.Np = p.Np;
    ga.m = m;
    ga.b0 = b0;
    ga.nb = nb;
    const Decomp& dc = p.dgather;
    ga.cols_per_cta = dc.cols_per_cta;
    const dim3 grid(dc.clusters, nb * n_m);
    ProfScope prof(FI_PROF_GATHER, s);
    const int stages = dc.stages;
    const size_t qb = sizeof(CT) == 2 ? dc.cols_per_cta * 2 + dc.cols_per_cta / 8
                                       : dc.cols_per_cta * 4;
    const size_t smem = align128(sizeof(GatherTerm) * p.l) +
                        static_cast<size_t>(stages) * (dc.cols_per_cta * sizeof(CT) + qb + 16);
    // FI_GATHER_PERS=1: the persistent form when the launch has more (span,
    // chunk) items than co-resident CTAs (2: always).  Off by default:
    // measured 10-25% slower per launch at config 3 (4.52 vs 3.68 ms per
    // step) -- each CTA stalls on its item's G-row epilogue loads while its
    // ring sits full, where one-shot CTAs overlap each other.
    static const int gpers = env_int("FI_GATHER_PERS", 0);
    bool launched = false;
    if (gpers) {
      const size_t stage_bytes = dc.cols_per_cta * sizeof(CT) + qb;
      const size_t psmem = static_cast<size_t>(stages) * (stage_bytes + 16) +
                           align128(sizeof(float) * stages) + sizeof(GatherTerm) * p.l + 64;
      const long long items = static_cast<long long>(nb) * n_m * dc.clusters;
      FI_TRY(dispatch_v(dc.v, [&](auto vc) {
        constexpr int V = decltype(vc)::value;
        if constexpr (V > 4) {
          return FI_OK;
        } else {
          auto kern = k_gather_bwd_pers<T, CT, V>;
          FI_TRY(set_smem(kern, psmem));
          int occ = 0;
          FI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 + dc.threads, psmem));
          const long long slots = static_cast<long long>(occ < 1 ? 1 : occ) * num_sms();
          if (gpers < 2 && items <= slots) return FI_OK;  // one round: the one-shot kernel
          static const int nprod = env_int("FI_GNPROD", 4);
          FI_TRY(launch_ex(kern, 1, dim3(static_cast<unsigned>(items < slots ? items : slots)),
                           dim3(32 + dc.threads), psmem, s, ga, stages, nprod, dc.clusters));
          launched = true;
          return FI_OK;
        }
      }));
    }
    if (launched) {
      FI_CUDA(cudaGetLastError());
      return FI_OK;
    }
    FI_TRY(dispatch_v(dc.v, [&](auto vc) {
      constexpr int V = decltype(vc)::value;
      if constexpr (V > 4) {
        return set_err(FI_ERR_UNSUPPORTED, "gather decomposition V=%d", V);
      } else {
        FI_TRY(set_smem(k_gather_bwd_bulk<T, CT, V>, smem));
        static const int nprod = env_int("FI_GNPROD", 4);
        return launch_ex(k_gather_bwd_bulk<T, CT, V>, 1, grid, dim3(32 + dc.threads), smem, s, ga,
                         stages, nprod);
      }
    }));
    FI_CUDA(cudaGetLastError());
    return FI_OK;
  };
  // outside-weight GEMM of child width m (dunary at m = 1) for sentences [b0, b0 + nb)
  auto dgrad = [&](int m, int b0, int nb, cudaStream_t s) -> int {
    const int n_m = p.l - m + 1;
    GemmEpi ep = {};
    ep.X = X;
    ep.Np = p.Np;
    ep.M = nb * n_m;
    ep.row0 = rowbase(m, p.B, p.l) + static_cast<long long>(b0) * n_m;
    ep.lengths = lengths;
    ep.width = m;
    ep.n_w = n_m;
    ep.b0 = b0;
    if (m >= 2) {
      ep.LQ = LQ;
      ep.LQS = LQS;
      constexpr int kEpiDgrad = sizeof(CT) == 2 ? EPI_DGRAD_H : EPI_DGRAD;
      return run_gemm<T, false, true, kEpiDgrad>(opGall, opWnnMN, ep.M, p.Np, 2 * p.Np,
                                                  static_cast<int>(ep.row0), ep, s);
    }
    ep.dunary = dunary;
    ep.vec4 = (p.P % 4 == 0 && reinterpret_cast<uintptr_t>(dunary) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(unary) % 16 == 0);
    ep.unary = unary;
    ep.P = p.P;
    ep.lmax = p.l;
    return run_gemm<T, false, true, EPI_DUNARY>(opGall, opWnpMN, ep.M, p.Pp, 2 * p.Np,
                                                 static_cast<int>(ep.row0), ep, s);
  };

  {
    Halves h;
    FI_TRY(make_halves(p, st, &h));
    // the narrow (wide-child) launches come first: two half-batch chains
    // until the child width's rows exceed the threshold, then one
    bool dual = dual_width(h, p, p.l - 1);
    if (dual) {
      FI_TRY(stream_wait(h.st[1], st));
      GemmStagesScope gs(dual_gemm_stages(h));
      for (int k = 0; k < 2; ++k) FI_TRY(gather(p.l - 1, h.b0[k], h.nb[k], h.st[k]));
    } else {
      FI_TRY(gather(p.l - 1, 0, p.B, st));
    }
    for (int m = p.l - 1; m >= 1; --m) {
      if (dual && !dual_width(h, p, m)) {
        FI_TRY(stream_wait(st, h.st[1]));  // join before the first full-batch launch
        dual = false;
      }
      if (!dual) {
        FI_TRY(dgrad(m, 0, p.B, st));
        if (m > 1) FI_TRY(gather(m - 1, 0, p.B, st));
        continue;
      }
      GemmStagesScope gs(dual_gemm_stages(h));
      for (int k = 0; k < 2; ++k) {
        KPartSelect kp(k);
        FI_TRY(dgrad(m, h.b0[k], h.nb[k], h.st[k]));
        if (m > 1) FI_TRY(gather(m - 1, h.b0[k], h.nb[k], h.st[k]));
      }
    }
    if (dual) FI_TRY(stream_wait(st, h.st[1]));
  }

  // weight gradients: dW = G^T E summed over every span, then * exp(table)
  GemmEpi ep = {};
  ep.Lsrc = L;
  ep.Rsrc = R;
  ep.dL = dL;
  ep.dR = dR;
  ep.n_nt = p.N;
  ep.ld_lr = p.N + p.P;
  ep.vec4 = ((p.N + p.P) % 4 == 0 && p.N % 4 == 0 && reinterpret_cast<uintptr_t>(L) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(R) % 16 == 0 && reinterpret_cast<uintptr_t>(dL) % 16 == 0 &&
             reinterpret_cast<uintptr_t>(dR) % 16 == 0);
  ep.Np = p.Np;
  ep.M = 2 * p.Np;
  const long long r2 = rowbase(2, p.B, p.l), rl = rowbase(p.l, p.B, p.l);
  // NN block (widths >= 2) over output rows [m0, m0 + m): m = 2Np both tables
  // in one GEMM; with dl_ready, dL's rows then dR's rows as two launches
  auto wgrad_nn = [&](int m0, int m) -> int {
    if (rl > r2) {
      const Operand opG{gall + r2 * 2 * p.Np + m0, static_cast<long long>(m), rl - r2,
                        2LL * p.Np, true, p.gall_lo};
      const Operand opE{eall + r2 * p.Np, p.Np, rl - r2, p.Np, true, p.eall_lo};
      ep.col_off = 0;
      ep.valid_cols = p.N;
      ep.M = m;
      ep.m_off = m0;
      FI_TRY((run_gemm<T, true, true, EPI_WGRAD>(opG, opE, m, p.Np, static_cast<int>(rl - r2), 0,
                                                  ep, st)));
    } else {  // l == 2: no width >= 2 span is ever projected
      for (int r = 0; r < p.N; ++r) {
        if (m0 < p.Np)
          FI_CUDA(cudaMemsetAsync(dL + static_cast<long long>(r) * (p.N + p.P), 0, 4ull * p.N, st));
        if (m0 + m > p.Np)
          FI_CUDA(cudaMemsetAsync(dR + static_cast<long long>(r) * (p.N + p.P), 0, 4ull * p.N, st));
      }
    }
    return FI_OK;
  };
  // NP block (width 1), both tables
  auto wgrad_np = [&]() -> int {
    const Operand opG{gall, 2LL * p.Np, static_cast<long long>(p.B) * p.l, 2LL * p.Np, true,
                      p.gall_lo};
    const Operand opE{e1, p.Pp, static_cast<long long>(p.B) * p.l, p.Pp, true, p.e1_lo};
    ep.col_off = p.N;
    ep.valid_cols = p.P;
    ep.M = 2 * p.Np;
    ep.m_off = 0;
    FI_TRY((run_gemm<T, true, true, EPI_WGRAD>(opG, opE, 2 * p.Np, p.Pp, p.B * p.l, 0, ep, st)));
    return FI_OK;
  };
  if (!dl_ready) {
    FI_TRY(wgrad_nn(0, 2 * p.Np));
    FI_TRY(wgrad_np());
    return FI_OK;
  }
  FI_TRY(wgrad_np());
  FI_TRY(wgrad_nn(0, p.Np));
  FI_CUDA(cudaEventRecord(dl_ready, st));  // dL (both blocks) is final from here
  FI_TRY(wgrad_nn(p.Np, p.Np));
  return FI_OK;
}

// ------------------------------------------------ parameterisation tables
// Workspace of fi_param_scores / fi_param_scores_backward (fi_param.cuh):
// packed operands (padded to 64 columns; bf16 hi + lo planes in fp32 mode,
// fp32 for tf32), the fp32 product / softmax-gradient operand, the padded
// gradient outputs and one split-K region.
struct ParamPlan {
  bool split;  // fp32 mode: bf16x3 split products
  int esz, planes, dp, cp;
  size_t a, b, c, g, da, db, kpart, total;
};

int param_plan(int mode, int rows, int cols, int d, ParamPlan* q) {
  if (rows < 1 || cols < 1 || d < 1)
    return set_err(FI_ERR_ARG, "score table needs rows, cols, d >= 1 (got %d, %d, %d)", rows, cols,
                   d);
  if (mode != FI_GEMM_BF16 && mode != FI_GEMM_TF32 && mode != FI_GEMM_FP32)
    return set_err(FI_ERR_ARG, "unknown gemm_dtype %d", mode);
  q->split = mode == FI_GEMM_FP32;
  q->esz = q->split ? 2 : 4;
  q->planes = q->split ? 2 : 1;
  q->dp = static_cast<int>(align_up(d, 64));
  q->cp = static_cast<int>(align_up(cols, 64));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 1024);
    return o;
  };
  const size_t e = static_cast<size_t>(q->esz) * q->planes;
  q->a = take(e * rows * q->dp);
  q->b = take(e * q->cp * q->dp);
  q->c = take(4ull * rows * q->cp);
  q->g = take(e * rows * q->cp);
  q->da = take(4ull * rows * q->dp);
  q->db = take(4ull * q->cp * q->dp);
  q->kpart = take(4ull * kKPartRegion);
  q->total = off;
  return FI_OK;
}

unsigned grid_for(long long n) {
  const long long b = (n + 255) / 256;
  return static_cast<unsigned>(b < 4LL * num_sms() ? (b < 1 ? 1 : b) : 4LL * num_sms());
}

// Row passes: threads per CTA and whether the register-resident float4 form applies.
struct RowLaunch {
  int threads;
  bool vec;
};
RowLaunch row_launch(int cols, int ld_a, int ld_b) {
  const int threads = cols > 4 * kRowVec * 256 ? 512 : 256;
  const bool vec = cols % 4 == 0 && ld_a % 4 == 0 && ld_b % 4 == 0 &&
                   cols <= 4 * kRowVec * threads;
  return {threads, vec};
}

// Operands already in the GEMM's format need no packing: fp32 (tf32) rows of
// a multiple of 64 elements are TMA-ready as they are.
bool param_direct(const ParamPlan& q, int d) { return !q.split && d % 64 == 0; }

template <typename T>
int param_forward(const ParamPlan& q, int rows, int cols, int d, const float* A, const float* B,
                  float* logp, void* ws, cudaStream_t st) {
  const bool direct = param_direct(q, d);
  const T* ap = direct ? reinterpret_cast<const T*>(A) : at<T>(ws, q.a);
  const T* bp = direct ? reinterpret_cast<const T*>(B) : at<T>(ws, q.b);
  const long long alo = q.split ? static_cast<long long>(rows) * q.dp : 0;
  const long long blo = q.split ? static_cast<long long>(cols) * q.dp : 0;
  ProfClassScope pc(FI_PROF_PARAM);
  if (!direct) {
    ProfScope prof(FI_PROF_PARAM, st);
    k_pack_rows<T><<<grid_for(1LL * rows * q.dp), 256, 0, st>>>(A, rows, d, at<T>(ws, q.a), q.dp,
                                                                alo);
    k_pack_rows<T><<<grid_for(1LL * cols * q.dp), 256, 0, st>>>(B, cols, d, at<T>(ws, q.b), q.dp,
                                                                blo);
    g_launches += 2;
    FI_CUDA(cudaGetLastError());
  }
  // the product lands in logp itself when its rows are 64-aligned (the row
  // pass then runs in place), else in the padded scratch
  const bool inplace = cols % 64 == 0;
  float* c = inplace ? logp : at<float>(ws, q.c);
  const int ldc = inplace ? cols : q.cp;
  GemmEpi ep = {};
  ep.M = rows;
  ep.C = c;
  ep.ldc = ldc;
  const Operand opA{ap, q.dp, rows, q.dp, false, alo};
  const Operand opB{bp, q.dp, cols, q.dp, false, blo};
  FI_TRY((run_gemm<T, false, false, EPI_STORE>(opA, opB, rows, q.cp, q.dp, 0, ep, st)));
  const RowLaunch rl = row_launch(cols, ldc, cols);
  ProfScope prof(FI_PROF_PARAM, st);
  if (rl.vec) k_row_log_softmax<true><<<rows, rl.threads, 0, st>>>(c, ldc, logp, cols);
  else k_row_log_softmax<false><<<rows, rl.threads, 0, st>>>(c, ldc, logp, cols);
  ++g_launches;
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

template <typename T>
int param_backward(const ParamPlan& q, int rows, int cols, int d, const float* A, const float* B,
                   const float* logp, const float* dlogp, float* dA, float* dB, void* ws,
                   cudaStream_t st) {
  const bool direct = param_direct(q, d);
  const T* ap = direct ? reinterpret_cast<const T*>(A) : at<T>(ws, q.a);
  const T* bp = direct ? reinterpret_cast<const T*>(B) : at<T>(ws, q.b);
  T* g = at<T>(ws, q.g);
  float* da = direct ? dA : at<float>(ws, q.da);
  float* db = direct && cols % 64 == 0 ? dB : at<float>(ws, q.db);
  const long long alo = q.split ? static_cast<long long>(rows) * q.dp : 0;
  const long long blo = q.split ? static_cast<long long>(cols) * q.dp : 0;
  const long long glo = q.split ? static_cast<long long>(rows) * q.cp : 0;
  ProfClassScope pc(FI_PROF_PARAM);
  if (!direct) {
    ProfScope prof(FI_PROF_PARAM, st);
    k_pack_rows<T><<<grid_for(1LL * rows * q.dp), 256, 0, st>>>(A, rows, d, at<T>(ws, q.a), q.dp,
                                                                alo);
    k_pack_rows<T><<<grid_for(1LL * cols * q.dp), 256, 0, st>>>(B, cols, d, at<T>(ws, q.b), q.dp,
                                                                blo);
    g_launches += 2;
  }
  const RowLaunch rl = row_launch(cols, cols, q.cp);
  {
  ProfScope prof(FI_PROF_PARAM, st);
  if (rl.vec)
    k_row_softmax_bwd<T, true><<<rows, rl.threads, 0, st>>>(logp, dlogp, cols, g, q.cp, glo);
  else
    k_row_softmax_bwd<T, false><<<rows, rl.threads, 0, st>>>(logp, dlogp, cols, g, q.cp, glo);
  }
  ++g_launches;
  FI_CUDA(cudaGetLastError());
  GemmEpi ep = {};
  // dA = g B: (rows x cp) K-major times B as MN-major (K = cols rows, N = dp)
  ep.M = rows;
  ep.C = da;
  ep.ldc = q.dp;
  FI_TRY((run_gemm<T, false, true, EPI_STORE>(Operand{g, q.cp, rows, q.cp, false, glo},
                                              Operand{bp, q.dp, cols, q.dp, true, blo}, rows, q.dp,
                                              q.cp, 0, ep, st)));
  // dB = g^T A: g as MN-major A (M = cp, K = rows), A as MN-major B (K = rows, N = dp)
  ep.M = db == dB ? cols : q.cp;
  ep.C = db;
  ep.ldc = q.dp;
  FI_TRY((run_gemm<T, true, true, EPI_STORE>(Operand{g, q.cp, rows, q.cp, true, glo},
                                             Operand{ap, q.dp, rows, q.dp, true, alo}, ep.M, q.dp,
                                             rows, 0, ep, st)));
  ProfScope prof(FI_PROF_PARAM, st);
  if (da != dA) {
    k_copy_cols<<<grid_for(1LL * rows * d), 256, 0, st>>>(da, q.dp, dA, rows, d);
    ++g_launches;
  }
  if (db != dB) {
    k_copy_cols<<<grid_for(1LL * cols * d), 256, 0, st>>>(db, q.dp, dB, cols, d);
    ++g_launches;
  }
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

size_t fi_workspace_bytes(const fi_shape* shape) {
  Plan p;
  if (make_plan(shape, &p) != FI_OK) return 0;
  return p.total;
}

int fi_get_chart_layout(const fi_shape* shape, fi_chart_layout* out) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  if (!out) return set_err(FI_ERR_ARG, "null layout");
  out->np = p.Np;
  out->pp = p.Pp;
  out->rows = p.rows;
  out->off_a = static_cast<int64_t>(p.a);
  out->off_b = static_cast<int64_t>(p.b);
  out->off_o = p.store_o ? static_cast<int64_t>(p.o) : -1;
  out->off_x = static_cast<int64_t>(p.x);
  out->off_lq = static_cast<int64_t>(p.lq);
  out->off_lqs = p.half_chart ? static_cast<int64_t>(p.lqs) : -1;
  out->off_flag = static_cast<int64_t>(p.flag);
  out->chart_fmt = p.half_chart ? FI_CHART_F16 : FI_CHART_F32;
  return FI_OK;
}

int fi_inside_forward(const fi_shape* shape, const float* L, const float* R, const float* root,
                      const float* unary, const int32_t* lengths, float* log_z, void* ws,
                      void* stream) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({L, R, root, unary, lengths, log_z, ws}));
  FI_TRY(load_encode());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KPartScope kps(at<float>(ws, p.kpart), st, 2);
  FI_TRY(kps.err);
  if (p.tf32) {
    if (p.half_chart) return forward_impl<float, __half>(p, L, R, root, unary, lengths, log_z, ws, st);
    return forward_impl<float, float>(p, L, R, root, unary, lengths, log_z, ws, st);
  }
  if (p.half_chart)
    return forward_impl<__nv_bfloat16, __half>(p, L, R, root, unary, lengths, log_z, ws, st);
  return forward_impl<__nv_bfloat16, float>(p, L, R, root, unary, lengths, log_z, ws, st);
}

int fi_inside_backward(const fi_shape* shape, const float* L, const float* R, const float* root,
                       const float* unary, const int32_t* lengths, const float* log_z,
                       const float* grad_log_z, float* dL, float* dR, float* droot,
                       float* dunary, void* ws, void* stream) {
  return fi_inside_backward_ex(shape, L, R, root, unary, lengths, log_z, grad_log_z, dL, dR,
                               droot, dunary, ws, stream, nullptr);
}

int fi_inside_backward_ex(const fi_shape* shape, const float* L, const float* R,
                          const float* root, const float* unary, const int32_t* lengths,
                          const float* log_z, const float* grad_log_z, float* dL, float* dR,
                          float* droot, float* dunary, void* ws, void* stream, void* dl_ready) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({L, R, root, unary, lengths, log_z, grad_log_z, dL, dR, droot, dunary, ws}));
  FI_TRY(load_encode());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KPartScope kps(at<float>(ws, p.kpart), st, 2);
  FI_TRY(kps.err);
#define FI_BWD(T, CT)                                                                      \
  return backward_impl<T, CT>(p, L, R, root, unary, lengths, log_z, grad_log_z, dL, dR, droot, \
                              dunary, ws, st, static_cast<cudaEvent_t>(dl_ready))
  if (p.tf32) {
    if (p.half_chart) FI_BWD(float, __half);
    FI_BWD(float, float);
  }
  if (p.half_chart) FI_BWD(__nv_bfloat16, __half);
  FI_BWD(__nv_bfloat16, float);
#undef FI_BWD
}

int fi_marginals(const fi_shape* shape, const int32_t* lengths, const float* grad_log_z,
                 float* mu, void* ws, void* stream) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({lengths, grad_log_z, mu, ws}));
  if (!p.store_o) return set_err(FI_ERR_ARG, "marginals need store_chart = 1");
  const long long nrows = p.rows - rowbase(2, p.B, p.l);
  if (nrows <= 0) return FI_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_check_lengths<<<(p.B + 255) / 256, 256, 0, st>>>(lengths, at<int>(ws, p.lens), nullptr,
                                                      nullptr, p.B, p.l);
  lengths = at<int>(ws, p.lens);
  (p.half_chart ? k_marginals<true> : k_marginals<false>)<<<static_cast<unsigned>(nrows), 256, 0, st>>>(
      at<float>(ws, p.lq), p.half_chart ? at<float>(ws, p.lqs) : nullptr, at<float>(ws, p.o),
      grad_log_z, lengths, mu, p.B, p.l, p.Np, p.N);
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

int fi_span_marginals(const fi_shape* shape, const int32_t* lengths, const float* grad_log_z,
                      float* mass, void* ws, void* stream) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({lengths, grad_log_z, mass, ws}));
  if (!p.store_o) return set_err(FI_ERR_ARG, "span marginals need store_chart = 1");
  const long long nrows = p.rows - rowbase(2, p.B, p.l);
  if (nrows <= 0) return FI_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_check_lengths<<<(p.B + 255) / 256, 256, 0, st>>>(lengths, at<int>(ws, p.lens), nullptr,
                                                      nullptr, p.B, p.l);
  lengths = at<int>(ws, p.lens);
  (p.half_chart ? k_span_mass<true> : k_span_mass<false>)<<<static_cast<unsigned>(nrows), 256, 0,
                                                             st>>>(
      at<float>(ws, p.lq), p.half_chart ? at<float>(ws, p.lqs) : nullptr, at<float>(ws, p.o),
      grad_log_z, lengths, mass, p.B, p.l, p.Np, p.N);
  ++g_launches;
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

int fi_mbr_decode(const fi_shape* shape, const int32_t* lengths, const float* mass,
                  float* score, int32_t* split, void* stream) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({lengths, mass, score, split}));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_mbr_cky<<<p.B, 128, 0, st>>>(mass, lengths, score, split, p.B, p.l);
  ++g_launches;
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

int fi_viterbi(const fi_shape* shape, const float* L, const float* R, const float* root,
               const float* unary, const int32_t* lengths, float* va, float* vb, float* vo,
               int32_t* nodes, float* best, void* stream) {
  Plan p;
  FI_TRY(make_plan(shape, &p));
  FI_TRY(check_ptrs({L, R, root, unary, lengths, va, vb, vo, nodes, best}));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int ld = p.N + p.P;
  // both tables' tropical projections of M rows in one launch: [L | R] rows
  // as the output columns.  64 x 128 tiles (2 CTAs per SM; measured 418 vs
  // 397 sentences/s for 128 x 128 tiles at one CTA per SM, |N| = 4096)
  static const int trop_v1 = env_int("FI_TROP_V1", 0);  // the 64 x 64 reference kernel
  auto trop = [&](const float* A, int lda, const float* Wl, const float* Wr, int M, int K,
                  float* outA, float* outB) {
    if (trop_v1) {
      const dim3 grid((p.N + kTropTile - 1) / kTropTile, (M + kTropTile - 1) / kTropTile);
      k_trop_gemm<<<grid, 256, 0, st>>>(A, lda, Wl, ld, M, p.N, K, outA, outA, p.N, p.Np);
      k_trop_gemm<<<grid, 256, 0, st>>>(A, lda, Wr, ld, M, p.N, K, outB, outB, p.N, p.Np);
      g_launches += 2;
      return cudaGetLastError();
    }
    const int vec = (lda % 4 == 0 && ld % 4 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(Wl) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(Wr) % 16 == 0) ? 1 : 0;
    const int gx = (2 * p.N + 127) / 128;
    static const int trop_bm = env_int("FI_TROP_BM", 64);
    if (trop_bm == 128 && static_cast<long long>(gx) * ((M + 127) / 128) >= 2LL * num_sms()) {
      k_trop_gemm2<128><<<dim3(gx, (M + 127) / 128), 256, 0, st>>>(
          A, lda, Wl, Wr, ld, M, p.N, K, outA, outB, p.Np, vec);
    } else {
      k_trop_gemm2<64><<<dim3(gx, (M + 63) / 64), 256, 0, st>>>(A, lda, Wl, Wr, ld, M, p.N, K,
                                                                  outA, outB, p.Np, vec);
    }
    ++g_launches;
    return cudaGetLastError();
  };
  // width 1: va/vb = max_t L/R[A, N + t] + unary[b, i, t]   (parse.py:56-57, :66-71)
  const int m1 = p.B * p.l;
  FI_CUDA(trop(unary, p.P, L + p.N, R + p.N, m1, p.P, va, vb));
  for (int w = 2; w <= p.l; ++w) {
    const int n_w = p.l - w + 1;
    const long long r0 = rowbase(w, p.B, p.l);
    k_vit_split<<<dim3((p.Np / 4 + 255) / 256, p.B * n_w), 256, 0, st>>>(va, vb, vo, lengths, p.B,
                                                                          p.l, w, p.Np);
    ++g_launches;
    FI_CUDA(cudaGetLastError());
    if (w < p.l) {  // parse.py:66-71 over the nonterminal block
      FI_CUDA(trop(vo + r0 * p.Np, p.Np, L, R, p.B * n_w, p.N, va + r0 * p.Np, vb + r0 * p.Np));
    }
  }
  k_vit_backtrack<<<p.B, 256, 0, st>>>(va, vb, vo, unary, L, R, root, lengths, nodes, best, p.B,
                                       p.l, p.N, p.P, p.Np, p.P);
  ++g_launches;
  FI_CUDA(cudaGetLastError());
  return FI_OK;
}

size_t fi_param_workspace_bytes(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d) {
  ParamPlan q;
  if (param_plan(gemm_dtype, rows, cols, d, &q) != FI_OK) return 0;
  return q.total;
}

int fi_param_scores(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d, const float* A,
                    const float* B, float* logp, void* ws, void* stream) {
  ParamPlan q;
  FI_TRY(param_plan(gemm_dtype, rows, cols, d, &q));
  FI_TRY(check_ptrs({A, B, logp, ws}));
  FI_TRY(load_encode());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KPartScope kps(at<float>(ws, q.kpart), st, 1);
  FI_TRY(kps.err);
  if (q.split) return param_forward<__nv_bfloat16>(q, rows, cols, d, A, B, logp, ws, st);
  return param_forward<float>(q, rows, cols, d, A, B, logp, ws, st);
}

int fi_param_scores_backward(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d,
                             const float* A, const float* B, const float* logp,
                             const float* dlogp, float* dA, float* dB, void* ws, void* stream) {
  ParamPlan q;
  FI_TRY(param_plan(gemm_dtype, rows, cols, d, &q));
  FI_TRY(check_ptrs({A, B, logp, dlogp, dA, dB, ws}));
  FI_TRY(load_encode());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  KPartScope kps(at<float>(ws, q.kpart), st, 1);
  FI_TRY(kps.err);
  if (q.split)
    return param_backward<__nv_bfloat16>(q, rows, cols, d, A, B, logp, dlogp, dA, dB, ws, st);
  return param_backward<float>(q, rows, cols, d, A, B, logp, dlogp, dA, dB, ws, st);
}

int fi_test_gemm(int32_t dtype, int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K,
                 const void* A, const void* B, float* C, void* stream) {
  FI_TRY(check_ptrs({A, B, C}));
  FI_TRY(load_encode());
  if (M < 1 || N < 64 || N % 64 || K < 1)
    return set_err(FI_ERR_ARG, "test GEMM needs M>=1, N%%64==0, K>=1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* scratch = nullptr;
  FI_CUDA(cudaMallocAsync(&scratch, 4 * kKPartRegion, st));
  struct Free {
    void* p;
    cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } free_scratch{scratch, st};
  KPartScope kps(static_cast<float*>(scratch), st, 1);
  FI_TRY(kps.err);
  GemmEpi ep = {};
  ep.M = M;
  ep.C = C;
  ep.ldc = N;
  const Operand opA = a_mn ? Operand{A, M, K, M, true, 0} : Operand{A, K, M, K, false, 0};
  const Operand opB = b_mn ? Operand{B, N, K, N, true, 0} : Operand{B, K, N, K, false, 0};
#define FI_GEMM_CASE(T, AMN, BMN) \
  if (!!a_mn == AMN && !!b_mn == BMN) return run_gemm<T, AMN, BMN, EPI_STORE>(opA, opB, M, N, K, 0, ep, st);
  if (dtype == FI_GEMM_TF32) {
    FI_GEMM_CASE(float, false, false)
    FI_GEMM_CASE(float, false, true)
    FI_GEMM_CASE(float, true, true)
  } else {
    FI_GEMM_CASE(__nv_bfloat16, false, false)
    FI_GEMM_CASE(__nv_bfloat16, false, true)
    FI_GEMM_CASE(__nv_bfloat16, true, true)
  }
#undef FI_GEMM_CASE
  return set_err(FI_ERR_ARG, "unsupported majorness combination (A MN-major needs B MN-major)");
}

int64_t fi_launch_count(void) { return g_launches.load(); }

void fi_profile_enable(int32_t on) { g_prof_on = on != 0; }

int fi_profile_collect(float* ms, int32_t* counts, int32_t n) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int c = 0; c < n; ++c) {
    if (ms) ms[c] = 0.f;
    if (counts) counts[c] = 0;
  }
  int rc = FI_OK;
  for (const ProfRec& r : g_prof) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) rc = set_err(FI_ERR_CUDA, "profile event: %s", cudaGetErrorString(e));
    if (r.cls >= 0 && r.cls < n) {
      if (ms) ms[r.cls] += t;
      if (counts) counts[r.cls] += 1;
    }
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof.clear();
  return rc;
}
int fi_profile_collect_launches(float* ms, int32_t* cls, int32_t n) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int k = 0;
  for (const ProfRec& r : g_prof) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess) cudaEventElapsedTime(&t, r.a, r.b);
    if (k < n) {
      if (ms) ms[k] = t;
      if (cls) cls[k] = r.cls;
    }
    ++k;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof.clear();
  return k;
}

const char* fi_last_error(void) { return g_err; }
int32_t fi_version(void) { return 1; }

}  // extern "C"
