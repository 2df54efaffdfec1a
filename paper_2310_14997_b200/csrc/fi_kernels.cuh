// Bandwidth-bound FlashInside kernels for sm_100a: weight exponentiation,
// width-1 preparation, the split-point contraction (forward), the seed of
// the outside pass, and the gather-form split backward.
//
// Chart layout in HBM, one row per span:
//   n_w        = lmax - w + 1                    spans of width w per sentence
//   rowbase(w) = B * sum_{v<w} n_v               first row of width w
//   row(w,b,i) = rowbase(w) + b * n_w + i        span (i, i+w) of sentence b
// Every per-symbol array has row stride Np (nonterminals padded to a multiple
// of 256 with -inf / zero-probability dummy symbols).
//
// Numerics: all log values are base 2 (log2 = ln * log2(e)), so every
// exp/log is one MUFU op, and every span row carries its large magnitude in
// ONE fp64 scalar X[row] = x†, the row max of the inside score
// (inside.py:205-206).  Per-symbol arrays hold small fp32 offsets from it:
//   A^, B^ : a[w] - x†, b[w] - x†   = log2(E W^T)       (inside.py:203-213)
//   O^     : o[w] - x† <= 0          (optional: chart export / marginals)
//   E      : exp2(O^) in the GEMM operand type (bf16, tf32, or bf16 hi+lo)
//   LQ^    : log2|go| - o + x†  = log2|G W|  (outside weight, backward)
//   G      : [ga*exp(x†-a) | gb*exp(x†-b)] per span, 2*Np wide (backward)
// Sums such as a[m][i] + b[w-m][i+m] - o[w][i] are then formed as
// (fp64 scalar difference, rounded once) + (two O(10) fp32 offsets), so no
// fp32 operation ever cancels two O(100) log values.
#pragma once
#include <cooperative_groups.h>
#include "fi_ptx.cuh"

namespace cg = cooperative_groups;

namespace fi {

constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kLowInit = -1.0e30f;  // finite "minus infinity" for online LSE
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2d = 0.6931471805599453;


__host__ __device__ __forceinline__ long long rowbase(int w, int B, int lmax) {
  const long long k = w - 1;
  return static_cast<long long>(B) * (k * (lmax + 1) - k * (k + 1) / 2);
}
__host__ __device__ __forceinline__ long long chart_row(int w, int b, int i, int B, int lmax) {
  return rowbase(w, B, lmax) + static_cast<long long>(b) * (lmax - w + 1) + i;
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <typename T>
__device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <>
__device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(to_tf32(a), to_tf32(b), to_tf32(c), to_tf32(d));
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, float a, float b, float c,
                                                      float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = u;
}
template <typename T>
__device__ __forceinline__ T cvt1(float x);
template <>
__device__ __forceinline__ float cvt1<float>(float x) {
  return to_tf32(x);
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt1<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// Split-precision stores: with lo != 0 (fp32 mode, bf16x3) a second plane
// at element offset `lo` receives the bf16 residual x - bf16(x).
template <typename T>
__device__ __forceinline__ void store4s(T* p, long long lo, float a, float b, float c, float d) {
  if constexpr (sizeof(T) == 2) {
    store4<T>(p, a, b, c, d);
    if (lo) {
      const float ha = __bfloat162float(__float2bfloat16_rn(a));
      const float hb = __bfloat162float(__float2bfloat16_rn(b));
      const float hc = __bfloat162float(__float2bfloat16_rn(c));
      const float hd = __bfloat162float(__float2bfloat16_rn(d));
      store4<T>(p + lo, a - ha, b - hb, c - hc, d - hd);
    }
  } else {
    store4<T>(p, a, b, c, d);
  }
}
template <typename T>
__device__ __forceinline__ void store1s(T* p, long long lo, float x) {
  const T h = cvt1<T>(x);
  *p = h;
  if constexpr (sizeof(T) == 2) {
    if (lo) p[lo] = cvt1<T>(x - __bfloat162float(h));
  }
}

__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}

// Block-wide reduction; result valid in every thread.  `red` holds >= 33 floats.
template <bool kMax>
__device__ __forceinline__ float block_reduce(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float t = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, t) : v + t;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    float u = lane < nw ? red[lane] : (kMax ? kNegInf : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float t = __shfl_xor_sync(0xffffffffu, u, o);
      u = kMax ? fmaxf(u, t) : u + t;
    }
    if (lane == 0) red[32] = u;
  }
  __syncthreads();
  return red[32];
}

// Reduce a block-uniform value over the CTAs of the cluster through DSMEM.
template <bool kMax>
__device__ __forceinline__ float cluster_reduce(float v, float* slot, float* bcast) {
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) *slot = v;
  cl.sync();
  if (threadIdx.x == 0) {
    float r = kMax ? kNegInf : 0.f;
    for (unsigned k = 0; k < cl.num_blocks(); ++k) {
      float t = *cl.map_shared_rank(slot, k);
      r = kMax ? fmaxf(r, t) : r + t;
    }
    *bcast = r;
  }
  cl.sync();
  return *bcast;
}

// ---------------------------------------------------------------------------
// K1: W_NN = exp([L_NN ; R_NN]) (2Np x Np), W_NP = exp([L_NP ; R_NP]) (2Np x Pp).
// Once per call, not per sentence (inside.py:194-200 recomputes it per call).
// One CTA per row; it also reduces the row's block sums into
// wsum = {max_A sum W_L,NN, max sum W_R,NN, max sum W_L,NP, max sum W_R,NP},
// the bounds that let the split contraction use a fixed per-span shift.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_prep_weights(
    const float* __restrict__ L, const float* __restrict__ R, T* __restrict__ wnn,
    T* __restrict__ wnp, float* __restrict__ wsum, int N, int P, int Np, int Pp,
    long long wnn_lo, long long wnp_lo, int vec) {
  pdl_wait();
  __shared__ float red[33];
  const int row = blockIdx.x;  // 0 .. 2Np-1
  const bool right = row >= Np;
  const int a = right ? row - Np : row;
  const float* src = (right ? R : L) + static_cast<long long>(a) * (N + P);
  float snn = 0.f, snp = 0.f;
  if (vec) {  // N, P multiples of 4 and 16-B rows: float4 in, 4-wide stores out
    for (int c = 4 * threadIdx.x; c < Np; c += 4 * blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a < N && c < N) {
        v = ldg4(src + c);
        v = make_float4(expf(v.x), expf(v.y), expf(v.z), expf(v.w));
      }
      snn += (v.x + v.y) + (v.z + v.w);
      store4s<T>(wnn + static_cast<long long>(row) * Np + c, wnn_lo, v.x, v.y, v.z, v.w);
    }
    for (int t = 4 * threadIdx.x; t < Pp; t += 4 * blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (a < N && t < P) {
        v = ldg4(src + N + t);
        v = make_float4(expf(v.x), expf(v.y), expf(v.z), expf(v.w));
      }
      snp += (v.x + v.y) + (v.z + v.w);
      store4s<T>(wnp + static_cast<long long>(row) * Pp + t, wnp_lo, v.x, v.y, v.z, v.w);
    }
  } else {
    for (int c = threadIdx.x; c < Np; c += blockDim.x) {
      const float v = (a < N && c < N) ? expf(src[c]) : 0.f;
      snn += v;
      store1s<T>(wnn + static_cast<long long>(row) * Np + c, wnn_lo, v);
    }
    for (int t = threadIdx.x; t < Pp; t += blockDim.x) {
      const float v = (a < N && t < P) ? expf(src[N + t]) : 0.f;
      snp += v;
      store1s<T>(wnp + static_cast<long long>(row) * Pp + t, wnp_lo, v);
    }
  }
  snn = block_reduce<false>(snn, red);
  snp = block_reduce<false>(snp, red);
  if (threadIdx.x == 0) {  // non-negative floats order like their bit patterns
    atomicMax(reinterpret_cast<int*>(wsum) + (right ? 1 : 0), __float_as_int(snn));
    atomicMax(reinterpret_cast<int*>(wsum) + (right ? 3 : 2), __float_as_int(snp));
  }
}

// ---------------------------------------------------------------------------
// Length guard (inside.py:113-121 refuses sentences shorter than 2; the
// batched op also needs lengths[b] <= lmax).  Writes the sanitized copy every
// later kernel reads: a length outside [2, lmax] becomes 0, which makes the
// sentence inert (no span is live, no log Z / seed / gradient contribution,
// every chart write stays inside the workspace); its log Z is NaN and the
// FI_FLAG_BAD_LENGTH bit is set for the host to raise on.
// ---------------------------------------------------------------------------
__global__ void k_check_lengths(const int* __restrict__ lengths, int* __restrict__ lens,
                                float* __restrict__ logZ, int* __restrict__ flag, int B,
                                int lmax) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int len = lengths[b];
  const bool ok = len >= 2 && len <= lmax;
  lens[b] = ok ? len : 0;
  if (!ok) {
    if (logZ) logZ[b] = __int_as_float(0x7fc00000);  // NaN
    if (flag) atomicOr(flag, FI_FLAG_BAD_LENGTH);
  }
}

// ---------------------------------------------------------------------------
// Width 1: o[1] = unary (inside.py:296-298); x† = max; E1 = exp(unary - x†).
// One CTA per (sentence, position).  Padded positions get E1 = 0, x† = 0.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_prep_width1(const float* __restrict__ unary,
                                                     const int* __restrict__ lengths,
                                                     T* __restrict__ e1, double* __restrict__ X,
                                                     int lmax, int P, int Pp, long long e1_lo,
                                                     int vec) {
  pdl_wait();
  __shared__ float red[33];
  const int r = blockIdx.x;  // = b * lmax + i = chart_row(1, b, i)
  const int b = r / lmax, i = r % lmax;
  const bool ok = i < lengths[b];
  const float* u = unary + static_cast<long long>(r) * P;
  T* dst = e1 + static_cast<long long>(r) * Pp;
  float mx = kNegInf;
  if (vec) {  // P a multiple of 4, 16-B rows: float4 loads, 4-wide stores
    const float4* u4 = reinterpret_cast<const float4*>(u);
    if (ok)
      for (int t = threadIdx.x; t < P / 4; t += blockDim.x) {
        const float4 x = __ldg(u4 + t);
        mx = fmaxf(mx, fmaxf(fmaxf(x.x * kLog2e, x.y * kLog2e), fmaxf(x.z * kLog2e, x.w * kLog2e)));
      }
    mx = block_reduce<true>(mx, red);
    const float xs = (mx == kNegInf) ? 0.f : mx;
    for (int t = threadIdx.x; t < Pp / 4; t += blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok && 4 * t < P) {
        const float4 x = __ldg(u4 + t);
        v = make_float4(ex2(fmaf(x.x, kLog2e, -xs)), ex2(fmaf(x.y, kLog2e, -xs)),
                        ex2(fmaf(x.z, kLog2e, -xs)), ex2(fmaf(x.w, kLog2e, -xs)));
      }
      store4s<T>(dst + 4 * t, e1_lo, v.x, v.y, v.z, v.w);
    }
    if (threadIdx.x == 0) X[r] = xs;
    return;
  }
  if (ok)
    for (int t = threadIdx.x; t < P; t += blockDim.x) mx = fmaxf(mx, u[t] * kLog2e);
  mx = block_reduce<true>(mx, red);
  const float xs = (mx == kNegInf) ? 0.f : mx;
  for (int t = threadIdx.x; t < Pp; t += blockDim.x)
    store1s<T>(dst + t, e1_lo, (ok && t < P) ? ex2(fmaf(u[t], kLog2e, -xs)) : 0.f);
  if (threadIdx.x == 0) X[r] = xs;
}

// ---------------------------------------------------------------------------
// Storage of the projected chart vectors a[w], b[w] (the GEMM forward
// epilogue's output, the bandwidth kernels' input).  Two formats:
//   float  : A^ = a - x† = log2(acc), fp32 base-2 log offsets ("fp32 chart",
//            used in fp32 mode, where every stored value must carry 24 bits)
//   __half : the LINEAR projection acc = (E W^T)[A] scaled by 2^kChartScale,
//            fp16 ("half chart", bf16/tf32 modes).  acc = sum_B W[A,B] E[B]
//            with E <= 1 and W rows summing to <= 1, so acc in [0, 1] and
//            the stored value in [0, 2^14]: fp16 keeps 11 significant bits
//            (2^-12 relative, 4x finer than the bf16 GEMM operands) down to
//            acc = 2^-28, below which terms are < 1e-8 of the row's largest
//            and flush gracefully.  Half the bytes of the fp32 chart in both
//            bandwidth-bound kernels, and the split contraction becomes two
//            FMULs per element instead of an EX2.
// ---------------------------------------------------------------------------
constexpr int kChartScale = 14;

template <typename CT>
__device__ __forceinline__ float4 chart4(const CT* p);  // 4 consecutive values as fp32
template <>
__device__ __forceinline__ float4 chart4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 chart4<__half>(const __half* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
template <typename CT>
__device__ __forceinline__ float4 chart4_ldg(const CT* p);
template <>
__device__ __forceinline__ float4 chart4_ldg<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <>
__device__ __forceinline__ float4 chart4_ldg<__half>(const __half* p) {
  uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
// "zero projection mass" test of one stored value (a = -inf in the reference)
template <typename CT>
__device__ __forceinline__ bool is_dead(float v) {
  if constexpr (sizeof(CT) == 4) return v == kNegInf;
  else return v == 0.f;
}

// ---------------------------------------------------------------------------
// K4/K5: split-point contraction for width w (inside.py:313-332) + logZ
// (inside.py:124-129).  One cluster of C CTAs per span row; each CTA owns a
// contiguous chunk of Np/C nonterminal columns.  Per split m the
// a[m][i] and b[w-m][i+m] row chunks are streamed from HBM into a
// STAGES-deep shared-memory ring with cp.async.bulk (warp 0, one lane:
// producer) while the consumer warps accumulate from shared memory; mbarrier
// full/empty pairs hand stages back and forth (~STAGES x 8 KB in flight per
// CTA with almost no registers, so the kernel sits on the HBM roofline).
// The row max x† is reduced across the cluster through DSMEM, then E is
// written in the GEMM operand type.  No (w-1, n, N) stack is materialised.
// ---------------------------------------------------------------------------
struct SplitArgs {
  const void* A;     // CT*: a[w] (A^ or scaled linear, see above)
  const void* Bc;    // CT*: b[w]
  float* O;          // O^ (nullable)
  void* E;           // T*, row stride Np (nullable at w == lmax)
  long long e_lo;    // element offset of the lo plane (fp32 mode), else 0
  double* X;
  const float* wsum; // K1 block row-sum bounds
  float* TOP;        // B x Np : log2 root + O^ at the top span (for d_root)
  float* TOPZ;       // B      : log2 Z - x†_top
  float* logZ;       // B      : natural-log partition (output)
  const float* root;
  const int* lengths;
  int B, lmax, N, Np, w, cols_per_cta;
  int b0, nb;        // this launch's sentences [b0, b0 + nb)
};

struct SplitTerm {
  long long ra, rb;  // chart rows of a[m][i] and b[w-m][i+m]
  double xs;         // x†(a) + x†(b)
  float d;           // xs - D, rounded once from fp64
  float c;           // half chart: 2^(d - 2*kChartScale), the term's linear weight
};

// Every term a[m][i,A] + b[w-m][i+m,A] is bounded by its two row shifts plus
// the log2 row-sum bounds of the projection blocks (a^ = log2 sum_B W E with
// E <= 1), so with D = max_m of those bounds every 2^(term - D) <= 1: the
// log-sum-exp over splits needs no running max -- one FADD pair, one EX2 and
// one FADD per element and split (fp32 chart), or one FMUL and one FFMA
// (half chart).  (inside.py:323-331 computes the max first.)
__host__ __device__ __forceinline__ size_t align128(size_t v) { return (v + 127) & ~size_t(127); }

struct BulkRing {
  uint8_t* buf;     // stages x stage_bytes
  uint64_t* full;   // stages
  uint64_t* empty;  // stages
  int stages, stage_bytes, off1;
};

__device__ __forceinline__ BulkRing carve_ring(uint8_t* base, int stages, int bytes0,
                                               int bytes1) {
  BulkRing r;
  r.buf = base;
  r.stage_bytes = bytes0 + bytes1;
  r.off1 = bytes0;
  r.full = reinterpret_cast<uint64_t*>(base + static_cast<size_t>(stages) * r.stage_bytes);
  r.empty = r.full + stages;
  r.stages = stages;
  return r;
}

__device__ __forceinline__ void ring_init(BulkRing& r, int consumer_warps) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < r.stages; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], consumer_warps);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

template <typename T, typename CT, int V>
__global__ void __launch_bounds__(288) k_split_fwd_bulk(SplitArgs a, int stages) {
  constexpr bool kHalf = sizeof(CT) == 2;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ float red[33];
  __shared__ float cl_slot, cl_bcast;
  __shared__ double dred[33];
  const int w = a.w;
  const int nsplit = w - 1;
  const int n_w = a.lmax - w + 1;
  const int local = a.b0 * n_w + blockIdx.y;
  const int b = local / n_w, i = local % n_w;
  const int len = a.lengths[b];
  const long long row = rowbase(w, a.B, a.lmax) + local;
  const int nthr = blockDim.x;
  const int ncons = nthr - 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpc = a.cols_per_cta;
  const int chunk0 = blockIdx.x * cpc;
  const int ci = threadIdx.x - 32;                 // consumer index
  const int col0 = chunk0 + ci * 4;
  const CT* Ach = static_cast<const CT*>(a.A);
  const CT* Bch = static_cast<const CT*>(a.Bc);
  T* E = reinterpret_cast<T*>(a.E);
  SplitTerm* terms = reinterpret_cast<SplitTerm*>(dsm);
  const int cbytes = cpc * static_cast<int>(sizeof(CT));
  BulkRing ring = carve_ring(dsm + align128(sizeof(SplitTerm) * nsplit), stages, cbytes, cbytes);

  // per-split rows and fixed shift D
  const float lnn = a.wsum[0] > 0.f ? log2f(a.wsum[0]) : 0.f;
  const float rnn = a.wsum[1] > 0.f ? log2f(a.wsum[1]) : 0.f;
  const float lnp = a.wsum[2] > 0.f ? log2f(a.wsum[2]) : 0.f;
  const float rnp = a.wsum[3] > 0.f ? log2f(a.wsum[3]) : 0.f;
  double ub = -1.0e300;
  for (int t = threadIdx.x; t < nsplit; t += nthr) {
    const int m = t + 1;
    const long long r1 = chart_row(m, b, i, a.B, a.lmax);
    const long long r2 = chart_row(w - m, b, i + m, a.B, a.lmax);
    const double xs = a.X[r1] + a.X[r2];
    terms[t].ra = r1;
    terms[t].rb = r2;
    terms[t].xs = xs;
    ub = fmax(ub, xs + (m == 1 ? lnp : lnn) + (w - m == 1 ? rnp : rnn));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ub = fmax(ub, __shfl_xor_sync(0xffffffffu, ub, o));
  if (lane == 0) dred[warp] = ub;
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = dred[0];
    for (int k = 1; k < (nthr + 31) >> 5; ++k) d = fmax(d, dred[k]);
    dred[32] = d;
  }
  __syncthreads();
  const double D = dred[32];
  for (int t = threadIdx.x; t < nsplit; t += nthr) {
    const float d = static_cast<float>(terms[t].xs - D);
    terms[t].d = d;
    terms[t].c = exp2f(d - 2.f * kChartScale);
  }
  // The term table above reads only X and the W bounds, written two or more
  // launches back in the PDL chain (complete before the previous launch
  // passed its own wait and released this one); the a / b rows of width
  // w-1 come from the previous GEMM, so the wait sits here, before any
  // chart read or write.
  pdl_wait();

  if (i + w > len) {  // span outside the sentence: never feeds a valid span
    if (ci >= 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = col0 + v * ncons * 4;
        if (a.O) *reinterpret_cast<float4*>(a.O + row * a.Np + c) =
            make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        if (E) store4s<T>(E + row * a.Np + c, a.e_lo, 0.f, 0.f, 0.f, 0.f);
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.X[row] = D;
    return;  // uniform across the cluster (same row)
  }
  ring_init(ring, ncons >> 5);  // also publishes the term table

  float S[4 * V];
#pragma unroll
  for (int k = 0; k < 4 * V; ++k) S[k] = 0.f;
  if (warp == 0) {
    if (lane == 0) {  // producer: a[m][i] and b[w-m][i+m] chunks of every split
      int s = 0;
      uint32_t ph = 0;  // ring position, advanced without integer division
      for (int t = 0; t < nsplit; ++t, s = (s + 1 == stages) ? (ph ^= 1u, 0) : s + 1) {
        mbar_wait(&ring.empty[s], ph ^ 1);
        mbar_expect_tx(&ring.full[s], 2u * cbytes);
        uint8_t* dst = ring.buf + static_cast<size_t>(s) * ring.stage_bytes;
        bulk_g2s(dst, Ach + terms[t].ra * a.Np + chunk0, cbytes, &ring.full[s]);
        bulk_g2s(dst + ring.off1, Bch + terms[t].rb * a.Np + chunk0, cbytes, &ring.full[s]);
      }
    }
  } else {
    int s = 0;
    uint32_t ph = 0;
    for (int t = 0; t < nsplit; ++t, s = (s + 1 == stages) ? (ph ^= 1u, 0) : s + 1) {
      mbar_wait(&ring.full[s], ph);
      const float dl = kHalf ? terms[t].c : terms[t].d;
      const CT* src = reinterpret_cast<const CT*>(ring.buf + static_cast<size_t>(s) * ring.stage_bytes) + ci * 4;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 x = chart4<CT>(src + v * ncons * 4);
        const float4 y = chart4<CT>(src + cpc + v * ncons * 4);
        if constexpr (kHalf) {
          S[4 * v + 0] = fmaf(x.x * dl, y.x, S[4 * v + 0]);
          S[4 * v + 1] = fmaf(x.y * dl, y.y, S[4 * v + 1]);
          S[4 * v + 2] = fmaf(x.z * dl, y.z, S[4 * v + 2]);
          S[4 * v + 3] = fmaf(x.w * dl, y.w, S[4 * v + 3]);
        } else {
          S[4 * v + 0] += ex2(x.x + y.x + dl);
          S[4 * v + 1] += ex2(x.y + y.y + dl);
          S[4 * v + 2] += ex2(x.z + y.z + dl);
          S[4 * v + 3] += ex2(x.w + y.w + dl);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[s]);
    }
  }
  float o[4 * V];  // o - D
  float mx = kNegInf;
#pragma unroll
  for (int k = 0; k < 4 * V; ++k) {
    o[k] = warp == 0 ? kNegInf : lg2(S[k]);  // S = 0 -> -inf
    mx = fmaxf(mx, o[k]);
  }
  mx = block_reduce<true>(mx, red);
  mx = cluster_reduce<true>(mx, &cl_slot, &cl_bcast);
  const float xs = (mx == kNegInf) ? 0.f : mx;  // inside.py:324-326
#pragma unroll
  for (int k = 0; k < 4 * V; ++k) o[k] -= xs;    // O^ = o - x†  (<= 0)
  if (ci >= 0) {
    if (a.O) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        *reinterpret_cast<float4*>(a.O + row * a.Np + col0 + v * ncons * 4) =
            make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    }
    if (E) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        store4s<T>(E + row * a.Np + col0 + v * ncons * 4, a.e_lo, ex2(o[4 * v]),
                   ex2(o[4 * v + 1]), ex2(o[4 * v + 2]), ex2(o[4 * v + 3]));
    }
  }
  const double xrow = D + static_cast<double>(xs);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.X[row] = xrow;

  if (i == 0 && w == len) {  // top span: logZ = LSE_A(root[A] + o[A])  (inside.py:124-129)
    float sc[4 * V];
    float smx = kNegInf;
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = col0 + v * ncons * 4 + k;
        sc[4 * v + k] = (ci >= 0 && c < a.N) ? fmaf(a.root[c], kLog2e, o[4 * v + k]) : kNegInf;
        if (ci >= 0) a.TOP[static_cast<long long>(b) * a.Np + c] = sc[4 * v + k];
        smx = fmaxf(smx, sc[4 * v + k]);
      }
    smx = block_reduce<true>(smx, red);
    smx = cluster_reduce<true>(smx, &cl_slot, &cl_bcast);
    float sum = 0.f;
    if (smx != kNegInf) {
#pragma unroll
      for (int k = 0; k < 4 * V; ++k) sum += exp2f(sc[k] - smx);
    }
    sum = block_reduce<false>(sum, red);
    sum = cluster_reduce<false>(sum, &cl_slot, &cl_bcast);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const float z = smx == kNegInf ? kNegInf : smx + log2f(sum);  // log2 Z - x†
      a.TOPZ[b] = z;
      a.logZ[b] = z == kNegInf ? kNegInf : static_cast<float>((xrow + z) * kLn2d);
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent split contraction (one CTA per span row, C = 1).  The CTA loops
// over rows blockIdx.x, blockIdx.x + gridDim.x, ... of width w.  Its producer
// warp computes each row's term table and fixed shift D (all 32 lanes), then
// `nprod` lanes issue the row's 2 (w-1) row-chunk copies into the ring, each
// stage carrying a small header (the term's weight, and D on a row's first
// term); the consumer warps accumulate, and at a row's last term reduce the
// row max, write E / X / logZ -- while the producer is already streaming the
// next row.  So the ring never drains between rows (the per-row prologue /
// epilogue latency of one-CTA-per-row launches is hidden), several lanes keep
// more bulk copies in flight per CTA than one issuing thread can, and the
// grid is sized to the SMs instead of leaving a partial last wave.  A row
// outside its sentence takes one header-only stage (dead = 1).
// ---------------------------------------------------------------------------
struct StageHdr {
  float scal;  // term weight: d (fp32 chart) or c = 2^(d - 2 kChartScale) (half chart)
  int dead;    // 1: the row is outside its sentence (no copies in this stage)
  double D;    // the row's fixed shift (valid on the row's first stage)
};

__device__ __forceinline__ void cons_bar(int nthreads) {  // consumer warps only (barrier 1)
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
template <bool kMax>
__device__ __forceinline__ float cons_reduce(float v, float* red, int ncons) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float t = __shfl_xor_sync(0xffffffffu, v, o);
    v = kMax ? fmaxf(v, t) : v + t;
  }
  const int cw = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;  // consumer warp index
  cons_bar(ncons);
  if (lane == 0) red[cw] = v;
  cons_bar(ncons);
  float u = kMax ? kNegInf : 0.f;
  for (int k = 0; k < (ncons >> 5); ++k) u = kMax ? fmaxf(u, red[k]) : u + red[k];
  cons_bar(ncons);  // red is reused by the next reduction
  return u;
}

template <typename T, typename CT, int V>
__global__ void __launch_bounds__(288, 3) k_split_fwd_pers(SplitArgs a, int stages, int nprod) {
  constexpr bool kHalf = sizeof(CT) == 2;
  nprod = nprod < 1 ? 1 : (nprod > stages ? stages : (nprod > 32 ? 32 : nprod));
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ float red[32];
  const int w = a.w;
  const int nsplit = w - 1;
  const int n_w = a.lmax - w + 1;
  const int nrows = a.nb * n_w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = blockDim.x - 32;
  const int cpc = a.Np;  // one CTA per row
  const int cbytes = cpc * static_cast<int>(sizeof(CT));
  const CT* Ach = static_cast<const CT*>(a.A);
  const CT* Bch = static_cast<const CT*>(a.Bc);
  T* E = reinterpret_cast<T*>(a.E);
  uint8_t* ring = dsm;
  const int stage_bytes = 2 * cbytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(stages) * stage_bytes);
  uint64_t* empty = full + stages;
  StageHdr* hdr = reinterpret_cast<StageHdr*>(empty + stages);
  double* ptab = reinterpret_cast<double*>(hdr + stages);  // producer-private: xs per term
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons >> 5);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const float lnn = a.wsum[0] > 0.f ? log2f(a.wsum[0]) : 0.f;
  const float rnn = a.wsum[1] > 0.f ? log2f(a.wsum[1]) : 0.f;
  const float lnp = a.wsum[2] > 0.f ? log2f(a.wsum[2]) : 0.f;
  const float rnp = a.wsum[3] > 0.f ? log2f(a.wsum[3]) : 0.f;
  // the producer's term table of row kk: fp64 shift sums xs of each split
  // (ptab) and the row's fixed shift D (their bound); dead rows feed nothing
  auto row_table = [&](int kk, bool& dead) -> double {
    const int local = a.b0 * n_w + kk;
    const int b = local / n_w, i = local % n_w;
    dead = i + w > a.lengths[b];
    double ub = -1.0e300;
    if (!dead) {
      for (int t = lane; t < nsplit; t += 32) {
        const int m = t + 1;
        const double xs = a.X[chart_row(m, b, i, a.B, a.lmax)] +
                          a.X[chart_row(w - m, b, i + m, a.B, a.lmax)];
        ptab[t] = xs;
        ub = fmax(ub, xs + (m == 1 ? lnp : lnn) + (w - m == 1 ? rnp : rnn));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ub = fmax(ub, __shfl_xor_sync(0xffffffffu, ub, o));
    __syncwarp();
    return ub;
  };
  // The first row's table is built before the dependency wait: X and the
  // W bounds come from launches at least two back in the PDL chain (the
  // splits of narrower widths, the weight prep), which had completed before
  // the previous launch passed its own wait and released this one; only the
  // a / b rows of width w-1 (read through the ring) need the wait.
  bool dead0 = true;
  double D0 = 0.0;
  if (warp == 0 && static_cast<int>(blockIdx.x) < nrows) D0 = row_table(blockIdx.x, dead0);
  pdl_wait();     // a / b of width w-1 (the previous GEMM) are visible from here
  pdl_trigger();  // persistent: the next kernel may queue behind this one

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // ring position of this row's first stage (the consumers walk the same
    // sequence); lanes derive theirs with at most one wrap (nprod <= stages)
    int rs = 0;
    uint32_t rph = 0;
    auto advance = [&](int by) {  // by >= 0; once per row / batch, not per term
      rph ^= static_cast<uint32_t>((by / stages) & 1);
      rs += by % stages;
      if (rs >= stages) {
        rs -= stages;
        rph ^= 1u;
      }
    };
    for (int kk = blockIdx.x; kk < nrows; kk += gridDim.x) {
      const int local = a.b0 * n_w + kk;
      const int b = local / n_w, i = local % n_w;
      bool dead = dead0;
      const double D = kk == static_cast<int>(blockIdx.x) ? D0 : row_table(kk, dead);
      if (dead) {
        if (lane == 0) {
          mbar_wait(&empty[rs], rph ^ 1);
          hdr[rs].dead = 1;
          hdr[rs].D = D;
          mbar_arrive(&full[rs]);
        }
        advance(1);
      } else {
        // lanes issue in lockstep batches of nprod consecutive terms (nprod <=
        // stages): a parity wait on empty[] is then never more than one phase
        // behind, so no lane can reuse a stage whose previous round is unread
        for (int t0 = 0; t0 < nsplit; t0 += nprod) {
          const int t = t0 + lane;
          if (lane < nprod && t < nsplit) {
            int s = rs + lane;
            uint32_t ph = rph;
            if (s >= stages) {
              s -= stages;
              ph ^= 1u;
            }
            mbar_wait(&empty[s], ph ^ 1);
            const int m = t + 1;
            const float d = static_cast<float>(ptab[t] - D);
            hdr[s].scal = kHalf ? exp2f(d - 2.f * kChartScale) : d;
            hdr[s].dead = 0;
            hdr[s].D = D;
            mbar_expect_tx(&full[s], static_cast<uint32_t>(stage_bytes));
            uint8_t* dst = ring + static_cast<size_t>(s) * stage_bytes;
            bulk_g2s(dst, Ach + chart_row(m, b, i, a.B, a.lmax) * a.Np, cbytes, &full[s]);
            bulk_g2s(dst + cbytes, Bch + chart_row(w - m, b, i + m, a.B, a.lmax) * a.Np, cbytes,
                     &full[s]);
          }
          __syncwarp();
          advance(nsplit - t0 < nprod ? nsplit - t0 : nprod);
        }
      }
      __syncwarp();  // the term table is rewritten for the next row
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int ci = threadIdx.x - 32;
  const int col0 = ci * 4;
  int s = 0;
  uint32_t ph = 0;  // ring position (same sequence as the producer's), no integer division
  auto advance = [&]() {
    if (++s == stages) {
      s = 0;
      ph ^= 1u;
    }
  };
  for (int kk = blockIdx.x; kk < nrows; kk += gridDim.x) {
    const int local = a.b0 * n_w + kk;
    const int b = local / n_w, i = local % n_w;
    const int len = a.lengths[b];
    const long long row = rowbase(w, a.B, a.lmax) + local;
    // first stage: D, or the dead marker
    mbar_wait(&full[s], ph);
    const double D = hdr[s].D;
    if (hdr[s].dead) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = col0 + v * ncons * 4;
        if (a.O) *reinterpret_cast<float4*>(a.O + row * a.Np + c) =
            make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        if (E) store4s<T>(E + row * a.Np + c, a.e_lo, 0.f, 0.f, 0.f, 0.f);
      }
      if (ci == 0) a.X[row] = D;
      advance();
      continue;
    }
    float S[4 * V];
#pragma unroll
    for (int k = 0; k < 4 * V; ++k) S[k] = 0.f;
    for (int t = 0; t < nsplit; ++t) {
      if (t) mbar_wait(&full[s], ph);
      const float dl = hdr[s].scal;
      const CT* src = reinterpret_cast<const CT*>(ring + static_cast<size_t>(s) * stage_bytes) + col0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 x = chart4<CT>(src + v * ncons * 4);
        const float4 y = chart4<CT>(src + cpc + v * ncons * 4);
        if constexpr (kHalf) {
          S[4 * v + 0] = fmaf(x.x * dl, y.x, S[4 * v + 0]);
          S[4 * v + 1] = fmaf(x.y * dl, y.y, S[4 * v + 1]);
          S[4 * v + 2] = fmaf(x.z * dl, y.z, S[4 * v + 2]);
          S[4 * v + 3] = fmaf(x.w * dl, y.w, S[4 * v + 3]);
        } else {
          S[4 * v + 0] += ex2(x.x + y.x + dl);
          S[4 * v + 1] += ex2(x.y + y.y + dl);
          S[4 * v + 2] += ex2(x.z + y.z + dl);
          S[4 * v + 3] += ex2(x.w + y.w + dl);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      advance();
    }
    float o[4 * V];  // o - D
    float mx = kNegInf;
#pragma unroll
    for (int k = 0; k < 4 * V; ++k) {
      o[k] = lg2(S[k]);  // S = 0 -> -inf
      mx = fmaxf(mx, o[k]);
    }
    mx = cons_reduce<true>(mx, red, ncons);
    const float xs = (mx == kNegInf) ? 0.f : mx;  // inside.py:324-326
#pragma unroll
    for (int k = 0; k < 4 * V; ++k) o[k] -= xs;  // O^ = o - x†  (<= 0)
    if (a.O) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        *reinterpret_cast<float4*>(a.O + row * a.Np + col0 + v * ncons * 4) =
            make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    }
    if (E) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        store4s<T>(E + row * a.Np + col0 + v * ncons * 4, a.e_lo, ex2(o[4 * v]),
                   ex2(o[4 * v + 1]), ex2(o[4 * v + 2]), ex2(o[4 * v + 3]));
    }
    const double xrow = D + static_cast<double>(xs);
    if (ci == 0) a.X[row] = xrow;
    if (i == 0 && w == len) {  // top span: logZ = LSE_A(root[A] + o[A])  (inside.py:124-129)
      float sc[4 * V];
      float smx = kNegInf;
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = col0 + v * ncons * 4 + k;
          sc[4 * v + k] = c < a.N ? fmaf(a.root[c], kLog2e, o[4 * v + k]) : kNegInf;
          a.TOP[static_cast<long long>(b) * a.Np + c] = sc[4 * v + k];
          smx = fmaxf(smx, sc[4 * v + k]);
        }
      smx = cons_reduce<true>(smx, red, ncons);
      float sum = 0.f;
      if (smx != kNegInf) {
#pragma unroll
        for (int k = 0; k < 4 * V; ++k) sum += exp2f(sc[k] - smx);
      }
      sum = cons_reduce<false>(sum, red, ncons);
      if (ci == 0) {
        const float z = smx == kNegInf ? kNegInf : smx + log2f(sum);  // log2 Z - x†
        a.TOPZ[b] = z;
        a.logZ[b] = z == kNegInf ? kNegInf : static_cast<float>((xrow + z) * kLn2d);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Backward seed (inside.py:400-404): the root posterior
//   post[A] = exp(root[A] + o[len][0, A] - logZ)
// seeds the outside pass at each sentence's top span as
//   LQ^ = log2|g post| - o + x† = log2 root - (log2 Z - x†) + log2|g|
// and is itself d_root (times g).  One thread per column; loops sentences.
// ---------------------------------------------------------------------------
template <bool kHalfLQ>
__global__ void k_seed_bwd(const float* __restrict__ root, const float* __restrict__ TOP,
                           const float* __restrict__ TOPZ, const float* __restrict__ g,
                           const int* __restrict__ lengths, void* __restrict__ LQv,
                           float* __restrict__ LQS, float* __restrict__ droot,
                           int* __restrict__ flag, int B, int lmax, int N, int Np) {
  pdl_wait();
  // grid (Np / blockDim, B): block (x, b) seeds sentence b's top span for
  // one column range; the blocks of b = 0 also sum d_root over all
  // sentences (in sentence order: deterministic).  blockDim is a multiple
  // of 32 and Np of 256: each warp owns one 32-column chunk.
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Np) return;
  if (blockIdx.y == 0 && c < N) {
    float acc = 0.f;
#pragma unroll 4
    for (int b = 0; b < B; ++b) {
      const float z = TOPZ[b];
      const float gb = g[b];
      if (lengths[b] >= 2 && isfinite(z) && gb != 0.f)
        acc += gb * exp2f(TOP[static_cast<long long>(b) * Np + c] - z);
    }
    droot[c] = acc;
  }
  {
    const int b = blockIdx.y;
    const float z = TOPZ[b];
    const float gb = g[b];
    const int len = lengths[b];  // sanitized: 0 marks an invalid sentence (k_check_lengths)
    if (len < 2) return;
    const bool finite = isfinite(z);
    if (!finite && c == 0) atomicOr(flag, FI_FLAG_ZERO_PROB);
    float lq = kNegInf;
    if (finite && gb != 0.f && c < N) lq = fmaf(root[c], kLog2e, -z) + log2f(fabsf(gb));
    const long long row = chart_row(len, b, 0, B, lmax);
    if constexpr (kHalfLQ) {  // fp16 outside weight with a per-chunk exponent
      float mx = lq;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      int sc = mx == kNegInf ? 0 : static_cast<int>(floorf(mx)) - 14;
      sc = sc < -126 ? -126 : sc;
      static_cast<__half*>(LQv)[row * Np + c] = __float2half_rn(exp2f(lq - sc));
      if ((threadIdx.x & 31) == 0) LQS[row * (Np / 32) + c / 32] = static_cast<float>(sc);
    } else {
      static_cast<float*>(LQv)[row * Np + c] = lq;
    }
  }
}

// ---------------------------------------------------------------------------
// K7: gather-form split backward for child width m (inside.py:406-417).
// For span (i, i+m) of sentence b (row r), with the outside weight
// LQ = log2|go| - o of each parent:
//   G_L = [a != -inf] * sum_{w>m}  2^(x†_r + b[w-m][i+m] + LQ[w][i])
//   G_R = [b != -inf] * sum_{s<i}  2^(x†_r + a[i-s][s]   + LQ[i+m-s][s])
// which is ga*exp(x† - a) (resp. gb*exp(x† - b)) of the reference -- the row
// of the dgrad/wgrad GEMM operand -- because the a (resp. b) factor of the
// split softmax exp(a + b - o) cancels against exp(-a).  With the shifted
// storage each term is 2^(d + B^ + LQ^) (fp32 chart) or
// sib * 2^(d - kChartScale + LQ^) (half chart), d an fp64 per-term scalar.
// One CTA per (span, column chunk); the sibling and parent row chunks of
// every term stream through a cp.async.bulk + mbarrier ring as in the split
// contraction.  Each accumulator is written once: deterministic, no atomics.
// ---------------------------------------------------------------------------
struct GatherArgs {
  const void* A;  // CT*
  const void* Bc; // CT*
  const void* LQ;   // fp32 LQ^ (fp32 chart) or fp16 scaled |q| (half chart)
  const float* LQS; // half chart: per 32-column exponents of LQ
  const double* X;
  void* G;  // T*, row stride 2*Np
  long long g_lo;
  const int* lengths;
  const float* g;
  int B, lmax, Np, m, cols_per_cta;
  int b0, nb;        // this launch's sentences [b0, b0 + nb)
};

struct GatherTerm {
  long long rs, rp;  // chart rows of the sibling and of the parent
  float d;           // x†(child) + x†(sibling) - x†(parent), rounded from fp64
  float pad;
};

template <typename T, typename CT, int V>
__global__ void __launch_bounds__(288) k_gather_bwd_bulk(GatherArgs a, int stages, int nprod) {
  constexpr bool kHalf = sizeof(CT) == 2;
  nprod = nprod < 1 ? 1 : (nprod > stages ? stages : (nprod > 32 ? 32 : nprod));
  extern __shared__ __align__(128) uint8_t dsm[];
  const int m = a.m;
  const int n_m = a.lmax - m + 1;
  const int local = a.b0 * n_m + blockIdx.y;
  const int b = local / n_m, i = local % n_m;
  const int len = a.lengths[b];
  const long long row = rowbase(m, a.B, a.lmax) + local;
  const int nthr = blockDim.x;
  const int ncons = nthr - 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpc = a.cols_per_cta;
  const int chunk0 = blockIdx.x * cpc;
  const int ci = threadIdx.x - 32;
  const int col0 = chunk0 + ci * 4;
  const CT* Ach = static_cast<const CT*>(a.A);
  const CT* Bch = static_cast<const CT*>(a.Bc);
  T* G = reinterpret_cast<T*>(a.G) + row * (2LL * a.Np);

  if (i + m > len) {
    pdl_wait();
    if (ci >= 0) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = col0 + v * ncons * 4;
        store4s<T>(G + c, a.g_lo, 0.f, 0.f, 0.f, 0.f);
        store4s<T>(G + a.Np + c, a.g_lo, 0.f, 0.f, 0.f, 0.f);
      }
    }
    return;
  }
  const int n_left = len - i - m;
  const int n_all = n_left + i;
  GatherTerm* gterms = reinterpret_cast<GatherTerm*>(dsm);
  const int sbytes = cpc * static_cast<int>(sizeof(CT));
  // parent chunk: fp32 LQ^, or fp16 |q| followed by its cpc/32 exponents
  const int qbytes = kHalf ? cpc * 2 : cpc * 4;
  const int sxbytes = kHalf ? cpc / 8 : 0;
  BulkRing ring = carve_ring(dsm + align128(sizeof(GatherTerm) * a.lmax), stages, sbytes,
                             qbytes + sxbytes);
  const double xm = a.X[row] - (kHalf ? kChartScale : 0);
  for (int t = threadIdx.x; t < n_all; t += nthr) {
    long long rs, rp;
    if (t < n_left) {  // left child (i, i+m) of parent (i, i+w): sibling b[w-m][i+m]
      const int w = m + 1 + t;
      rs = chart_row(w - m, b, i + m, a.B, a.lmax);
      rp = chart_row(w, b, i, a.B, a.lmax);
    } else {           // right child of parent (s, i+m): sibling a[i-s][s]
      const int sidx = t - n_left;
      rs = chart_row(i - sidx, b, sidx, a.B, a.lmax);
      rp = chart_row(i + m - sidx, b, sidx, a.B, a.lmax);
    }
    gterms[t].rs = rs;
    gterms[t].rp = rp;
    gterms[t].d = static_cast<float>(xm + a.X[rs] - a.X[rp]);
  }
  // The term table reads only forward-pass data (X, the sanitized lengths);
  // the parents' LQ rows come from the previous dgrad launches, so the
  // dependency wait sits here, before the ring streams them.
  pdl_wait();
  ring_init(ring, ncons >> 5);

  float gl[4 * V], gr[4 * V];
#pragma unroll
  for (int k = 0; k < 4 * V; ++k) gl[k] = gr[k] = 0.f;
  if (warp == 0) {
    // `nprod` lanes issue in lockstep batches of consecutive terms (nprod <=
    // stages, so a parity wait is never more than one phase behind): a CTA
    // keeps more bulk copies in flight than one issuing thread can
    const unsigned imask = (1u << nprod) - 1u;
    int bs = 0;
    uint32_t bph = 0;  // ring position of the batch's first term (no per-term division)
    for (int t0 = 0; t0 < n_all && lane < nprod; t0 += nprod) {
      const int t = t0 + lane;
      if (t < n_all) {
        int s = bs + lane;
        uint32_t ph = bph;
        if (s >= stages) {  // at most one wrap: nprod <= stages
          s -= stages;
          ph ^= 1u;
        }
        mbar_wait(&ring.empty[s], ph ^ 1);
        mbar_expect_tx(&ring.full[s], static_cast<uint32_t>(ring.stage_bytes));
        uint8_t* dst = ring.buf + static_cast<size_t>(s) * ring.stage_bytes;
        const CT* sib = t < n_left ? Bch : Ach;
        bulk_g2s(dst, sib + gterms[t].rs * a.Np + chunk0, sbytes, &ring.full[s]);
        if constexpr (kHalf) {
          bulk_g2s(dst + ring.off1,
                   static_cast<const __half*>(a.LQ) + gterms[t].rp * a.Np + chunk0, qbytes,
                   &ring.full[s]);
          bulk_g2s(dst + ring.off1 + qbytes, a.LQS + gterms[t].rp * (a.Np / 32) + chunk0 / 32,
                   sxbytes, &ring.full[s]);
        } else {
          bulk_g2s(dst + ring.off1, static_cast<const float*>(a.LQ) + gterms[t].rp * a.Np + chunk0,
                   qbytes, &ring.full[s]);
        }
      }
      __syncwarp(imask);
      bs += nprod;
      if (bs >= stages) {
        bs -= stages;
        bph ^= 1u;
      }
    }
  } else {
    int s = 0;
    uint32_t ph = 0;  // ring position, advanced without integer division
    for (int t = 0; t < n_all; ++t, s = (s + 1 == stages) ? (ph ^= 1u, 0) : s + 1) {
      mbar_wait(&ring.full[s], ph);
      const float d = gterms[t].d;
      const uint8_t* stg = ring.buf + static_cast<size_t>(s) * ring.stage_bytes;
      const CT* src = reinterpret_cast<const CT*>(stg) + ci * 4;
      float* acc = t < n_left ? gl : gr;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 x = chart4<CT>(src + v * ncons * 4);
        if constexpr (kHalf) {
          // term = sib * q * 2^(d + s_chunk): one EX2 per 4 columns
          const __half* qh = reinterpret_cast<const __half*>(stg + ring.off1);
          const float* sx = reinterpret_cast<const float*>(stg + ring.off1 + qbytes);
          const int cl = ci * 4 + v * ncons * 4;  // column within the CTA chunk
          const float4 q = chart4<__half>(qh + cl);
          const float f = ex2(d + sx[cl >> 5]);
          if (t < n_left) {
            gl[4 * v + 0] = fmaf(x.x * q.x, f, gl[4 * v + 0]);
            gl[4 * v + 1] = fmaf(x.y * q.y, f, gl[4 * v + 1]);
            gl[4 * v + 2] = fmaf(x.z * q.z, f, gl[4 * v + 2]);
            gl[4 * v + 3] = fmaf(x.w * q.w, f, gl[4 * v + 3]);
          } else {
            gr[4 * v + 0] = fmaf(x.x * q.x, f, gr[4 * v + 0]);
            gr[4 * v + 1] = fmaf(x.y * q.y, f, gr[4 * v + 1]);
            gr[4 * v + 2] = fmaf(x.z * q.z, f, gr[4 * v + 2]);
            gr[4 * v + 3] = fmaf(x.w * q.w, f, gr[4 * v + 3]);
          }
        } else {
          const float* srq = reinterpret_cast<const float*>(stg + ring.off1) + ci * 4;
          const float4 q = *reinterpret_cast<const float4*>(srq + v * ncons * 4);
          if (t < n_left) {
            gl[4 * v + 0] += ex2(x.x + q.x + d);
            gl[4 * v + 1] += ex2(x.y + q.y + d);
            gl[4 * v + 2] += ex2(x.z + q.z + d);
            gl[4 * v + 3] += ex2(x.w + q.w + d);
          } else {
            gr[4 * v + 0] += ex2(x.x + q.x + d);
            gr[4 * v + 1] += ex2(x.y + q.y + d);
            gr[4 * v + 2] += ex2(x.z + q.z + d);
            gr[4 * v + 3] += ex2(x.w + q.w + d);
          }
        }
      }
      (void)acc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[s]);
    }
    // zero-mass projections carry no gradient (inside.py:441-443 NaN guard)
    const float sg = a.g[b] < 0.f ? -1.f : 1.f;
    const CT* pam = Ach + row * a.Np;
    const CT* pbm = Bch + row * a.Np;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = col0 + v * ncons * 4;
      const float4 am = chart4_ldg<CT>(pam + c), bm = chart4_ldg<CT>(pbm + c);
      store4s<T>(G + c, a.g_lo, is_dead<CT>(am.x) ? 0.f : sg * gl[4 * v + 0],
                 is_dead<CT>(am.y) ? 0.f : sg * gl[4 * v + 1],
                 is_dead<CT>(am.z) ? 0.f : sg * gl[4 * v + 2],
                 is_dead<CT>(am.w) ? 0.f : sg * gl[4 * v + 3]);
      store4s<T>(G + a.Np + c, a.g_lo, is_dead<CT>(bm.x) ? 0.f : sg * gr[4 * v + 0],
                 is_dead<CT>(bm.y) ? 0.f : sg * gr[4 * v + 1],
                 is_dead<CT>(bm.z) ? 0.f : sg * gr[4 * v + 2],
                 is_dead<CT>(bm.w) ? 0.f : sg * gr[4 * v + 3]);
    }
  }
}

// Persistent gather (the k_gather_bwd_bulk work, one CTA looping over
// work items (span row, column chunk) blockIdx.x, blockIdx.x + gridDim.x,
// ...).  As in k_split_fwd_pers: the producer warp builds an item's term
// table (all 32 lanes), `nprod` lanes issue its sibling / parent copies into
// the ring, each stage carrying the term's weight d, and goes straight on to
// the next item while the consumers still accumulate -- so the ring does
// not drain between items, and the per-CTA prologue (barrier init, term
// table) is paid once per CTA instead of once per item.  Items outside a
// sentence take no stage (both sides know it from the lengths).
// ---------------------------------------------------------------------------
template <typename T, typename CT, int V>
__global__ void __launch_bounds__(288, 3) k_gather_bwd_pers(GatherArgs a, int stages, int nprod,
                                                            int chunks) {
  constexpr bool kHalf = sizeof(CT) == 2;
  nprod = nprod < 1 ? 1 : (nprod > stages ? stages : (nprod > 32 ? 32 : nprod));
  extern __shared__ __align__(128) uint8_t dsm[];
  const int m = a.m;
  const int n_m = a.lmax - m + 1;
  const int items = a.nb * n_m * chunks;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = blockDim.x - 32;
  const int cpc = a.cols_per_cta;
  const CT* Ach = static_cast<const CT*>(a.A);
  const CT* Bch = static_cast<const CT*>(a.Bc);
  const int sbytes = cpc * static_cast<int>(sizeof(CT));
  const int qbytes = kHalf ? cpc * 2 : cpc * 4;
  const int sxbytes = kHalf ? cpc / 8 : 0;
  const int stage_bytes = sbytes + qbytes + sxbytes;
  uint8_t* ring = dsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(stages) * stage_bytes);
  uint64_t* empty = full + stages;
  float* hdr = reinterpret_cast<float*>(empty + stages);            // term weight per stage
  GatherTerm* ptab = reinterpret_cast<GatherTerm*>(
      reinterpret_cast<uint8_t*>(hdr) + align128(sizeof(float) * stages));  // producer-private
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], ncons >> 5);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();     // LQ / chart rows of the previous kernels visible from here
  pdl_trigger();  // persistent: the next kernel may queue behind this one

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    long long g0 = 0;
    for (int kk = blockIdx.x; kk < items; kk += gridDim.x) {
      const int local = a.b0 * n_m + kk / chunks;
      const int chunk0 = (kk % chunks) * cpc;
      const int b = local / n_m, i = local % n_m;
      const int len = a.lengths[b];
      if (i + m > len) continue;  // dead span: no stages
      const long long row = rowbase(m, a.B, a.lmax) + local;
      const int n_left = len - i - m;
      const int n_all = n_left + i;
      const double xm = a.X[row] - (kHalf ? kChartScale : 0);
      for (int t = lane; t < n_all; t += 32) {
        long long rs, rp;
        if (t < n_left) {  // left child (i, i+m) of parent (i, i+w): sibling b[w-m][i+m]
          const int w = m + 1 + t;
          rs = chart_row(w - m, b, i + m, a.B, a.lmax);
          rp = chart_row(w, b, i, a.B, a.lmax);
        } else {           // right child of parent (s, i+m): sibling a[i-s][s]
          const int sidx = t - n_left;
          rs = chart_row(i - sidx, b, sidx, a.B, a.lmax);
          rp = chart_row(i + m - sidx, b, sidx, a.B, a.lmax);
        }
        ptab[t].rs = rs;
        ptab[t].rp = rp;
        ptab[t].d = static_cast<float>(xm + a.X[rs] - a.X[rp]);
      }
      __syncwarp();
      // lanes issue in lockstep batches of nprod consecutive terms (nprod <=
      // stages: a parity wait is never more than one phase behind)
      for (int t0 = 0; t0 < n_all; t0 += nprod) {
        const int t = t0 + lane;
        if (lane < nprod && t < n_all) {
          const long long gg = g0 + t;
          const int st = static_cast<int>(gg % stages);
          mbar_wait(&empty[st], static_cast<uint32_t>((gg / stages) & 1) ^ 1);
          hdr[st] = ptab[t].d;
          mbar_expect_tx(&full[st], static_cast<uint32_t>(stage_bytes));
          uint8_t* dst = ring + static_cast<size_t>(st) * stage_bytes;
          const CT* sib = t < n_left ? Bch : Ach;
          bulk_g2s(dst, sib + ptab[t].rs * a.Np + chunk0, sbytes, &full[st]);
          if constexpr (kHalf) {
            bulk_g2s(dst + sbytes, static_cast<const __half*>(a.LQ) + ptab[t].rp * a.Np + chunk0,
                     qbytes, &full[st]);
            bulk_g2s(dst + sbytes + qbytes, a.LQS + ptab[t].rp * (a.Np / 32) + chunk0 / 32,
                     sxbytes, &full[st]);
          } else {
            bulk_g2s(dst + sbytes, static_cast<const float*>(a.LQ) + ptab[t].rp * a.Np + chunk0,
                     qbytes, &full[st]);
          }
        }
        __syncwarp();
      }
      g0 += n_all;
      __syncwarp();  // the term table is rewritten for the next item
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int ci = threadIdx.x - 32;
  long long g0 = 0;
  for (int kk = blockIdx.x; kk < items; kk += gridDim.x) {
    const int local = a.b0 * n_m + kk / chunks;
    const int chunk0 = (kk % chunks) * cpc;
    const int b = local / n_m, i = local % n_m;
    const int len = a.lengths[b];
    const long long row = rowbase(m, a.B, a.lmax) + local;
    const int col0 = chunk0 + ci * 4;
    T* G = reinterpret_cast<T*>(a.G) + row * (2LL * a.Np);
    if (i + m > len) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int c = col0 + v * ncons * 4;
        store4s<T>(G + c, a.g_lo, 0.f, 0.f, 0.f, 0.f);
        store4s<T>(G + a.Np + c, a.g_lo, 0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    const int n_left = len - i - m;
    const int n_all = n_left + i;
    float gl[4 * V], gr[4 * V];
#pragma unroll
    for (int k = 0; k < 4 * V; ++k) gl[k] = gr[k] = 0.f;
    for (int t = 0; t < n_all; ++t) {
      const long long gg = g0 + t;
      const int st = static_cast<int>(gg % stages);
      mbar_wait(&full[st], static_cast<uint32_t>((gg / stages) & 1));
      const float d = hdr[st];
      const uint8_t* stg = ring + static_cast<size_t>(st) * stage_bytes;
      const CT* src = reinterpret_cast<const CT*>(stg) + ci * 4;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 x = chart4<CT>(src + v * ncons * 4);
        if constexpr (kHalf) {
          // term = sib * q * 2^(d + s_chunk): one EX2 per 4 columns
          const __half* qh = reinterpret_cast<const __half*>(stg + sbytes);
          const float* sx = reinterpret_cast<const float*>(stg + sbytes + qbytes);
          const int cl = ci * 4 + v * ncons * 4;  // column within the item's chunk
          const float4 q = chart4<__half>(qh + cl);
          const float f = ex2(d + sx[cl >> 5]);
          // (explicit branches keep gl / gr in registers)
          if (t < n_left) {
            gl[4 * v + 0] = fmaf(x.x * q.x, f, gl[4 * v + 0]);
            gl[4 * v + 1] = fmaf(x.y * q.y, f, gl[4 * v + 1]);
            gl[4 * v + 2] = fmaf(x.z * q.z, f, gl[4 * v + 2]);
            gl[4 * v + 3] = fmaf(x.w * q.w, f, gl[4 * v + 3]);
          } else {
            gr[4 * v + 0] = fmaf(x.x * q.x, f, gr[4 * v + 0]);
            gr[4 * v + 1] = fmaf(x.y * q.y, f, gr[4 * v + 1]);
            gr[4 * v + 2] = fmaf(x.z * q.z, f, gr[4 * v + 2]);
            gr[4 * v + 3] = fmaf(x.w * q.w, f, gr[4 * v + 3]);
          }
        } else {
          const float* srq = reinterpret_cast<const float*>(stg + sbytes) + ci * 4;
          const float4 q = *reinterpret_cast<const float4*>(srq + v * ncons * 4);
          if (t < n_left) {
            gl[4 * v + 0] += ex2(x.x + q.x + d);
            gl[4 * v + 1] += ex2(x.y + q.y + d);
            gl[4 * v + 2] += ex2(x.z + q.z + d);
            gl[4 * v + 3] += ex2(x.w + q.w + d);
          } else {
            gr[4 * v + 0] += ex2(x.x + q.x + d);
            gr[4 * v + 1] += ex2(x.y + q.y + d);
            gr[4 * v + 2] += ex2(x.z + q.z + d);
            gr[4 * v + 3] += ex2(x.w + q.w + d);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    g0 += n_all;
    // zero-mass projections carry no gradient (inside.py:441-443 NaN guard)
    const float sg = a.g[b] < 0.f ? -1.f : 1.f;
    const CT* pam = Ach + row * a.Np;
    const CT* pbm = Bch + row * a.Np;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = col0 + v * ncons * 4;
      const float4 am = chart4_ldg<CT>(pam + c), bm = chart4_ldg<CT>(pbm + c);
      store4s<T>(G + c, a.g_lo, is_dead<CT>(am.x) ? 0.f : sg * gl[4 * v + 0],
                 is_dead<CT>(am.y) ? 0.f : sg * gl[4 * v + 1],
                 is_dead<CT>(am.z) ? 0.f : sg * gl[4 * v + 2],
                 is_dead<CT>(am.w) ? 0.f : sg * gl[4 * v + 3]);
      store4s<T>(G + a.Np + c, a.g_lo, is_dead<CT>(bm.x) ? 0.f : sg * gr[4 * v + 0],
                 is_dead<CT>(bm.y) ? 0.f : sg * gr[4 * v + 1],
                 is_dead<CT>(bm.z) ? 0.f : sg * gr[4 * v + 2],
                 is_dead<CT>(bm.w) ? 0.f : sg * gr[4 * v + 3]);
    }
  }
}

// Span marginals mu_sym[w][i, A] = go / |g| = 2^(LQ^ + O^ - log2|g|)  (inside.py:425-430)
template <bool kHalfLQ>
__global__ void k_marginals(const void* __restrict__ LQv, const float* __restrict__ LQS,
                            const float* __restrict__ O, const float* __restrict__ g,
                            const int* __restrict__ lengths, float* __restrict__ mu, int B,
                            int lmax, int Np, int N) {
  const long long row = rowbase(2, B, lmax) + blockIdx.x;  // rows of widths >= 2
  int w = 2;
  while (w < lmax && row >= rowbase(w + 1, B, lmax)) ++w;
  const int n_w = lmax - w + 1;
  const long long local = row - rowbase(w, B, lmax);
  const int b = static_cast<int>(local / n_w), i = static_cast<int>(local % n_w);
  const bool ok = i + w <= lengths[b] && g[b] != 0.f;
  const float lg = ok ? log2f(fabsf(g[b])) : 0.f;
  float* out = mu + (row - rowbase(2, B, lmax)) * N;
  if ((N & 3) == 0 && (reinterpret_cast<uintptr_t>(mu) & 15) == 0) {  // 4 columns per thread
    for (int c = 4 * threadIdx.x; c < N; c += 4 * blockDim.x) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) {
        const float4 o = __ldg(reinterpret_cast<const float4*>(O + row * Np + c));
        if constexpr (kHalfLQ) {
          const uint2 u = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(LQv) +
                                                               row * Np + c));
          const float2 q01 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          const float2 q23 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
          const float e = LQS[row * (Np / 32) + c / 32] - lg;
          v = make_float4(q01.x * exp2f(e + o.x), q01.y * exp2f(e + o.y), q23.x * exp2f(e + o.z),
                          q23.y * exp2f(e + o.w));
        } else {
          const float4 q = __ldg(reinterpret_cast<const float4*>(
              static_cast<const float*>(LQv) + row * Np + c));
          v = make_float4(exp2f(q.x + o.x - lg), exp2f(q.y + o.y - lg), exp2f(q.z + o.z - lg),
                          exp2f(q.w + o.w - lg));
        }
      }
      *reinterpret_cast<float4*>(out + c) = v;
    }
    return;
  }
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    float v = 0.f;
    if (ok) {
      if constexpr (kHalfLQ) {
        const float q = __half2float(static_cast<const __half*>(LQv)[row * Np + c]);
        v = q * exp2f(LQS[row * (Np / 32) + c / 32] + O[row * Np + c] - lg);
      } else {
        v = exp2f(static_cast<const float*>(LQv)[row * Np + c] + O[row * Np + c] - lg);
      }
    }
    out[c] = v;
  }
}

}  // namespace fi
