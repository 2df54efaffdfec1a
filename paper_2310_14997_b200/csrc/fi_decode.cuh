// Decoders over the inside chart: span posterior mass and
// minimum-Bayes-risk CKY (parse.py:98-131), batched over sentences.
#pragma once
#include "fi_kernels.cuh"

namespace fi {

// mass[r] = sum_A mu(span r, A) for the rows of widths >= 2 (MarginalTable.mu,
// inside.py:355-372 / :425-430), mu = go / |g| = 2^(LQ^ + O^ - log2|g|).
// One CTA per span row.
template <bool kHalfLQ>
__global__ void __launch_bounds__(256) k_span_mass(const void* __restrict__ LQv,
                                                   const float* __restrict__ LQS,
                                                   const float* __restrict__ O,
                                                   const float* __restrict__ g,
                                                   const int* __restrict__ lengths,
                                                   float* __restrict__ mass, int B, int lmax,
                                                   int Np, int N) {
  __shared__ float red[33];
  const long long row = rowbase(2, B, lmax) + blockIdx.x;
  int w = 2;
  while (w < lmax && row >= rowbase(w + 1, B, lmax)) ++w;
  const int n_w = lmax - w + 1;
  const long long local = row - rowbase(w, B, lmax);
  const int b = static_cast<int>(local / n_w), i = static_cast<int>(local % n_w);
  const bool ok = i + w <= lengths[b] && g[b] != 0.f;
  const float lg = ok ? log2f(fabsf(g[b])) : 0.f;
  float s = 0.f;
  if (ok && (N & 3) == 0) {  // 4 columns per thread: 8-B / 16-B loads
    const float* orow = O + row * Np;
    for (int c = 4 * threadIdx.x; c < N; c += 4 * blockDim.x) {
      const float4 o = __ldg(reinterpret_cast<const float4*>(orow + c));
      if constexpr (kHalfLQ) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(LQv) +
                                                             row * Np + c));
        const float2 q01 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
        const float2 q23 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
        const float e = LQS[row * (Np / 32) + c / 32] - lg;
        s += q01.x * exp2f(e + o.x) + q01.y * exp2f(e + o.y) + q23.x * exp2f(e + o.z) +
             q23.y * exp2f(e + o.w);
      } else {
        const float4 q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(LQv) +
                                                               row * Np + c));
        s += exp2f(q.x + o.x - lg) + exp2f(q.y + o.y - lg) + exp2f(q.z + o.z - lg) +
             exp2f(q.w + o.w - lg);
      }
    }
  } else if (ok) {
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      if constexpr (kHalfLQ) {
        const float q = __half2float(static_cast<const __half*>(LQv)[row * Np + c]);
        s += q * exp2f(LQS[row * (Np / 32) + c / 32] + O[row * Np + c] - lg);
      } else {
        s += exp2f(static_cast<const float*>(LQv)[row * Np + c] + O[row * Np + c] - lg);
      }
    }
  }
  s = block_reduce<false>(s, red);
  if (threadIdx.x == 0) mass[blockIdx.x] = s;
}

// MBR CKY per sentence (parse.py:98-131): score(i,i+1) = 0,
// score(i,j) = mass(i,j) + max_k score(i,k) + score(k,j), ties -> smallest k.
// One CTA per sentence; score / split tables are (lmax) x (lmax + 1), index
// i * (lmax + 1) + j; widths are a sequential sweep (block barrier each).
__global__ void __launch_bounds__(256) k_mbr_cky(const float* __restrict__ mass,
                                                 const int* __restrict__ lengths,
                                                 float* __restrict__ score,
                                                 int* __restrict__ split, int B, int lmax) {
  const int b = blockIdx.x;
  const int len = lengths[b];
  if (len < 2 || len > lmax) return;  // invalid sentence: no tree (the host refuses it)
  const int ld = lmax + 1;
  float* sc = score + static_cast<long long>(b) * lmax * ld;
  int* sp = split + static_cast<long long>(b) * lmax * ld;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    sc[i * ld + i + 1] = 0.f;
    sp[i * ld + i + 1] = 0;
  }
  __syncthreads();
  const long long base2 = rowbase(2, B, lmax);
  for (int w = 2; w <= len; ++w) {
    const int n_w = lmax - w + 1;
    const float* mw = mass + (rowbase(w, B, lmax) - base2) + static_cast<long long>(b) * n_w;
    for (int i = threadIdx.x; i + w <= len; i += blockDim.x) {
      const int j = i + w;
      int best_k = i + 1;
      float best = -__builtin_huge_valf();
      for (int k = i + 1; k < j; ++k) {
        const float s = sc[i * ld + k] + sc[k * ld + j];
        if (s > best) {
          best = s;
          best_k = k;
        }
      }
      sc[i * ld + j] = mw[i] + best;
      sp[i * ld + j] = best_k;
    }
    __syncthreads();
  }
}

}  // namespace fi

namespace fi {

// ---------------------------------------------------------------------------
// Viterbi (parse.py:33-95): the inside recursion in the (max, +) semiring.
// Chart rows as in the inside pass (row(w, b, i)); log values in fp32 (no
// shifts: max-plus never exponentiates).
//   project:  va[r, A] = max_k (L[A, k] + vo[r, k]), vb likewise with R
//             (k over the live block: preterminals at width 1, else
//             nonterminals) -- a tropical GEMM on the CUDA cores
//   split:    vo[r, A] = max_m va[m][i, A] + vb[w-m][i+m, A]
//   root:     argmax_A root[A] + vo[top][A]
//   backtrack per sentence on the device: smallest maximising split, then
//             the maximising child symbols (ties -> smallest index).
// ---------------------------------------------------------------------------

// C[r, c] = max_k A[r, k] + W[c, k] for r < M, c < Ncols; A row stride lda,
// W row stride ldw (K-major both).  64 x 64 tile per CTA, 256 threads x 4x4
// outputs, K staged through shared memory in slices of 32.  Output columns
// [0, Nhalf) go to outA, [Nhalf, 2 Nhalf) to outB (row stride ldo).
constexpr int kTropTile = 64;
constexpr int kTropK = 32;
__global__ void __launch_bounds__(256) k_trop_gemm(const float* __restrict__ A, int lda,
                                                   const float* __restrict__ W, int ldw, int M,
                                                   int Ncols, int K, float* __restrict__ outA,
                                                   float* __restrict__ outB, int Nhalf,
                                                   int ldo) {
  __shared__ float sa[kTropK][kTropTile + 4];
  __shared__ float sw[kTropK][kTropTile + 4];
  const int r0 = blockIdx.y * kTropTile, c0 = blockIdx.x * kTropTile;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = kNegInf;
  for (int k0 = 0; k0 < K; k0 += kTropK) {
    // stage a 64 x 32 slice of A and of W (transposed: [k][row])
    for (int e = threadIdx.x; e < kTropTile * kTropK; e += 256) {
      const int rr = e / kTropK, kk = e % kTropK;
      const int gr = r0 + rr, gc = c0 + rr, gk = k0 + kk;
      sa[kk][rr] = (gr < M && gk < K) ? A[static_cast<long long>(gr) * lda + gk] : kNegInf;
      sw[kk][rr] = (gc < Ncols && gk < K) ? W[static_cast<long long>(gc) * ldw + gk] : kNegInf;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kTropK; ++kk) {
      float av[4], wv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[kk][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) wv[b] = sw[kk][tx * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaxf(acc[a][b], av[a] + wv[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = r0 + ty * 4 + a;
    if (r >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = c0 + tx * 4 + b;
      if (c >= Ncols) continue;
      if (c < Nhalf) outA[static_cast<long long>(r) * ldo + c] = acc[a][b];
      else outB[static_cast<long long>(r) * ldo + c - Nhalf] = acc[a][b];
    }
  }
}

// Register-tiled tropical GEMM for the Viterbi projections, both tables in
// one launch:  out[r, c] = max_k A[r, k] + W(c)[k]  with W(c) = W0 row c for
// c < Nhalf (-> outA) and W1 row c - Nhalf (-> outB).  BM x 128 tiles,
// K slices of 16 staged in shared memory as k-PAIRS ([k/2][row][k%2]; the
// next slice prefetched into registers during the current one), 256 threads
// with (BM/16) x 8 results each in 4 x 4 blocks (rows ty*4 (+BM/2), cols
// tx*4 (+64)).  Two K steps of one result cost one packed FADD2 (the two
// sums) and one three-input FMNMX3 (sm_100): 1 instruction per max-plus op
// instead of 2.  `vec`: A, W rows 16-B aligned (float4 global loads).
__device__ __forceinline__ float2 trop_add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float trop_max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int BM>
__global__ void __launch_bounds__(256, BM == 64 ? 2 : 1) k_trop_gemm2(const float* __restrict__ A, int lda,
                                                    const float* __restrict__ W0,
                                                    const float* __restrict__ W1, int ldw, int M,
                                                    int Nhalf, int K, float* __restrict__ outA,
                                                    float* __restrict__ outB, int ldo, int vec) {
  constexpr int BN = 128, BK = 16, KP = BK / 2;
  constexpr int RB = BM / 64;            // row blocks of 4 per thread (1 or 2)
  constexpr int NA = BM * BK / 4 / 256;  // float4 loads of A per thread per slice
  constexpr int NW = BN * BK / 4 / 256;
  __shared__ __align__(16) float sa[KP][2 * BM + 8];  // [k pair][row][k % 2]
  __shared__ __align__(16) float sw[KP][2 * BN + 8];
  const int Ncols = 2 * Nhalf;
  const int r0 = blockIdx.y * BM, c0 = blockIdx.x * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4 * RB][8];
#pragma unroll
  for (int i = 0; i < 4 * RB; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = kNegInf;
  float4 ra[NA], rw[NW];
  auto ld4 = [&](const float* row, int gk, bool ok) -> float4 {
    if (!ok) return make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
    if (vec && gk + 3 < K) return __ldg(reinterpret_cast<const float4*>(row + gk));
    float4 v;
    v.x = gk < K ? __ldg(row + gk) : kNegInf;
    v.y = gk + 1 < K ? __ldg(row + gk + 1) : kNegInf;
    v.z = gk + 2 < K ? __ldg(row + gk + 2) : kNegInf;
    v.w = gk + 3 < K ? __ldg(row + gk + 3) : kNegInf;
    return v;
  };
  auto gload = [&](int k0) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = threadIdx.x + q * 256, rr = e / 4, gk = k0 + (e % 4) * 4;
      const int gr = r0 + rr;
      ra[q] = ld4(A + static_cast<long long>(gr < M ? gr : 0) * lda, gk, gr < M);
    }
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const int e = threadIdx.x + q * 256, cc = e / 4, gk = k0 + (e % 4) * 4;
      const int gc = c0 + cc;
      const float* wr = gc < Nhalf ? W0 + static_cast<long long>(gc) * ldw
                                   : W1 + static_cast<long long>(gc < Ncols ? gc - Nhalf : 0) * ldw;
      rw[q] = ld4(wr, gk, gc < Ncols);
    }
  };
  auto sstore = [&]() {  // four consecutive k of one row -> two k pairs
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      const int e = threadIdx.x + q * 256, rr = e / 4, kp = (e % 4) * 2;
      *reinterpret_cast<float2*>(&sa[kp][2 * rr]) = make_float2(ra[q].x, ra[q].y);
      *reinterpret_cast<float2*>(&sa[kp + 1][2 * rr]) = make_float2(ra[q].z, ra[q].w);
    }
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const int e = threadIdx.x + q * 256, cc = e / 4, kp = (e % 4) * 2;
      *reinterpret_cast<float2*>(&sw[kp][2 * cc]) = make_float2(rw[q].x, rw[q].y);
      *reinterpret_cast<float2*>(&sw[kp + 1][2 * cc]) = make_float2(rw[q].z, rw[q].w);
    }
  };
  gload(0);
  for (int k0 = 0; k0 < K; k0 += BK) {
    __syncthreads();  // the previous slice is consumed
    sstore();
    __syncthreads();
    if (k0 + BK < K) gload(k0 + BK);  // in flight during this slice
#pragma unroll
    for (int kp = 0; kp < KP; ++kp) {
      float2 a[4 * RB], w[8];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        const float4* src = reinterpret_cast<const float4*>(&sa[kp][2 * (ty * 4 + rb * (BM / 2))]);
        const float4 u = src[0], v = src[1];
        a[4 * rb] = make_float2(u.x, u.y);
        a[4 * rb + 1] = make_float2(u.z, u.w);
        a[4 * rb + 2] = make_float2(v.x, v.y);
        a[4 * rb + 3] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        const float4* src = reinterpret_cast<const float4*>(&sw[kp][2 * (tx * 4 + cb * 64)]);
        const float4 u = src[0], v = src[1];
        w[4 * cb] = make_float2(u.x, u.y);
        w[4 * cb + 1] = make_float2(u.z, u.w);
        w[4 * cb + 2] = make_float2(v.x, v.y);
        w[4 * cb + 3] = make_float2(v.z, v.w);
      }
#pragma unroll
      for (int i = 0; i < 4 * RB; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 t = trop_add2(a[i], w[j]);
          acc[i][j] = trop_max3(acc[i][j], t.x, t.y);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 4 * RB; ++i) {
    const int r = r0 + ty * 4 + (i & 3) + (i >> 2) * (BM / 2);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + tx * 4 + (j & 3) + (j >> 2) * 64;
      if (c >= Ncols) continue;
      if (c < Nhalf) outA[static_cast<long long>(r) * ldo + c] = acc[i][j];
      else outB[static_cast<long long>(r) * ldo + c - Nhalf] = acc[i][j];
    }
  }
}

// vo[row(w, b, i), A] = max_m va[m][b, i, A] + vb[w-m][b, i+m, A]; padded spans -inf.
__global__ void __launch_bounds__(256) k_vit_split(const float* __restrict__ VA,
                                                   const float* __restrict__ VB,
                                                   float* __restrict__ VO,
                                                   const int* __restrict__ lengths, int B,
                                                   int lmax, int w, int Np) {
  const int local = blockIdx.y;
  const int n_w = lmax - w + 1;
  const int b = local / n_w, i = local % n_w;
  const long long row = rowbase(w, B, lmax) + local;
  const int c = 4 * (blockIdx.x * blockDim.x + threadIdx.x);  // 4 columns per thread (Np % 4 == 0)
  if (c >= Np) return;
  float4 best = make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
  if (i + w <= lengths[b]) {
    for (int m = 1; m < w; ++m) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(VA + chart_row(m, b, i, B, lmax) * Np + c));
      const float4 y =
          __ldg(reinterpret_cast<const float4*>(VB + chart_row(w - m, b, i + m, B, lmax) * Np + c));
      best.x = fmaxf(best.x, x.x + y.x);
      best.y = fmaxf(best.y, x.y + y.y);
      best.z = fmaxf(best.z, x.z + y.z);
      best.w = fmaxf(best.w, x.w + y.w);
    }
  }
  *reinterpret_cast<float4*>(VO + row * Np + c) = best;
}

// Per sentence: root argmax, then the derivation top-down.  Output per
// sentence: nodes[b][k] = (i, j, sym) for the 2 len - 1 nodes (internal
// nodes carry a nonterminal, leaves a preterminal index), root first.
// L/R are the (N, N+P) log tables; VO width-1 rows hold the unary
// (preterminal) scores in columns [0, P) (row stride Pp), wider rows the
// nonterminal scores (row stride Np).
__global__ void __launch_bounds__(256) k_vit_backtrack(
    const float* __restrict__ VA, const float* __restrict__ VB, const float* __restrict__ VO,
    const float* __restrict__ VO1, const float* __restrict__ L, const float* __restrict__ R,
    const float* __restrict__ root, const int* __restrict__ lengths, int* __restrict__ nodes,
    float* __restrict__ best_score, int B, int lmax, int N, int P, int Np, int Pp) {
  __shared__ float sval[256];
  __shared__ int sidx[256];
  __shared__ int stack[3 * 1024];
  __shared__ int top;
  const int b = blockIdx.x;
  const int len = lengths[b];
  int* out = nodes + static_cast<long long>(b) * (2 * lmax) * 3;
  auto argmax = [&](float v, int idx) {  // block argmax, ties -> smallest index
    sval[threadIdx.x] = v;
    sidx[threadIdx.x] = idx;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) {
        const float o = sval[threadIdx.x + s];
        const int oi = sidx[threadIdx.x + s];
        if (o > sval[threadIdx.x] || (o == sval[threadIdx.x] && oi < sidx[threadIdx.x])) {
          sval[threadIdx.x] = o;
          sidx[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    const int r = sidx[0];
    const float rv = sval[0];
    __syncthreads();
    return make_float2(rv, __int_as_float(r));
  };
  if (len < 2 || len > lmax) {  // invalid sentence: NaN score, no nodes (the host refuses it)
    if (threadIdx.x == 0) best_score[b] = __int_as_float(0x7fc00000);
    for (int k = threadIdx.x; k < 2 * lmax * 3; k += blockDim.x) out[k] = -1;
    return;
  }
  // root symbol
  float v = kNegInf;
  int vi = 0x7fffffff;
  const long long top_row = chart_row(len, b, 0, B, lmax);
  for (int a = threadIdx.x; a < N; a += blockDim.x) {
    const float s = (len == 1 ? kNegInf : root[a] + VO[top_row * Np + a]);
    if (s > v || (s == v && a < vi)) {
      v = s;
      vi = a;
    }
  }
  float2 r = argmax(v, vi);
  if (threadIdx.x == 0) {
    best_score[b] = r.x;
    stack[0] = 0;
    stack[1] = len;
    stack[2] = __float_as_int(r.y);
    top = 1;
  }
  __syncthreads();
  int nout = 0;
  while (true) {
    __syncthreads();
    if (top == 0) break;
    const int i = stack[3 * (top - 1)], j = stack[3 * (top - 1) + 1],
              sym = stack[3 * (top - 1) + 2];
    __syncthreads();
    if (threadIdx.x == 0) {
      --top;
      out[3 * nout] = i;
      out[3 * nout + 1] = j;
      out[3 * nout + 2] = sym;
    }
    ++nout;
    const int w = j - i;
    if (w == 1) continue;  // leaf: sym is a preterminal index
    // smallest maximising split (parse.py:62-64 argmax over m)
    v = kNegInf;
    vi = 0x7fffffff;
    for (int m = 1 + threadIdx.x; m < w; m += blockDim.x) {
      const float s = VA[chart_row(m, b, i, B, lmax) * Np + sym] +
                      VB[chart_row(w - m, b, i + m, B, lmax) * Np + sym];
      if (s > v || (s == v && m < vi)) {
        v = s;
        vi = m;
      }
    }
    const int k = __float_as_int(argmax(v, vi).y);
    // children: argmax over the live symbols of L[sym, s] + vo[k][i, s]
    int child[2];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int ci = side ? i + k : i;
      const int cw = side ? w - k : k;
      const float* tab = (side ? R : L) + static_cast<long long>(sym) * (N + P);
      v = kNegInf;
      vi = 0x7fffffff;
      if (cw == 1) {  // preterminal child: columns N + t
        const float* u = VO1 + (static_cast<long long>(b) * lmax + ci) * Pp;
        for (int t = threadIdx.x; t < P; t += blockDim.x) {
          const float s = tab[N + t] + u[t];
          if (s > v || (s == v && t < vi)) {
            v = s;
            vi = t;
          }
        }
      } else {
        const float* o = VO + chart_row(cw, b, ci, B, lmax) * Np;
        for (int a = threadIdx.x; a < N; a += blockDim.x) {
          const float s = tab[a] + o[a];
          if (s > v || (s == v && a < vi)) {
            v = s;
            vi = a;
          }
        }
      }
      child[side] = __float_as_int(argmax(v, vi).y);
    }
    if (threadIdx.x == 0) {  // push right then left: left subtree is emitted first
      stack[3 * top] = i + k;
      stack[3 * top + 1] = j;
      stack[3 * top + 2] = child[1];
      stack[3 * top + 3] = i;
      stack[3 * top + 4] = i + k;
      stack[3 * top + 5] = child[0];
      top += 2;
    }
  }
}

}  // namespace fi
