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
  if (ok) {
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
