// Score tables of the grammar parameterisations: the
// row log-softmax of a product A B^T and its backward, around the engine's
// own tcgen05 GEMM (fi_gemm.cuh).  Reference: neuralparam.py:185-189
// (log_left = log_softmax(f3 f2^T), log_right = log_softmax(f3 f4^T)) and the
// matching part of backward_params (neuralparam.py:242-320: the softmax
// backward, then the gradients of the two embedding factors).
//
// Kernels here are the bandwidth passes; the products are k_gemm launches:
//   forward   C = A B^T (EPI_STORE, fp32, padded columns), then
//             k_row_log_softmax: logp = C - logsumexp_row(C)
//   backward  k_row_softmax_bwd: g = dlogp - exp(logp) * rowsum(dlogp)
//             (written in the GEMM operand type: fp32 for tf32, bf16 hi / lo
//             planes for the fp32 mode's split products), then
//             dA = g B (K-major g, MN-major B) and dB = g^T A (both MN-major).
#pragma once

#include "fi_kernels.cuh"

namespace fi {

// x -> (hi, lo) bf16 planes (hi = bf16(x), lo = bf16(x - hi)) of a row-major
// (rows x cols) matrix into a (rows x ld) padded destination; padding = 0.
// T = float copies (tf32 operands), lo unused.
template <typename T>
__global__ void __launch_bounds__(256) k_pack_rows(const float* __restrict__ src, int rows,
                                                   int cols, T* __restrict__ dst, int ld,
                                                   long long lo) {
  const long long n = static_cast<long long>(rows) * ld;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / ld), c = static_cast<int>(i % ld);
    store1s<T>(dst + i, lo, c < cols ? src[static_cast<long long>(r) * cols + c] : 0.f);
  }
}

// One CTA per row: logp[r, :cols] = x[r, :cols] - logsumexp(x[r, :cols])
// (x row stride ldx, logp row stride cols; x may alias logp).  Rows of up
// to kRowVec x 4 x blockDim columns (a multiple of 4, 16-B aligned rows) are
// read once into registers as float4 (VEC); other shapes take three strided
// passes.  An all -inf row stays -inf.
constexpr int kRowVec = 8;
template <bool VEC>
__global__ void __launch_bounds__(512) k_row_log_softmax(const float* x, int ldx, float* logp,
                                                         int cols) {
  __shared__ float red[33];
  const float* xr = x + static_cast<long long>(blockIdx.x) * ldx;
  float* out = logp + static_cast<long long>(blockIdx.x) * cols;
  if constexpr (VEC) {
    float4 v[kRowVec];
    float mx = kNegInf;
#pragma unroll
    for (int k = 0; k < kRowVec; ++k) {
      const int c = 4 * (threadIdx.x + k * blockDim.x);
      v[k] = c < cols ? *reinterpret_cast<const float4*>(xr + c)
                      : make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
      mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
    }
    mx = block_reduce<true>(mx, red);
    const float sh = mx == kNegInf ? 0.f : mx;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kRowVec; ++k)
      s += (expf(v[k].x - sh) + expf(v[k].y - sh)) + (expf(v[k].z - sh) + expf(v[k].w - sh));
    s = block_reduce<false>(s, red);
    const float lse = sh + logf(s);
#pragma unroll
    for (int k = 0; k < kRowVec; ++k) {
      const int c = 4 * (threadIdx.x + k * blockDim.x);
      if (c < cols)
        *reinterpret_cast<float4*>(out + c) =
            make_float4(v[k].x - lse, v[k].y - lse, v[k].z - lse, v[k].w - lse);
    }
  } else {
    float mx = kNegInf;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, xr[c]);
    mx = block_reduce<true>(mx, red);
    const float sh = mx == kNegInf ? 0.f : mx;
    float s = 0.f;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) s += expf(xr[c] - sh);
    s = block_reduce<false>(s, red);
    const float lse = sh + logf(s);
    for (int c = threadIdx.x; c < cols; c += blockDim.x) out[c] = xr[c] - lse;
  }
}

// One CTA per row: g[r, c] = dlogp[r, c] - exp(logp[r, c]) * sum_c' dlogp[r, c']
// (the log-softmax backward), written into the GEMM operand (row stride ldg,
// padding columns 0; T = bf16 writes hi / lo planes `lo` elements apart).
// VEC: dlogp held in registers as float4 (cols and ldg multiples of 4,
// cols <= kRowVec x 4 x blockDim).
template <typename T, bool VEC>
__global__ void __launch_bounds__(512) k_row_softmax_bwd(const float* __restrict__ logp,
                                                         const float* __restrict__ dlogp,
                                                         int cols, T* __restrict__ g, int ldg,
                                                         long long lo) {
  __shared__ float red[33];
  const long long r = blockIdx.x;
  const float* lp = logp + r * cols;
  const float* dl = dlogp + r * cols;
  T* gr = g + r * ldg;
  if constexpr (VEC) {
    float4 v[kRowVec];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kRowVec; ++k) {
      const int c = 4 * (threadIdx.x + k * blockDim.x);
      v[k] = c < cols ? __ldg(reinterpret_cast<const float4*>(dl + c)) : make_float4(0, 0, 0, 0);
      s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    }
    s = block_reduce<false>(s, red);
#pragma unroll
    for (int k = 0; k < kRowVec; ++k) {
      const int c = 4 * (threadIdx.x + k * blockDim.x);
      if (c < cols) {
        const float4 p = __ldg(reinterpret_cast<const float4*>(lp + c));
        store4s<T>(gr + c, lo, fmaf(-expf(p.x), s, v[k].x), fmaf(-expf(p.y), s, v[k].y),
                   fmaf(-expf(p.z), s, v[k].z), fmaf(-expf(p.w), s, v[k].w));
      } else if (c < ldg) {
        store4s<T>(gr + c, lo, 0.f, 0.f, 0.f, 0.f);
      }
    }
    for (int c = 4 * (threadIdx.x + kRowVec * blockDim.x); c < ldg; c += 4 * blockDim.x)
      store4s<T>(gr + c, lo, 0.f, 0.f, 0.f, 0.f);
  } else {
    float s = 0.f;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) s += dl[c];
    s = block_reduce<false>(s, red);
    for (int c = threadIdx.x; c < ldg; c += blockDim.x)
      store1s<T>(gr + c, lo, c < cols ? fmaf(-expf(lp[c]), s, dl[c]) : 0.f);
  }
}

// dst (rows x cols) = src (rows x lds) columns [0, cols).
__global__ void __launch_bounds__(256) k_copy_cols(const float* __restrict__ src, int lds,
                                                   float* __restrict__ dst, int rows, int cols) {
  const long long n = static_cast<long long>(rows) * cols;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cols;
    dst[i] = src[r * lds + i % cols];
  }
}

}  // namespace fi
