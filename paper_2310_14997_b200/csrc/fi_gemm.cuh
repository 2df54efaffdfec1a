// Persistent, warp-specialised tcgen05 GEMM for sm_100a with fused
// FlashInside epilogues.
//
//   C[M, N] = A[M, K] * B[N, K]^T        (fp32 accumulate in TMEM)
//
// A and B are staged by TMA into 128B-swizzled shared memory; either operand
// may be K-major (rows of K contiguous) or MN-major (rows of MN contiguous,
// i.e. the K index is the outer, strided dimension).  One elected thread
// issues tcgen05.mma (K=16 for bf16 / 8 for tf32) into one of two TMEM
// accumulators, so the epilogue of tile t overlaps the main loop of tile
// t+1 (N tiles up to 256).  N tiles of 320..512 (BN = 512 kernels, pairs
// only) issue two MMAs per K step (sub-tiles of 256 + the rest) into one
// TMEM-filling accumulator: 25% fewer operand bytes per flop than 256-wide
// tiles, which are bound by the per-SM L2 -> shared fill rate, at the cost
// of a serialized epilogue.  The epilogue reads TMEM with tcgen05.ld and
// applies one of the inside-algorithm transforms (see EpiMode) before
// writing to HBM.
//
// PAIR: a cluster of two CTAs (one TPC) computes a 256 x bn tile with
// tcgen05.mma.cta_group::2 -- each CTA stages its own 128 rows of A and
// half (bn/2 rows) of B, so the L2 -> SM operand traffic per flop drops by a
// third against single-CTA 128 x bn tiles (the measured limit of those: the
// chip's TMA/L2 read rate, not the tensor pipe).  The leader CTA (rank 0)
// issues the MMAs; both CTAs' TMA loads complete on the leader's full
// barriers, MMA commits multicast to both CTAs' empty / TMEM-full barriers,
// and both CTAs' epilogue warps release the leader's TMEM-empty barrier.
//
// Warp roles (256 threads): w0 = TMA producer, w1 = MMA issuer,
// w2 = TMEM allocator, w4..w7 = epilogue (TMEM lane quadrant = warp % 4).
#pragma once
#include "fi_ptx.cuh"

namespace fi {

// All log values are base 2 and stored as fp32 offsets from the span row's
// fp64 shift x† (see fi_kernels.cuh), so the epilogues below need no x†.
enum EpiMode : int {
  EPI_FWD = 0,     // [a | b] - x† = log2(acc)                     (inside.py:203-213)
  EPI_DGRAD = 1,   // LQ^ = log2|acc| (= log2|go| - o + x†)        (inside.py:433-447)
  EPI_DUNARY = 2,  // dunary = acc * exp(unary - x†) (width-1 go)  (inside.py:420-423)
  EPI_WGRAD = 3,   // d{L,R} = exp({L,R}) * acc                    (inside.py:446)
  EPI_STORE = 4,   // plain C = acc (GEMM unit tests)
  EPI_FWD_H = 5,   // [a | b] as fp16 acc * 2^kChartScale (half chart, fi_kernels.cuh)
  EPI_DGRAD_H = 6, // |acc| as fp16 per-32-column scaled + exponent (half chart)
};

struct GemmShape {
  int M, N, K;    // logical problem; rows >= M are masked in the epilogue
  int a_row0;     // K-major A: first row coordinate inside the tensor map
  int b_row0;     // K-major B: first row coordinate (TR: the chart rows are the B operand)
  int num_m, num_n, num_k;  // tiles of (128 or 256 for pairs) x bn x BK
  int bn;         // N tile (runtime, <= the kernel's BN bound, multiple of 32)
  int stages;     // smem ring depth (runtime: as many as fit in shared memory)
  int b_stage;    // bytes of one B stage in this CTA (128 B of K x bn / NCTA rows)
  // split-K (ksplit > 1): work unit u = (tile tile_begin + u / ksplit, K part
  // u % ksplit); each unit stores its raw fp32 partial tile, dense
  // (tile_rows x bn), at part + ((kpart * T_split + tile - tile_begin) *
  // tile_rows * bn); the parts are summed in order (deterministic) by the
  // tile's own CTAs (sem != null, below) or by k_gemm_fixup, which then
  // apply the epilogue.
  int ksplit;
  float* part;
  // non-null (FI_GEMM_INKERNEL_RED=1; default: the k_gemm_fixup kernel): the
  // ksplit CTAs (x NCTA) of a split tile reduce it in-kernel --
  // each publishes its partial, waits on the tile's counter sem[tile - tile_begin]
  // (zero on entry, left zero on exit) and then sums every part, in part
  // order, over its own 1/ksplit of the tile's columns and runs the epilogue.
  // Needs all units resident (units <= slots; one unit per CTA).
  int* sem;
  // tiles [tile_begin, tile_end) only (tile_end 0: all; a "waves + split-K
  // tail" GEMM is two launches over one shape: whole waves, then the tail
  // split over K)
  int tile_begin, tile_end;
  // stream-K (sk > 0: the persistent slot count, ksplit 1): tiles
  // [0, sk_first) run whole (sk_first is a multiple of sk, so every slot
  // gets the same number), and the K iterations of the last tiles
  // [sk_first, T) (at most sk of them) are cut into sk equal contiguous
  // runs, one per slot.  A run spans at most two tiles; each of its
  // segments that does not end its tile stores a raw partial at
  // part + (slot + seg * sk) * tile_rows * bn and counts itself on
  // sem[tile - sk_first]; the segment that ends the tile waits for its
  // tile's other segments, adds their partials to its accumulator in slot
  // order and runs the epilogue (and re-arms the counter).  A slot runs its
  // non-final segment first, so no wait ever waits on a waiting CTA.
  int sk, sk_first;
};

// Work unit i of persistent slot `slot`: tile, K range [k0, k1) (empty:
// skip) and the partial-tile slot (-1: the epilogue writes the output).
struct GemmUnit {
  int tile, k0, k1, pidx;
  int skt;  // stream-K: tile index within the stream-K tiles, else -1
};
__device__ __forceinline__ bool gemm_unit(const GemmShape& sh, int slot, int nslot, int i, int ks,
                                          int k_iters, int tb, int tile_e, GemmUnit& x) {
  x.skt = -1;
  x.pidx = -1;
  if (sh.sk > 0) {
    const int ndp = sh.sk_first / nslot;  // whole tiles per slot
    if (i < ndp) {
      x.tile = slot + i * nslot;
      x.k0 = 0;
      x.k1 = k_iters;
      return true;
    }
    const int j = i - ndp;
    if (j >= 2) return false;
    const long long W = static_cast<long long>(tile_e - sh.sk_first) * k_iters;
    const long long st = W * slot / nslot, en = W * (slot + 1) / nslot;
    const int ta = static_cast<int>(st / k_iters);
    const bool two = en > static_cast<long long>(ta + 1) * k_iters;
    // order: the segment in the next tile (never final unless it fills it) first
    const int seg = two ? 1 - j : (j == 0 ? 0 : -1);
    if (seg < 0 || en <= st) {
      x.tile = tb;
      x.k0 = x.k1 = 0;
      return true;
    }
    const long long t0 = static_cast<long long>(ta + seg) * k_iters;
    const long long a = seg == 0 ? st : t0;
    const long long b = en < t0 + k_iters ? en : t0 + k_iters;
    x.skt = ta + seg;
    x.tile = sh.sk_first + x.skt;
    x.k0 = static_cast<int>(a - t0);
    x.k1 = static_cast<int>(b - t0);
    x.pidx = slot + seg * nslot;
    return true;
  }
  const int u = slot + i * nslot;
  if (u >= (tile_e - tb) * ks) return false;
  const int tu = u / ks, kp = u - tu * ks;
  x.tile = tb + tu;
  x.k0 = k_iters * kp / ks;
  x.k1 = k_iters * (kp + 1) / ks;
  x.pidx = ks > 1 ? kp * (tile_e - tb) + tu : -1;
  return true;
}

// Stream-K: the partial slots of stream-K tile `skt`'s segments, in slot
// order, except `own`; returns their count (<= 15).
__device__ __forceinline__ int sk_parts(const GemmShape& sh, int skt, int nslot, int k_iters,
                                        int tile_e, int own, int (&pid)[16]) {
  const long long W = static_cast<long long>(tile_e - sh.sk_first) * k_iters;
  const long long lo = static_cast<long long>(skt) * k_iters, hi = lo + k_iters;
  long long s = lo * nslot / W;
  s = s > 0 ? s - 1 : 0;
  int n = 0;
  for (; s < nslot && n < 16; ++s) {
    const long long st = W * s / nslot, en = W * (s + 1) / nslot;
    if (st >= hi) break;
    if (en <= lo || en <= st) continue;
    const int p = static_cast<int>(s) + (st >= lo ? 0 : 1) * nslot;
    if (p != own) pid[n++] = p;
  }
  return n;
}

struct GemmEpi {
  int M;              // valid output rows
  long long row0;     // global chart row of output row 0 (X / chart indexing)
  const double* X;    // per-row log2 shift x† (indexed by global row)
  // EPI_FWD
  float* outA;
  float* outB;
  int Np;             // padded nonterminal count == row stride of chart arrays
  // EPI_DGRAD (EPI_DGRAD_H: LQ is the fp16 array, LQS its per-32-column exponents)
  float* LQ;
  float* LQS;
  const int* lengths;
  int width;
  int n_w;
  int b0;             // first sentence of this launch's row range (DGRAD top-span check)
  // EPI_DUNARY
  float* dunary;
  const float* unary;
  int P;
  int lmax;
  // EPI_WGRAD
  const float* Lsrc;
  const float* Rsrc;
  float* dL;
  float* dR;
  int n_nt;
  int ld_lr;          // row stride of L/R/dL/dR (= N + P)
  int col_off;        // 0 for the NN block, N for the NP block
  int valid_cols;     // N or P
  int m_off;          // output row of this launch's row 0 (0..2Np: a launch may cover
                      // only the dR half, so dL can be all-reduced while it runs)
  // EPI_STORE
  float* C;
  int ldc;
  int vec4;           // EPI_DUNARY / EPI_WGRAD rows 16-B aligned: vector loads/stores
};

template <typename T, int BN>  // BN: the largest N tile the smem ring is sized for
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int kElt = static_cast<int>(sizeof(T));
  static constexpr int BK = 128 / kElt;            // one 128-B swizzle row of K
  static constexpr int UK = 32 / kElt;             // K per tcgen05.mma
  static constexpr int ATOM = 128 / kElt;          // MN elements per 128-B atom
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024 / STAGE_BYTES) > 8 ? 8 : (200 * 1024 / STAGE_BYTES);
  // accumulator columns: two buffers of BN (double-buffered) up to BN = 256;
  // BN = 512 (pair tiles 256 x 512) fills TMEM with one buffer
  static constexpr int TMEM_COLS = 2 * BN > 512 ? 512 : 2 * BN;
  static constexpr int TMEM_HALF = TMEM_COLS / 2;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr bool TF32 = (kElt == 4);
};

// Row-wise epilogue for one 32-column chunk of one accumulator row.
template <int EPI>
__device__ __forceinline__ void epi_chunk(const GemmEpi& ep, int lrow, long long grow, int col,
                                          const float (&v)[32], float xv, bool row_ok,
                                          float* rowptr, int aux) {
  if (!row_ok) return;
  if constexpr (EPI == EPI_FWD) {
    float4* dst = reinterpret_cast<float4*>(rowptr + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 o;
      o.x = lg2(v[4 * q + 0]);
      o.y = lg2(v[4 * q + 1]);
      o.z = lg2(v[4 * q + 2]);
      o.w = lg2(v[4 * q + 3]);
      dst[q] = o;
    }
  } else if constexpr (EPI == EPI_FWD_H) {
    // rowptr is a __half row; the linear projection is already the stored value
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(rowptr) + col);
    constexpr float kScale = 16384.f;  // 2^kChartScale
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __half2 p2 = __floats2half2_rn(v[8 * q + 2 * h] * kScale, v[8 * q + 2 * h + 1] * kScale);
        w[h] = *reinterpret_cast<uint32_t*>(&p2);
      }
      dst[q] = u;
    }
  } else if constexpr (EPI == EPI_DGRAD_H) {
    float m = 0.f;
#pragma unroll
    for (int t = 0; t < 32; ++t) m = fmaxf(m, fabsf(v[t]));
    const int sc = lq_chunk_exp(m);
    const float f = exp2_int(-sc);
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(rowptr) + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __half2 p2 = __floats2half2_rn(fabsf(v[8 * q + 2 * h]) * f,
                                       fabsf(v[8 * q + 2 * h + 1]) * f);
        w[h] = *reinterpret_cast<uint32_t*>(&p2);
      }
      dst[q] = u;
    }
    ep.LQS[grow * (ep.Np / 32) + col / 32] = static_cast<float>(sc);
  } else if constexpr (EPI == EPI_DGRAD) {
    float4* dst = reinterpret_cast<float4*>(rowptr + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 o;
      o.x = lg2(fabsf(v[4 * q + 0]));
      o.y = lg2(fabsf(v[4 * q + 1]));
      o.z = lg2(fabsf(v[4 * q + 2]));
      o.w = lg2(fabsf(v[4 * q + 3]));
      dst[q] = o;
    }
  } else if constexpr (EPI == EPI_DUNARY) {
    // rowptr = dunary row, aux = 1 if the token position is inside the sentence
    const float* un = ep.unary + static_cast<long long>(lrow) * ep.P;
    if (ep.vec4 && col + 32 <= ep.P) {  // 16-B loads/stores (one 128-B line per thread)
      const float4* u4 = reinterpret_cast<const float4*>(un + col);
      float4* d4 = reinterpret_cast<float4*>(rowptr + col);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 u = __ldg(u4 + q);
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (aux) {
          o.x = v[4 * q + 0] * ex2(fmaf(u.x, 1.4426950408889634f, -xv));
          o.y = v[4 * q + 1] * ex2(fmaf(u.y, 1.4426950408889634f, -xv));
          o.z = v[4 * q + 2] * ex2(fmaf(u.z, 1.4426950408889634f, -xv));
          o.w = v[4 * q + 3] * ex2(fmaf(u.w, 1.4426950408889634f, -xv));
        }
        d4[q] = o;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        int c = col + t;
        if (c < ep.P) rowptr[c] = aux ? v[t] * ex2(fmaf(un[c], 1.4426950408889634f, -xv)) : 0.f;
      }
    }
  } else if constexpr (EPI == EPI_WGRAD) {
    // rowptr = d{L,R} row start; aux selects the right table; lrow = table row
    const float* lr = (aux ? ep.Rsrc : ep.Lsrc) + static_cast<long long>(lrow) * ep.ld_lr;
    if (ep.vec4 && col + 32 <= ep.valid_cols) {
      const float4* l4 = reinterpret_cast<const float4*>(lr + ep.col_off + col);
      float4* d4 = reinterpret_cast<float4*>(rowptr + ep.col_off + col);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 u = __ldg(l4 + q);
        d4[q] = make_float4(expf(u.x) * v[4 * q], expf(u.y) * v[4 * q + 1],
                            expf(u.z) * v[4 * q + 2], expf(u.w) * v[4 * q + 3]);
      }
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        int c = col + t;
        if (c < ep.valid_cols) {
          long long off = static_cast<long long>(ep.col_off + c);
          rowptr[off] = expf(lr[off]) * v[t];
        }
      }
    }
  } else {  // EPI_STORE (test hook; ldc is a multiple of 64, rows 16-B aligned)
    float4* dst = reinterpret_cast<float4*>(rowptr + col);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}

// Per-row epilogue state: where row `lrow` of this GEMM goes and what the
// fused transform needs (shared by the GEMM epilogue and the split-K reductions).
struct EpiRow {
  float* rowptr;    // row base (EPI_FWD/_H: the a row)
  float* rowptr_b;  // EPI_FWD/_H: the b row
  long long grow;   // global chart row
  float xv;
  int aux, erow;
  bool ok;
};

template <int EPI>
__device__ __forceinline__ EpiRow epi_row(const GemmEpi& ep, int lrow) {
  EpiRow r;
  r.grow = ep.row0 + lrow;
  r.xv = 0.f;
  r.aux = 0;
  r.rowptr = nullptr;
  r.rowptr_b = nullptr;
  const bool row_ok = lrow < ep.M;
  const long long grow = r.grow;
  if (row_ok) {
    if constexpr (EPI == EPI_FWD) {
      r.rowptr = ep.outA + grow * ep.Np;
      r.rowptr_b = ep.outB + grow * ep.Np;
    } else if constexpr (EPI == EPI_FWD_H) {
      r.rowptr = reinterpret_cast<float*>(reinterpret_cast<__half*>(ep.outA) + grow * ep.Np);
      r.rowptr_b = reinterpret_cast<float*>(reinterpret_cast<__half*>(ep.outB) + grow * ep.Np);
    } else if constexpr (EPI == EPI_DGRAD) {
      r.rowptr = ep.LQ + grow * ep.Np;
    } else if constexpr (EPI == EPI_DGRAD_H) {
      r.rowptr = reinterpret_cast<float*>(reinterpret_cast<__half*>(ep.LQ) + grow * ep.Np);
    } else if constexpr (EPI == EPI_DUNARY) {
      // width-1 rows: grow = b * lmax + i (rowbase(1) = 0)
      r.xv = static_cast<float>(ep.X[grow]);
      const int b = static_cast<int>(grow / ep.lmax), i = static_cast<int>(grow % ep.lmax);
      r.aux = i < ep.lengths[b];
      r.rowptr = ep.dunary + grow * ep.P;
    } else if constexpr (EPI == EPI_WGRAD) {
      const int mrow = lrow + ep.m_off;
      r.aux = mrow >= ep.Np;  // 0 -> left table, 1 -> right table
      const int arow = r.aux ? mrow - ep.Np : mrow;
      r.rowptr = (r.aux ? ep.dR : ep.dL) + static_cast<long long>(arow) * ep.ld_lr;
      if (arow >= ep.n_nt) r.rowptr = nullptr;
    } else {
      r.rowptr = ep.C + static_cast<long long>(lrow) * ep.ldc;
    }
  }
  r.ok = row_ok && r.rowptr != nullptr;
  if constexpr (EPI == EPI_DGRAD || EPI == EPI_DGRAD_H) {
    // the seed kernel owns the top span of each sentence (inside.py:400-404)
    if (r.ok) {
      const int b = ep.b0 + lrow / ep.n_w, i = lrow % ep.n_w;
      if (i == 0 && ep.lengths[b] == ep.width) r.ok = false;
    }
  }
  r.erow = EPI == EPI_WGRAD ? (r.aux ? lrow + ep.m_off - ep.Np : lrow + ep.m_off)
           : EPI == EPI_DUNARY ? static_cast<int>(grow) : lrow;
  return r;
}

// Epilogue of one 32-column chunk starting at GEMM column `col` (skips the N
// tail; the forward's [a | b] columns split at Np, possibly inside a tile).
template <int EPI>
__device__ __forceinline__ void epi_emit(const GemmEpi& ep, const EpiRow& r, int col, int N,
                                         const float (&v)[32]) {
  if (col >= N) return;
  float* rp = r.rowptr;
  if constexpr (EPI == EPI_FWD || EPI == EPI_FWD_H) {
    if (col >= ep.Np) {
      col -= ep.Np;
      rp = r.rowptr_b;
    }
  }
  epi_chunk<EPI>(ep, r.erow, r.grow, col, v, r.xv, r.ok, rp, r.aux);
}

// SPLIT (fp32 mode, bf16x3): each operand is stored as hi + lo bf16 planes
// (x = hi + lo to ~2^-17 relative).  One ring stage holds the hi and lo
// tiles of A and B for a K block and the MMA issuer runs its three products
// from it: lo*hi and hi*lo into a "small" accumulator, hi*hi into a "big"
// one (two TMEM accumulators per buffer, so the small terms never round
// against the big sum); the epilogue adds small + big per chunk.  Staging
// the four tiles once per K block moves 2/3 of the operand bytes of three
// separate passes (the per-SM fill rate is the GEMM's limit).
//
// CHUNK > 0: the tensor core accumulates in fp32 with truncation, a
// downward bias that grows with the number of MMA steps into one
// accumulator (~1.5e-5 relative at K = 8192) and compounds through the 40
// levels of the outside pass.  With CHUNK, every CHUNK K-iterations the
// accumulator is handed to the epilogue warps, which add it into a
// round-to-nearest fp32 register sum and hand it back (double-buffered), so
// the bias is bounded by the chunk length whatever K is.  Requires BN <= 128.
// Epilogue warps: one per TMEM lane quadrant (measured: a second set of 4
// splitting the columns does not shorten the step).
template <int CHUNK>
constexpr int gemm_epi_warps() { return 4; }
template <int CHUNK>
constexpr int gemm_threads() { return 128 + 32 * gemm_epi_warps<CHUNK>(); }

// MC (multicast clusters): a cluster of FOUR CTAs = two CTA pairs that work
// on the same 256 A rows and adjacent N tiles (a 256 x 2bn cluster tile).
// Each CTA loads only half of its 128 A rows and multicasts them to the CTA
// at the same pair position in the other pair, so a CTA fetches 8 KB of A +
// bn/2 rows of B per K step (24 KB at bn = 256) -- the bytes per MMA of a
// 256 x 512 pair tile -- while keeping the double-buffered 2 x 256 TMEM
// accumulator (epilogue overlapped with the next tile) and 256-column N
// granularity.  A stage is released only when both pairs' MMAs consumed it.
//
// TR (transposed output): the launch computes C^T = B A^T -- the kernel's A
// operand is the weight table (the MMA's M side: 128 / 256 W rows per
// tile, output columns) and its B operand the chart rows (the MMA's N side,
// N tile = any multiple of 32 up to 256, output rows).  Few chart rows then
// need no re-read of the 64 MB weight table per row tile, and the N tile can
// divide the row count exactly (the wave-quantisation fix of the library
// GEMMs on these shapes).  The epilogue transposes each warp's 32 x 32
// accumulator chunk through shared memory and runs the ordinary row
// epilogue on the output rows.
template <typename T, int BN, bool A_MN, bool B_MN, int EPI, bool SPLIT, int CHUNK, bool PAIR,
          bool MC = false, bool TR = false>
__global__ void __launch_bounds__(gemm_threads<CHUNK>(), 1)
    k_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
           const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
           GemmShape sh, GemmEpi ep) {
  using C = GemmCfg<T, BN>;
  constexpr int NCTA = PAIR ? 2 : 1;
  constexpr int CL = MC ? 4 : NCTA;  // CTAs per cluster
  static_assert(!MC || (PAIR && !A_MN && !SPLIT && CHUNK == 0 && BN <= 256),
                "multicast clusters: bf16/tf32 K-major A, double-buffered pair tiles");
  static_assert(!TR || (!B_MN && !SPLIT && CHUNK == 0 && BN <= 256 && !MC),
                "transposed output: K-major chart rows as B, double-buffered tiles");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int NS = sh.stages;
  // SPLIT: A stage = [hi | lo] tiles; B stage (sh.b_stage) = [hi | lo] halves
  constexpr int kAStage = (SPLIT ? 2 : 1) * C::A_BYTES;
  constexpr int kTmemCols = SPLIT ? 4 * BN : C::TMEM_COLS;  // SPLIT: small + big per buffer
  constexpr int kTmemHalf = kTmemCols / 2;
  static_assert(kTmemCols <= 512, "TMEM holds 512 columns");
  uint8_t* smA = smem;
  uint8_t* smB = smem + NS * kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smB + NS * sh.b_stage);
  uint64_t* empty = full + NS;
  uint64_t* tfull = empty + NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  // TR: one 32 x 33 transpose tile per epilogue warp, behind the 256-B barrier block
  float* tbuf = reinterpret_cast<float*>(smB + NS * sh.b_stage + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // MC: a unit's tile index counts cluster tiles (M block, pair of N tiles)
  const int num_tiles = sh.num_m * (MC ? (sh.num_n + 1) / 2 : sh.num_n);
  const int k_iters = sh.num_k;
  const int ks = sh.ksplit > 1 ? sh.ksplit : 1;
  const int tb = sh.tile_begin;
  const int tile_e = sh.tile_end > 0 ? sh.tile_end : num_tiles;
  const int bn = sh.bn;                       // runtime N tile <= BN
  const int bn_cta = bn / NCTA;               // B rows staged by this CTA
  const int nbuf = SPLIT || bn <= C::TMEM_HALF ? 2 : 1;  // accumulator buffers in TMEM
  const uint32_t crank = PAIR ? cluster_rank() : 0;
  const uint32_t rank = crank & 1u;               // position in the CTA pair
  const uint32_t pidx = MC ? (crank >> 1) : 0u;   // which pair of the cluster
  const uint32_t lead = crank & ~1u;              // cluster rank of this pair's leader
  const int tile0 = blockIdx.x / CL;
  const int tstep = gridDim.x / CL;
  auto tile_mn = [&](int tile, int& m_blk, int& n_blk) {
    m_blk = tile % sh.num_m;
    n_blk = MC ? 2 * (tile / sh.num_m) + static_cast<int>(pidx) : tile / sh.num_m;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (SPLIT) {
      tma_prefetch_desc(&tmA2);
      tma_prefetch_desc(&tmB2);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);  // MC: both pairs' MMAs read this stage's A
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], gemm_epi_warps<CHUNK>() * NCTA);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc2<kTmemCols>(tslot);
    else tmem_alloc<kTmemCols>(tslot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // barrier inits visible to the peer
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  pdl_wait();     // operands written by the previous kernel are visible from here
  pdl_trigger();  // persistent: every CTA is resident, so the next kernel may queue

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t stage_tx = NCTA * (kAStage + sh.b_stage);
      GemmUnit un;
      for (int ui = 0; gemm_unit(sh, tile0, tstep, ui, ks, k_iters, tb, tile_e, un); ++ui) {
        const int k0 = un.k0, k1 = un.k1;
        if (k0 >= k1) continue;
        int m_blk, n_blk;
        tile_mn(un.tile, m_blk, n_blk);
        const int m0 = m_blk * (C::BM * NCTA) + rank * C::BM;  // this CTA's A rows
        const int n0 = n_blk * bn + rank * bn_cta;              // this CTA's B rows
        for (int it = k0; it < k1; ++it) {
          const int kb = it;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a_dst = smA + stage * kAStage;
          uint8_t* b_dst = smB + stage * sh.b_stage;
          // completion is counted on the leader's full barrier (both CTAs' bytes)
          uint32_t fb = smem_u32(&full[stage]);
          if constexpr (PAIR) {
            fb = mapa_rank(&full[stage], lead);
            if (rank == 0) mbar_expect_tx(&full[stage], stage_tx);
          } else {
            mbar_expect_tx(&full[stage], stage_tx);
          }
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if constexpr (PAIR) tma_load_2d_pair(dst, m, fb, c0, c1);
            else tma_load_2d(dst, m, &full[stage], c0, c1);
          };
          auto load_a = [&](uint8_t* dst, const CUtensorMap* ma) {
            if constexpr (!A_MN) {
              load(dst, ma, kb * C::BK, sh.a_row0 + m0);
            } else {
#pragma unroll
              for (int j = 0; j < C::BM / C::ATOM; ++j)
                load(dst + j * C::BK * 128, ma, m0 + j * C::ATOM, kb * C::BK);
            }
          };
          auto load_b = [&](uint8_t* dst, const CUtensorMap* mb) {
            if constexpr (!B_MN) {
              load(dst, mb, kb * C::BK, sh.b_row0 + n0);
            } else {
              for (int j = 0; j < bn_cta / C::ATOM; ++j)
                load(dst + j * C::BK * 128, mb, n0 + j * C::ATOM, kb * C::BK);
            }
          };
          if constexpr (MC) {  // this CTA's half of the A rows, to both pairs
            constexpr int kHalfRows = C::BM / 2;
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
            tma_load_2d_pair_mc(a_dst + pidx * kHalfRows * 128, &tmA,
                                pair_leader_addr(&full[stage]), mask, kb * C::BK,
                                sh.a_row0 + m0 + static_cast<int>(pidx) * kHalfRows);
          } else {
            load_a(a_dst, &tmA);
          }
          load_b(b_dst, &tmB);
          if constexpr (SPLIT) {  // the lo planes behind the hi tiles
            load_a(a_dst + C::A_BYTES, &tmA2);
            load_b(b_dst + sh.b_stage / 2, &tmB2);
          }
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ------------------------------------------------ MMA issuer (leader)
      // The whole warp runs the loop (waits, bookkeeping, descriptor math:
      // warp-uniform values the compiler keeps in uniform registers); one
      // elected lane issues the MMAs and commits.
      // N tiles above 256 are two MMAs per K step (sub-tiles of 256 + the rest)
      const uint32_t idesc0 = make_idesc<C::TF32>(bn > 256 ? 256 : bn, A_MN, B_MN, C::BM * NCTA);
      const uint32_t idesc1 = make_idesc<C::TF32>(bn > 256 ? bn - 256 : 64, A_MN, B_MN, C::BM * NCTA);
      constexpr uint32_t sub_b_off = 256 / NCTA * 128;  // B bytes of sub-tile 0 in this CTA
      constexpr uint32_t a_lbo = A_MN ? C::BK * 128 : 16;
      constexpr uint32_t b_lbo = B_MN ? C::BK * 128 : 16;
      // tf32 MN-major operands use the 32B-atom 128B swizzle (4-row groups)
      constexpr uint32_t a_lay = (A_MN && C::TF32) ? kLayoutSW128Base32B : kLayoutSW128;
      constexpr uint32_t b_lay = (B_MN && C::TF32) ? kLayoutSW128Base32B : kLayoutSW128;
      constexpr uint32_t a_sbo = (A_MN && C::TF32) ? 512 : 1024;
      constexpr uint32_t b_sbo = (B_MN && C::TF32) ? 512 : 1024;
      constexpr uint32_t a_kstep = A_MN ? C::UK * 128 : C::UK * C::kElt;
      constexpr uint32_t b_kstep = B_MN ? C::UK * 128 : C::UK * C::kElt;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      GemmUnit un;
      for (int ui = 0; gemm_unit(sh, tile0, tstep, ui, ks, k_iters, tb, tile_e, un); ++ui) {
        const int k0 = un.k0, k1 = un.k1;
        if (k0 >= k1) continue;
        const int cl = CHUNK > 0 ? CHUNK : k1 - k0;
        uint32_t d_tmem = tmem_base;
        int kc = 0;  // K iteration within the accumulator chunk (no per-iteration division)
        for (int kb = k0; kb < k1; ++kb, kc = (kc + 1 == cl) ? 0 : kc + 1) {
          if (kc == 0) {  // start a chunk in a drained accumulator
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            d_tmem = tmem_base + static_cast<uint32_t>(acc * kTmemHalf);
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * kAStage);
          const uint32_t b_base = smem_u32(smB + stage * sh.b_stage);
          auto mma = [&](uint32_t dt, uint64_t ad, uint64_t bd, uint32_t id, uint32_t accum) {
            if constexpr (PAIR) umma2<C::TF32>(dt, ad, bd, id, accum);
            else umma<C::TF32>(dt, ad, bd, id, accum);
          };
          // K step k of a stage: the start-address field (bits 0-13, 16-B units)
          // advances by kstep / 16 -- no carry within a stage
          const uint64_t ad0 = make_sdesc(a_base, a_lbo, a_sbo, a_lay);
          const uint64_t bd0 = make_sdesc(b_base, b_lbo, b_sbo, b_lay);
          const bool issuer = elect_one();
          if (!issuer) {
            // the other lanes only keep the bookkeeping in step
          } else if constexpr (SPLIT) {  // small (lo*hi + hi*lo) at +0, big (hi*hi) at +BN
            const uint32_t b_lo = static_cast<uint32_t>(sh.b_stage / 2);
#pragma unroll
            for (int k = 0; k < C::BK / C::UK; ++k) {
              const uint64_t ah = make_sdesc(a_base + k * a_kstep, a_lbo, a_sbo, a_lay);
              const uint64_t al = make_sdesc(a_base + C::A_BYTES + k * a_kstep, a_lbo, a_sbo, a_lay);
              const uint64_t bh = make_sdesc(b_base + k * b_kstep, b_lbo, b_sbo, b_lay);
              const uint64_t bl = make_sdesc(b_base + b_lo + k * b_kstep, b_lbo, b_sbo, b_lay);
              const uint32_t accum = (kc | k) != 0 ? 1u : 0u;
              mma(d_tmem, al, bh, idesc0, accum);
              mma(d_tmem, ah, bl, idesc0, 1u);
              mma(d_tmem + static_cast<uint32_t>(BN), ah, bh, idesc0, accum);
            }
          } else if constexpr (BN <= 256) {  // BN > 256 kernels run only N tiles above 256
#pragma unroll
            for (int k = 0; k < C::BK / C::UK; ++k)
              mma(d_tmem, ad0 + static_cast<uint64_t>(k * (a_kstep >> 4)),
                  bd0 + static_cast<uint64_t>(k * (b_kstep >> 4)), idesc0,
                  (kc | k) != 0 ? 1u : 0u);
          } else {
            constexpr uint64_t kSubB = sub_b_off >> 4;
#pragma unroll
            for (int k = 0; k < C::BK / C::UK; ++k) {
              const uint64_t ad = ad0 + static_cast<uint64_t>(k * (a_kstep >> 4));
              const uint64_t bd = bd0 + static_cast<uint64_t>(k * (b_kstep >> 4));
              const uint32_t accum = (kc | k) != 0 ? 1u : 0u;
              mma(d_tmem, ad, bd, idesc0, accum);
              mma(d_tmem + 256u, ad, bd + kSubB, idesc1, accum);
            }
          }
          const bool chunk_end = kc == cl - 1 || kb == k1 - 1;
          if (issuer) {
            if constexpr (MC) umma_commit2_mask(&empty[stage], 0xF);  // both pairs' stages
            else if constexpr (PAIR) umma_commit2(&empty[stage]);
            else umma_commit(&empty[stage]);
            if (chunk_end) {
              if constexpr (MC) umma_commit2_mask(&tfull[acc], static_cast<uint16_t>(3u << lead));
              else if constexpr (PAIR) umma_commit2(&tfull[acc]);
              else umma_commit(&tfull[acc]);
            }
          }
          __syncwarp();
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
          if (chunk_end) {
            if (++acc == nbuf) {
              acc = 0;
              acc_phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int ehalf = (warp - 4) >> 2;  // which chunk pairs this warp drains (CHUNK == 0)
    const int r = quad * 32 + lane;  // accumulator row (TMEM lane)
    int acc = 0;
    uint32_t acc_phase = 0;
    // TMEM-empty arrivals go to the leader (its MMA issuer reuses the buffer)
    uint32_t te[2];
    te[0] = PAIR ? mapa_rank(&tempty[0], lead) : smem_u32(&tempty[0]);
    te[1] = PAIR ? mapa_rank(&tempty[1], lead) : smem_u32(&tempty[1]);
    auto release = [&](int a) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(te[a]);
        else mbar_arrive(&tempty[a]);
      }
    };
    GemmUnit un;
    for (int ui = 0; gemm_unit(sh, tile0, tstep, ui, ks, k_iters, tb, tile_e, un); ++ui) {
      const int k0 = un.k0, k1 = un.k1;
      if (k0 >= k1) continue;
      const int u = tile0 + ui * tstep;
      const int tu = un.tile - tb, kpart = u - tu * ks;  // (in-kernel reduction only)
      int m_blk, n_blk;
      tile_mn(un.tile, m_blk, n_blk);
      const int lrow = m_blk * (C::BM * NCTA) + rank * C::BM + r;  // row within this GEMM
      // (TR: rows are output columns; the row epilogue runs after the transpose)
      const EpiRow er = TR ? EpiRow{} : epi_row<EPI>(ep, lrow);
      const int col_base = n_blk * bn;
      // tile column of TMEM column chunk j: with two sub-tiles in a pair, each
      // CTA stages B rows [0, 128) of sub-tile 0 then the rest of its half,
      // so sub-tile s's columns are [half 0 | half 1] of that range
      auto tile_col = [&](int j) -> int {
        const int c = j * 32;
        if (!PAIR || BN <= 256) return c;
        const int sb = c >> 8, w = c & 255;
        const int hs = (sb ? bn - 256 : 256) / 2;
        const int q = w >= hs ? 1 : 0;  // w < 2 hs: the CTA half, without a division
        return q * bn_cta + sb * 128 + (w - q * hs);
      };
      // stream-K: the segment that ends its tile sums the others' partials
      const bool sk_final = un.skt >= 0 && un.k1 == k_iters;
      int sk_pid[16];
      const int sk_np = sk_final ? sk_parts(sh, un.skt, tstep, k_iters, tile_e, un.pidx, sk_pid) : 0;
      const bool to_part = un.pidx >= 0 && !sk_final;
      int* sk_cnt = un.skt >= 0 ? sh.sem + un.skt : nullptr;
      constexpr int kEpiThreadsAll = 32 * gemm_epi_warps<CHUNK>();
      constexpr int tile_rows_u = C::BM * NCTA;
      if (sk_np > 0) {  // wait until every other segment of the tile has published
        if (threadIdx.x == 128)
          while (ld_acquire_gpu(sk_cnt) < sk_np * NCTA) __nanosleep(64);
        epi_bar_sync(kEpiThreadsAll);
      }
      // the final segment is this CTA's last unit: once its accumulator is
      // full the smem ring is idle and holds the other segments' sum
      // (128 x bn, rows padded by 16 B), read with coalesced loads
      const uint32_t sk_tile = smem_u32(smem);
      constexpr int kSkDepth = 16;
      auto sk_stage = [&]() {
        // a partial row-block is contiguous (tile_rows_u x bn floats per part):
        // kSkDepth float4 loads in flight per thread per part, then st.shared
        const int n4 = C::BM * bn / 4;
        const float4* base = reinterpret_cast<const float4*>(
            sh.part + static_cast<long long>(rank * C::BM) * bn);
        const long long pstr4 = static_cast<long long>(tile_rows_u) * bn / 4;
        for (int i0 = threadIdx.x - 128; i0 < n4; i0 += kSkDepth * kEpiThreadsAll) {
          float4 a[kSkDepth];
#pragma unroll
          for (int u = 0; u < kSkDepth; ++u) {
            const int i = i0 + u * kEpiThreadsAll;
            a[u] = i < n4 ? __ldcg(base + sk_pid[0] * pstr4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int pi = 1; pi < sk_np; ++pi) {  // slot order: deterministic
            const float4* pp = base + sk_pid[pi] * pstr4;
            float4 w[kSkDepth];
#pragma unroll
            for (int u = 0; u < kSkDepth; ++u) {
              const int i = i0 + u * kEpiThreadsAll;
              w[u] = i < n4 ? __ldcg(pp + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < kSkDepth; ++u) {
              a[u].x += w[u].x;
              a[u].y += w[u].y;
              a[u].z += w[u].z;
              a[u].w += w[u].w;
            }
          }
#pragma unroll
          for (int u = 0; u < kSkDepth; ++u) {
            const int i = i0 + u * kEpiThreadsAll;
            if (i < n4) {
              const int row = i / (bn / 4), c4 = i - row * (bn / 4);
              st_shared_v4(sk_tile + static_cast<uint32_t>((row * (bn + 4) + c4 * 4) * 4), a[u]);
            }
          }
        }
        epi_bar_sync(kEpiThreadsAll);
      };
      auto emit = [&](int j, const float (&v0)[32]) {
        const int tc = tile_col(j);
        if (to_part) {  // split-K / stream-K: raw fp32 partial, summed + transformed
          float4* dst = reinterpret_cast<float4*>(    // below or by k_gemm_fixup
              sh.part + (static_cast<long long>(un.pidx) * tile_rows_u + rank * C::BM + r) * bn + tc);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(v0[4 * q], v0[4 * q + 1], v0[4 * q + 2], v0[4 * q + 3]);
          return;
        }
        float v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = v0[t];
        if (sk_np > 0) {  // + the other segments' sum, staged in the idle ring (below)
          const uint32_t src = sk_tile + static_cast<uint32_t>((r * (bn + 4) + tc) * 4);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 w = ld_shared_v4(src + 16u * q);
            v[4 * q] += w.x;
            v[4 * q + 1] += w.y;
            v[4 * q + 2] += w.z;
            v[4 * q + 3] += w.w;
          }
        }
        if constexpr (TR) {  // v = 32 output rows of output column lrow: transpose
          float* tw = tbuf + (warp - 4) * (32 * 33);
#pragma unroll
          for (int q = 0; q < 32; ++q) tw[lane * 33 + q] = v[q];
          __syncwarp();
          float w[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) w[q] = tw[q * 33 + lane];
          __syncwarp();
          const int orow = col_base + tc + lane;                         // output row
          const int ocol = m_blk * (C::BM * NCTA) + rank * C::BM + quad * 32;  // first column
          const EpiRow ert = epi_row<EPI>(ep, orow);
          epi_emit<EPI>(ep, ert, ocol, sh.M, w);
        } else {
          epi_emit<EPI>(ep, er, col_base + tc, sh.N, v);
        }
      };
      const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
      if constexpr (CHUNK == 0) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (sk_np > 0) sk_stage();
        const uint32_t t_row = t_lane + static_cast<uint32_t>(acc * kTmemHalf);
        const int nch = bn / 32;
        constexpr int kHalves = gemm_epi_warps<CHUNK>() / 4;
#pragma unroll 1
        for (int j = 2 * ehalf; j + 1 < nch; j += 2 * kHalves) {
          float v0[32], v1[32];
          tmem_ld32x2(t_row + j * 32, t_row + j * 32 + 32, v0, v1);
          emit(j, v0);
          emit(j + 1, v1);
        }
        if ((nch & 1) && ((nch - 1) / 2) % kHalves == ehalf) {
          float v[32];
          tmem_ld32(t_row + (nch - 1) * 32, v);
          emit(nch - 1, v);
        }
        release(acc);
        if (++acc == nbuf) {
          acc = 0;
          acc_phase ^= 1;
        }
        if (un.skt >= 0 && !sk_final) {  // publish this segment's partial rows
          __threadfence();
          epi_bar_sync(kEpiThreadsAll);
          if (threadIdx.x == 128) atomicAdd(sk_cnt, 1);
        } else if (sk_np > 0) {  // the last CTA of the finalizing pair re-arms the counter
          epi_bar_sync(kEpiThreadsAll);
          if (threadIdx.x == 128 && atomicAdd(sk_cnt, 1) == sk_np * NCTA + NCTA - 1)
            atomicExch(sk_cnt, 0);
        }
        if (ks > 1 && sh.sem && sh.sk == 0) {
          constexpr int tile_rows = C::BM * NCTA;
          constexpr int kEpiThreads = 32 * gemm_epi_warps<CHUNK>();
          const long long tsplit = tile_e - tb;
          int* cnt = sh.sem + tu;
          const int parts = ks * NCTA;
          __threadfence();  // this thread's partial rows -> visible GPU-wide
          epi_bar_sync(kEpiThreads);
          if (threadIdx.x == 128) {
            atomicAdd(cnt, 1);
            while (ld_acquire_gpu(cnt) < parts) __nanosleep(64);
          }
          epi_bar_sync(kEpiThreads);
          const int c0 = nch * kpart / ks, c1 = nch * (kpart + 1) / ks;
          const float* prow = sh.part + (tu * tile_rows + rank * C::BM + r) * static_cast<long long>(bn);
          const long long pstride = tsplit * tile_rows * static_cast<long long>(bn);
#pragma unroll 1
          for (int c = c0; c < c1; ++c) {
            float v[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) v[t] = 0.f;
            for (int k = 0; k < ks; ++k) {
              const float4* src = reinterpret_cast<const float4*>(prow + k * pstride + c * 32);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 w = __ldcg(src + q);
                v[4 * q] += w.x;
                v[4 * q + 1] += w.y;
                v[4 * q + 2] += w.z;
                v[4 * q + 3] += w.w;
              }
            }
            epi_emit<EPI>(ep, er, col_base + c * 32, sh.N, v);
          }
          // second round of arrivals: the last one re-arms the counter
          epi_bar_sync(kEpiThreads);
          if (threadIdx.x == 128 && atomicAdd(cnt, 1) == 2 * parts - 1) atomicExch(cnt, 0);
        }
      } else {
        static_assert(BN <= 128, "chunked accumulation keeps BN fp32 sums per thread");
        float sum[BN / 32][32];
#pragma unroll
        for (int j = 0; j < BN / 32; ++j)
#pragma unroll
          for (int t = 0; t < 32; ++t) sum[j][t] = 0.f;
        const int nchunks = (k1 - k0 + CHUNK - 1) / CHUNK;
        for (int c = 0; c < nchunks; ++c) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t t_row = t_lane + static_cast<uint32_t>(acc * kTmemHalf);
#pragma unroll
          for (int j = 0; j < BN / 32; ++j) {
            if (j < bn / 32) {
              float v[32];
              if constexpr (SPLIT) {  // small + big, then into the running sum
                float vb[32];
                tmem_ld32x2(t_row + j * 32, t_row + BN + j * 32, v, vb);
#pragma unroll
                for (int t = 0; t < 32; ++t) v[t] += vb[t];
              } else {
                tmem_ld32(t_row + j * 32, v);
              }
#pragma unroll
              for (int t = 0; t < 32; ++t) sum[j][t] += v[t];
            }
          }
          release(acc);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
#pragma unroll
        for (int j = 0; j < BN / 32; ++j)
          if (j < bn / 32) emit(j, sum[j]);
      }
    }
  }

  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();  // the peer's MMAs / arrivals are done
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (PAIR) tmem_dealloc2<kTmemCols>(tmem_base);
    else tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// Split-K fixup (FI_GEMM_INKERNEL_RED=0, or more split tiles than counters):
// sum the ksplit raw partials of the tiles [tile_begin, T) in part order and
// run the launch's epilogue.  One CTA per (tile, block of kFixRows rows):
// the partial rows are read as coalesced float4 runs (each warp streams 512
// contiguous bytes per load), summed in registers in part order
// (deterministic), staged in shared memory, and the epilogue then runs one
// thread per (row, 32-column chunk) from there.
constexpr int kFixRows = 8;
template <int EPI>
__global__ void __launch_bounds__(256) k_gemm_fixup(const float* __restrict__ part, int ksplit,
                                                    int M, int N, int num_m, int tile_rows,
                                                    int bn, int tile_begin, int num_tiles,
                                                    GemmEpi ep) {
  pdl_wait();
  extern __shared__ __align__(16) float fix_sm[];  // kFixRows x bn
  const int blocks_per_tile = tile_rows / kFixRows;
  const int tile = tile_begin + static_cast<int>(blockIdx.x) / blocks_per_tile;
  const int r0 = (static_cast<int>(blockIdx.x) % blocks_per_tile) * kFixRows;
  const long long tsplit = num_tiles - tile_begin;
  const int row_base = (tile % num_m) * tile_rows + r0;   // GEMM row of smem row 0
  const int col_base = (tile / num_m) * bn;
  const long long pstride = tsplit * tile_rows * static_cast<long long>(bn);
  // shared layout [row][chunk][36 floats]: 32 values + 4 pad, so the
  // epilogue threads' 16-B reads of consecutive chunks hit distinct banks
  const int chunks = bn / 32;
  const int n4 = kFixRows * bn / 4;
  const float4* src = reinterpret_cast<const float4*>(
      part + ((tile - tile_begin) * static_cast<long long>(tile_rows) + r0) * bn);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) {
    float4 acc = __ldcg(src + i);
    for (int k = 1; k < ksplit; ++k) {
      const float4 w = __ldcg(src + k * (pstride / 4) + i);
      acc.x += w.x;
      acc.y += w.y;
      acc.z += w.z;
      acc.w += w.w;
    }
    const int c4 = i % (bn / 4), rr = i / (bn / 4);
    *reinterpret_cast<float4*>(fix_sm + (rr * chunks + c4 / 8) * 36 + (c4 % 8) * 4) = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kFixRows * chunks; t += blockDim.x) {
    const int rr = t / chunks, ch = t % chunks;
    const int lrow = row_base + rr, col = col_base + ch * 32;
    if (lrow >= M || col >= N) continue;
    float v[32];
    const float4* p4 = reinterpret_cast<const float4*>(fix_sm + t * 36);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 x = p4[q];
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
    const EpiRow er = epi_row<EPI>(ep, lrow);
    epi_emit<EPI>(ep, er, col, N, v);
  }
}

// Split-K fixup of a TR launch: the partial tiles are in kernel layout
// (W rows x chart rows); one CTA per (tile, 32 kernel rows) sums them in
// part order into shared memory and each thread then emits one output row
// (a kernel column) for those 32 output columns.
template <int EPI>
__global__ void __launch_bounds__(256) k_gemm_fixup_tr(const float* __restrict__ part, int ksplit,
                                                       int M, int N, int num_m, int tile_rows,
                                                       int bn, int tile_begin, int num_tiles,
                                                       GemmEpi ep) {
  pdl_wait();
  extern __shared__ __align__(16) float fix_sm[];  // 32 x (bn + 1)
  const int blocks_per_tile = tile_rows / 32;
  const int tile = tile_begin + static_cast<int>(blockIdx.x) / blocks_per_tile;
  const int r0 = (static_cast<int>(blockIdx.x) % blocks_per_tile) * 32;
  const long long tsplit = num_tiles - tile_begin;
  const int krow0 = (tile % num_m) * tile_rows + r0;   // kernel row = output column
  const int kcol0 = (tile / num_m) * bn;               // kernel column = output row
  const long long pstride = tsplit * tile_rows * static_cast<long long>(bn);
  const float* src = part + ((tile - tile_begin) * static_cast<long long>(tile_rows) + r0) * bn;
  for (int i = threadIdx.x; i < 32 * bn; i += blockDim.x) {
    float acc = __ldcg(src + i);
    for (int k = 1; k < ksplit; ++k) acc += __ldcg(src + k * pstride + i);
    fix_sm[(i / bn) * (bn + 1) + i % bn] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < bn; t += blockDim.x) {
    const int orow = kcol0 + t;
    if (orow >= ep.M || krow0 >= M) continue;
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = fix_sm[q * (bn + 1) + t];
    const EpiRow er = epi_row<EPI>(ep, orow);
    epi_emit<EPI>(ep, er, krow0, M, v);
  }
}

}  // namespace fi
