/*
 * flashinside.h -- C ABI of the B200-native FlashInside engine (sm_100a).
 *
 * This is the drop-in boundary for the reference's inside-algorithm engine
 * API.  The reference is pure Python/NumPy; its plug-in seam is the engine
 * registry ENGINES (pkg/src/flashpcfg/inside.py:343-348) whose entries have
 * the signature  engine(g, tokens, meter=None) -> InsideChart
 * (inside.py:150-151, :216-217, :274-275), plus the backward
 * inside_backward(g, tokens, chart) -> (GrammarGrad, MarginalTable)
 * (inside.py:375-376).  A ctypes binding calls the
 * entry points below; the Python package paper_2310_14997_b200 does exactly
 * that and re-exposes the reference's names.
 *
 * Conventions
 *   - All pointers are DEVICE pointers on the current CUDA device unless the
 *     name says otherwise; all arrays are C-contiguous fp32 / int32.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t, may be NULL)
 *     and returns FI_OK or an error code; fi_last_error() gives the message
 *     (thread-local).  No C++ exception crosses this boundary.
 *   - The workspace `ws` (fi_workspace_bytes) is caller-allocated device
 *     memory.  The forward leaves the chart in it; the backward consumes it.
 *     The library never allocates or frees caller memory.
 *   - Calls on different streams (and threads) may run concurrently, each
 *     with its own workspace.  (The opt-in FI_GEMM_INKERNEL_RED=1 schedule
 *     assumes one stream at a time: its split-K units wait for each other.)
 *
 * Shapes (N = n_nt, P = n_pt, B = batch, l = max_len):
 *   L, R      : (N, N+P)   log_left / log_right  (grammar.py:99-100)
 *   root      : (N,)       log_root
 *   unary     : (B, l, P)  unary[b, i, T] = log_emit[T, tokens[b][i]]
 *                          (the width-1 chart row, inside.py:296-298)
 *   lengths   : (B,)       2 <= lengths[b] <= l; a length outside that range
 *                          is caught on the device (FI_FLAG_BAD_LENGTH below)
 *   log_z     : (B,)       per-sentence log partition (InsideChart.log_z)
 *   grad_log_z: (B,)       upstream gradient dLoss/dlog_z
 *   dL, dR    : (N, N+P)   sum_b grad_log_z[b] * dlog_z[b]/dL  (GrammarGrad)
 *   droot     : (N,)
 *   dunary    : (B, l, P)  gradient w.r.t. unary (d_emit = scatter of it,
 *                          inside.py:420-423)
 */
#ifndef FLASHINSIDE_H_
#define FLASHINSIDE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FI_OK 0
#define FI_ERR_ARG 1         /* invalid shape / pointer (InsideError analogue) */
#define FI_ERR_CUDA 2        /* CUDA runtime / driver failure                  */
#define FI_ERR_UNSUPPORTED 3 /* no sm_100a device or unsupported size          */

#define FI_GEMM_BF16 0 /* projection GEMM operands bf16, fp32 accumulate      */
#define FI_GEMM_TF32 1 /* projection GEMM operands tf32 (single pass)           */
#define FI_GEMM_FP32 2 /* "fp32 mode": bf16x3 split operands (hi*hi + lo*hi +
                          hi*lo), ~2^-16 relative per product, fp32 accumulate */

/* Storage of the projected chart vectors a[w], b[w] between the projection
 * GEMM and the bandwidth-bound split kernels (see fi_chart_layout). */
#define FI_CHART_AUTO 0 /* fp16 linear with bf16/tf32 GEMM operands, fp32 log in fp32 mode */
#define FI_CHART_F32 1  /* fp32 base-2 log offsets a^ = log2(acc)                         */
#define FI_CHART_F16 2  /* fp16 linear acc * 2^14 (acc = (E W^T) in [0, 1])               */

/* Bits of the int32 flag word at fi_chart_layout.off_flag (cleared by every
 * fi_inside_forward / fi_inside_backward call, then set on the stream):
 *   FI_FLAG_ZERO_PROB  (backward) a sentence with log Z = -inf: it gets no
 *                      gradient (inside.py:392-393 raises InsideError here)
 *   FI_FLAG_BAD_LENGTH a lengths[b] outside [2, l] (inside.py:113-121): that
 *                      sentence is inert -- log_z[b] = NaN, zero gradients,
 *                      no chart write outside its own rows. */
#define FI_FLAG_ZERO_PROB 1
#define FI_FLAG_BAD_LENGTH 2

typedef struct fi_shape {
  int32_t n_nt;        /* N */
  int32_t n_pt;        /* P */
  int32_t batch;       /* B */
  int32_t max_len;     /* l */
  int32_t gemm_dtype;  /* FI_GEMM_BF16 | FI_GEMM_TF32 | FI_GEMM_FP32 */
  int32_t store_chart; /* 1: keep o[w] for every span (chart export, marginals) */
  int32_t chart_dtype; /* FI_CHART_AUTO | FI_CHART_F32 | FI_CHART_F16 */
} fi_shape;

/* Byte offsets of the chart arrays inside the workspace, for chart export.
 * Row r of an array with row stride `np` lives at offset + 4*r*np.
 *   row(w, b, i) = rowbase(w) + b*(l-w+1) + i,
 *   rowbase(w)   = B * ((w-1)*(l+1) - (w-1)*w/2).
 * Storage is base-2 and shifted: the natural-log value of a chart entry is
 *   ln2 * (x[row] + stored[row, A])
 * with x[row] the fp64 per-span shift (off_x) and the stored fp32 offsets
 * a^, b^, o^ (o^ <= 0) and, after a backward, lq^ = log2|go| - log2 o + x.
 * With chart_fmt == FI_CHART_F16 the a/b arrays hold fp16 s = acc * 2^14
 * (row stride np halves), i.e. a^ = log2(s) - 14, and lq holds fp16 q with
 * lq^ = log2(q) + e[row, A / 32] (e: fp32 exponents at off_lqs). */
typedef struct fi_chart_layout {
  int64_t np;       /* padded N (row stride, floats)          */
  int64_t pp;       /* padded P                               */
  int64_t rows;     /* total span rows = rowbase(l) + B       */
  int64_t off_a;    /* a[w]  fp32, widths 1..l-1              */
  int64_t off_b;    /* b[w]  fp32, widths 1..l-1              */
  int64_t off_o;    /* o[w]  fp32, widths 2..l (-1 if absent) */
  int64_t off_x;    /* x†    fp64 per row (log2 units)        */
  int64_t off_lq;   /* log|go|-o, widths 2..l (after backward)*/
  int64_t off_flag; /* int32 error flags (FI_FLAG_ZERO_PROB | FI_FLAG_BAD_LENGTH) */
  int64_t chart_fmt; /* FI_CHART_F32 or FI_CHART_F16: storage of a, b, lq */
  int64_t off_lqs;   /* FI_CHART_F16: fp32 exponent per 32 columns of lq (-1 otherwise) */
} fi_chart_layout;

/* Workspace bytes needed for `shape` (0 on invalid shape). */
size_t fi_workspace_bytes(const fi_shape* shape);

/* Chart layout of the workspace for `shape`. */
int fi_get_chart_layout(const fi_shape* shape, fi_chart_layout* out);

/* Forward inside pass (replaces inside_flash, inside.py:274-340, batched).
 * Writes log_z[B]; keeps the chart in ws for fi_inside_backward. */
int fi_inside_forward(const fi_shape* shape, const float* L, const float* R, const float* root,
                      const float* unary, const int32_t* lengths, float* log_z, void* ws,
                      void* stream);

/* Backward / outside pass (replaces inside_backward + _projection_backward,
 * inside.py:375-447) by recomputation from the chart in ws. */
int fi_inside_backward(const fi_shape* shape, const float* L, const float* R, const float* root,
                       const float* unary, const int32_t* lengths, const float* log_z,
                       const float* grad_log_z, float* dL, float* dR, float* droot,
                       float* dunary, void* ws, void* stream);

/* fi_inside_backward for the data-parallel step (the sum of
 * per-sentence GrammarGrads across ranks replaces train.py:206-218's loop):
 * the weight-gradient GEMMs run as [width-1 block of dL and dR] -> [dL's
 * width >= 2 block] -> record `dl_ready` (a cudaEvent_t, may be NULL) on
 * `stream` -> [dR's width >= 2 block], so a caller can all-reduce dL on
 * another stream while dR's GEMM still runs.  droot is final before it too.
 * With dl_ready == NULL this is exactly fi_inside_backward. */
int fi_inside_backward_ex(const fi_shape* shape, const float* L, const float* R,
                          const float* root, const float* unary, const int32_t* lengths,
                          const float* log_z, const float* grad_log_z, float* dL, float* dR,
                          float* droot, float* dunary, void* ws, void* stream, void* dl_ready);

/* Span marginals mu_sym (MarginalTable, inside.py:425-430) for widths >= 2,
 * rows ordered like the chart from rowbase(2); shape (rows - rowbase(2), N).
 * Requires store_chart = 1 and a completed backward with the same grad_log_z. */
int fi_marginals(const fi_shape* shape, const int32_t* lengths, const float* grad_log_z,
                 float* mu, void* ws, void* stream);

/* Span posterior mass mu(i, j) = sum_A mu_sym (MarginalTable.mu, inside.py:355-372)
 * for widths >= 2, one float per chart row from rowbase(2) (same order as
 * fi_marginals).  Requires store_chart = 1 and a completed backward. */
int fi_span_marginals(const fi_shape* shape, const int32_t* lengths, const float* grad_log_z,
                      float* mass, void* ws, void* stream);

/* Minimum-Bayes-risk CKY over span masses (mbr_decode, parse.py:98-131),
 * batched: for every sentence b and span (i, j), split[b, i, j] is the best
 * split point (ties -> smallest) and score[b, i, j] the best total mass; both
 * (B, l, l + 1) with index (b * l + i) * (l + 1) + j.  The tree is read off
 * split from (0, len) down. */
int fi_mbr_decode(const fi_shape* shape, const int32_t* lengths, const float* mass,
                  float* score, int32_t* split, void* stream);

/* Viterbi parse (viterbi_decode, parse.py:33-95), batched: the inside
 * recursion in the (max, +) semiring with fp32 natural-log scores.  The
 * caller provides va, vb, vo: (rows, np) fp32 scratch charts (rows / np of
 * fi_get_chart_layout); outputs per sentence b: best[b] = the best
 * derivation's log probability, and nodes[b, k, 0:3] = (i, j, sym) for the
 * 2 len - 1 nodes of that derivation in preorder (internal nodes carry a
 * nonterminal index, leaves a preterminal index); nodes is (B, 2 l, 3).
 * Ties prefer the smallest split, then the smallest symbol index. */
int fi_viterbi(const fi_shape* shape, const float* L, const float* R, const float* root,
               const float* unary, const int32_t* lengths, float* va, float* vb, float* vo,
               int32_t* nodes, float* best, void* stream);

/* Score tables of the grammar parameterisations (
 * replaces the float64 products + row log-softmax of neuralparam.py:185-189
 * and the matching softmax backward of backward_params, :242-320):
 *   logp = log_softmax(A B^T, rows)     A (rows, d), B (cols, d), logp (rows, cols)
 * e.g. log_left = log_softmax(f3 f2^T) with rows = N, cols = N + P.  The
 * product runs on the engine's tcgen05 GEMM: tf32 operands for
 * FI_GEMM_BF16 / FI_GEMM_TF32, bf16x3 split operands for FI_GEMM_FP32 (the
 * 1e-4 parity mode).  ws: fi_param_workspace_bytes device bytes (scratch;
 * the backward does not need the forward's). */
size_t fi_param_workspace_bytes(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d);
int fi_param_scores(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d, const float* A,
                    const float* B, float* logp, void* ws, void* stream);
/* Backward of fi_param_scores given dlogp = dLoss/dlogp:
 *   g = dlogp - exp(logp) * rowsum(dlogp);  dA = g B;  dB = g^T A. */
int fi_param_scores_backward(int32_t gemm_dtype, int32_t rows, int32_t cols, int32_t d,
                             const float* A, const float* B, const float* logp,
                             const float* dlogp, float* dA, float* dB, void* ws, void* stream);

/* Test hook: C[M,N] = A * B^T in the engine's tcgen05 GEMM (fp32 out).
 * a_mn / b_mn select MN-major operands: A is (M,K) K-major or (K,M) MN-major,
 * B is (N,K) K-major or (K,N) MN-major; elements bf16 (dtype 0) or fp32/tf32. */
int fi_test_gemm(int32_t dtype, int32_t a_mn, int32_t b_mn, int32_t M, int32_t N, int32_t K,
                 const void* A, const void* B, float* C, void* stream);

/* Cumulative number of kernels this library has enqueued in the process
 * (bench accounting: difference before/after the timed region). */
int64_t fi_launch_count(void);

/* Optional per-kernel-class timing with CUDA events recorded on the launch
 * stream around every launch of this thread (bench.py roofline).  Collect
 * synchronizes on the recorded events, returns total ms and launch counts per
 * class (arrays of n >= FI_PROF_NCLASS) and clears the record. */
#define FI_PROF_PREP 0       /* exp of [L|R], width-1 prep (and test GEMMs) */
#define FI_PROF_SPLIT 1      /* k_split_fwd: split-point contraction         */
#define FI_PROF_GEMM_FWD 2   /* projection GEMM, EPI_FWD                      */
#define FI_PROF_SEED 3       /* k_seed_bwd                                    */
#define FI_PROF_GATHER 4     /* k_gather_bwd: split backward                  */
#define FI_PROF_GEMM_DGRAD 5 /* dgrad GEMMs (EPI_DGRAD, EPI_DUNARY)           */
#define FI_PROF_GEMM_WGRAD 6 /* wgrad GEMMs (EPI_WGRAD)                       */
#define FI_PROF_PARAM 7      /* fi_param_scores(_backward): GEMMs + row passes */
#define FI_PROF_NCLASS 8
void fi_profile_enable(int32_t on);
int fi_profile_collect(float* ms, int32_t* counts, int32_t n);
/* Same record, per launch in issue order: ms[k] and class cls[k] for the
 * first n launches; returns the number of recorded launches and clears. */
int fi_profile_collect_launches(float* ms, int32_t* cls, int32_t n);

const char* fi_last_error(void);
int32_t fi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLASHINSIDE_H_ */
