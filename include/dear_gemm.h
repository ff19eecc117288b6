/*
 * dear_gemm.h — hand-written sm_100a tcgen05/TMA GEMM for the synthetic
 * per-layer compute that DeAR's collectives overlap with.
 *
 * The reference has no layer math (LayerSpec carries only t_ff / t_bp
 * durations, model.hpp:30-31); BASELINE.json asks for "synthetic layer
 * compute" with a tcgen05 GEMM so feed-forward / backprop are real dense
 * contractions on the tensor cores.
 *
 *   D[m, n] (+)= sum_k A[m, k] * B[n, k]        bf16 x bf16 -> fp32 accumulate
 *
 *   A : K-major, element (m, k) at A[m * lda + k]
 *   B : K-major (b_mn_major = 0): (n, k) at B[n * ldb + k]
 *       MN-major (b_mn_major = 1): (n, k) at B[k * ldb + n]
 *   D : row-major, (m, n) at D[m * ldd + n], fp32 (d_fp32 = 1) or bf16.
 *       Elements with m * ldd + n >= d_limit are not written (d_limit < 0:
 *       no flat bound) — lets a weight gradient land in a flat parameter
 *       tensor whose last row is partial.
 *   accumulate = 1: D += result with fp32 reductions (requires fp32 D; the
 *       K dimension may then be split across CTAs, split_k = 0 picks it).
 *   Leading dimensions must be multiples of 8 elements, bases 16 B aligned.
 */
#ifndef DEAR_GEMM_H_
#define DEAR_GEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dear_gemm_plan dear_gemm_plan;

int dear_gemm_plan_create(const void* A, int64_t lda, const void* B, int64_t ldb,
                          int32_t b_mn_major, void* D, int64_t ldd, int32_t d_fp32, int64_t M,
                          int64_t N, int64_t K, int64_t d_limit, int32_t accumulate,
                          int32_t split_k, dear_gemm_plan** out);
/* Enqueue on `stream` (cudaStream_t as void*). Launches are persistent (one
 * CTA per SM) and use programmatic dependent launch. */
int dear_gemm_run(dear_gemm_plan* plan, void* stream);
/* One launch computing n (1 or 2) independent plans on a shared persistent
 * grid, e.g. the weight- and data-gradient GEMMs of one layer. */
int dear_gemm_run_group(dear_gemm_plan* const* plans, int32_t n, void* stream);
/* Tile geometry actually used: BN, grid.x (N tiles), grid.y (M tiles), splits. */
int dear_gemm_plan_info(dear_gemm_plan* plan, int32_t* bn, int32_t* n_tiles, int32_t* m_tiles,
                        int32_t* splits);
/* Cluster shape (cm x cn CTAs sharing operands by TMA multicast) and how
 * many such clusters are resident at once. */
int dear_gemm_plan_cluster(dear_gemm_plan* plan, int32_t* cm, int32_t* cn, int32_t* resident);
/* Plan flags (dear_gemm_plan_set_flags).
 * DEAR_GEMM_EARLY_OPERANDS: the caller guarantees A and B are not written by
 * any kernel that may still be running when this GEMM starts (e.g. operands
 * that stay read-only across a chain of GEMM launches on the stream). The
 * GEMM then streams its operands while the preceding kernel drains under
 * programmatic dependent launch; D is still touched only after it completes. */
#define DEAR_GEMM_EARLY_OPERANDS 1
/* DEAR_GEMM_RED_ADD: accumulate fp32 D with per-thread red.global.add instead
 * of staged TMA reduce-add (a tuning choice; the sums are the same up to
 * fp32 addition order, as with any split-K). */
#define DEAR_GEMM_RED_ADD 2
/* Override the cost model's tile choice: bn (multiple of 16, <= 256) and
 * single-CTA (pair = 0) or 2-CTA pair (pair = 1) tiles; multicast clusters
 * off. Used by the plan-time autotuner (paper_2302_12445_b200.gemm.autotune). */
int dear_gemm_plan_set_tile(dear_gemm_plan* plan, int32_t bn, int32_t pair);
/* Override the split-K count of an accumulating plan (>= 1; clipped to the
 * number of 64-deep k-blocks). */
int dear_gemm_plan_set_splits(dear_gemm_plan* plan, int32_t split_k);
int dear_gemm_plan_set_flags(dear_gemm_plan* plan, int32_t flags);
/* 1 when the plan runs as 2-CTA pairs (cta_group::2 MMAs on 256-row tiles;
 * reported by dear_gemm_plan_cluster as cm = 2, cn = 1), else 0. */
int dear_gemm_plan_pair(dear_gemm_plan* plan, int32_t* pair);
/* Profiling: when set, every subsequent launch writes 8 %globaltimer stamps
 * per CTA into this device buffer (CTA start, prologue done, dependency
 * released, first stage landed, last MMA issued, epilogue done, CTA end);
 * NULL turns it off (the default). */
int dear_gemm_set_trace(void* device_buffer);
int dear_gemm_plan_destroy(dear_gemm_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* DEAR_GEMM_H_ */
