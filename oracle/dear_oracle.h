/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's DeAR hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this (as the checker). The product library never links it.
 *
 * Parity status: PINNED. Every function below is checked by tests/ against
 *   (a) golden fixtures produced by the reference itself (oracle/_ref, built
 *       from /root/reference/proj/src unmodified; tests/golden/make_golden.py),
 *   (b) the reference's own known-answer tests (test_collective.cpp,
 *       test_model_fusion.cpp, acceptance.cpp criterion 2), restated in
 *       tests/test_oracle.py.
 * Exceptions, labelled UNPINNED: momentum / weight decay / nesterov (the
 * reference's SgdState has only lr, collective.hpp:77-80), and the fp32
 * variants (the reference is fp64).
 */
#ifndef DEAR_ORACLE_H_
#define DEAR_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + std::uniform_real_distribution<double>(-1,1)
 * as used by the reference's tests (test_collective.cpp:27-37). */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;
void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
double or_uniform_pm1(or_mt64* g);
/* P*d values, worker-major, one generator — random_vectors() of the tests. */
void or_random_vectors(int P, int64_t d, uint64_t seed, double* out);
void or_random_vectors_f32(int P, int64_t d, uint64_t seed, float* out);

/* ---- Model presets (model.cpp:80-168). profile 0 = Uniform, 1 = Imbalanced.
 * Returns L (tensor count) or -1 on unknown name / cap too small. */
int or_preset_params(const char* name, int profile, int64_t* out, int cap);

/* ---- Fusion partitioner (fusion.cpp:29-70). layer_bytes[0] is layer 1.
 * buffer_bytes == 0 -> per-layer plan. Groups are written in BP issue order
 * (groups[0] holds layer L). Returns group count, -1 on invalid input. */
int or_build_fusion_plan(const int64_t* layer_bytes, int L, int64_t buffer_bytes,
                         int32_t* low, int32_t* high);

/* ---- chunk_ranges (collective.cpp:39-57): begin has P+1 entries. */
int or_chunk_ranges(int64_t d, int P, int64_t* begin);
/* Owner of chunk c after ring reduce-scatter (collective.cpp:94): (c-1) mod P. */
int or_chunk_owner(int c, int P);

/* ---- ring reduce-scatter (collective.cpp:59-101) restated as the sum it
 * computes: chunk c = v_c + v_{c+1} + ... + v_{c-1} folded left in ring
 * arrival order. in: P x d (worker-major); out: d (chunk c at its range). */
void or_ring_reduce_scatter(int P, int64_t d, const double* in, double* out);
/* all_reduce_average (collective.cpp:159-164): sum then * (1.0/P). */
void or_all_reduce_average(int P, int64_t d, const double* in, double* out);
/* sgd_step (collective.cpp:166-194): w -= lr * mean; identical replicas, so
 * one weight vector is carried. Returns -1 on bad args. */
int or_sgd_step(int P, int64_t d, double lr, double* w, const double* grads);

/* ---- UNPINNED extension: PyTorch SGD semantics for momentum / dampening /
 * weight decay / nesterov, applied to the averaged gradient exactly where the
 * reference applies its update. `buf` has d entries; *has_buf 0 on the first
 * step (buf initialised from the gradient, as torch.optim.SGD does). */
int or_sgd_step_momentum(int P, int64_t d, double lr, double momentum, double dampening,
                         double weight_decay, int nesterov, double* w, double* buf,
                         int* has_buf, const double* grads);

/* ---- fp32 variants with the same per-element operation order (the GPU
 * computes in fp32). `prescale` = apply 1/P before the ring sum (exact for
 * P = 2^k, SURVEY §7 hard parts) instead of after it. */
void or_ring_reduce_scatter_f32(int P, int64_t d, const float* in, float* out);
int or_sgd_step_f32(int P, int64_t d, float lr, float momentum, float dampening,
                    float weight_decay, int nesterov, float* w, float* buf, int* has_buf,
                    const float* grads, int prescale);

#ifdef __cplusplus
}
#endif
#endif
