// Internal interface between the host runtime (runtime.cpp) and the sm_100a
// kernels (kernels.cu). Not part of the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace dear {

// One contiguous run of a bucket op: the intersection of one layer tensor
// with one chunk, cut into pieces of at most kUnitElems elements so every CTA
// gets a similar share. Pointer roles per op:
//   pack   : a = grad + j (src)        b = buf + off (dst)
//   update : a = param + j (w, read)   b = buf + off (grad in, w' out)
//            c = momentum + off'       (nullptr without momentum)
//   unpack : a = buf + off (src)       b = param + j (dst)
//            c = bf16 shadow + j       (nullptr when not registered)
struct Unit {
  const float* a;
  float* b;
  void* c;
  int64_t len;
};

constexpr int64_t kUnitElems = 8192;

// Device-resident optimizer hyper-parameters (graph-safe lr changes).
struct HyperParams {
  float lr;
  float momentum;
  float one_minus_dampening;
  float weight_decay;
  float inv_p;       // 1/P applied in update when !prescaled
  int32_t nesterov;
  int32_t prescaled; // 1/P already applied by pack (P = 2^k)
  int32_t pad;
};

// Launchers (stream-ordered, no host sync). n_units may be 0.
cudaError_t launch_pack(const Unit* units, int n_units, float scale, cudaStream_t s);
cudaError_t launch_update(const Unit* units, int n_units, const HyperParams* hp,
                          int has_momentum_buf, int use_momentum, int use_wd, cudaStream_t s);
cudaError_t launch_unpack(const Unit* units, int n_units, int with_shadow, cudaStream_t s);

// Local-group collectives over P same-device buffers (ring order, in place):
// rs: bufs[r][r*stride + i] = fold_k bufs[(r+1+k)%P][r*stride + i], k = 0..P-1
//     — slot r carries chunk c = (r+1)%P, folded left starting at rank c, then
//     c+1, ..., c-1: the reference's ring-arrival order (collective.cpp:70-90).
// ag: bufs[r][s*stride + i] = bufs[s][s*stride + i] for all r != s.
cudaError_t launch_local_reduce_scatter(float* const* bufs_dev, int P, int64_t stride,
                                        int64_t count, cudaStream_t s);
cudaError_t launch_local_all_gather(float* const* bufs_dev, int P, int64_t stride,
                                    int64_t count, cudaStream_t s);

// Order-independent 64-bit hash of float bit patterns (sum of mixed words),
// accumulated into *acc with atomics. Used by dear_check_replicas.
cudaError_t launch_hash(const float* x, int64_t n, uint64_t salt,
                        unsigned long long* acc, cudaStream_t s);

}  // namespace dear
