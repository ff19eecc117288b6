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
  int64_t start;  // prefix sum of len over the op's unit list
  int32_t peer;   // unpack units: rank whose slot `a` points into (peer backend)
  int32_t pad;
};

// Units are cut at this length only to bound the per-unit index arithmetic;
// load balance comes from giving every CTA an equal slice of the op's total
// elements: the host precomputes, per CTA, the unit and offset its slice
// starts at (a Slice table next to the units).
constexpr int64_t kUnitElems = 1 << 20;

// Grid of every bucket-op launch: 4 resident 256-thread CTAs on each of the
// 148 SMs, one wave, equal element slices.
#ifndef DEAR_SLICES_PER_SM
#define DEAR_SLICES_PER_SM 4
#endif
constexpr int kSlices = 148 * DEAR_SLICES_PER_SM;
// The update kernels stream two inputs per round (run_unit_pre) and need more
// registers: 3 CTAs per SM for the shard update, 2 for the P = 1 direct update
// (graph-chained A/B, profiles/r01e_hbm_kernels_ab.log). Their slice tables use
// the first kUpdSlices / kDirSlices entries of a kSlices-sized region.
#ifndef DEAR_UPD_CTAS_PER_SM
#define DEAR_UPD_CTAS_PER_SM 3
#endif
#ifndef DEAR_DIR_CTAS_PER_SM
#define DEAR_DIR_CTAS_PER_SM 2
#endif
#ifndef DEAR_PACK_CTAS_PER_SM
#define DEAR_PACK_CTAS_PER_SM 4
#endif
#ifndef DEAR_UNPACK_CTAS_PER_SM
#define DEAR_UNPACK_CTAS_PER_SM 4
#endif
// Waves of CTAs per launch (slices = resident CTAs x waves; > 1 lets the
// block scheduler balance short slices as CTAs retire).
#ifndef DEAR_HBM_WAVES
#define DEAR_HBM_WAVES 1
#endif
constexpr int kPackSlices = 148 * DEAR_PACK_CTAS_PER_SM * DEAR_HBM_WAVES;
constexpr int kUnpackSlices = 148 * DEAR_UNPACK_CTAS_PER_SM * DEAR_HBM_WAVES;
static_assert(kPackSlices <= kSlices && kUnpackSlices <= kSlices, "slice regions are kSlices long");
constexpr int kUpdSlices = 148 * DEAR_UPD_CTAS_PER_SM * DEAR_HBM_WAVES;
constexpr int kDirSlices = 148 * DEAR_DIR_CTAS_PER_SM * DEAR_HBM_WAVES;
static_assert(kUpdSlices <= kSlices && kDirSlices <= kSlices, "slice regions are kSlices long");
// NVLink-bound peer kernels need far fewer CTAs to saturate the links
// (~1.2 MB in flight); a small grid leaves the SMs to the concurrent GEMMs.
#ifndef DEAR_PEER_SLICES
#define DEAR_PEER_SLICES 64
#endif
constexpr int kPeerSlices = DEAR_PEER_SLICES;
// Zero-copy peer kernels: one CTA per SM (the reduce-scatter is bound by
// NVLink round trips, so more requests in flight shorten it — and the time it
// shares the SMs with the backprop GEMMs; profiles/r01e_zc_n2_sweep.log).
#ifndef DEAR_ZC_SLICES
#define DEAR_ZC_SLICES 148
#endif
constexpr int kZcSlices = DEAR_ZC_SLICES;
// Peer-backend pack: one CTA per SM, one contiguous slice per CTA.
constexpr int kPackPeerSlices = 148;

struct Slice {
  Unit first;     // the slice's first piece, pointers pre-offset (one load per CTA)
  int32_t unit;   // index of that unit; later pieces continue at unit + 1
  int32_t pad;
  int64_t count;  // elements in the slice (multiple of 4 except the last)
};

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

// Launchers (stream-ordered, no host sync). n_units may be 0; total is the
// sum of the units' lengths.
// `grid` <= kSlices CTAs (each walks slices blockIdx.x, +grid, ...); 0 = kSlices.
cudaError_t launch_pack(const Unit* units, const Slice* slices, int64_t total, float scale,
                        int grid, cudaStream_t s);
cudaError_t launch_update(const Unit* units, const Slice* slices, int64_t total,
                          const HyperParams* hp, int has_momentum_buf, int use_momentum,
                          int use_wd, int grid, cudaStream_t s);
cudaError_t launch_unpack(const Unit* units, const Slice* slices, int64_t total, int with_shadow,
                          int grid, cudaStream_t s);
// Host: the Slice table (n_slices entries, one per CTA) for a unit list with
// prefix starts.
// c_elem_bytes: element size behind Unit::c (4 momentum, 2 bf16 shadow, 0 none).
void make_slices(const Unit* units, int n_units, int64_t total, Slice* out,
                 int n_slices, int c_elem_bytes);

// Local-group collectives over P same-device buffers (ring order, in place):
// rs: bufs[r][r*stride + i] = fold_k bufs[(r+1+k)%P][r*stride + i], k = 0..P-1
//     — slot r carries chunk c = (r+1)%P, folded left starting at rank c, then
//     c+1, ..., c-1: the reference's ring-arrival order (collective.cpp:70-90).
// ag: bufs[r][s*stride + i] = bufs[s][s*stride + i] for all r != s.
cudaError_t launch_local_reduce_scatter(float* const* bufs_dev, int P, int64_t stride,
                                        int64_t count, cudaStream_t s);
cudaError_t launch_local_all_gather(float* const* bufs_dev, int P, int64_t stride,
                                    int64_t count, cudaStream_t s);

// ---- Peer (NVLink P2P) backend -------------------------------------------
// Every rank's arena is IPC-mapped by every other rank; the same object lives
// at address p + delta[k] in rank k's arena. Per bucket, each rank keeps three
// monotonically increasing completion counters in its arena (packs, updates,
// gathers done); ordering across GPUs is "wait until every peer's counter
// reaches mine", so no host-side epoch is baked into CUDA graphs.
constexpr int kMaxPeers = 16;
struct PeerArgs {
  int64_t delta[kMaxPeers];  // peer arena base - own arena base (bytes)
  int32_t P;
  int32_t rank;
  long long spin_limit;  // clock64 cycles a cross-GPU wait may spin before __trap (0: forever)
};
struct BucketFlags {
  uint32_t packed;
  uint32_t updated;
  uint32_t gathered;
  uint32_t pad;
  uint32_t done[4];  // per-op CTA completion counters (last CTA signals)
};

// One-warp kernel: waits until, for every peer k, the counter at
// watch + delta[k] >= *mine (acquire, system scope).
cudaError_t launch_wait_peers(const uint32_t* mine, const uint32_t* watch, const PeerArgs& pa,
                              cudaStream_t s);
// pack with a completion signal (flags->packed += 1 after all CTAs finish).
// P = 1, no momentum: w <- sgd(w, grad) and the bf16 copy, from the layers.
cudaError_t launch_update_direct(const Unit* units, const Slice* slices, int64_t total,
                                 const HyperParams* hp, int use_wd, int with_shadow,
                                 cudaStream_t s);
// `slices` holds kPackPeerSlices entries (one per CTA).
cudaError_t launch_pack_signal(const Unit* units, const Slice* slices, int64_t total, float scale,
                               BucketFlags* flags, const PeerArgs& pa, cudaStream_t s);
// Push reduce-scatter (DEAR_PUSH_RS=1 on the zero-copy layout): every chunk of
// our gradients (x scale) to slot `rank` of its owner's bucket buffer (unit
// peer = owner, reached at U.b + pa.delta[owner]) once every owner reduced
// our previous push; then flags->packed += 1. `slices`: kPackPeerSlices.
cudaError_t launch_pack_push(const Unit* units, const Slice* slices, float scale,
                             BucketFlags* flags, const PeerArgs& pa, cudaStream_t s);
// Fused reduce-scatter + shard SGD update: for each own-shard element, sum the
// peers' slot-`rank` values in ring order (rank+1, ..., rank), update, write
// w' into the own slot; then flags->updated += 1.
cudaError_t launch_rs_update_peer(const Unit* units, const Slice* slices, int64_t total,
                                  const HyperParams* hp, int has_momentum_buf, int use_momentum,
                                  int use_wd, const PeerArgs& pa, BucketFlags* flags,
                                  cudaStream_t s);
// Fused all-gather + unpack: every element read from its owner's slot (remote
// over NVLink unless owned), written to the params (+ bf16 copy); then
// flags->gathered += 1.
// `sa`: where unit sources live on each rank (the arena deltas for bucket
// slots; the parameter-allocation deltas for zero-copy).
// `n_slices`: entries of `slices` (kPeerSlices, or kZcSlices for zero-copy),
// one CTA each.
cudaError_t launch_ag_unpack_peer(const Unit* units, const Slice* slices, int64_t total,
                                  int with_shadow, const PeerArgs& pa, const PeerArgs& sa,
                                  BucketFlags* flags, int n_slices, cudaStream_t s);
// Zero-copy fused reduce-scatter + update: the owned chunk of every rank's
// gradients (at ga.delta[k]) summed in ring order, 1/P, SGD, written into
// the own parameters (+ bf16 copy); announces / waits on flags->packed and
// bumps flags->updated. mom_base: the bucket's momentum shard (or null).
// announce = 0 (push reduce-scatter): the pack already announced; ga then
// holds the local slot offsets (slot k = rank k's pushed contribution).
cudaError_t launch_rs_update_zc(const Unit* units, const Slice* slices, const HyperParams* hp,
                                int has_momentum_buf, float* mom_base, int use_momentum,
                                int use_wd, int with_shadow, const PeerArgs& pa,
                                const PeerArgs& ga, BucketFlags* flags, cudaStream_t s,
                                int announce = 1);

// Comm-kernel phase trace (profiling): records of 40 B {t0, t_arrived, t_end,
// kind, tag, epoch, cta}; buf = null turns it off; the count restarts at 0.
cudaError_t set_comm_trace(void* buf, uint32_t cap);
cudaError_t comm_trace_count(uint32_t* n);

// hp->lr = lr, stream-ordered (dear_set_lr; graph-capturable).
cudaError_t launch_set_lr(HyperParams* hp, float lr, cudaStream_t s);

// ---- NVLS (NVLink SHARP multicast) backend --------------------------------
// Per-bucket counters in the symmetric heap; every rank's copy is bumped at
// once through the multicast alias (multimem.red), polled locally.
struct NvlsFlags {
  uint32_t packed;    // += 1 per rank whose gradients of the bucket are complete
  uint32_t updated;   // += 1 per owner whose reduce-scatter + update finished
  uint32_t gathered;  // += 1 per owner whose broadcast (all-gather) finished
  uint32_t pad[13];   // 64 B per bucket
};
struct NvlsArgs {
  int64_t mc_delta;   // multicast alias - local address (bytes), heap-wide
  NvlsFlags* ucf;     // this bucket's counters, local address
  NvlsFlags* mcf;     // ... multicast alias
  int32_t P;
  int32_t pad;
  long long spin_limit;
};
// Owned-chunk units (a = grad, b = param, c = bf16 copy; the zero-copy RS
// tables). RS: multimem.ld_reduce of the gradients + SGD into the parameters;
// bumps flags->updated (local epoch) and na.mcf->updated (every rank).
cudaError_t launch_rs_update_nvls(const Unit* units, const Slice* slices, const HyperParams* hp,
                                  int has_momentum_buf, float* mom_base, int use_momentum,
                                  int use_wd, const NvlsArgs& na, BucketFlags* flags,
                                  cudaStream_t s);
// AG: multicast stores of the owned chunk (+ bf16 copy) into every rank, then
// waits until every owner's broadcast of the bucket landed.
cudaError_t launch_ag_nvls(const Unit* units, const Slice* slices, int with_shadow,
                           const NvlsArgs& na, BucketFlags* flags, cudaStream_t s);
// One warp: until every owner's RS of this bucket (epoch *epoch) finished.
cudaError_t launch_nvls_wait_updated(const uint32_t* epoch, const NvlsArgs& na, cudaStream_t s);

// Same-device peer group (LocalGroup "peer"): one rank's arguments of a peer
// kernel. The group runs each reduce-scatter / all-gather as ONE cooperative
// launch holding every rank's CTAs (nb per rank), so the kernels' cross-rank
// waits are between co-resident CTAs of one grid.
struct GroupOp {
  const Unit* units;
  const Slice* slices;
  const HyperParams* hp;
  float* mom;          // zero-copy RS: the bucket's momentum shard (or null)
  BucketFlags* flags;
  PeerArgs pa;         // arena deltas (counters, slot buffers)
  PeerArgs sa;         // zero-copy RS: gradient deltas; AG: source deltas
  int32_t n_slices;
  int32_t pad;
};
cudaError_t launch_group_rs_zc(const GroupOp* ops, int P, int nb, int has_buf, int use_momentum,
                               int use_wd, int with_shadow, cudaStream_t s);
cudaError_t launch_group_rs_peer(const GroupOp* ops, int P, int nb, int has_buf,
                                 int use_momentum, int use_wd, cudaStream_t s);
cudaError_t launch_group_ag(const GroupOp* ops, int P, int nb, int with_shadow, cudaStream_t s);

// Order-independent 64-bit hash of float bit patterns (sum of mixed words),
// accumulated into *acc with atomics. Used by dear_check_replicas.
cudaError_t launch_hash(const float* x, int64_t n, uint64_t salt,
                        unsigned long long* acc, cudaStream_t s);

}  // namespace dear
