// DeAR runtime: tensor registration, bucket layout in HBM, the BackPipe /
// FeedPipe schedule on a dedicated high-priority comm stream, and the two
// collective backends (NCCL over NVLink/NVSwitch; a local group emulating P
// ranks on one device).
//
// Schedule contract (the reference's task DAG, task_graph.cpp:127-210, with
// the two-stream semantics of simulate.cpp:65-159):
//   BackPipe  : bucket g complete (all its layers' grads reported)
//               -> [comm] wait grad events, pack_g, RS_g, update_g
//               buckets are issued strictly in plan order (:186-194); NCCL
//               additionally requires every rank to issue collectives in the
//               same order, which plan order guarantees.
//   BARRIER   : dear_step — comm stream waits for the caller's stream.
//   FeedPipe  : AG_g + unpack_g in reverse plan order (:199-206); FF_l waits
//               on ag_done[g(l)] only (:207).
//   WFBP      : RS_g, update_g, AG_g, unpack_g back to back during BackPipe
//               (all-reduce as RS + AG).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <thread>
#include <cstdio>
#include <deque>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dear.h"
#include "dear_internal.h"
#include "dear_kernels.h"

namespace dear {

namespace {

thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(DEAR_EINTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    throw Error(DEAR_EINTERNAL, std::string(what) + ": " + ncclGetErrorString(r));
  }
}

void invalid(const std::string& m) { throw Error(DEAR_EINVAL, m); }

bool is_fused(int policy) {
  return policy == DEAR_POLICY_WFBP_FUSED || policy == DEAR_POLICY_DEAR_FUSED;
}
bool is_dear(int policy) {
  return policy == DEAR_POLICY_DEAR || policy == DEAR_POLICY_DEAR_FUSED;
}
bool is_pp(int policy) { return policy == DEAR_POLICY_PRIORITY_PARTITION; }

enum OpKind { OP_FENCE_READY, OP_FENCE_STEP, OP_PACK, OP_RS, OP_UPDATE, OP_AG, OP_UNPACK,
              OP_AG_DONE, OP_CALLER_WAIT_PACKED, OP_SET_LR };

struct Op {
  OpKind kind;
  int bucket;
  cudaStream_t stream;  // OP_CALLER_WAIT_PACKED
  float value = 0.f;    // OP_SET_LR
  bool collective() const { return kind == OP_RS || kind == OP_AG; }
};

enum TimingEv { T_PACK0, T_PACK1, T_RS1, T_UPD1, T_AG0, T_AG1, T_UNPACK1, T_COUNT };

struct LayerReg {
  float* param = nullptr;
  float* grad = nullptr;
  void* shadow = nullptr;
  int64_t numel = -1;
  int bucket = -1;
  int64_t off = 0;  // offset of the layer inside its bucket's flat order
  int n_parts = 1;  // PRIORITY_PARTITION: buckets bucket .. bucket + n_parts - 1
  bool ready = false;
};

struct Bucket {
  int low = 0, high = 0;
  int part = 0;     // PRIORITY_PARTITION: 1-based part of layer `low` (== high)
  int64_t e0 = 0;   // ... covering elements [e0, e0 + d) of that layer
  int64_t d = 0, stride = 0;
  float* buf = nullptr;  // P * stride: slot r holds chunk (r+1)%P
  float* mom = nullptr;  // stride (own shard's momentum), or null
  int layers_left = 0;
  bool complete = false;
  std::vector<cudaStream_t> ready_streams;
  std::vector<cudaEvent_t> ready_events;
  Unit *pack_u = nullptr, *upd_u = nullptr, *unpack_u = nullptr;
  int n_pack = 0, n_upd = 0, n_unpack = 0;
  int64_t e_pack = 0, e_upd = 0, e_unpack = 0;  // elements per op
  Slice *pack_s = nullptr, *upd_s = nullptr, *unpack_s = nullptr;  // kSlices each
  Slice *upd_ps = nullptr, *unpack_ps = nullptr;  // kPeerSlices each (peer kernels)
  Slice* pack_ps = nullptr;                        // kPackPeerSlices (peer pack)
  // Zero-copy peer path: RS units over the owned chunk (a = grad, b = param,
  // c = bf16 copy) and AG units over the other chunks (a = b = param on the
  // owner `peer`, c = bf16 copy); kPeerSlices slices each.
  Unit *zrs_u = nullptr, *zag_u = nullptr;
  int n_zrs = 0, n_zag = 0;
  int64_t e_zrs = 0, e_zag = 0;
  Slice *zrs_ps = nullptr, *zag_ps = nullptr;
  Unit* dir_u = nullptr;                           // P = 1 direct update (grad -> param)
  int n_dir = 0;
  int64_t e_dir = 0;
  Slice* dir_s = nullptr;                          // kSlices
  // Push reduce-scatter: P slots of pstride fp32 (slot k = rank k's pushed
  // copy of this rank's chunk; pieces padded so each starts in its
  // parameter's 16 B phase), pack units (a = grad, b = slot `rank` in the
  // owner's buffer, peer = owner) and RS units (a = slot 0 position, b =
  // param, c = bf16 copy).
  int64_t pstride = 0;
  float* pbuf = nullptr;
  Unit *ppk_u = nullptr, *prs_u = nullptr;
  int n_ppk = 0, n_prs = 0;
  int64_t e_ppk = 0, e_prs = 0;
  Slice *ppk_ps = nullptr, *prs_ps = nullptr;
  BucketFlags* flags = nullptr;  // peer backend completion counters (in the arena)
  bool any_shadow = false;
  bool mom_init = false;
  cudaEvent_t ag_done = nullptr;
  unsigned long long ag_capture = 0;  // capture id ag_done was recorded in (0: eager)
  bool ag_live = false;          // an AG for this bucket is enqueued
  cudaStream_t waited = nullptr; // last stream that waited on ag_done
  bool waited_valid = false;
  cudaEvent_t t[T_COUNT] = {};
  bool t_rec[T_COUNT] = {};
};

}  // namespace
}  // namespace dear

using namespace dear;

struct dear_local_group {
  int P = 0;
  int transport = DEAR_LOCAL_RING;
  // PEER transport: per bucket, the P ranks' GroupOp records of its
  // reduce-scatter and all-gather kernels (device), nb CTAs per rank.
  GroupOp* ops_dev = nullptr;
  int nb = 0;
  bool connected = false;
  std::vector<dear_ctx*> ranks;
  std::map<int, float**> bufs_dev;  // bucket -> device array of P buffers
  cudaEvent_t arrive[64] = {};
  cudaEvent_t done = nullptr;
  bool draining = false;
  ~dear_local_group();
  void drain();
  void run_collective(const Op& op);
};

struct dear_ctx {
  bool local = false;
  ncclComm_t comm = nullptr;
  dear_local_group* group = nullptr;
  int rank = 0, P = 1;
  int device = 0;
  cudaStream_t compute = nullptr;
  cudaStream_t comm_stream = nullptr;
  dear_cfg cfg{};
  bool finalized = false;
  std::vector<LayerReg> layers;  // index layer-1
  std::vector<Bucket> buckets;   // plan order
  int rs_cursor = 0;
  int reported = 0;
  bool ags_deferred = false;
  int64_t iteration = 0;
  HyperParams hp_host{};
  HyperParams* hp_dev = nullptr;
  char* arena = nullptr;
  float pack_scale = 1.f;
  cudaEvent_t packed_ev = nullptr;
  cudaEvent_t step_ev = nullptr;
  cudaEvent_t join_ev = nullptr;
  unsigned long long* hash_dev = nullptr;
  size_t arena_bytes = 0;
  bool peer = false;             // NVLink peer backend (fused RS+update, AG+unpack)
  // P = 1 without momentum: the reduce-scatter / all-gather are the identity,
  // so one kernel updates the parameters (and their bf16 copy) straight from
  // the gradients — 14 B/element instead of pack + update + unpack's 30.
  bool direct = false;
  PeerArgs pa{};
  // Zero-copy (peer backend): every rank's gradient and parameter allocations
  // are IPC-mapped too; ga / qa hold the per-rank deltas of those tensors.
  bool zc = false;
  bool zc_tables = false;  // finalize built the zero-copy unit tables
  PeerArgs ga{}, qa{};
  // Push reduce-scatter (DEAR_PUSH_RS=1, multi-process zero-copy): each rank
  // writes every chunk of its gradients into slot `rank` of the chunk owner's
  // push buffer (posted NVLink stores); the owner sums its P slots locally in
  // ring order and updates. The all-gather stays the zero-copy pull.
  bool push_tables = false;
  bool push = false;
  // Same-device peer group (dear_local_group_create_ex(.., DEAR_LOCAL_PEER)):
  // the P ranks are contexts of this process on one device, and the peer
  // kernels address each other's memory with in-process deltas instead of
  // IPC mappings.
  bool same_dev = false;
  // NVLS backend (dear_nvls_connect): multicast reduce-scatter / broadcast
  // all-gather on the symmetric heap; na.ucf / na.mcf point at bucket 0's
  // counters (bucket g at + g).
  bool nvls = false;
  NvlsArgs na{};
  NvlsArgs nvls_args(int g) const {
    NvlsArgs a = na;
    a.ucf += g;
    a.mcf += g;
    return a;
  }
  std::vector<void*> peer_maps;  // cudaIpcOpenMemHandle mappings to close
  bool timing = false;
  std::vector<std::string> trace;
  std::deque<Op> queue;  // local mode: ops not yet executed
  // dear_group_dependency: comm-stream dispatch sequence of one iteration
  // (>0: RS of bucket v-1, <0: AG of bucket -v-1), dear_set_comm_order.
  std::vector<int32_t> comm_order;
  size_t order_cursor = 0;
  size_t order_tail = 0;  // first entry after the last RS: the step-time AGs

  ~dear_ctx();
  void enqueue(Op op);
  void exec(const Op& op);
  void complete_bucket(int b);
  void enqueue_backpipe(int b);
  void enqueue_feedpipe(cudaStream_t fence_stream);
  void enqueue_ag(int g);
  void enqueue_ordered_ags();
  void record_t(int b, int which);
  std::string label(const char* kind, int b) const;
};

namespace {

void free_events(std::vector<cudaEvent_t>& evs) {
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  evs.clear();
}

// Id of the CUDA-graph capture `s` is part of, 0 when not capturing.
unsigned long long capture_id(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  cuda_check(cudaStreamGetCaptureInfo(s, &st, &id), "cudaStreamGetCaptureInfo");
  return st == cudaStreamCaptureStatusActive ? id : 0;
}

cudaEvent_t new_event(bool timing) {
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming),
             "cudaEventCreate");
  return e;
}

// Units for one bucket op: the intersections of the bucket's layers (in
// ascending layer order, the flatten order) with chunk range [cb, ce), cut at
// kUnitElems. emit(layer, j0, len, pos) where pos is the offset inside the
// chunk.
template <typename Emit>
void for_each_piece(const dear_ctx& ctx, const Bucket& B, int64_t cb, int64_t ce, Emit&& emit) {
  if (B.part > 0) {  // one part of one layer: its elements e0 ..
    const int64_t s = std::max<int64_t>(0, cb), e = std::min(B.d, ce);
    for (int64_t p = s; p < e; p += kUnitElems)
      emit(B.low, B.e0 + p, std::min(kUnitElems, e - p), p - cb);
    return;
  }
  for (int l = B.low; l <= B.high; ++l) {
    const LayerReg& L = ctx.layers[static_cast<size_t>(l - 1)];
    const int64_t lb = L.off, le = L.off + L.numel;
    const int64_t s = std::max(lb, cb), e = std::min(le, ce);
    for (int64_t p = s; p < e; p += kUnitElems) {
      const int64_t len = std::min(kUnitElems, e - p);
      emit(l, p - lb, len, p - cb);
    }
  }
}

// Prefix offsets of the units from `first` to the end; returns the total.
int64_t set_starts(std::vector<Unit>& u, size_t first) {
  int64_t at = 0;
  for (size_t i = first; i < u.size(); ++i) {
    u[i].start = at;
    at += u[i].len;
  }
  return at;
}

}  // namespace

dear_local_group::~dear_local_group() {
  if (ops_dev) cudaFree(ops_dev);
  for (auto& kv : bufs_dev) cudaFree(kv.second);
  for (cudaEvent_t e : arrive)
    if (e) cudaEventDestroy(e);
  if (done) cudaEventDestroy(done);
}

void dear_local_group::run_collective(const Op& op) {
  dear_ctx* c0 = ranks[0];
  const Bucket& B0 = c0->buckets[static_cast<size_t>(op.bucket)];
  if (transport == DEAR_LOCAL_PEER) {
    // Every rank's comm stream reached this collective: ONE cooperative launch
    // of the peer kernel over all ranks' data on rank 0's comm stream.
    if (!connected) invalid("local group: call dear_local_group_connect before the first step");
    for (int r = 0; r < P; ++r) {
      if (!arrive[r]) arrive[r] = new_event(false);
      cuda_check(cudaEventRecord(arrive[r], ranks[static_cast<size_t>(r)]->comm_stream), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(c0->comm_stream, arrive[r], 0), "cudaStreamWaitEvent");
    }
    const GroupOp* ops = ops_dev + (static_cast<size_t>(op.bucket) * 2 + (op.kind == OP_AG ? 1 : 0)) *
                                       static_cast<size_t>(P);
    const dear_cfg& cf = c0->cfg;
    if (op.kind == OP_RS) {
      cuda_check(c0->zc ? launch_group_rs_zc(ops, P, nb, B0.mom_init ? 1 : 0, cf.momentum != 0.0,
                                             cf.weight_decay != 0.0, B0.any_shadow ? 1 : 0,
                                             c0->comm_stream)
                        : launch_group_rs_peer(ops, P, nb, B0.mom_init ? 1 : 0,
                                               cf.momentum != 0.0, cf.weight_decay != 0.0,
                                               c0->comm_stream),
                 "group reduce-scatter kernel");
    } else {
      cuda_check(launch_group_ag(ops, P, nb, B0.any_shadow ? 1 : 0, c0->comm_stream),
                 "group all-gather kernel");
    }
    if (!done) done = new_event(false);
    cuda_check(cudaEventRecord(done, c0->comm_stream), "cudaEventRecord");
    for (int r = 1; r < P; ++r)
      cuda_check(cudaStreamWaitEvent(ranks[static_cast<size_t>(r)]->comm_stream, done, 0), "cudaStreamWaitEvent");
    return;
  }
  auto it = bufs_dev.find(op.bucket);
  if (it == bufs_dev.end()) {
    std::vector<float*> h(static_cast<size_t>(P));
    for (int r = 0; r < P; ++r) h[static_cast<size_t>(r)] = ranks[static_cast<size_t>(r)]->buckets[static_cast<size_t>(op.bucket)].buf;
    float** d = nullptr;
    cuda_check(cudaMalloc(&d, sizeof(float*) * static_cast<size_t>(P)), "cudaMalloc");
    cuda_check(cudaMemcpy(d, h.data(), sizeof(float*) * static_cast<size_t>(P), cudaMemcpyHostToDevice),
               "cudaMemcpy");
    it = bufs_dev.emplace(op.bucket, d).first;
  }
  for (int r = 0; r < P; ++r) {
    if (!arrive[r]) arrive[r] = new_event(false);
    cuda_check(cudaEventRecord(arrive[r], ranks[static_cast<size_t>(r)]->comm_stream), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(c0->comm_stream, arrive[r], 0), "cudaStreamWaitEvent");
  }
  const int64_t count = B0.stride;
  if (op.kind == OP_RS) {
    cuda_check(launch_local_reduce_scatter(it->second, P, B0.stride, count, c0->comm_stream),
               "local reduce-scatter");
  } else {
    cuda_check(launch_local_all_gather(it->second, P, B0.stride, count, c0->comm_stream),
               "local all-gather");
  }
  if (!done) done = new_event(false);
  cuda_check(cudaEventRecord(done, c0->comm_stream), "cudaEventRecord");
  for (int r = 1; r < P; ++r)
    cuda_check(cudaStreamWaitEvent(ranks[static_cast<size_t>(r)]->comm_stream, done, 0), "cudaStreamWaitEvent");
}

// Executes every rank's queued ops up to its next collective; a collective
// runs once all P ranks have it at the head of their queues (the lock-step
// rounds of collective.cpp:70-90, with the host as the round driver).
void dear_local_group::drain() {
  if (draining) return;
  draining = true;
  try {
    for (;;) {
      bool progress = false;
      for (dear_ctx* c : ranks) {
        if (!c) continue;
        while (!c->queue.empty() && !c->queue.front().collective()) {
          const Op op = c->queue.front();
          c->queue.pop_front();
          c->exec(op);
          progress = true;
        }
      }
      bool all_head = true;
      for (dear_ctx* c : ranks) {
        if (!c || c->queue.empty()) {
          all_head = false;
          break;
        }
      }
      if (all_head) {
        const Op& h = ranks[0]->queue.front();
        for (dear_ctx* c : ranks) {
          const Op& o = c->queue.front();
          if (o.kind != h.kind || o.bucket != h.bucket) {
            invalid("local group: ranks issued different collectives (out of lock-step)");
          }
        }
        const Op op = h;
        run_collective(op);
        for (dear_ctx* c : ranks) {
          c->queue.pop_front();
          c->exec(op);  // post-collective bookkeeping (timing, trace)
        }
        progress = true;
      }
      if (!progress) break;
    }
  } catch (...) {
    draining = false;
    throw;
  }
  draining = false;
}

dear_ctx::~dear_ctx() {
  // Same-device peer group: the other ranks' kernels read this context's
  // memory; the caller synchronised every rank, so this only drains the device.
  if (same_dev) cudaDeviceSynchronize();
  if (comm_stream) cudaStreamSynchronize(comm_stream);
  for (Bucket& b : buckets) {
    free_events(b.ready_events);
    if (b.ag_done) cudaEventDestroy(b.ag_done);
    for (cudaEvent_t e : b.t)
      if (e) cudaEventDestroy(e);
  }
  if (packed_ev) cudaEventDestroy(packed_ev);
  if (step_ev) cudaEventDestroy(step_ev);
  if (join_ev) cudaEventDestroy(join_ev);
  for (void* m : peer_maps) cudaIpcCloseMemHandle(m);
  if (arena) cudaFree(arena);
  if (comm_stream) cudaStreamDestroy(comm_stream);
  if (group) {
    for (auto& r : group->ranks)
      if (r == this) r = nullptr;
  }
}

std::string dear_ctx::label(const char* kind, int b) const {
  // task_label (task_graph.cpp:51-58): fused tasks name the group (gi+1);
  // per-layer WFBP names the layer (subject = high_layer, :170).
  const Bucket& B = buckets[static_cast<size_t>(b)];
  if (B.part > 0)  // task_label: "AR l<layer> p<part>" (task_graph.cpp:51-58)
    return std::string(kind) + " l" + std::to_string(B.high) + " p" + std::to_string(B.part);
  if (!is_fused(cfg.policy) && !is_dear(cfg.policy)) {
    return std::string(kind) + " l" + std::to_string(B.high);
  }
  return std::string(kind) + " g" + std::to_string(b + 1);
}

void dear_ctx::record_t(int b, int which) {
  if (!timing) return;
  Bucket& B = buckets[static_cast<size_t>(b)];
  // Inside a CUDA-graph capture the stamp must be an external event node to
  // be timed after a replay (graph-mode timelines, tools/graph_timeline.py).
  if (capture_id(comm_stream) != 0)
    cuda_check(cudaEventRecordWithFlags(B.t[which], comm_stream, cudaEventRecordExternal),
               "cudaEventRecordWithFlags");
  else
    cuda_check(cudaEventRecord(B.t[which], comm_stream), "cudaEventRecord");
  B.t_rec[which] = true;
}

void dear_ctx::exec(const Op& op) {
  Bucket* B = op.bucket >= 0 ? &buckets[static_cast<size_t>(op.bucket)] : nullptr;
  switch (op.kind) {
    case OP_FENCE_READY:
      for (cudaEvent_t e : B->ready_events)
        cuda_check(cudaStreamWaitEvent(comm_stream, e, 0), "cudaStreamWaitEvent");
      break;
    case OP_FENCE_STEP:
      cuda_check(cudaStreamWaitEvent(comm_stream, step_ev, 0), "cudaStreamWaitEvent");
      break;
    case OP_PACK:
      if (direct && !nvls) break;  // P = 1: the update reads the gradients in place
      record_t(op.bucket, T_PACK0);
      if (push) {
        cuda_check(launch_pack_push(B->ppk_u, B->ppk_ps, pack_scale, B->flags, pa, comm_stream),
                   "push pack kernel");
        cuda_check(cudaEventRecord(packed_ev, comm_stream), "cudaEventRecord");
        record_t(op.bucket, T_PACK1);
        break;
      }
      if (zc || nvls) {  // zero-copy: the reduce-scatter reads the gradients in place
        record_t(op.bucket, T_PACK1);
        break;
      }
      if (peer) {
        // The kernel first waits (in-kernel) until every peer gathered from
        // our buffer, which it then rewrites. One CTA per SM, one contiguous
        // slice each: the pack overlaps backprop GEMMs and the fused peer
        // kernels; a full 4-CTA/SM grid would hold every SM's register file
        // and stall the persistent GEMM (profiles/r01_n4_interference_matrix.log).
#ifdef DEAR_PEER_PACK_FULL
        cuda_check(launch_pack_signal(B->pack_u, B->pack_s, B->e_pack, pack_scale, B->flags, pa,
                                      comm_stream),
#else
        cuda_check(launch_pack_signal(B->pack_u, B->pack_ps, B->e_pack, pack_scale, B->flags, pa,
                                      comm_stream),
#endif
                   "pack kernel");
      } else {
        cuda_check(launch_pack(B->pack_u, B->pack_s, B->e_pack, pack_scale, 0, comm_stream),
                   "pack kernel");
      }
      cuda_check(cudaEventRecord(packed_ev, comm_stream), "cudaEventRecord");
      record_t(op.bucket, T_PACK1);
      break;
    case OP_RS:
      if (local && same_dev) {
        // The group already ran every rank's reduce-scatter (run_collective).
        if (cfg.momentum != 0.0) B->mom_init = true;
      } else if (nvls) {
        // The switch sums the owned chunk over the ranks (multimem.ld_reduce).
        cuda_check(launch_rs_update_nvls(B->zrs_u, B->zrs_ps, hp_dev, B->mom_init ? 1 : 0, B->mom,
                                         cfg.momentum != 0.0, cfg.weight_decay != 0.0,
                                         nvls_args(op.bucket), B->flags, comm_stream),
                   "nvls rs+update kernel");
        if (cfg.momentum != 0.0) B->mom_init = true;
      } else if (push) {
        // Our P slots (slot k = rank k's push), summed in ring order; the
        // pack already announced, so the kernel only waits.
        PeerArgs sa = pa;
        for (int k = 0; k < P; ++k)
          sa.delta[k] = static_cast<int64_t>(k) * B->pstride * static_cast<int64_t>(sizeof(float));
        cuda_check(launch_rs_update_zc(B->prs_u, B->prs_ps, hp_dev, B->mom_init ? 1 : 0, B->mom,
                                       cfg.momentum != 0.0, cfg.weight_decay != 0.0,
                                       B->any_shadow ? 1 : 0, pa, sa, B->flags, comm_stream, 0),
                   "push rs+update kernel");
        if (cfg.momentum != 0.0) B->mom_init = true;
      } else if (zc) {
        cuda_check(launch_rs_update_zc(B->zrs_u, B->zrs_ps, hp_dev, B->mom_init ? 1 : 0, B->mom,
                                       cfg.momentum != 0.0, cfg.weight_decay != 0.0,
                                       B->any_shadow ? 1 : 0, pa, ga, B->flags, comm_stream),
                   "zero-copy rs+update kernel");
        if (cfg.momentum != 0.0) B->mom_init = true;
      } else if (peer) {
        // Fused reduce-scatter + update over NVLink (OP_UPDATE becomes a no-op);
        // it waits in-kernel for every rank's pack of this bucket.
        cuda_check(launch_rs_update_peer(B->upd_u, B->upd_ps, B->e_upd, hp_dev, B->mom_init ? 1 : 0,
                                         cfg.momentum != 0.0, cfg.weight_decay != 0.0, pa,
                                         B->flags, comm_stream),
                   "rs+update kernel");
        if (cfg.momentum != 0.0) B->mom_init = true;
      } else if (!local && P > 1 && B->stride > 0) {
        nccl_check(ncclReduceScatter(B->buf, B->buf + static_cast<int64_t>(rank) * B->stride,
                                     static_cast<size_t>(B->stride), ncclFloat32, ncclSum, comm,
                                     comm_stream),
                   "ncclReduceScatter");
      }
      record_t(op.bucket, T_RS1);
      break;
    case OP_UPDATE:
      if (peer || nvls) break;
      if (direct) {
        cuda_check(launch_update_direct(B->dir_u, B->dir_s, B->e_dir, hp_dev,
                                        cfg.weight_decay != 0.0, B->any_shadow ? 1 : 0,
                                        comm_stream),
                   "direct update kernel");
        cuda_check(cudaEventRecord(packed_ev, comm_stream), "cudaEventRecord");
        record_t(op.bucket, T_UPD1);
        break;
      }
      cuda_check(launch_update(B->upd_u, B->upd_s, B->e_upd, hp_dev, B->mom_init ? 1 : 0,
                               cfg.momentum != 0.0, cfg.weight_decay != 0.0, 0, comm_stream),
                 "update kernel");
      if (cfg.momentum != 0.0) B->mom_init = true;
      record_t(op.bucket, T_UPD1);
      break;
    case OP_AG:
      if (!local) record_t(op.bucket, T_AG0);
      if (local && same_dev) {
        // run by the group (run_collective)
      } else if (nvls) {
        // The owner's multicast stores broadcast its chunk to every rank.
        cuda_check(launch_ag_nvls(B->zrs_u, B->zrs_ps, B->any_shadow ? 1 : 0,
                                  nvls_args(op.bucket), B->flags, comm_stream),
                   "nvls all-gather kernel");
      } else if (zc) {
        // Each owner's updated parameters, read over NVLink into ours.
        cuda_check(launch_ag_unpack_peer(B->zag_u, B->zag_ps, B->e_zag, B->any_shadow ? 1 : 0,
                                         pa, qa, B->flags, kZcSlices, comm_stream),
                   "zero-copy ag kernel");
      } else if (peer) {
        // Fused all-gather + unpack over NVLink (OP_UNPACK becomes a no-op);
        // it waits in-kernel for every owner's update of this bucket.
        cuda_check(launch_ag_unpack_peer(B->unpack_u, B->unpack_ps, B->e_unpack,
                                         B->any_shadow ? 1 : 0, pa, pa, B->flags, kPeerSlices,
                                         comm_stream),
                   "ag+unpack kernel");
      } else if (!local && P > 1 && B->stride > 0) {
        nccl_check(ncclAllGather(B->buf + static_cast<int64_t>(rank) * B->stride, B->buf,
                                 static_cast<size_t>(B->stride), ncclFloat32, comm, comm_stream),
                   "ncclAllGather");
      }
      record_t(op.bucket, T_AG1);
      break;
    case OP_UNPACK:
      if (peer || direct || nvls) break;
      cuda_check(launch_unpack(B->unpack_u, B->unpack_s, B->e_unpack, B->any_shadow ? 1 : 0, 0,
                               comm_stream),
                 "unpack kernel");
      record_t(op.bucket, T_UNPACK1);
      break;
    case OP_AG_DONE:
      cuda_check(cudaEventRecord(B->ag_done, comm_stream), "cudaEventRecord");
      B->ag_capture = capture_id(comm_stream);
      break;
    case OP_CALLER_WAIT_PACKED:
      if (nvls && !buckets.empty()) {
        // Every owner's reduce-scatter of the last bucket (so of all) read
        // our gradients.
        const int last = static_cast<int>(buckets.size()) - 1;
        cuda_check(launch_nvls_wait_updated(&buckets.back().flags->updated, nvls_args(last),
                                            comm_stream),
                   "nvls wait kernel");
        cuda_check(cudaEventRecord(packed_ev, comm_stream), "cudaEventRecord");
      } else if (zc && !push && !buckets.empty()) {
        // Zero-copy: peers read our gradients in their reduce-scatters, so
        // "consumed" means every rank's last (plan-order) RS has finished.
        const BucketFlags* f = buckets.back().flags;
        cuda_check(launch_wait_peers(&f->updated, &f->updated, pa, comm_stream), "wait kernel");
        cuda_check(cudaEventRecord(packed_ev, comm_stream), "cudaEventRecord");
      }
      cuda_check(cudaStreamWaitEvent(op.stream, packed_ev, 0), "cudaStreamWaitEvent");
      break;
    case OP_SET_LR:
      cuda_check(launch_set_lr(hp_dev, op.value, comm_stream), "set-lr kernel");
      break;
  }
}

void dear_ctx::enqueue(Op op) {
  if (!local) {
    exec(op);
    return;
  }
  queue.push_back(op);
}

void dear_ctx::enqueue_backpipe(int b) {
  Bucket& B = buckets[static_cast<size_t>(b)];
  enqueue({OP_FENCE_READY, b, nullptr});
  enqueue({OP_PACK, b, nullptr});
  enqueue({OP_RS, b, nullptr});
  enqueue({OP_UPDATE, b, nullptr});
  if (is_dear(cfg.policy)) {
    trace.push_back(label("RS", b));
    if (!comm_order.empty()) enqueue_ordered_ags();
  } else {
    trace.push_back(label("AR", b));
    enqueue({OP_AG, b, nullptr});
    enqueue({OP_UNPACK, b, nullptr});
    enqueue({OP_AG_DONE, b, nullptr});
    B.ag_live = true;
    B.waited_valid = false;
  }
  if (local) group->drain();
}

void dear_ctx::enqueue_feedpipe(cudaStream_t fence_stream) {
  // BARRIER: the all-gathers (which rewrite parameters) start after the work
  // already enqueued on `fence_stream` (the end of backprop, or — when
  // deferred — the start of the next forward, which keeps the comm stream
  // inside a CUDA-graph capture of that stream).
  cuda_check(cudaEventRecord(step_ev, fence_stream), "cudaEventRecord");
  enqueue({OP_FENCE_STEP, -1, nullptr});
  if (!comm_order.empty()) {
    // Group dependency: the all-gathers not dispatched during backprop, in
    // the simulated dispatch order.
    for (; order_cursor < comm_order.size(); ++order_cursor)
      enqueue_ag(-comm_order[order_cursor] - 1);
    order_cursor = 0;
  } else {
    // Reverse plan order = feed-forward order (task_graph.cpp:199-206).
    for (int g = static_cast<int>(buckets.size()) - 1; g >= 0; --g) enqueue_ag(g);
  }
  ags_deferred = false;
  if (local) group->drain();
}

void dear_ctx::enqueue_ag(int g) {
  Bucket& B = buckets[static_cast<size_t>(g)];
  enqueue({OP_AG, g, nullptr});
  enqueue({OP_UNPACK, g, nullptr});
  enqueue({OP_AG_DONE, g, nullptr});
  trace.push_back(label("AG", g));
  B.ag_live = true;
  B.waited_valid = false;
}

// After RS_g was enqueued: the all-gathers the dispatch order puts before the
// next reduce-scatter run now, behind it on the comm stream (AG_g <- RS_g,
// task_graph.cpp:201-203; their layers are already backpropagated).
void dear_ctx::enqueue_ordered_ags() {
  ++order_cursor;  // the RS just enqueued
  while (order_cursor < order_tail && comm_order[order_cursor] < 0) {
    enqueue_ag(-comm_order[order_cursor] - 1);
    ++order_cursor;
  }
}

void dear_ctx::complete_bucket(int b) {
  Bucket& B = buckets[static_cast<size_t>(b)];
  B.complete = true;
  if (is_pp(cfg.policy) && !comm_order.empty()) {
    // PRIORITY_PARTITION: the reference scheduler's dispatch sequence; a part
    // goes once it and every part before it in the sequence is ready.
    while (order_cursor < comm_order.size() &&
           buckets[static_cast<size_t>(comm_order[order_cursor] - 1)].complete) {
      enqueue_backpipe(comm_order[order_cursor] - 1);
      ++order_cursor;
      ++rs_cursor;  // parts issued
    }
    return;
  }
  // Issue RS in plan order only (task_graph.cpp:186-194; NCCL ordering).
  while (rs_cursor < static_cast<int>(buckets.size()) &&
         buckets[static_cast<size_t>(rs_cursor)].complete) {
    enqueue_backpipe(rs_cursor);
    ++rs_cursor;
  }
}

extern "C" {

const char* dear_last_error(void) { return g_last_error.c_str(); }

int dear_comm_unique_id(uint8_t id[128]) {
  DEAR_API_BEGIN
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  nccl_check(ncclGetUniqueId(&u), "ncclGetUniqueId");
  memcpy(id, &u, 128);
  DEAR_API_END
}

int dear_comm_init(void** comm, int32_t nranks, const uint8_t id[128], int32_t rank) {
  DEAR_API_BEGIN
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) invalid("dear_comm_init: bad args");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclComm_t c = nullptr;
  nccl_check(ncclCommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
  *comm = c;
  DEAR_API_END
}

int dear_comm_destroy(void* comm) {
  DEAR_API_BEGIN
  if (comm) nccl_check(ncclCommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  DEAR_API_END
}

int dear_local_group_create(int32_t P, dear_local_group** group) {
  return dear_local_group_create_ex(P, DEAR_LOCAL_RING, group);
}

int dear_local_group_create_ex(int32_t P, int32_t transport, dear_local_group** group) {
  DEAR_API_BEGIN
  if (P < 1 || P > 64 || !group) invalid("dear_local_group_create: P must be in 1..64");
  if (transport != DEAR_LOCAL_RING && transport != DEAR_LOCAL_PEER)
    invalid("dear_local_group_create_ex: transport must be DEAR_LOCAL_RING or DEAR_LOCAL_PEER");
  if (transport == DEAR_LOCAL_PEER && P > kMaxPeers)
    invalid("dear_local_group_create_ex: the peer transport supports at most 16 ranks");
  auto* g = new dear_local_group();
  g->P = P;
  g->transport = transport;
  g->ranks.assign(static_cast<size_t>(P), nullptr);
  *group = g;
  DEAR_API_END
}

int dear_local_group_destroy(dear_local_group* group) {
  DEAR_API_BEGIN
  if (group) {
    for (dear_ctx* c : group->ranks)
      if (c) invalid("dear_local_group_destroy: destroy the rank contexts first");
    delete group;
  }
  DEAR_API_END
}

static void validate_cfg(const dear_cfg* cfg) {
  if (!cfg) invalid("dear_create: cfg is null");
  const int k = cfg->policy;
  if (k != DEAR_POLICY_WFBP && k != DEAR_POLICY_WFBP_FUSED && k != DEAR_POLICY_DEAR &&
      k != DEAR_POLICY_DEAR_FUSED && k != DEAR_POLICY_PRIORITY_PARTITION)
    invalid("unknown policy kind " + std::to_string(k));
  if (is_pp(k) && cfg->partition_bytes <= 0)
    invalid("PRIORITY_PARTITION requires partition_bytes > 0");
  if (is_fused(k) && cfg->fusion_buffer_bytes <= 0) {
    invalid(std::string(k == DEAR_POLICY_WFBP_FUSED ? "WFBP_FUSED" : "DEAR_FUSED") +
            " requires fusion_buffer_bytes > 0");
  }
  if (!(cfg->lr >= 0.0)) invalid("lr must be >= 0");
  if (!(cfg->momentum >= 0.0)) invalid("momentum must be >= 0");
  if (!(cfg->weight_decay >= 0.0)) invalid("weight_decay must be >= 0");
  if (cfg->nesterov && (cfg->momentum <= 0.0 || cfg->dampening != 0.0))
    invalid("Nesterov momentum requires a momentum and zero dampening");
}

static int create_common(dear_ctx* c, int32_t rank, int32_t P, void* compute_stream,
                         const dear_cfg* cfg) {
  validate_cfg(cfg);
  if (P < 1 || rank < 0 || rank >= P) invalid("dear_create: rank must be in [0, P)");
  c->rank = rank;
  c->P = P;
  c->cfg = *cfg;
  c->compute = static_cast<cudaStream_t>(compute_stream);
  cuda_check(cudaGetDevice(&c->device), "cudaGetDevice");
  int lo = 0, hi = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
  // DEAR_COMM_PRIORITY=low|high (default high): block-scheduling priority of
  // the comm stream's kernels against the compute stream's GEMMs.
  const char* pe = std::getenv("DEAR_COMM_PRIORITY");
  const int prio = (pe && pe[0] == 'l') ? lo : hi;
  cuda_check(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio),
             "cudaStreamCreateWithPriority");
  return DEAR_OK;
}

int dear_create(void* nccl_comm, int32_t rank, int32_t P, void* compute_stream, const dear_cfg* cfg,
                dear_ctx** out) {
  DEAR_API_BEGIN
  if (!out) invalid("dear_create: out is null");
  if (P > 1 && !nccl_comm) invalid("dear_create: an NCCL communicator is required when P > 1");
  std::unique_ptr<dear_ctx> c(new dear_ctx());
  create_common(c.get(), rank, P, compute_stream, cfg);
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  if (c->comm) {
    int n = 0, r = 0;
    nccl_check(ncclCommCount(c->comm, &n), "ncclCommCount");
    nccl_check(ncclCommUserRank(c->comm, &r), "ncclCommUserRank");
    if (n != P || r != rank) invalid("dear_create: communicator size/rank do not match P/rank");
  }
  *out = c.release();
  DEAR_API_END
}

int dear_create_local(dear_local_group* group, int32_t rank, void* compute_stream,
                      const dear_cfg* cfg, dear_ctx** out) {
  DEAR_API_BEGIN
  if (!group || !out) invalid("dear_create_local: null argument");
  if (rank < 0 || rank >= group->P) invalid("dear_create_local: rank out of range");
  if (group->ranks[static_cast<size_t>(rank)]) invalid("dear_create_local: rank already created");
  std::unique_ptr<dear_ctx> c(new dear_ctx());
  create_common(c.get(), rank, group->P, compute_stream, cfg);
  // Ops queue and the group drains them in lock-step; a collective runs once
  // every rank reached it (ring kernels, or the peer kernels as one
  // cooperative group launch).
  c->local = true;
  c->same_dev = group->transport == DEAR_LOCAL_PEER;
  c->group = group;
  group->ranks[static_cast<size_t>(rank)] = c.get();
  *out = c.release();
  DEAR_API_END
}

static dear_ctx* need(dear_ctx* ctx, bool finalized) {
  if (!ctx) invalid("null context");
  if (finalized && !ctx->finalized) invalid("context is not finalized (call dear_finalize)");
  if (!finalized && ctx->finalized) invalid("context is already finalized");
  return ctx;
}

static void check_aligned(const void* p, const char* what, int32_t layer) {
  if (reinterpret_cast<uintptr_t>(p) & 15) {
    invalid(std::string(what) + " of layer " + std::to_string(layer) +
            " must be 16-byte aligned");
  }
}

int dear_register_tensor(dear_ctx* ctx, int32_t layer, float* param, float* grad, int64_t numel) {
  DEAR_API_BEGIN
  need(ctx, false);
  if (layer < 1) invalid("dear_register_tensor: layer indices are 1-based");
  if (numel < 0) invalid("model: param_count must be >= 0");
  if (numel > 0 && (!param || !grad)) invalid("dear_register_tensor: null param/grad");
  check_aligned(param, "param", layer);
  check_aligned(grad, "grad", layer);
  if (static_cast<size_t>(layer) > ctx->layers.size()) ctx->layers.resize(static_cast<size_t>(layer));
  LayerReg& L = ctx->layers[static_cast<size_t>(layer - 1)];
  if (L.numel >= 0) invalid("dear_register_tensor: layer " + std::to_string(layer) + " registered twice");
  L.param = param;
  L.grad = grad;
  L.numel = numel;
  DEAR_API_END
}

int dear_register_shadow(dear_ctx* ctx, int32_t layer, void* bf16_copy) {
  DEAR_API_BEGIN
  need(ctx, false);
  if (layer < 1 || static_cast<size_t>(layer) > ctx->layers.size() ||
      ctx->layers[static_cast<size_t>(layer - 1)].numel < 0)
    invalid("dear_register_shadow: register the tensor first");
  check_aligned(bf16_copy, "bf16 copy", layer);
  ctx->layers[static_cast<size_t>(layer - 1)].shadow = bf16_copy;
  DEAR_API_END
}

static uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ULL;
  }
  return h;
}

int dear_finalize(dear_ctx* ctx) {
  DEAR_API_BEGIN
  need(ctx, false);
  dear_ctx& c = *ctx;
  const int L = static_cast<int>(c.layers.size());
  if (L == 0) invalid("build_fusion_plan: empty model");
  for (int i = 0; i < L; ++i) {
    if (c.layers[static_cast<size_t>(i)].numel < 0) {
      invalid("model: layer indices must be exactly 1..L; layer " + std::to_string(i + 1) +
              " was not registered");
    }
  }
  std::vector<int64_t> bytes(static_cast<size_t>(L));
  for (int i = 0; i < L; ++i) bytes[static_cast<size_t>(i)] = c.layers[static_cast<size_t>(i)].numel * 4;
  std::vector<Group> plan;
  if (is_pp(c.cfg.policy)) {
    // PRIORITY_PARTITION (task_graph.cpp:215-258): layer L down to 1, each in
    // ceil(bytes / partition_bytes) parts (one for an empty layer) of balanced
    // element ranges; every part is its own bucket, all-reduced on its own.
    for (int l = L; l >= 1; --l) {
      LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
      const int64_t b = bytes[static_cast<size_t>(l - 1)];
      const int64_t parts = b == 0 ? 1 : (b + c.cfg.partition_bytes - 1) / c.cfg.partition_bytes;
      if (parts > (1 << 20)) invalid("PRIORITY_PARTITION: partition_bytes too small for layer " +
                                     std::to_string(l));
      const std::vector<int64_t> pb = chunk_begins(R.numel, static_cast<int>(parts));
      R.bucket = static_cast<int>(c.buckets.size());
      R.n_parts = static_cast<int>(parts);
      R.off = 0;
      for (int64_t k = 0; k < parts; ++k) {
        Bucket B;
        B.low = B.high = l;
        B.part = static_cast<int>(k + 1);
        B.e0 = pb[static_cast<size_t>(k)];
        B.d = pb[static_cast<size_t>(k) + 1] - pb[static_cast<size_t>(k)];
        B.any_shadow = R.shadow != nullptr;
        c.buckets.push_back(std::move(B));
        plan.push_back(Group{l, l});
      }
    }
  } else {
    plan = build_plan(bytes, is_fused(c.cfg.policy) ? c.cfg.fusion_buffer_bytes : 0);
    c.buckets.resize(plan.size());
  }

  // Bucket geometry and HBM layout: one arena holding every bucket buffer
  // (P slots of `stride` fp32 each), the momentum shards and the unit tables.
  const bool mom = c.cfg.momentum != 0.0;
  size_t floats = 0, units = 0;
  for (size_t g = 0; g < plan.size(); ++g) {
    Bucket& B = c.buckets[g];
    if (B.part == 0) {
      B.low = plan[g].low;
      B.high = plan[g].high;
      int64_t off = 0;
      for (int l = B.low; l <= B.high; ++l) {
        LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
        R.bucket = static_cast<int>(g);
        R.off = off;
        off += R.numel;
        if (R.shadow) B.any_shadow = true;
      }
      B.d = off;
    }
    B.stride = slot_stride(B.d, c.P);
    floats += static_cast<size_t>(B.stride) * static_cast<size_t>(c.P) + (mom ? static_cast<size_t>(B.stride) : 0);
  }
  // DEAR_DIRECT=0 keeps the pack/update/unpack kernels at P = 1 (tools that
  // measure those kernels on one GPU).
  const char* dir_env = std::getenv("DEAR_DIRECT");
  c.direct = c.P == 1 && !c.peer && c.cfg.momentum == 0.0 && !(dir_env && dir_env[0] == '0');
  // Zero-copy tables for a later dear_peer_connect (multi-process only).
  // (also at P = 1 outside local groups: the NVLS kernels run on one GPU too)
  c.zc_tables = (!c.local && !c.same_dev) || (c.same_dev && c.P > 1);
  const char* push_env = std::getenv("DEAR_PUSH_RS");
  c.push_tables = !c.local && !c.same_dev && c.P > 1 && push_env && push_env[0] == '1';
  // Unit tables.
  std::vector<Unit> host_units;
  struct Span { size_t pack, upd, unpack; };
  std::vector<Span> spans(plan.size());
  std::vector<std::vector<int64_t>> begins(plan.size());
  for (size_t g = 0; g < plan.size(); ++g) begins[g] = chunk_begins(c.buckets[g].d, c.P);
  // Push slot position of a piece: the running offset advanced to the phase
  // of the piece's parameter (layer offset j; tensors are 16 B aligned).
  auto push_pos = [](int64_t& so, int64_t j, int64_t len) {
    so += ((j - so) % 4 + 4) % 4;
    const int64_t at = so;
    so += len;
    return at;
  };
  if (c.push_tables) {
    for (size_t g = 0; g < plan.size(); ++g) {
      Bucket& B = c.buckets[g];
      int64_t mx = 0;
      for (int ch = 0; ch < c.P; ++ch) {
        int64_t so = 0;
        for_each_piece(c, B, begins[g][static_cast<size_t>(ch)], begins[g][static_cast<size_t>(ch) + 1],
                       [&](int, int64_t j, int64_t len, int64_t) { push_pos(so, j, len); });
        mx = std::max(mx, so);
      }
      B.pstride = (mx + 63) / 64 * 64;
      floats += static_cast<size_t>(B.pstride) * static_cast<size_t>(c.P);
    }
  }
  // First pass only counts; pointers are filled once the arena exists.
  for (size_t g = 0; g < plan.size(); ++g) {
    const Bucket& B = c.buckets[g];
    const auto& bg = begins[g];
    size_t n = 0;
    for (int ch = 0; ch < c.P; ++ch)
      for_each_piece(c, B, bg[static_cast<size_t>(ch)], bg[static_cast<size_t>(ch) + 1],
                     [&](int, int64_t, int64_t, int64_t) { ++n; });
    const int own = (c.rank + 1) % c.P;
    size_t nu = 0;
    for_each_piece(c, B, bg[static_cast<size_t>(own)], bg[static_cast<size_t>(own) + 1],
                   [&](int, int64_t, int64_t, int64_t) { ++nu; });
    units += 2 * n + nu + (c.direct ? n : 0) + (c.zc_tables ? 2 * n : 0) +
             (c.push_tables ? n + nu : 0);
  }
  const size_t float_bytes = (floats * sizeof(float) + 255) / 256 * 256;
  const size_t unit_bytes = (units * sizeof(Unit) + 255) / 256 * 256;
  const size_t per_bucket_slices = 3 * static_cast<size_t>(kSlices) + 2 * kPeerSlices +
                                   kPackPeerSlices + (c.direct ? kSlices : 0) +
                                   (c.zc_tables ? 2 * kZcSlices : 0) +
                                   (c.push_tables ? kPackPeerSlices + kZcSlices : 0);
  const size_t n_slices = plan.size() * per_bucket_slices;
  const size_t slice_bytes = (n_slices * sizeof(Slice) + 255) / 256 * 256;
  // Layout: [bucket buffers + momentum][flags] is identical on every rank (the
  // region peers address through IPC); unit/slice tables (rank-specific)
  // follow.
  const size_t flag_bytes = (plan.size() * sizeof(BucketFlags) + 255) / 256 * 256;
  const size_t total = float_bytes + flag_bytes + unit_bytes + slice_bytes + 256 + 256;
  cuda_check(cudaMalloc(&c.arena, total), "cudaMalloc(bucket arena)");
  cuda_check(cudaMemset(c.arena, 0, float_bytes), "cudaMemset");
  float* fp = reinterpret_cast<float*>(c.arena);
  Unit* up = reinterpret_cast<Unit*>(c.arena + float_bytes + flag_bytes);
  BucketFlags* fl = reinterpret_cast<BucketFlags*>(c.arena + float_bytes);
  Slice* sp = reinterpret_cast<Slice*>(c.arena + float_bytes + flag_bytes + unit_bytes);
  c.hp_dev = reinterpret_cast<HyperParams*>(c.arena + float_bytes + flag_bytes + unit_bytes +
                                            slice_bytes);
  c.hash_dev = reinterpret_cast<unsigned long long*>(c.arena + float_bytes + flag_bytes +
                                                      unit_bytes + slice_bytes + 256);
  c.arena_bytes = float_bytes + flag_bytes;  // the rank-independent (peer-shared) prefix
  cuda_check(cudaMemset(fl, 0, flag_bytes), "cudaMemset(flags)");
  for (size_t g = 0; g < plan.size(); ++g) c.buckets[g].flags = fl + g;
  std::vector<Slice> host_slices(n_slices);
  for (size_t g = 0; g < plan.size(); ++g) {
    Bucket& B = c.buckets[g];
    B.buf = fp;
    fp += B.stride * c.P;
    if (mom) {
      B.mom = fp;
      fp += B.stride;
    }
    if (c.push_tables) {
      B.pbuf = fp;
      fp += B.pstride * c.P;
    }
  }
  host_units.reserve(units);
  for (size_t g = 0; g < plan.size(); ++g) {
    Bucket& B = c.buckets[g];
    const auto& bg = begins[g];
    // pack: every chunk c to slot owner(c) = (c-1) mod P.
    B.pack_u = up + host_units.size();
    for (int ch = 0; ch < c.P; ++ch) {
      const int slot = (ch - 1 + c.P) % c.P;
      for_each_piece(c, B, bg[static_cast<size_t>(ch)], bg[static_cast<size_t>(ch) + 1],
                     [&](int l, int64_t j, int64_t len, int64_t pos) {
                       const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                       host_units.push_back({R.grad + j, B.buf + slot * B.stride + pos, nullptr, len, 0, 0, 0});
                     });
    }
    B.n_pack = static_cast<int>(host_units.size() - static_cast<size_t>(B.pack_u - up));
    B.e_pack = set_starts(host_units, static_cast<size_t>(B.pack_u - up));
    // update: own chunk (rank+1) mod P, in slot `rank`.
    B.upd_u = up + host_units.size();
    const int own = (c.rank + 1) % c.P;
    for_each_piece(c, B, bg[static_cast<size_t>(own)], bg[static_cast<size_t>(own) + 1],
                   [&](int l, int64_t j, int64_t len, int64_t pos) {
                     const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                     host_units.push_back({R.param + j, B.buf + c.rank * B.stride + pos,
                                           B.mom ? static_cast<void*>(B.mom + pos) : nullptr, len, 0, 0, 0});
                   });
    B.n_upd = static_cast<int>(host_units.size() - static_cast<size_t>(B.upd_u - up));
    B.e_upd = set_starts(host_units, static_cast<size_t>(B.upd_u - up));
    // unpack: every slot back to the layers (and their bf16 copies).
    B.unpack_u = up + host_units.size();
    for (int ch = 0; ch < c.P; ++ch) {
      const int slot = (ch - 1 + c.P) % c.P;
      for_each_piece(c, B, bg[static_cast<size_t>(ch)], bg[static_cast<size_t>(ch) + 1],
                     [&](int l, int64_t j, int64_t len, int64_t pos) {
                       const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                       void* sh = R.shadow ? static_cast<void*>(static_cast<uint16_t*>(R.shadow) + j) : nullptr;
                       host_units.push_back({B.buf + slot * B.stride + pos, R.param + j, sh, len, 0, slot, 0});
                     });
    }
    B.n_unpack = static_cast<int>(host_units.size() - static_cast<size_t>(B.unpack_u - up));
    B.e_unpack = set_starts(host_units, static_cast<size_t>(B.unpack_u - up));
    if (c.direct) {
      // P = 1: gradient -> parameter (+ bf16 copy), layer by layer.
      B.dir_u = up + host_units.size();
      for_each_piece(c, B, bg[0], bg[1], [&](int l, int64_t j, int64_t len, int64_t) {
        const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
        void* sh = R.shadow ? static_cast<void*>(static_cast<uint16_t*>(R.shadow) + j) : nullptr;
        host_units.push_back({R.grad + j, R.param + j, sh, len, 0, 0, 0});
      });
      B.n_dir = static_cast<int>(host_units.size() - static_cast<size_t>(B.dir_u - up));
      B.e_dir = set_starts(host_units, static_cast<size_t>(B.dir_u - up));
    }
    if (c.zc_tables) {
      // Zero-copy RS: the owned chunk, gradient -> parameter (+ bf16 copy).
      B.zrs_u = up + host_units.size();
      for_each_piece(c, B, bg[static_cast<size_t>(own)], bg[static_cast<size_t>(own) + 1],
                     [&](int l, int64_t j, int64_t len, int64_t) {
                       const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                       void* sh = R.shadow ? static_cast<void*>(static_cast<uint16_t*>(R.shadow) + j) : nullptr;
                       host_units.push_back({R.grad + j, R.param + j, sh, len, 0, 0, 0});
                     });
      B.n_zrs = static_cast<int>(host_units.size() - static_cast<size_t>(B.zrs_u - up));
      B.e_zrs = set_starts(host_units, static_cast<size_t>(B.zrs_u - up));
      // Zero-copy AG: every other chunk from its owner's parameters.
      B.zag_u = up + host_units.size();
      for (int ch = 0; ch < c.P; ++ch) {
        if (ch == own) continue;
        const int owner = (ch - 1 + c.P) % c.P;
        for_each_piece(c, B, bg[static_cast<size_t>(ch)], bg[static_cast<size_t>(ch) + 1],
                       [&](int l, int64_t j, int64_t len, int64_t) {
                         const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                         void* sh = R.shadow ? static_cast<void*>(static_cast<uint16_t*>(R.shadow) + j) : nullptr;
                         host_units.push_back({R.param + j, R.param + j, sh, len, 0, owner, 0});
                       });
      }
      B.n_zag = static_cast<int>(host_units.size() - static_cast<size_t>(B.zag_u - up));
      B.e_zag = set_starts(host_units, static_cast<size_t>(B.zag_u - up));
    }
    // Equal element slices per CTA for each op (one wave of kSlices CTAs).
    Slice* hs = host_slices.data() + g * per_bucket_slices;
    make_slices(host_units.data() + (B.pack_u - up), B.n_pack, B.e_pack, hs, kPackSlices, 0);
    make_slices(host_units.data() + (B.upd_u - up), B.n_upd, B.e_upd, hs + kSlices, kUpdSlices, 4);
    make_slices(host_units.data() + (B.unpack_u - up), B.n_unpack, B.e_unpack, hs + 2 * kSlices,
                kUnpackSlices, 2);
    make_slices(host_units.data() + (B.upd_u - up), B.n_upd, B.e_upd, hs + 3 * kSlices,
                kPeerSlices, 4);
    make_slices(host_units.data() + (B.unpack_u - up), B.n_unpack, B.e_unpack,
                hs + 3 * kSlices + kPeerSlices, kPeerSlices, 2);
    make_slices(host_units.data() + (B.pack_u - up), B.n_pack, B.e_pack,
                hs + 3 * kSlices + 2 * kPeerSlices, kPackPeerSlices, 0);
    if (c.direct)
      make_slices(host_units.data() + (B.dir_u - up), B.n_dir, B.e_dir,
                  hs + 3 * kSlices + 2 * kPeerSlices + kPackPeerSlices, kDirSlices, 2);
    B.pack_s = sp + g * per_bucket_slices;
    B.upd_s = B.pack_s + kSlices;
    B.unpack_s = B.upd_s + kSlices;
    B.upd_ps = B.unpack_s + kSlices;
    B.unpack_ps = B.upd_ps + kPeerSlices;
    B.pack_ps = B.unpack_ps + kPeerSlices;
    B.dir_s = c.direct ? B.pack_ps + kPackPeerSlices : nullptr;
    if (c.zc_tables) {
      const size_t z0 = 3 * kSlices + 2 * kPeerSlices + kPackPeerSlices + (c.direct ? kSlices : 0);
      make_slices(host_units.data() + (B.zrs_u - up), B.n_zrs, B.e_zrs, hs + z0, kZcSlices, 2);
      make_slices(host_units.data() + (B.zag_u - up), B.n_zag, B.e_zag, hs + z0 + kZcSlices,
                  kZcSlices, 2);
      B.zrs_ps = B.pack_s + z0;
      B.zag_ps = B.zrs_ps + kZcSlices;
    }
    if (c.push_tables) {
      // Push pack: chunk ch to slot `rank` of its owner's push buffer.
      B.ppk_u = up + host_units.size();
      for (int ch = 0; ch < c.P; ++ch) {
        const int owner = (ch - 1 + c.P) % c.P;
        int64_t so = 0;
        for_each_piece(c, B, bg[static_cast<size_t>(ch)], bg[static_cast<size_t>(ch) + 1],
                       [&](int l, int64_t j, int64_t len, int64_t) {
                         const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                         const int64_t at = push_pos(so, j, len);
                         host_units.push_back({R.grad + j, B.pbuf + c.rank * B.pstride + at, nullptr,
                                               len, 0, owner, 0});
                       });
      }
      B.n_ppk = static_cast<int>(host_units.size() - static_cast<size_t>(B.ppk_u - up));
      B.e_ppk = set_starts(host_units, static_cast<size_t>(B.ppk_u - up));
      // Push RS: the own chunk, slot 0 position -> parameter (+ bf16 copy).
      B.prs_u = up + host_units.size();
      int64_t so = 0;
      for_each_piece(c, B, bg[static_cast<size_t>(own)], bg[static_cast<size_t>(own) + 1],
                     [&](int l, int64_t j, int64_t len, int64_t) {
                       const LayerReg& R = c.layers[static_cast<size_t>(l - 1)];
                       void* sh = R.shadow ? static_cast<void*>(static_cast<uint16_t*>(R.shadow) + j) : nullptr;
                       host_units.push_back({B.pbuf + push_pos(so, j, len), R.param + j, sh, len, 0, 0, 0});
                     });
      B.n_prs = static_cast<int>(host_units.size() - static_cast<size_t>(B.prs_u - up));
      B.e_prs = set_starts(host_units, static_cast<size_t>(B.prs_u - up));
      const size_t p0 = 3 * kSlices + 2 * kPeerSlices + kPackPeerSlices + (c.direct ? kSlices : 0) +
                        (c.zc_tables ? 2 * kZcSlices : 0);
      make_slices(host_units.data() + (B.ppk_u - up), B.n_ppk, B.e_ppk, hs + p0, kPackPeerSlices, 0);
      make_slices(host_units.data() + (B.prs_u - up), B.n_prs, B.e_prs, hs + p0 + kPackPeerSlices,
                  kZcSlices, 2);
      B.ppk_ps = B.pack_s + p0;
      B.prs_ps = B.ppk_ps + kPackPeerSlices;
    }
    B.ag_done = new_event(false);
    for (int k = 0; k < T_COUNT; ++k) B.t[k] = new_event(true);
    B.layers_left = B.high - B.low + 1;
  }
  if (!host_units.empty()) {
    cuda_check(cudaMemcpy(up, host_units.data(), host_units.size() * sizeof(Unit), cudaMemcpyHostToDevice),
               "cudaMemcpy(units)");
  }
  cuda_check(cudaMemcpy(sp, host_slices.data(), n_slices * sizeof(Slice), cudaMemcpyHostToDevice),
             "cudaMemcpy(slices)");
  // Hyper-parameters; 1/P folded into pack when it is exact (P = 2^k).
  const bool pow2 = (c.P & (c.P - 1)) == 0;
  c.pack_scale = pow2 ? 1.0f / static_cast<float>(c.P) : 1.0f;
  c.hp_host.lr = static_cast<float>(c.cfg.lr);
  c.hp_host.momentum = static_cast<float>(c.cfg.momentum);
  c.hp_host.one_minus_dampening = 1.0f - static_cast<float>(c.cfg.dampening);
  c.hp_host.weight_decay = static_cast<float>(c.cfg.weight_decay);
  c.hp_host.inv_p = 1.0f / static_cast<float>(c.P);
  c.hp_host.nesterov = c.cfg.nesterov ? 1 : 0;
  c.hp_host.prescaled = pow2 ? 1 : 0;
  cuda_check(cudaMemcpy(c.hp_dev, &c.hp_host, sizeof(HyperParams), cudaMemcpyHostToDevice), "cudaMemcpy(hp)");
  c.packed_ev = new_event(false);
  c.step_ev = new_event(false);
  c.join_ev = new_event(false);

  // Every rank must have registered the same model (the precondition the
  // reference checks as vector-length / replica equality, collective.cpp:172-186).
  uint64_t h = 1469598103934665603ULL;
  h = fnv(h, static_cast<uint64_t>(L));
  for (const LayerReg& R : c.layers) h = fnv(h, static_cast<uint64_t>(R.numel));
  h = fnv(h, static_cast<uint64_t>(c.cfg.policy));
  h = fnv(h, static_cast<uint64_t>(c.cfg.fusion_buffer_bytes));
  h = fnv(h, static_cast<uint64_t>(is_pp(c.cfg.policy) ? c.cfg.partition_bytes : 0));
  if (c.local || c.same_dev) {
    for (dear_ctx* o : c.group->ranks) {
      if (o && o != &c && o->finalized) {
        if (o->buckets.size() != c.buckets.size())
          invalid("dear_finalize: ranks registered different models");
        for (size_t g = 0; g < c.buckets.size(); ++g)
          if (o->buckets[g].d != c.buckets[g].d || o->buckets[g].low != c.buckets[g].low)
            invalid("dear_finalize: ranks registered different models");
      }
    }
  } else if (c.P > 1) {
    unsigned long long hv[2] = {h, ~h};
    cuda_check(cudaMemcpy(c.hash_dev, hv, sizeof hv, cudaMemcpyHostToDevice), "cudaMemcpy");
    nccl_check(ncclAllReduce(c.hash_dev, c.hash_dev, 2, ncclUint64, ncclMax, c.comm, c.comm_stream),
               "ncclAllReduce(registration check)");
    cuda_check(cudaMemcpyAsync(hv, c.hash_dev, sizeof hv, cudaMemcpyDeviceToHost, c.comm_stream), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
    if (hv[0] != h || hv[1] != ~h) invalid("dear_finalize: ranks registered different models");
  }
  cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  c.finalized = true;
  DEAR_API_END
}

int dear_grad_ready(dear_ctx* ctx, int32_t layer, void* stream) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (layer < 1 || static_cast<size_t>(layer) > c.layers.size())
    invalid("dear_grad_ready: layer " + std::to_string(layer) + " out of range");
  LayerReg& R = c.layers[static_cast<size_t>(layer - 1)];
  if (R.ready) invalid("dear_grad_ready: layer " + std::to_string(layer) + " reported twice in one iteration");
  if (c.ags_deferred) invalid("dear_grad_ready: backward started before the deferred all-gathers were flushed");
  R.ready = true;
  ++c.reported;
  if (c.reported == 1) c.trace.clear();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // A layer is one bucket's member, or (PRIORITY_PARTITION) n_parts buckets.
  for (int g = R.bucket; g < R.bucket + R.n_parts; ++g) {
    Bucket& B = c.buckets[static_cast<size_t>(g)];
    if (std::find(B.ready_streams.begin(), B.ready_streams.end(), s) == B.ready_streams.end())
      B.ready_streams.push_back(s);
    if (--B.layers_left == 0) {
      // All of the bucket's gradients are enqueued: fence each producing stream.
      while (B.ready_events.size() < B.ready_streams.size()) B.ready_events.push_back(new_event(false));
      for (size_t i = 0; i < B.ready_streams.size(); ++i)
        cuda_check(cudaEventRecord(B.ready_events[i], B.ready_streams[i]), "cudaEventRecord");
      B.ready_events.resize(B.ready_streams.size());
      c.complete_bucket(g);
    }
  }
  DEAR_API_END
}

int dear_set_comm_order(dear_ctx* ctx, const int32_t* seq, int32_t n) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (c.reported != 0 || c.ags_deferred)
    invalid("dear_set_comm_order: call between iterations");
  const int G = static_cast<int>(c.buckets.size());
  if (is_pp(c.cfg.policy)) {
    // every part once, any order (the scheduler's priority dispatch)
    if (n == 0) {
      c.comm_order.clear();
      c.order_cursor = 0;
      return DEAR_OK;
    }
    if (!seq || n != G) invalid("dear_set_comm_order: PRIORITY_PARTITION needs every part once");
    std::vector<char> seen(static_cast<size_t>(G), 0);
    for (int32_t i = 0; i < n; ++i) {
      if (seq[i] < 1 || seq[i] > G || seen[static_cast<size_t>(seq[i] - 1)])
        invalid("dear_set_comm_order: PRIORITY_PARTITION needs every part once");
      seen[static_cast<size_t>(seq[i] - 1)] = 1;
    }
    c.comm_order.assign(seq, seq + n);
    c.order_cursor = 0;
    return DEAR_OK;
  }
  if (!is_dear(c.cfg.policy)) invalid("dear_set_comm_order: needs a DEAR policy");
  if (!c.cfg.dear_group_dependency)
    invalid("dear_set_comm_order: needs dear_group_dependency (AG_g waits on RS_g only)");
  if (n == 0) {
    c.comm_order.clear();
    c.order_cursor = c.order_tail = 0;
    return DEAR_OK;
  }
  if (!seq || n != 2 * G) invalid("dear_set_comm_order: need 2 x buckets entries");
  // Reduce-scatters in plan order; every all-gather once, after its RS.
  std::vector<char> rs_seen(static_cast<size_t>(G), 0), ag_seen(static_cast<size_t>(G), 0);
  int next_rs = 0;
  if (seq[0] != 1) invalid("dear_set_comm_order: must start with RS of bucket 1");
  for (int32_t i = 0; i < n; ++i) {
    const int32_t v = seq[i];
    if (v > 0) {
      if (v > G) invalid("dear_set_comm_order: entry out of range");
      if (v != next_rs + 1) invalid("dear_set_comm_order: reduce-scatters must follow plan order");
      rs_seen[static_cast<size_t>(next_rs++)] = 1;
    } else if (v < 0 && -v <= G) {
      const int g = -v - 1;
      if (!rs_seen[static_cast<size_t>(g)]) invalid("dear_set_comm_order: AG before its RS");
      if (ag_seen[static_cast<size_t>(g)]) invalid("dear_set_comm_order: AG listed twice");
      ag_seen[static_cast<size_t>(g)] = 1;
    } else {
      invalid("dear_set_comm_order: entry out of range");
    }
  }
  c.comm_order.assign(seq, seq + n);
  c.order_cursor = 0;
  c.order_tail = 0;
  for (int32_t i = 0; i < n; ++i)
    if (seq[i] > 0) c.order_tail = static_cast<size_t>(i) + 1;
  DEAR_API_END
}

int dear_step(dear_ctx* ctx, void* stream) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (c.rs_cursor != static_cast<int>(c.buckets.size())) {
    std::string missing;
    for (size_t i = 0; i < c.layers.size(); ++i)
      if (!c.layers[i].ready) missing += (missing.empty() ? "" : ",") + std::to_string(i + 1);
    invalid("dear_step: gradients not reported for layers [" + missing + "]");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Both directions of the barrier: gradients are consumed (packed) before the
  // caller may overwrite them; parameters are rewritten only after the
  // caller's backward work.
  c.enqueue({OP_CALLER_WAIT_PACKED, -1, s});
  if (is_dear(c.cfg.policy)) {
    if (!c.comm_order.empty() && c.order_cursor >= c.comm_order.size()) {
      c.order_cursor = 0;  // every all-gather already dispatched during backprop
      if (c.local) c.group->drain();
    } else if (c.cfg.defer_allgather) {
      c.ags_deferred = true;
    } else {
      c.enqueue_feedpipe(s);
    }
  } else if (c.local) {
    c.group->drain();
  }
  for (LayerReg& R : c.layers) R.ready = false;
  for (Bucket& B : c.buckets) {
    B.complete = false;
    B.layers_left = B.high - B.low + 1;
    B.ready_streams.clear();
  }
  c.rs_cursor = 0;
  if (is_pp(c.cfg.policy)) c.order_cursor = 0;
  c.reported = 0;
  ++c.iteration;
  DEAR_API_END
}

int dear_param_wait(dear_ctx* ctx, int32_t layer, void* stream) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (layer < 1 || static_cast<size_t>(layer) > c.layers.size())
    invalid("dear_param_wait: layer " + std::to_string(layer) + " out of range");
  if (c.ags_deferred) {
    if (c.local) {
      // The group flushes together: a local collective needs every rank.
      for (dear_ctx* o : c.group->ranks)
        if (o && o->ags_deferred) o->enqueue_feedpipe(o == &c ? static_cast<cudaStream_t>(stream) : o->compute);
    } else {
      c.enqueue_feedpipe(static_cast<cudaStream_t>(stream));
    }
  }
  const LayerReg& R = c.layers[static_cast<size_t>(layer - 1)];
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int g = R.bucket; g < R.bucket + R.n_parts; ++g) {  // PRIORITY_PARTITION: every part
    Bucket& B = c.buckets[static_cast<size_t>(g)];
    if (!B.ag_live) continue;
    if (B.waited_valid && B.waited == s) continue;
    // An all-gather recorded in another capture context than this wait (inside
    // a capture: the previous iteration of a WFBP schedule, or one issued during
    // the previous graph's backprop under dear_group_dependency; eagerly: one
    // recorded while capturing the previous graph) is ordered before this work
    // by that graph's / this capture's trailing dear_join on the caller's
    // stream. Waiting on it is illegal, so it is dropped.
    const unsigned long long cap = capture_id(s);
    if (B.ag_capture != cap) continue;
    if (c.local) {
      c.group->drain();
      if (!c.queue.empty()) invalid("dear_param_wait: local group ranks are out of lock-step");
    }
    cuda_check(cudaStreamWaitEvent(s, B.ag_done, 0), "cudaStreamWaitEvent");
    B.waited = s;
    B.waited_valid = true;
  }
  DEAR_API_END
}

int dear_join(dear_ctx* ctx, void* stream) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (ctx->local) ctx->group->drain();
  cuda_check(cudaEventRecord(ctx->join_ev, ctx->comm_stream), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ctx->join_ev, 0), "cudaStreamWaitEvent");
  DEAR_API_END
}

// Host wait for the comm stream that watches the communicator (SURVEY §5,
// failure detection): NCCL reports a peer's failure asynchronously
// (ncclCommGetAsyncError) while its kernels may never finish, so poll both;
// on an error, or after DEAR_SYNC_TIMEOUT_S seconds (0 / unset = no limit),
// abort the communicator (ncclCommAbort unblocks its kernels) and fail with
// DEAR_EINTERNAL instead of hanging.
static void wait_comm_stream(dear_ctx& c) {
  if (!c.comm) {
    cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
    return;
  }
  const char* e = std::getenv("DEAR_SYNC_TIMEOUT_S");
  const double limit = e ? std::atof(e) : 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(c.comm_stream);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) cuda_check(q, "comm stream");
    ncclResult_t async = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(c.comm, &async), "ncclCommGetAsyncError");
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((async != ncclSuccess && async != ncclInProgress) || (limit > 0.0 && s > limit)) {
      const std::string why = async != ncclSuccess && async != ncclInProgress
                                  ? std::string("NCCL reported ") + ncclGetErrorString(async)
                                  : "no progress within DEAR_SYNC_TIMEOUT_S";
      ncclCommAbort(c.comm);
      c.comm = nullptr;
      throw Error(DEAR_EINTERNAL, "dear_synchronize: " + why + "; communicator aborted");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int dear_synchronize(dear_ctx* ctx) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (ctx->local) {
    for (dear_ctx* o : ctx->group->ranks)
      if (o && o->ags_deferred) o->enqueue_feedpipe(o->compute);
    ctx->group->drain();
    if (!ctx->queue.empty()) invalid("dear_synchronize: other ranks of the local group lag behind");
  }
  else if (ctx->ags_deferred) {
    ctx->enqueue_feedpipe(ctx->compute);
  }
  wait_comm_stream(*ctx);
  DEAR_API_END
}

int dear_set_comm_trace(void* device_buffer, int64_t capacity) {
  DEAR_API_BEGIN
  if (capacity < 0 || capacity > 0xffffffffLL) invalid("dear_set_comm_trace: bad capacity");
  cuda_check(set_comm_trace(device_buffer, device_buffer ? static_cast<uint32_t>(capacity) : 0u),
             "dear_set_comm_trace");
  DEAR_API_END
}

int dear_comm_trace_count(int64_t* n) {
  DEAR_API_BEGIN
  if (!n) invalid("dear_comm_trace_count: null output");
  uint32_t v = 0;
  cuda_check(comm_trace_count(&v), "dear_comm_trace_count");
  *n = v;
  DEAR_API_END
}

int dear_comm_error(dear_ctx* ctx, int32_t* failed) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (!failed) invalid("dear_comm_error: null output");
  *failed = 0;
  if (ctx->comm) {
    ncclResult_t async = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(ctx->comm, &async), "ncclCommGetAsyncError");
    if (async != ncclSuccess && async != ncclInProgress) *failed = 1;
  }
  DEAR_API_END
}

int dear_destroy(dear_ctx* ctx) {
  DEAR_API_BEGIN
  delete ctx;
  DEAR_API_END
}

int dear_set_lr(dear_ctx* ctx, double lr) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (!(lr >= 0.0)) invalid("lr must be >= 0");
  ctx->cfg.lr = lr;
  ctx->hp_host.lr = static_cast<float>(lr);
  // A one-thread kernel on the comm stream (value passed by argument): updates
  // enqueued before keep the old rate, later ones see the new; no host sync,
  // and legal inside a CUDA-graph capture. Local-group contexts queue it in
  // order with their pending ops.
  Op op{OP_SET_LR, -1, nullptr};
  op.value = static_cast<float>(lr);
  ctx->enqueue(op);
  DEAR_API_END
}

// ---- zero-copy span: one allocation holding every layer's tensor ----------
namespace {
struct TensorSpan {
  bool ok = false;
  char* lo = nullptr;    // lowest tensor address
  char* base = nullptr;  // allocation base
  uint64_t layout = 0;   // hash of every tensor's offset from `lo`
};

using MemGetAddressRange = int (*)(uintptr_t*, size_t*, uintptr_t);

// need_alloc: the tensors must lie in one device allocation (the IPC export
// unit); the same-device peer group only needs their relative layout.
TensorSpan tensor_span(const dear_ctx& c, bool grads, bool need_alloc = true) {
  TensorSpan sp;
  static MemGetAddressRange range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess)
      return static_cast<MemGetAddressRange>(nullptr);
    return reinterpret_cast<MemGetAddressRange>(fn);
  }();
  if (need_alloc && !range) return sp;
  char *lo = nullptr, *hi = nullptr;
  for (const LayerReg& R : c.layers) {
    char* p = reinterpret_cast<char*>(grads ? R.grad : R.param);
    if (!p || R.numel <= 0) continue;
    if (!lo || p < lo) lo = p;
    if (!hi || p + R.numel * 4 > hi) hi = p + R.numel * 4;
  }
  if (!lo) return sp;
  uintptr_t base = reinterpret_cast<uintptr_t>(lo);
  size_t size = 0;
  if (need_alloc) {
    if (range(&base, &size, reinterpret_cast<uintptr_t>(lo)) != 0) return sp;
    if (reinterpret_cast<uintptr_t>(hi) > base + size) return sp;  // several allocations
  }
  uint64_t h = 1469598103934665603ULL;
  for (const LayerReg& R : c.layers) {
    const char* p = reinterpret_cast<const char*>(grads ? R.grad : R.param);
    h = fnv(h, p && R.numel > 0 ? static_cast<uint64_t>(p - lo) : ~0ULL);
  }
  sp.ok = true;
  sp.lo = lo;
  sp.base = reinterpret_cast<char*>(base);
  sp.layout = h;
  return sp;
}

// Handle record (DEAR_PEER_HANDLE_BYTES):
//   [0,64) arena IPC handle  [64,72) arena bytes  [72,76) rank  [76,80) zero-copy ok
//   [80,144) gradient allocation handle  [144,208) parameter allocation handle
//   [208,216) grad lo - base  [216,224) param lo - base
//   [224,232) gradient layout hash  [232,240) parameter layout hash
constexpr size_t kH_ZC = 76, kH_G = 80, kH_Q = 144, kH_GOFF = 208, kH_QOFF = 216,
                 kH_GLAY = 224, kH_QLAY = 232, kH_PUSH = 240;
}  // namespace

namespace {
// DEAR_PEER_TIMEOUT_S (default 600 s, torch's NCCL watchdog default; 0 =
// wait forever): how long a cross-GPU wait spins before the kernel traps. A
// rank doing rank-local work (eval, checkpoint) for longer must barrier first.
long long peer_spin_limit(int device) {
  const char* e = std::getenv("DEAR_PEER_TIMEOUT_S");
  const double s = e ? std::atof(e) : 600.0;
  if (!(s > 0.0)) return 0;
  int khz = 0;
  if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device) != cudaSuccess || khz <= 0)
    khz = 2000000;
  return static_cast<long long>(s * static_cast<double>(khz) * 1000.0);
}

// Switches a finalized context to the peer kernels: pa = arena deltas, ga / qa
// = gradient / parameter deltas (zero-copy only).
void enable_peer(dear_ctx& c, PeerArgs pa, PeerArgs ga, PeerArgs qa, bool zc) {
  pa.spin_limit = peer_spin_limit(c.device);
  ga.spin_limit = qa.spin_limit = pa.spin_limit;
  c.pa = pa;
  c.ga = ga;
  c.qa = qa;
  c.peer = true;
  if (zc) {
    // No pack, so no pre-scaling: the update applies 1/P after the ring sum
    // (collective.cpp:159-164's order; for P = 2^k the same bits either way).
    // The push reduce-scatter's pack pre-scales like the slot path.
    c.zc = true;
    c.push = c.push_tables;
    c.hp_host.prescaled = c.push && (c.P & (c.P - 1)) == 0 ? 1 : 0;
    cuda_check(cudaMemcpy(c.hp_dev, &c.hp_host, sizeof(HyperParams), cudaMemcpyHostToDevice),
               "cudaMemcpy(hp)");
  }
}
}  // namespace

int dear_local_group_connect(dear_local_group* group, int32_t allow_zero_copy) {
  DEAR_API_BEGIN
  if (!group || group->transport != DEAR_LOCAL_PEER)
    invalid("dear_local_group_connect: needs a group created with DEAR_LOCAL_PEER");
  const int P = group->P;
  for (dear_ctx* c : group->ranks) {
    if (!c || !c->finalized) invalid("dear_local_group_connect: create and finalize every rank first");
    if (c->peer) invalid("dear_local_group_connect: already connected");
  }
  // Zero-copy when every rank's gradients (and parameters) have the same
  // layout relative to its lowest tensor address, in the same 16 B phase.
  const char* env = std::getenv("DEAR_ZERO_COPY");
  bool zc = allow_zero_copy && P > 1 && !(env && env[0] == '0');
  std::vector<TensorSpan> gs(static_cast<size_t>(P)), qs(static_cast<size_t>(P));
  for (int r = 0; r < P && zc; ++r) {
    const dear_ctx& c = *group->ranks[static_cast<size_t>(r)];
    gs[static_cast<size_t>(r)] = tensor_span(c, true, false);
    qs[static_cast<size_t>(r)] = tensor_span(c, false, false);
    const TensorSpan &g = gs[static_cast<size_t>(r)], &q = qs[static_cast<size_t>(r)];
    zc = g.ok && q.ok && g.layout == gs[0].layout && q.layout == qs[0].layout &&
         ((reinterpret_cast<uintptr_t>(g.lo) ^ reinterpret_cast<uintptr_t>(gs[0].lo)) & 15) == 0 &&
         ((reinterpret_cast<uintptr_t>(q.lo) ^ reinterpret_cast<uintptr_t>(qs[0].lo)) & 15) == 0;
  }
  int sms = 148;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount,
                                    group->ranks[0]->device), "cudaDeviceGetAttribute");
  for (int r = 0; r < P; ++r) {
    dear_ctx& c = *group->ranks[static_cast<size_t>(r)];
    PeerArgs pa{}, ga{}, qa{};
    pa.P = ga.P = qa.P = P;
    pa.rank = ga.rank = qa.rank = r;
    for (int k = 0; k < P; ++k) {
      const dear_ctx& o = *group->ranks[static_cast<size_t>(k)];
      pa.delta[k] = static_cast<int64_t>(o.arena - c.arena);
      if (zc) {
        ga.delta[k] = static_cast<int64_t>(gs[static_cast<size_t>(k)].lo - gs[static_cast<size_t>(r)].lo);
        qa.delta[k] = static_cast<int64_t>(qs[static_cast<size_t>(k)].lo - qs[static_cast<size_t>(r)].lo);
      }
    }
    enable_peer(c, pa, ga, qa, zc);
  }
  // The group launch records: per bucket, [RS: P ranks][AG: P ranks]. One
  // cooperative grid of P x nb CTAs (one per SM in total) runs all ranks.
  const size_t G = group->ranks[0]->buckets.size();
  std::vector<GroupOp> ops(G * 2 * static_cast<size_t>(P));
  for (size_t g = 0; g < G; ++g) {
    for (int r = 0; r < P; ++r) {
      const dear_ctx& c = *group->ranks[static_cast<size_t>(r)];
      const Bucket& B = c.buckets[g];
      GroupOp& rs = ops[(g * 2) * static_cast<size_t>(P) + static_cast<size_t>(r)];
      GroupOp& ag = ops[(g * 2 + 1) * static_cast<size_t>(P) + static_cast<size_t>(r)];
      rs.hp = ag.hp = c.hp_dev;
      rs.flags = ag.flags = B.flags;
      rs.pa = ag.pa = c.pa;
      if (c.zc) {
        rs.units = B.zrs_u, rs.slices = B.zrs_ps, rs.mom = B.mom, rs.sa = c.ga;
        rs.n_slices = kZcSlices;
        ag.units = B.zag_u, ag.slices = B.zag_ps, ag.sa = c.qa, ag.n_slices = kZcSlices;
      } else {
        rs.units = B.upd_u, rs.slices = B.upd_ps, rs.sa = c.pa, rs.n_slices = kPeerSlices;
        ag.units = B.unpack_u, ag.slices = B.unpack_ps, ag.sa = c.pa, ag.n_slices = kPeerSlices;
      }
    }
  }
  if (group->ops_dev) cudaFree(group->ops_dev);
  group->ops_dev = nullptr;
  if (!ops.empty()) {
    cuda_check(cudaMalloc(&group->ops_dev, ops.size() * sizeof(GroupOp)), "cudaMalloc(group ops)");
    cuda_check(cudaMemcpy(group->ops_dev, ops.data(), ops.size() * sizeof(GroupOp),
                          cudaMemcpyHostToDevice), "cudaMemcpy(group ops)");
  }
  group->nb = std::max(1, sms / P);
  group->connected = true;
  DEAR_API_END
}

int dear_peer_handle(dear_ctx* ctx, uint8_t out[DEAR_PEER_HANDLE_BYTES]) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (ctx->local || ctx->same_dev)
    invalid("dear_peer_handle: local-group contexts connect with dear_local_group_connect");
  if (!out) invalid("dear_peer_handle: null output");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t h;
  cuda_check(cudaIpcGetMemHandle(&h, ctx->arena), "cudaIpcGetMemHandle");
  memset(out, 0, DEAR_PEER_HANDLE_BYTES);
  memcpy(out, &h, 64);
  const uint64_t sz = ctx->arena_bytes;
  memcpy(out + 64, &sz, 8);
  const int32_t r = ctx->rank;
  memcpy(out + 72, &r, 4);
  // Zero-copy: the gradients and parameters each in one exportable allocation.
  const char* env = std::getenv("DEAR_ZERO_COPY");
  int32_t zc = ctx->zc_tables && !(env && env[0] == '0');
  TensorSpan gs, qs;
  cudaIpcMemHandle_t gh{}, qh{};
  if (zc) {
    gs = tensor_span(*ctx, true);
    qs = tensor_span(*ctx, false);
    zc = gs.ok && qs.ok && cudaIpcGetMemHandle(&gh, gs.base) == cudaSuccess &&
         cudaIpcGetMemHandle(&qh, qs.base) == cudaSuccess;
    cudaGetLastError();  // a non-exportable allocation only disables zero-copy
  }
  memcpy(out + kH_ZC, &zc, 4);
  const int32_t push = ctx->push_tables ? 1 : 0;
  memcpy(out + kH_PUSH, &push, 4);
  if (zc) {
    memcpy(out + kH_G, &gh, 64);
    memcpy(out + kH_Q, &qh, 64);
    const uint64_t goff = static_cast<uint64_t>(gs.lo - gs.base), qoff = static_cast<uint64_t>(qs.lo - qs.base);
    memcpy(out + kH_GOFF, &goff, 8);
    memcpy(out + kH_QOFF, &qoff, 8);
    memcpy(out + kH_GLAY, &gs.layout, 8);
    memcpy(out + kH_QLAY, &qs.layout, 8);
  }
  DEAR_API_END
}

int dear_peer_connect(dear_ctx* ctx, const uint8_t* handles, int32_t n) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (c.local || c.same_dev)
    invalid("dear_peer_connect: local-group contexts connect with dear_local_group_connect");
  if (c.peer) invalid("dear_peer_connect: already connected");
  if (!handles || n != c.P) invalid("dear_peer_connect: need one handle per rank");
  if (c.P > kMaxPeers) invalid("dear_peer_connect: at most 16 ranks");
  PeerArgs pa{}, ga{}, qa{};
  pa.P = ga.P = qa.P = c.P;
  pa.rank = ga.rank = qa.rank = c.rank;
  // Zero-copy only when every rank offers it with the same tensor layouts
  // (and the same 16 B phase, so the kernels' float4 streams line up).
  bool zc = true;
  uint64_t glay = 0, qlay = 0, goff0 = 0, qoff0 = 0;
  for (int k = 0; k < c.P; ++k) {
    const uint8_t* h = handles + static_cast<size_t>(k) * DEAR_PEER_HANDLE_BYTES;
    int32_t z = 0;
    uint64_t gl = 0, ql = 0, go = 0, qo = 0;
    memcpy(&z, h + kH_ZC, 4);
    int32_t push = 0;
    memcpy(&push, h + kH_PUSH, 4);
    if ((push != 0) != c.push_tables)
      invalid("dear_peer_connect: ranks disagree on DEAR_PUSH_RS (set it on every rank before "
              "dear_finalize)");
    memcpy(&gl, h + kH_GLAY, 8);
    memcpy(&ql, h + kH_QLAY, 8);
    memcpy(&go, h + kH_GOFF, 8);
    memcpy(&qo, h + kH_QOFF, 8);
    if (k == 0) {
      glay = gl, qlay = ql, goff0 = go, qoff0 = qo;
    }
    zc = zc && z && gl == glay && ql == qlay && (go & 15) == (goff0 & 15) &&
         (qo & 15) == (qoff0 & 15);
  }
  const TensorSpan gs = zc ? tensor_span(c, true) : TensorSpan{};
  const TensorSpan qs = zc ? tensor_span(c, false) : TensorSpan{};
  zc = zc && gs.ok && qs.ok;
  std::vector<void*> maps;
  try {
    for (int k = 0; k < c.P; ++k) {
      const uint8_t* h = handles + static_cast<size_t>(k) * DEAR_PEER_HANDLE_BYTES;
      uint64_t sz = 0;
      int32_t r = -1;
      memcpy(&sz, h + 64, 8);
      memcpy(&r, h + 72, 4);
      if (r != k) invalid("dear_peer_connect: handles must be in rank order");
      if (sz != c.arena_bytes) invalid("dear_peer_connect: ranks registered different models");
      if (k == c.rank) continue;
      auto open = [&](size_t at) {
        cudaIpcMemHandle_t ih;
        memcpy(&ih, h + at, 64);
        void* p = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
        maps.push_back(p);
        return static_cast<char*>(p);
      };
      pa.delta[k] = static_cast<int64_t>(open(0) - c.arena);
      if (zc) {
        uint64_t go = 0, qo = 0;
        memcpy(&go, h + kH_GOFF, 8);
        memcpy(&qo, h + kH_QOFF, 8);
        char* gbase = open(kH_G);
        // Gradients and parameters in one allocation: map it once.
        char* qbase = memcmp(h + kH_G, h + kH_Q, 64) == 0 ? gbase : open(kH_Q);
        ga.delta[k] = static_cast<int64_t>(gbase + go - gs.lo);
        qa.delta[k] = static_cast<int64_t>(qbase + qo - qs.lo);
      }
    }
  } catch (...) {
    for (void* m : maps) cudaIpcCloseMemHandle(m);
    throw;
  }
  c.peer_maps = std::move(maps);
  enable_peer(c, pa, ga, qa, zc);
  DEAR_API_END
}

int dear_nvls_connect(dear_ctx* ctx, dear_symm* heap) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (!heap) invalid("dear_nvls_connect: null heap");
  if (c.local || c.same_dev) invalid("dear_nvls_connect: needs one process per GPU");
  if (c.peer || c.nvls) invalid("dear_nvls_connect: already connected");
  if (!symm_bound(heap)) invalid("dear_nvls_connect: the heap is not bound (dear_symm_bind)");
  if (symm_size(heap) != c.P || symm_rank(heap) != c.rank)
    invalid("dear_nvls_connect: heap and context disagree on rank / world size");
  if (c.P > 1 && !c.comm) invalid("dear_nvls_connect: needs the NCCL communicator for the layout check");
  // Every tensor in the heap, at offsets identical on every rank.
  const uintptr_t base = symm_base(heap);
  uint64_t h = 1469598103934665603ULL;
  for (size_t i = 0; i < c.layers.size(); ++i) {
    const LayerReg& R = c.layers[i];
    if (R.numel <= 0) continue;
    const size_t nb = static_cast<size_t>(R.numel) * 4;
    if (!symm_contains(heap, R.grad, nb) || !symm_contains(heap, R.param, nb) ||
        (R.shadow && !symm_contains(heap, R.shadow, nb / 2)))
      invalid("dear_nvls_connect: layer " + std::to_string(i + 1) +
              "'s gradient / parameter / bf16 copy is not inside the symmetric heap");
    h = fnv(h, reinterpret_cast<uintptr_t>(R.grad) - base);
    h = fnv(h, reinterpret_cast<uintptr_t>(R.param) - base);
    h = fnv(h, R.shadow ? reinterpret_cast<uintptr_t>(R.shadow) - base : ~0ULL);
  }
  const size_t G = c.buckets.size();
  const size_t at = symm_take_flags(heap, G * sizeof(NvlsFlags));
  h = fnv(h, at);
  if (c.P > 1) {
    unsigned long long hv[2] = {h, ~h};
    cuda_check(cudaMemcpy(c.hash_dev, hv, sizeof hv, cudaMemcpyHostToDevice), "cudaMemcpy");
    nccl_check(ncclAllReduce(c.hash_dev, c.hash_dev, 2, ncclUint64, ncclMax, c.comm, c.comm_stream),
               "ncclAllReduce(nvls layout check)");
    cuda_check(cudaMemcpyAsync(hv, c.hash_dev, sizeof hv, cudaMemcpyDeviceToHost, c.comm_stream),
               "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
    if (hv[0] != h || hv[1] != ~h)
      invalid("dear_nvls_connect: ranks placed their tensors at different heap offsets");
  }
  const int64_t d = symm_mc_delta(heap);
  NvlsArgs na{};
  na.mc_delta = d;
  na.ucf = reinterpret_cast<NvlsFlags*>(base + at);
  na.mcf = reinterpret_cast<NvlsFlags*>(base + at + d);
  na.P = c.P;
  na.spin_limit = peer_spin_limit(c.device);
  c.na = na;
  c.nvls = true;
  c.peer = true;  // no pack / update / unpack kernels (fused in the NVLS pair)
  // 1/P after the switch's sum (same bits as pre-scaling for P = 2^k).
  c.hp_host.prescaled = 0;
  cuda_check(cudaMemcpy(c.hp_dev, &c.hp_host, sizeof(HyperParams), cudaMemcpyHostToDevice),
             "cudaMemcpy(hp)");
  DEAR_API_END
}

int dear_nvls_enabled(dear_ctx* ctx, int32_t* on) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (!on) invalid("dear_nvls_enabled: null output");
  *on = ctx->nvls ? 1 : 0;
  DEAR_API_END
}

int dear_peer_zero_copy(dear_ctx* ctx, int32_t* on) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (!on) invalid("dear_peer_zero_copy: null output");
  *on = ctx->zc ? (ctx->push ? 2 : 1) : 0;
  DEAR_API_END
}

int dear_bench_stage(dear_ctx* ctx, int32_t stage, int32_t reps, void* stream) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (stage < 0 || stage > 3 || reps < 0) invalid("dear_bench_stage: stage in 0..3, reps >= 0");
  if (stage == 3 && !c.direct) invalid("dear_bench_stage: no direct-update tables (P > 1 or DEAR_DIRECT=0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool wd = c.cfg.weight_decay != 0.0, mom = c.cfg.momentum != 0.0;
  for (int r = 0; r < reps; ++r) {
    for (Bucket& B : c.buckets) {
      cudaError_t e = cudaSuccess;
      switch (stage) {
        case 0: e = launch_pack(B.pack_u, B.pack_s, B.e_pack, c.pack_scale, 0, s); break;
        // has_buf = 0: momentum (if any) is re-seeded each launch, the same traffic
        case 1: e = launch_update(B.upd_u, B.upd_s, B.e_upd, c.hp_dev, 0, mom, wd, 0, s); break;
        case 2: e = launch_unpack(B.unpack_u, B.unpack_s, B.e_unpack, B.any_shadow ? 1 : 0, 0, s); break;
        default: e = launch_update_direct(B.dir_u, B.dir_s, B.e_dir, c.hp_dev, wd,
                                          B.any_shadow ? 1 : 0, s); break;
      }
      cuda_check(e, "dear_bench_stage");
    }
  }
  DEAR_API_END
}

int dear_num_buckets(dear_ctx* ctx, int32_t* n) {
  DEAR_API_BEGIN
  need(ctx, true);
  *n = static_cast<int32_t>(ctx->buckets.size());
  DEAR_API_END
}

int dear_bucket_info(dear_ctx* ctx, int32_t g, int32_t* low, int32_t* high, int64_t* elems,
                     int64_t* stride) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (g < 0 || static_cast<size_t>(g) >= ctx->buckets.size()) invalid("bucket index out of range");
  const Bucket& B = ctx->buckets[static_cast<size_t>(g)];
  if (low) *low = B.low;
  if (high) *high = B.high;
  if (elems) *elems = B.d;
  if (stride) *stride = B.stride;
  DEAR_API_END
}

int dear_trace(dear_ctx* ctx, char* buf, int64_t cap, int64_t* needed) {
  DEAR_API_BEGIN
  if (!ctx) invalid("null context");
  std::string s;
  for (const auto& t : ctx->trace) s += t + "\n";
  if (needed) *needed = static_cast<int64_t>(s.size()) + 1;
  if (buf && cap > 0) {
    const size_t n = std::min(static_cast<size_t>(cap - 1), s.size());
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  DEAR_API_END
}

int dear_set_timing(dear_ctx* ctx, int32_t enable) {
  DEAR_API_BEGIN
  need(ctx, true);
  ctx->timing = enable != 0;
  for (Bucket& B : ctx->buckets)
    for (bool& r : B.t_rec) r = false;
  DEAR_API_END
}

int dear_get_timings(dear_ctx* ctx, float* out, int32_t n_buckets) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (n_buckets != static_cast<int32_t>(ctx->buckets.size())) invalid("dear_get_timings: bucket count mismatch");
  auto span = [&](const Bucket& B, int a, int b) -> float {
    if (!B.t_rec[a] || !B.t_rec[b]) return -1.f;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, B.t[a], B.t[b]) != cudaSuccess) return -1.f;
    return ms;
  };
  for (size_t g = 0; g < ctx->buckets.size(); ++g) {
    const Bucket& B = ctx->buckets[g];
    float* o = out + g * 5;
    o[0] = span(B, T_PACK0, T_PACK1);
    o[1] = span(B, T_PACK1, T_RS1);
    o[2] = span(B, T_RS1, T_UPD1);
    o[3] = span(B, T_AG0, T_AG1);
    o[4] = span(B, T_AG1, T_UNPACK1);
  }
  DEAR_API_END
}

int dear_get_timeline(dear_ctx* ctx, void* base_event, float* out, int32_t n_buckets) {
  DEAR_API_BEGIN
  need(ctx, true);
  if (!base_event || !out) invalid("dear_get_timeline: null argument");
  if (n_buckets != static_cast<int32_t>(ctx->buckets.size()))
    invalid("dear_get_timeline: bucket count mismatch");
  cudaEvent_t base = static_cast<cudaEvent_t>(base_event);
  for (size_t g = 0; g < ctx->buckets.size(); ++g) {
    const Bucket& B = ctx->buckets[g];
    for (int k = 0; k < T_COUNT; ++k) {
      float ms = -1.f;
      if (B.t_rec[k] && cudaEventElapsedTime(&ms, base, B.t[k]) != cudaSuccess) {
        (void)cudaGetLastError();
        ms = -1.f;
      }
      out[g * T_COUNT + k] = ms;
    }
  }
  DEAR_API_END
}

static unsigned long long hash_params(dear_ctx& c) {
  cuda_check(cudaMemsetAsync(c.hash_dev, 0, sizeof(unsigned long long), c.comm_stream), "cudaMemsetAsync");
  for (size_t i = 0; i < c.layers.size(); ++i)
    cuda_check(launch_hash(c.layers[i].param, c.layers[i].numel, 0x9E3779B97F4A7C15ULL * (i + 1),
                           c.hash_dev, c.comm_stream),
               "hash kernel");
  unsigned long long h = 0;
  cuda_check(cudaMemcpyAsync(&h, c.hash_dev, sizeof h, cudaMemcpyDeviceToHost, c.comm_stream), "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
  return h;
}

int dear_check_replicas(dear_ctx* ctx, int32_t* identical) {
  DEAR_API_BEGIN
  need(ctx, true);
  dear_ctx& c = *ctx;
  if (c.ags_deferred) c.enqueue_feedpipe(c.compute);
  cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
  const unsigned long long h = hash_params(c);
  if (c.local || c.same_dev) {
    bool same = true;
    for (dear_ctx* o : c.group->ranks) {
      if (!o || o == &c) continue;
      cuda_check(cudaStreamSynchronize(o->comm_stream), "cudaStreamSynchronize");
      if (hash_params(*o) != h) same = false;
    }
    *identical = same ? 1 : 0;
  } else if (c.P > 1) {
    unsigned long long hv[2] = {h, ~h};
    cuda_check(cudaMemcpy(c.hash_dev, hv, sizeof hv, cudaMemcpyHostToDevice), "cudaMemcpy");
    nccl_check(ncclAllReduce(c.hash_dev, c.hash_dev, 2, ncclUint64, ncclMax, c.comm, c.comm_stream),
               "ncclAllReduce(replica check)");
    unsigned long long out[2];
    cuda_check(cudaMemcpyAsync(out, c.hash_dev, sizeof out, cudaMemcpyDeviceToHost, c.comm_stream), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(c.comm_stream), "cudaStreamSynchronize");
    *identical = (out[0] == h && out[1] == ~h) ? 1 : 0;
  } else {
    *identical = 1;
  }
  DEAR_API_END
}

}  // extern "C"
