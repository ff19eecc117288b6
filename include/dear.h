/*
 * dear.h — C ABI of the B200-native DeAR decoupled all-reduce runtime.
 *
 * The reference (/root/reference/proj, a C++20 simulator + fp64 oracle) has no
 * runtime FFI; its interface for this path is the value-type C++ API in
 * proj/include/dearsim/{model,fusion,policy,collective,task_graph}.hpp, and
 * the paper describes the runtime as "a communication library using C/C++
 * based on NCCL [exposing] APIs for high-level scripts in Python" wrapped by a
 * DistOptim. Each entry point below cites the reference
 * interface it realises. INTEGRATION.md shows the ctypes binding.
 *
 * Conventions (mirroring the reference's error model):
 *   return 0 (DEAR_OK), 1 (DEAR_EINVAL: std::invalid_argument in the
 *   reference, e.g. "build_fusion_plan: empty model", fusion.cpp:33) or
 *   2 (DEAR_EINTERNAL: CUDA/NCCL failure; std::runtime_error in the
 *   reference). dear_last_error() returns the calling thread's last message.
 *   Layers are 1-based: layer 1 is the input side, layer L the output side
 *   (model.hpp:24-34). A context is not thread-safe; serialise calls.
 *   Streams are cudaStream_t passed as void* (NULL = legacy default stream).
 */
#ifndef DEAR_H_
#define DEAR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DEAR_OK 0
#define DEAR_EINVAL 1
#define DEAR_EINTERNAL 2

/* PolicyKind (policy.hpp:34), same numbering. PRIORITY_PARTITION (the
 * ByteScheduler baseline, task_graph.cpp:215-258): every layer's all-reduce in
 * ceil(bytes / partition_bytes) parts, dispatched by ascending layer (the
 * order the forward consumes them) instead of gradient-readiness order. */
#define DEAR_POLICY_WFBP 0
#define DEAR_POLICY_WFBP_FUSED 1
#define DEAR_POLICY_PRIORITY_PARTITION 2
#define DEAR_POLICY_DEAR 3
#define DEAR_POLICY_DEAR_FUSED 4

typedef struct dear_ctx dear_ctx;
typedef struct dear_local_group dear_local_group;

/* PolicySpec (policy.hpp:36-45) + the optimizer of SgdState
 * (collective.hpp:77-80). momentum / dampening / weight_decay / nesterov
 * follow torch.optim.SGD and are an UNPINNED extension (the reference's
 * update is plain lr-SGD, collective.cpp:190-192). */
typedef struct {
  int32_t policy;               /* DEAR_POLICY_* */
  int64_t fusion_buffer_bytes;  /* > 0 for *_FUSED (policy.cpp:53-66) */
  int32_t dear_group_dependency;/* policy.hpp:44: AG_g waits on RS_g only */
  double lr;
  double momentum;
  double dampening;
  double weight_decay;
  int32_t nesterov;
  int32_t defer_allgather;      /* 1: AGs are enqueued by the next
                                   dear_param_wait (CUDA-graph friendly);
                                   0: by dear_step */
  int64_t partition_bytes;      /* > 0 for PRIORITY_PARTITION (policy.cpp:58-61) */
} dear_cfg;

/* ---------------------------------------------------------------------------
 * Pure host functions (no GPU needed).
 * ------------------------------------------------------------------------ */

/* build_fusion_plan (fusion.cpp:29-57); buffer_bytes == 0 selects
 * per_layer_plan (fusion.cpp:59-70). layer_bytes[0] is layer 1. Groups are
 * written in backprop issue order (low[0]/high[0] hold layer L); low/high
 * need room for L entries. Bit-exact with the reference. */
int dear_plan_build(const int64_t* layer_bytes, int32_t L, int64_t buffer_bytes,
                    int32_t* low, int32_t* high, int32_t* n_groups);

/* chunk_ranges (collective.cpp:39-57): begin[0..P] (P+1 entries), chunk c is
 * [begin[c], begin[c+1]). *slot_elems = ceil(d/P), the per-rank NCCL count
 * before alignment padding. Chunk c is owned (fully reduced) by rank
 * (c-1) mod P (collective.cpp:94), so NCCL slot r carries chunk (r+1) mod P. */
int dear_chunk_layout(int64_t d, int32_t P, int64_t* begin, int64_t* slot_elems);

/* Stride (elements) between rank slots in a bucket buffer: ceil(d/P) rounded
 * up to a multiple of 64 elements (256 B). */
int64_t dear_slot_stride(int64_t d, int32_t P);

const char* dear_last_error(void);

/* ---------------------------------------------------------------------------
 * Communicators. NCCL over NVLink/NVSwitch for one process per GPU; a local
 * group emulates P ranks inside one process (one device), with collectives
 * executed as ring-order kernels over all ranks' buffers — used to exercise
 * the P > 1 path on a single GPU.
 * ------------------------------------------------------------------------ */
int dear_comm_unique_id(uint8_t id[128]);
int dear_comm_init(void** comm, int32_t nranks, const uint8_t id[128], int32_t rank);
int dear_comm_destroy(void* comm);
int dear_local_group_create(int32_t P, dear_local_group** group);
int dear_local_group_destroy(dear_local_group* group);

/* Local-group transports (P ranks as contexts of ONE process on ONE device,
 * driven in lock-step; each rank's ops queue, and a collective runs once every
 * rank reached it). RING: ring-order kernels over all ranks' buffers
 * (collective.cpp:59-152). PEER: the multi-GPU NVLink peer kernels themselves
 * (zero-copy or slot reduce-scatter + update, all-gather) with the other
 * ranks' memory addressed by in-process deltas instead of IPC mappings — a
 * one-GPU box runs the N > 1 data path. Their cross-rank counter waits stay
 * inside ONE cooperative launch holding every rank's CTAs, so no kernel ever
 * waits on another launch. */
#define DEAR_LOCAL_RING 0
#define DEAR_LOCAL_PEER 1
int dear_local_group_create_ex(int32_t P, int32_t transport, dear_local_group** group);
/* PEER transport, after dear_finalize on every rank: connect the ranks.
 * allow_zero_copy = 1 selects the zero-copy kernels when every rank's
 * gradients and parameters share one relative layout (as dear_peer_connect);
 * 0 forces the slot path. dear_peer_zero_copy reports the outcome. */
int dear_local_group_connect(dear_local_group* group, int32_t allow_zero_copy);

/* ---------------------------------------------------------------------------
 * Runtime context (the DistOptim of PAPER.md:183-188).
 * ------------------------------------------------------------------------ */

/* nccl_comm: an ncclComm_t from dear_comm_init (NULL allowed when P == 1).
 * compute_stream: the stream forward/backward run on (recorded for joins).
 * Validates cfg like validate(PolicySpec) (policy.cpp:53-66). */
int dear_create(void* nccl_comm, int32_t rank, int32_t P, void* compute_stream,
                const dear_cfg* cfg, dear_ctx** out);
/* Same, as rank `rank` of a local group. */
int dear_create_local(dear_local_group* group, int32_t rank, void* compute_stream,
                      const dear_cfg* cfg, dear_ctx** out);

/* Tensor registration: LayerSpec (model.hpp:26-34). `layer` must end up
 * exactly 1..L (model.cpp:50-56). param/grad are caller-owned device fp32
 * buffers of `numel` elements. */
int dear_register_tensor(dear_ctx* ctx, int32_t layer, float* param, float* grad,
                         int64_t numel);
/* Optional bf16 compute copy of a layer's parameters; the fused unpack
 * kernel refreshes it together with the fp32 parameters. */
int dear_register_shadow(dear_ctx* ctx, int32_t layer, void* bf16_copy);
/* Builds the fusion plan, bucket buffers, unit tables, events; checks (when
 * P > 1) that every rank registered the same model. */
int dear_finalize(dear_ctx* ctx);

/* Backward hook: layer's gradient is complete on `stream`. When the bucket
 * holding it is complete (all its layers reported), its pack -> RS -> update
 * is enqueued on the comm stream, in plan order (task_graph.cpp:186-194,
 * RS_g deps = BP of g's layers :148-154). WFBP kinds also enqueue AG + unpack
 * right behind (task_graph.cpp:163-176). */
int dear_grad_ready(dear_ctx* ctx, int32_t layer, void* stream);

/* Forward pre-hook: `stream` waits for the all-gather + unpack of the bucket
 * holding `layer` (FF_l <- AG_{g(l)}, task_graph.cpp:207) — never a global
 * barrier. Enqueues deferred all-gathers first when defer_allgather = 1. */
int dear_param_wait(dear_ctx* ctx, int32_t layer, void* stream);

/* End of backprop: the BARRIER of task_graph.cpp:195-198. All layers must
 * have been reported. DEAR kinds enqueue AG_g + unpack in feed-forward order
 * (reverse plan order, :199-206) unless deferred. `stream` (the caller's
 * compute stream) is fenced both ways: the comm stream's all-gathers wait for
 * work already on `stream`, and `stream` waits until every gradient has been
 * packed (so gradients may be zeroed / overwritten afterwards). */
int dear_step(dear_ctx* ctx, void* stream);
/* dear_group_dependency (policy.hpp:44; task_graph.cpp:195-206): AG_g depends
 * on RS_g only and the comm resource dispatches ready work by issue order
 * (simulate.cpp:65-159), so all-gathers back-fill the comm stream during
 * backprop. A CUDA stream is in-order, so the dispatch sequence is fixed per
 * iteration: seq[0..2G) lists the comm tasks as the reference's scheduler
 * dispatches them (v > 0: RS of bucket v, v < 0: AG of bucket -v, 1-based plan
 * order; RS in plan order, each AG after its RS), e.g. from simulating the
 * iteration on measured times (costmodel.predict_iteration). AGs between two
 * RS entries are enqueued right behind the first during backprop; the AGs
 * after the last RS at dear_step (or, deferred, at the next dear_param_wait),
 * in seq order, where they overlap the next feed-forward. n = 0 restores the default (all AGs at dear_step in feed-forward
 * order). Requires a DEAR policy with dear_group_dependency; call between
 * iterations. */
int dear_set_comm_order(dear_ctx* ctx, const int32_t* seq, int32_t n);
/* PRIORITY_PARTITION uses the same call: seq lists every part (1-based, plan
 * order: layer L's parts first) once, in the order the reference scheduler
 * dispatches them (costmodel.predict_iteration(..., "PRIORITY_PARTITION")
 * ["comm_order"]); a part is enqueued once it and every part before it in seq
 * is ready. n = 0: gradient-readiness order. The negotiation of the reference
 * (a modelled latency) has no runtime counterpart: ranks agree on seq. */

/* `stream` waits for all comm-stream work enqueued so far (graph capture
 * join point). */
int dear_join(dear_ctx* ctx, void* stream);

/* Host-blocking: flush deferred all-gathers and wait until parameters are
 * fully updated ("forced to synchronize ... before evaluating"). */
int dear_synchronize(dear_ctx* ctx);

/* Failure detection: *failed = 1 when the NCCL communicator
 * reported an asynchronous error (ncclCommGetAsyncError). dear_synchronize
 * polls the same while it waits, and with DEAR_SYNC_TIMEOUT_S set also bounds
 * the wait; either way it aborts the communicator (ncclCommAbort) and returns
 * DEAR_EINTERNAL instead of hanging. The NVLink peer / NVLS kernels bound
 * their cross-GPU waits with DEAR_PEER_TIMEOUT_S (default 600 s; they trap). */
int dear_comm_error(dear_ctx* ctx, int32_t* failed);

/* Profiling aid: the zero-copy reduce-scatter / all-gather CTAs append 40-byte
 * records {u64 t_start, u64 t_peers_arrived, u64 t_end (%globaltimer ns),
 * u32 kind (0 RS, 1 AG), u32 bucket tag, u32 epoch, u32 cta} to a device
 * buffer of `capacity` records (NULL = off); dear_comm_trace_count reads how
 * many were written since the last dear_set_comm_trace (process-wide). */
int dear_set_comm_trace(void* device_buffer, int64_t capacity);
int dear_comm_trace_count(int64_t* n);

int dear_destroy(dear_ctx* ctx);

/* Learning-rate change (device-resident; CUDA-graph safe). */
int dear_set_lr(dear_ctx* ctx, double lr);

/* ---------------------------------------------------------------------------
 * NVLink peer backend (one process per GPU, after dear_finalize on every rank).
 * Each rank exports an IPC handle of its bucket arena; once every rank has
 * connected to all handles, each bucket's reduce-scatter runs as ONE kernel
 * that reads every rank's slot over NVLink, sums in the reference's ring
 * order (collective.cpp:70-90, bit-exact with the fp32 restatement) and
 * applies the SGD update; the all-gather runs as ONE kernel that reads each
 * owner's updated slot over NVLink straight into the parameters (+ bf16 copy).
 * Cross-GPU ordering uses per-bucket completion counters in each arena
 * (graph-safe). The NCCL communicator is still used for dear_finalize's and
 * dear_check_replicas' cross-rank checks.
 * ------------------------------------------------------------------------ */
#define DEAR_PEER_HANDLE_BYTES 256
int dear_peer_handle(dear_ctx* ctx, uint8_t out[DEAR_PEER_HANDLE_BYTES]);
/* handles: n = P records of DEAR_PEER_HANDLE_BYTES, in rank order.
 * Zero-copy: when every rank's registered gradients lie in one device
 * allocation and its parameters in another (e.g. flat buffers viewed per
 * layer), with the same relative layout on every rank, those allocations are
 * IPC-mapped as well. The reduce-scatter kernel then reads the owned chunk of
 * every rank's gradients in place (no pack, no bucket buffer) and writes the
 * updated shard into the owner's parameters, and the all-gather kernel reads
 * the owners' parameters: 14 B of HBM traffic per element and rank instead of
 * 24 (P = 4). Same sums in the same order, so results are unchanged. The
 * environment variable DEAR_ZERO_COPY=0 disables it. Gradients are then
 * "consumed" (dear_step's fence) once every rank's reduce-scatters finished. */
int dear_peer_connect(dear_ctx* ctx, const uint8_t* handles, int32_t n);
/* *on = 1 when dear_peer_connect enabled the zero-copy path, 2 when it also
 * took the push reduce-scatter (DEAR_PUSH_RS=1 set on every rank before
 * dear_finalize: each rank writes every chunk of its gradients into slot
 * `rank` of the chunk owner's push buffer over NVLink; the owner sums its P
 * slots locally in ring order — same sums, same bits; the all-gather stays
 * the zero-copy pull). */
int dear_peer_zero_copy(dear_ctx* ctx, int32_t* on);

/* ---------------------------------------------------------------------------
 * NVLS backend (NVLink SHARP through the NVSwitch, one process per GPU).
 * Gradients, parameters and bf16 copies live in a symmetric heap: per rank one
 * physical allocation mapped locally and through ONE multicast object over
 * all P GPUs. The owner of a chunk reduces it with multimem.ld_reduce (the
 * switch sums the P ranks' values), applies the SGD update, and the
 * all-gather broadcasts the updated chunk with multicast stores; cross-rank
 * order uses counters bumped on every rank by multimem.red and polled
 * locally. The switch's fp32 summation order is unspecified: exact at P = 2,
 * within the 1e-5 tolerance otherwise (like NCCL). The schedule (RS during
 * backprop, AG gating each layer's forward) is unchanged.
 * ------------------------------------------------------------------------ */
typedef struct dear_symm dear_symm;
/* *ok = 1 when `device` supports multicast objects. */
int dear_nvls_supported(int32_t device, int32_t* ok);
/* Collective heap setup: every rank calls dear_symm_create (rank 0 returns the
 * (pid, fd) of the exported multicast handle; others get -1), the caller
 * broadcasts rank 0's pair, every rank calls dear_symm_join (imports it with
 * pidfd_getfd; no-op on rank 0), barrier, dear_symm_bind, barrier. */
int dear_symm_create(int32_t rank, int32_t P, int64_t bytes, dear_symm** out, int64_t* pid,
                     int64_t* fd);
int dear_symm_join(dear_symm* heap, int64_t pid, int64_t fd);
int dear_symm_bind(dear_symm* heap);
/* The caller's region: local and multicast base addresses, bytes (>= the
 * requested size). Carve identical layouts on every rank. */
int dear_symm_ptr(dear_symm* heap, void** local, void** multicast, int64_t* bytes);
/* Collective: every rank synchronizes and barriers first (peers store into
 * this rank's memory through the multicast alias). */
int dear_symm_destroy(dear_symm* heap);
/* After dear_finalize: switch ctx to the NVLS kernels. Every registered
 * gradient, parameter and bf16 copy must lie in `heap`'s region at the same
 * offsets on every rank (checked across ranks over the NCCL communicator). */
int dear_nvls_connect(dear_ctx* ctx, dear_symm* heap);
/* *on = 1 when ctx runs the NVLS kernels. */
int dear_nvls_enabled(dear_ctx* ctx, int32_t* on);

/* ---------------------------------------------------------------------------
 * Introspection, timing and checks.
 * ------------------------------------------------------------------------ */
int dear_num_buckets(dear_ctx* ctx, int32_t* n);
/* Bucket g (0-based, plan order): layers low..high, d elements, slot stride. */
int dear_bucket_info(dear_ctx* ctx, int32_t g, int32_t* low, int32_t* high, int64_t* elems,
                     int64_t* slot_stride);
/* Collective issue log of the current/last iteration, reference task labels
 * (task_graph.cpp:51-58), e.g. "RS g1\nRS g2\nAG g2\nAG g1\n". Writes at most
 * cap bytes (NUL-terminated); *needed gets the full length + 1. */
int dear_trace(dear_ctx* ctx, char* buf, int64_t cap, int64_t* needed);
/* Enable per-bucket CUDA-event timing of pack / RS / update / AG / unpack. */
int dear_set_timing(dear_ctx* ctx, int32_t enable);
/* After dear_synchronize: milliseconds per bucket and stage for the last
 * timed iteration; out is n_buckets x 5 (pack, rs, update, ag, unpack),
 * -1 where a stage did not run. */
int dear_get_timings(dear_ctx* ctx, float* out, int32_t n_buckets);
/* Measured timeline of the last timed iteration: for every bucket the
 * milliseconds from `base_event` (a cudaEvent_t recorded earlier, as void*)
 * to its 7 comm-stream stamps: pack start, pack end (= RS start), RS end,
 * update end, AG start, AG end (= unpack start), unpack end; -1 where a stage
 * did not run. out is n_buckets x 7. */
int dear_get_timeline(dear_ctx* ctx, void* base_event, float* out, int32_t n_buckets);
/* Replica check — the GPU analogue of sgd_step's "replica divergence"
 * rejection (collective.cpp:172-181): hashes every registered parameter
 * and compares across ranks. *identical = 1 when all ranks agree. */
int dear_check_replicas(dear_ctx* ctx, int32_t* identical);
/* Measurement hook (bench.py's kernel rooflines): enqueue `reps` rounds of
 * one bucket-kernel stage over every bucket on `stream`, outside the schedule
 * — stage 0 pack, 1 update, 2 unpack, 3 direct update (P = 1). Capturable in
 * a CUDA graph, so a chain of launches is timed without host launch gaps.
 * It rewrites the bucket buffers / parameters like the real stages do
 * (values are not meaningful afterwards: re-register or re-seed). */
int dear_bench_stage(dear_ctx* ctx, int32_t stage, int32_t reps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DEAR_H_ */
