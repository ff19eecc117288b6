// sm_100a kernels for the DeAR bucket pipeline: pack (grad -> NCCL slot
// layout, fused 1/P scale), shard-local SGD update (between reduce-scatter
// and all-gather), unpack (slot layout -> fp32 params + bf16 compute copy).
//
// All three are HBM-streaming kernels: pack and unpack move
// 8 B/elem (+2 B/elem for the bf16 copy), update 12 B/shard-elem (20 with a
// momentum buffer). The host cuts every bucket op into Units (one layer x
// chunk intersection each) and gives each of the kSlices CTAs (4 per SM, one
// wave) an equal contiguous slice of the op's elements, which it walks across
// units. Inside a unit the destination is peeled to 16 B alignment
// and every access is a 128-bit vector; when the source is misaligned
// relative to the destination (layer boundaries fall anywhere inside a
// bucket), each lane loads its aligned float4 and takes the next lane's via
// __shfl_down_sync, so both sides stay 128-bit and fully coalesced.
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdlib>

#include "dear_kernels.h"

namespace dear {
namespace {

#ifndef DEAR_KTHREADS
#define DEAR_KTHREADS 256
#endif
constexpr int kThreads = DEAR_KTHREADS;
// Zero-copy / peer kernels: a register cap so one comm CTA (256 threads x 96)
// still fits on an SM next to the GEMM's two resident CTAs (2 x 6 warps x 88
// registers); at P = 2 BERT-L this took the step from 8.64 to 8.40 ms
// (profiles/r01e/tl4j_2_*.jsonl).
#ifndef DEAR_ZC_MAXNREG
#define DEAR_ZC_MAXNREG 96
#endif
#if DEAR_ZC_MAXNREG > 0
#define DEAR_ZC_BOUNDS __maxnreg__(DEAR_ZC_MAXNREG)
#else
#define DEAR_ZC_BOUNDS __launch_bounds__(kThreads, 1)
#endif
#ifndef DEAR_HBM_UNROLL
#define DEAR_HBM_UNROLL 4
#endif
constexpr int kUnroll = DEAR_HBM_UNROLL;
// Remote (NVLink) source streams: float4 loads in flight per lane in the
// all-gather. 4, not the 8 that minimise the kernel in isolation: the comm
// kernels run next to L2-bound GEMMs, and a gentler stream costs the GEMMs less
// than it costs itself (BERT-L N = 4 step 8.25 vs 8.96 ms with KU below,
// profiles/r02v2_comm_throttle.log).
#ifndef DEAR_PEER_UNROLL
#define DEAR_PEER_UNROLL 4
#endif
constexpr int kPeerUnroll = DEAR_PEER_UNROLL;

constexpr int kSms = 148;

__device__ __forceinline__ float4 shfl_down4(float4 v) {
  v.x = __shfl_down_sync(0xffffffffu, v.x, 1);
  v.y = __shfl_down_sync(0xffffffffu, v.y, 1);
  v.z = __shfl_down_sync(0xffffffffu, v.z, 1);
  v.w = __shfl_down_sync(0xffffffffu, v.w, 1);
  return v;
}

template <int M>
__device__ __forceinline__ float4 realign(float4 a, float4 b) {
  if constexpr (M == 0) {
    return a;
  } else if constexpr (M == 1) {
    return make_float4(a.y, a.z, a.w, b.x);
  } else if constexpr (M == 2) {
    return make_float4(a.z, a.w, b.x, b.y);
  } else {
    return make_float4(a.w, b.x, b.y, b.z);
  }
}

enum class Hint { kStream, kKeep };

// Realignment of a source that is not in the destination's 16 B phase by a
// second (cache-hit) load per vector in the local HBM kernels (pack, update,
// direct update, unpack); 0 keeps the shuffle exchange.
#ifndef DEAR_REALIGN_LD2
#define DEAR_REALIGN_LD2 1
#endif
constexpr bool kRealignLd2 = DEAR_REALIGN_LD2 != 0;

// Streaming (evict-first) stores for the pack / unpack destinations:
// graph-chained ResNet-50 buckets, pack 0.636 -> 0.660 and unpack 0.666 ->
// 0.708 of HBM peak (tools/micro/hbm_stage.py, profiles/r02h5_hbm_ab.log).
#ifndef DEAR_HBM_NO_ST_CS
#define HBM_ST4(p, v) __stcs(p, v)
#else
#define HBM_ST4(p, v) (*(p) = (v))
#endif
template <Hint H>
__device__ __forceinline__ float4 ld4(const float4* p) {
  if constexpr (H == Hint::kStream) {
    return __ldcs(p);
  } else {
    return __ldg(p);
  }
}

// Warp-cooperative walk over destination vectors q in [0, n4). The source
// element for destination element 4q+e is src_floor[M + 4q + e]; src_floor is
// 16 B aligned and vectors up to index qmax hold at least one valid element.
// body(q, v) runs on every lane whose q < n4. All loads of one round (kUnroll
// vectors per lane, plus the one vector past the round that lane 31 needs
// when M != 0) are issued before any is consumed: no dependent second trip.
// `pre` (optional, kPre): a second stream indexed like the destination
// (pre[q] pairs with destination vector q), loaded in the same round as the
// source so the body never starts a dependent second memory trip; the body
// then receives it as its third argument.
// kLd2 (local sources only): each lane loads its next source vector itself
// (an L1 / L2 hit — the neighbour lane loads it too) instead of taking it
// from the neighbour with 8 shuffles per vector.
template <int M, Hint H, int kUnroll, bool kPre = false, bool kLd2 = false, typename Body>
__device__ __forceinline__ void warp_stream(const float* src_floor, int64_t n4, int64_t qmax,
                                            Body&& body, const float4* pre = nullptr) {
  const float4* s4 = reinterpret_cast<const float4*>(src_floor);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = static_cast<int64_t>(warp) * 32 * kUnroll; base < n4;
       base += static_cast<int64_t>(kWarps) * 32 * kUnroll) {
    float4 a[kUnroll];
    float4 p[kPre ? kUnroll : 1];
    constexpr bool kTwo = kLd2 && M != 0;
    float4 a2[kTwo ? kUnroll : 1];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int64_t q = base + k * 32 + lane;
      a[k] = q <= qmax ? ld4<H>(s4 + q) : zero;
      if constexpr (kTwo) a2[k] = q + 1 <= qmax ? ld4<H>(s4 + q + 1) : zero;
      if constexpr (kPre) p[k] = q < n4 ? __ldcs(pre + q) : zero;
    }
    float4 extra = zero;
    if constexpr (M != 0 && !kTwo) {
      const int64_t qx = base + kUnroll * 32;
      if (lane == 31 && qx <= qmax) extra = ld4<H>(s4 + qx);
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int64_t q = base + k * 32 + lane;
      float4 b = a[k];
      if constexpr (kTwo) {
        b = a2[k];
      } else if constexpr (M != 0) {
        b = shfl_down4(a[k]);
        float4 nxt = extra;
        if (k + 1 < kUnroll) {
          nxt.x = __shfl_sync(0xffffffffu, a[k + 1 < kUnroll ? k + 1 : k].x, 0);
          nxt.y = __shfl_sync(0xffffffffu, a[k + 1 < kUnroll ? k + 1 : k].y, 0);
          nxt.z = __shfl_sync(0xffffffffu, a[k + 1 < kUnroll ? k + 1 : k].z, 0);
          nxt.w = __shfl_sync(0xffffffffu, a[k + 1 < kUnroll ? k + 1 : k].w, 0);
        }
        if (lane == 31) b = nxt;
      }
      if constexpr (kPre) {
        if (q < n4) body(q, realign<M>(a[k], b), p[k]);
      } else {
        if (q < n4) body(q, realign<M>(a[k], b));
      }
    }
  }
}

// Peels `dst` to 16 B alignment (scalar head via head_fn), then dispatches the
// vector walk on the source misalignment, then the scalar tail.
template <Hint H, int KU = kUnroll, bool kLd2 = false, typename HeadFn, typename VecFn>
__device__ __forceinline__ void run_unit(const float* src, const float* dst, int64_t len,
                                         HeadFn&& scalar_fn, VecFn&& vec_fn) {
  int64_t head = ((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) >> 2;
  if (head > len) head = len;
  if (threadIdx.x < head) scalar_fn(static_cast<int64_t>(threadIdx.x));
  const int64_t rest = len - head;
  const int64_t n4 = rest >> 2;
  if (n4 > 0) {
    const float* s = src + head;
    const int m = static_cast<int>((reinterpret_cast<uintptr_t>(s) & 15) >> 2);
    const float* floor = s - m;
    const int64_t qmax = (m + rest - 1) >> 2;
    switch (m) {
      case 0:
        warp_stream<0, H, KU, false, kLd2>(floor, n4, qmax, [&](int64_t q, float4 v) { vec_fn(head, q, v); });
        break;
      case 1:
        warp_stream<1, H, KU, false, kLd2>(floor, n4, qmax, [&](int64_t q, float4 v) { vec_fn(head, q, v); });
        break;
      case 2:
        warp_stream<2, H, KU, false, kLd2>(floor, n4, qmax, [&](int64_t q, float4 v) { vec_fn(head, q, v); });
        break;
      default:
        warp_stream<3, H, KU, false, kLd2>(floor, n4, qmax, [&](int64_t q, float4 v) { vec_fn(head, q, v); });
        break;
    }
  }
  for (int64_t i = head + n4 * 4 + threadIdx.x; i < len; i += kThreads) scalar_fn(i);
}

// run_unit with a second destination-aligned input stream `pre` (element i
// of `pre` pairs with dst[i]); vec_fn(head, q, v_src, v_pre).
template <Hint H, int KU = kUnroll, bool kLd2 = false, typename HeadFn, typename VecFn>
__device__ __forceinline__ void run_unit_pre(const float* src, const float* dst, const float* pre,
                                             int64_t len, HeadFn&& scalar_fn, VecFn&& vec_fn) {
  int64_t head = ((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) >> 2;
  if (head > len) head = len;
  if ((reinterpret_cast<uintptr_t>(pre + head) & 15) != 0) {
    // `pre` out of phase with the destination (not produced by the runtime's
    // layouts): per-lane scalar gathers of it inside the body.
    run_unit<H, KU, kLd2>(src, dst, len, scalar_fn, [&](int64_t h, int64_t q, float4 v) {
      const float* pp = pre + h + 4 * q;
      vec_fn(h, q, v, make_float4(pp[0], pp[1], pp[2], pp[3]));
    });
    return;
  }
  if (threadIdx.x < head) scalar_fn(static_cast<int64_t>(threadIdx.x));
  const int64_t rest = len - head;
  const int64_t n4 = rest >> 2;
  if (n4 > 0) {
    const float* s = src + head;
    const int m = static_cast<int>((reinterpret_cast<uintptr_t>(s) & 15) >> 2);
    const float* floor = s - m;
    const int64_t qmax = (m + rest - 1) >> 2;
    const float4* p4 = reinterpret_cast<const float4*>(pre + head);
    auto body = [&](int64_t q, float4 v, float4 w) { vec_fn(head, q, v, w); };
    switch (m) {
      case 0: warp_stream<0, H, KU, true, kLd2>(floor, n4, qmax, body, p4); break;
      case 1: warp_stream<1, H, KU, true, kLd2>(floor, n4, qmax, body, p4); break;
      case 2: warp_stream<2, H, KU, true, kLd2>(floor, n4, qmax, body, p4); break;
      default: warp_stream<3, H, KU, true, kLd2>(floor, n4, qmax, body, p4); break;
    }
  }
  for (int64_t i = head + n4 * 4 + threadIdx.x; i < len; i += kThreads) scalar_fn(i);
}

// Every CTA walks its equal slice of the op's elements across units. The
// first piece travels inside the Slice record (pointers already offset), so
// the common single-unit slice costs one descriptor load.
template <typename F>
__device__ __forceinline__ void walk_one(const Unit* __restrict__ units, const Slice& sl, F&& f) {
  if (sl.count <= 0) return;
  const int64_t n0 = min(sl.first.len, sl.count);
  f(sl.first, int64_t{0}, n0);
  int64_t left = sl.count - n0;
  for (int u = sl.unit + 1; left > 0; ++u) {
    const Unit U = units[u];
    const int64_t n = min(U.len, left);
    if (n > 0) f(U, int64_t{0}, n);
    left -= n;
  }
}

// A CTA's place in the grid of ONE rank's kernel: (blockIdx.x, gridDim.x) for
// a normal launch; in a same-device group launch (all ranks' CTAs in one
// cooperative grid) the index within its rank's share.
struct Blk {
  int id;
  int n;
};
__device__ __forceinline__ Blk this_blk() {
  return Blk{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x)};
}

// Each CTA walks slices b.id, b.id + b.n, ... of the op's n_slices equal
// slices (one slice per CTA at the full grid).
template <typename F>
__device__ __forceinline__ void walk_slice(const Unit* __restrict__ units,
                                           const Slice* __restrict__ slices, int n_slices,
                                           F&& f, Blk b = this_blk()) {
  for (int i = b.id; i < n_slices; i += b.n) walk_one(units, slices[i], f);
}

// --------------------------------------- programmatic dependent launch ----
// The local bucket kernels (pack / update / unpack / direct update) launch
// with programmatic stream serialization: each lets the next kernel of the
// stream start as its own CTAs retire (launch_dependents at entry), and waits
// (griddepcontrol.wait: the previous grid completed and its writes are
// visible) before touching memory — the next launch's ramp overlaps this
// one's tail. DEAR_PDL=0 launches them plainly.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------ comm-kernel phase trace ----
// Profiling aid (dear_set_comm_trace): the zero-copy reduce-scatter and
// all-gather CTAs record %globaltimer at entry, when every peer has arrived,
// and at exit, so an in-step trace separates waiting on other GPUs from
// moving data. Off (null) by default: one predicated load per CTA.
struct CommTraceRec {
  unsigned long long t0, t_arrived, t_end;
  uint32_t kind;   // 0 reduce-scatter, 1 all-gather
  uint32_t tag;    // low bits of the bucket's counter block (identifies the bucket)
  uint32_t epoch;  // the bucket's iteration count on this rank
  uint32_t cta;
};
__device__ CommTraceRec* g_comm_trace = nullptr;
__device__ uint32_t g_comm_trace_cap = 0;
__device__ uint32_t g_comm_trace_n = 0;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The two stamps live in shared memory (thread 0 only), not registers: the
// register-capped peer kernels must not spill for a profiling aid.
__device__ __forceinline__ unsigned long long* trace_slots() {
  __shared__ unsigned long long t[2];
  return t;
}
__device__ __forceinline__ void trace_stamp(int which) {
  if (threadIdx.x == 0 && g_comm_trace) trace_slots()[which] = gtimer();
}
__device__ __forceinline__ void trace_finish(uint32_t kind, const void* flags, uint32_t epoch,
                                             int cta) {
  if (threadIdx.x != 0 || !g_comm_trace) return;
  const uint32_t i = atomicAdd(&g_comm_trace_n, 1u);
  if (i >= g_comm_trace_cap) return;
  CommTraceRec r;
  r.t0 = trace_slots()[0];
  r.t_arrived = trace_slots()[1];
  r.t_end = gtimer();
  r.kind = kind;
  r.tag = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(flags) & 0xffffffffu);
  r.epoch = epoch;
  r.cta = static_cast<uint32_t>(cta);
  g_comm_trace[i] = r;
}

// ------------------------------------------------------ peer signalling ----
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__device__ __forceinline__ const T* at_peer(const T* p, int64_t delta) {
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(p) + delta);
}

// Last CTA of the launch bumps `counter` (release, system scope) once every
// CTA's writes are visible. Each CTA orders its writes before its `done`
// increment at GPU scope (peers read this GPU's memory through its L2); the
// last CTA, which observed every increment, then releases at system scope,
// which is cumulative over what it observed (PTX memory model), so one
// system-scope fence per launch suffices.
__device__ __forceinline__ void signal_done(uint32_t* done, uint32_t* counter,
                                            Blk b = this_blk()) {
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef DEAR_SIGNAL_SYS_FENCE_ALL
    __threadfence_system();
#else
    __threadfence();
#endif
    const uint32_t prev = atomicAdd(done, 1u);
    if (prev == static_cast<uint32_t>(b.n) - 1) {
      *done = 0;
      __threadfence_system();
      atomicAdd_system(counter, 1u);
    }
  }
}

__global__ void wait_peers_kernel(const uint32_t* mine, const uint32_t* watch, PeerArgs pa) {
  const uint32_t target = ld_acquire_sys(mine);
  const int k = threadIdx.x;
  if (k < pa.P && k != pa.rank) {
    const uint32_t* f = at_peer(watch, pa.delta[k]);
    const long long t0 = clock64();
    while (static_cast<int32_t>(ld_acquire_sys(f) - target) < 0) {
      __nanosleep(256);
      // A peer that never arrives fails loudly after pa.spin_limit cycles
      // (DEAR_PEER_TIMEOUT_S; 0 = wait forever, like NCCL).
      if (pa.spin_limit > 0 && clock64() - t0 > pa.spin_limit) __trap();
    }
  }
}

// In-kernel form of wait_peers_kernel: warp 0 of every CTA spins until each
// peer's `watch` counter reached our own `mine`, then the CTA proceeds (the
// acquire + CTA barrier order the CTA's later peer reads after the peers'
// released writes). Saves a dependent launch per stage on the comm stream.
__device__ __forceinline__ void cta_wait_peers(const uint32_t* mine, const uint32_t* watch,
                                               const PeerArgs& pa) {
  if (threadIdx.x < 32) {
    const uint32_t target = ld_acquire_sys(mine);
    const int k = threadIdx.x;
    if (k < pa.P && k != pa.rank) {
      const uint32_t* f = at_peer(watch, pa.delta[k]);
      const long long t0 = clock64();
      while (static_cast<int32_t>(ld_acquire_sys(f) - target) < 0) {
        __nanosleep(128);
        if (pa.spin_limit > 0 && clock64() - t0 > pa.spin_limit) __trap();
      }
    }
    __syncwarp();
#ifdef DEAR_WAIT_SYS_FENCE
    asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
  }
  __syncthreads();  // the acquires of warp 0 order the whole CTA's later reads
}

// ---------------------------------------------------------------- pack ----
// Peer backend (kSignal): one CTA per SM next to the GEMMs, so each lane keeps
// kPackPeerUnroll vectors in flight instead of relying on occupancy.
#ifndef DEAR_PACK_PEER_UNROLL
#define DEAR_PACK_PEER_UNROLL 16
#endif
constexpr int kPackPeerUnroll = DEAR_PACK_PEER_UNROLL;
// Push reduce-scatter pack: vectors per lane per round (posted NVLink stores);
// in-step BERT-L N = 4: 16 -> 8.92 ms, 4 -> 8.43, 1 -> 8.15 (pull: 7.47-7.60).
#ifndef DEAR_PUSH_UNROLL
#define DEAR_PUSH_UNROLL 1
#endif
#ifdef DEAR_PEER_PACK_FULL
constexpr bool kPeerPackLight = false;  // experiment: peer pack on the full grid
#else
constexpr bool kPeerPackLight = true;
#endif
#ifndef DEAR_PACK_UNROLL
#define DEAR_PACK_UNROLL kUnroll
#endif
#ifndef DEAR_UNPACK_UNROLL
#define DEAR_UNPACK_UNROLL kUnroll
#endif
// kPush (push reduce-scatter, DEAR_PUSH_RS): the destination is slot `rank`
// of the chunk owner's bucket buffer, U.b + pa.delta[U.peer] (posted stores
// over NVLink; the own chunk stays local).
template <bool kSignal, bool kPush = false>
__global__ void __launch_bounds__(kThreads, (kSignal && kPeerPackLight) ? 1 : DEAR_PACK_CTAS_PER_SM) pack_kernel(const Unit* __restrict__ units,
                                                           const Slice* __restrict__ slices,
                                                           float scale, BucketFlags* flags,
                                                           PeerArgs pa, int n_slices) {
  if (!kSignal) pdl_enter();
  // Peer backend: our slots may be rewritten once every peer gathered them.
  // Push: the owners' slots may be rewritten once every owner has reduced
  // (and so read) what we pushed last time.
  if (kSignal) cta_wait_peers(&flags->packed, kPush ? &flags->updated : &flags->gathered, pa);
  walk_slice(units, slices, n_slices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* src = U.a + off;
    float* dst = kPush ? const_cast<float*>(at_peer(U.b + off, pa.delta[U.peer])) : U.b + off;
    run_unit<Hint::kStream,
             kPush ? DEAR_PUSH_UNROLL
                   : ((kSignal && kPeerPackLight) ? kPackPeerUnroll : DEAR_PACK_UNROLL),
             kRealignLd2>(
        src, dst, n, [&](int64_t i) { dst[i] = __fmul_rn(src[i], scale); },
        [&](int64_t head, int64_t q, float4 v) {
          v.x = __fmul_rn(v.x, scale);
          v.y = __fmul_rn(v.y, scale);
          v.z = __fmul_rn(v.z, scale);
          v.w = __fmul_rn(v.w, scale);
          HBM_ST4(reinterpret_cast<float4*>(dst + head) + q, v);
        });
  });
  if (kPush) {
    // Remote stores: every CTA fences at system scope before it counts.
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
  if (kSignal) signal_done(&flags->done[0], &flags->packed);
}

// -------------------------------------------------------------- update ----
// torch.optim.SGD per element on the averaged gradient; with momentum = wd = 0
// it is exactly w - lr * (sum * 1/P) (collective.cpp:159-164, :190-192). Each
// operation is separately rounded (no FMA contraction), in the order of
// oracle/dear_oracle.c:or_sgd_step_f32.
template <bool kMom, bool kWd>
__device__ __forceinline__ float sgd_elem(float g, float w, float& m, const HyperParams& hp,
                                          bool has_buf) {
  float dp = hp.prescaled ? g : __fmul_rn(g, hp.inv_p);
  if (kWd) dp = __fadd_rn(dp, __fmul_rn(hp.weight_decay, w));
  if (kMom) {
    m = has_buf ? __fadd_rn(__fmul_rn(m, hp.momentum), __fmul_rn(hp.one_minus_dampening, dp))
                : dp;
    dp = hp.nesterov ? __fadd_rn(dp, __fmul_rn(hp.momentum, m)) : m;
  }
  return __fsub_rn(w, __fmul_rn(hp.lr, dp));
}

template <bool kMom, bool kWd>
__global__ void __launch_bounds__(kThreads, DEAR_UPD_CTAS_PER_SM) update_kernel(const Unit* __restrict__ units,
                                                             const Slice* __restrict__ slices,
                                                             const HyperParams* __restrict__ hpp,
                                                             int has_buf) {
  pdl_enter();
  const HyperParams hp = *hpp;
  walk_slice(units, slices, kUpdSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* w = U.a + off;
    float* g = U.b + off;
    float* mom = kMom ? static_cast<float*>(U.c) + off : nullptr;
    run_unit_pre<Hint::kKeep, kUnroll, kRealignLd2>(
        w, g, g, n,
        [&](int64_t i) {
          float m = kMom ? mom[i] : 0.f;
          g[i] = sgd_elem<kMom, kWd>(g[i], w[i], m, hp, has_buf);
          if (kMom) mom[i] = m;
        },
        [&](int64_t head, int64_t q, float4 wv, float4 gv) {
          float4* g4 = reinterpret_cast<float4*>(g + head);
          float4 mv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (kMom && has_buf) mv = reinterpret_cast<float4*>(mom + head)[q];
          gv.x = sgd_elem<kMom, kWd>(gv.x, wv.x, mv.x, hp, has_buf);
          gv.y = sgd_elem<kMom, kWd>(gv.y, wv.y, mv.y, hp, has_buf);
          gv.z = sgd_elem<kMom, kWd>(gv.z, wv.z, mv.z, hp, has_buf);
          gv.w = sgd_elem<kMom, kWd>(gv.w, wv.w, mv.w, hp, has_buf);
          g4[q] = gv;
          if (kMom) reinterpret_cast<float4*>(mom + head)[q] = mv;
        });
  });
}

// ------------------------------------------------------- direct (P = 1) ---
// One rank: the reduce-scatter and all-gather are the identity, so the
// parameters are updated straight from the gradients (and the bf16 copy
// refreshed) — 14 B per element. Same per-element operations as update_kernel
// (sum * 1/P with P = 1 is exact), so the result is bit-identical.
template <bool kWd, bool kShadow>
__global__ void __launch_bounds__(kThreads, DEAR_DIR_CTAS_PER_SM) update_direct_kernel(
    const Unit* __restrict__ units, const Slice* __restrict__ slices,
    const HyperParams* __restrict__ hpp) {
  pdl_enter();
  const HyperParams hp = *hpp;
  walk_slice(units, slices, kDirSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* g = U.a + off;
    float* w = U.b + off;
    __nv_bfloat16* sh = (kShadow && U.c) ? static_cast<__nv_bfloat16*>(U.c) + off : nullptr;
    run_unit_pre<Hint::kStream, kUnroll, kRealignLd2>(
        g, w, w, n,
        [&](int64_t i) {
          float m = 0.f;
          const float v = sgd_elem<false, kWd>(g[i], w[i], m, hp, false);
          w[i] = v;
          if (kShadow && sh) sh[i] = __float2bfloat16_rn(v);
        },
        [&](int64_t head, int64_t q, float4 gv, float4 v) {
          float4* w4 = reinterpret_cast<float4*>(w + head);
          float m = 0.f;
          v.x = sgd_elem<false, kWd>(gv.x, v.x, m, hp, false);
          v.y = sgd_elem<false, kWd>(gv.y, v.y, m, hp, false);
          v.z = sgd_elem<false, kWd>(gv.z, v.z, m, hp, false);
          v.w = sgd_elem<false, kWd>(gv.w, v.w, m, hp, false);
          w4[q] = v;
          if (kShadow && sh) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
            uint2 packed;
            packed.x = *reinterpret_cast<uint32_t*>(&lo);
            packed.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(sh + head)[q] = packed;
          }
        });
  });
}

// -------------------------------------------------------------- unpack ----
template <bool kShadow>
__global__ void __launch_bounds__(kThreads, DEAR_UNPACK_CTAS_PER_SM) unpack_kernel(const Unit* __restrict__ units,
                                                             const Slice* __restrict__ slices) {
  pdl_enter();
  walk_slice(units, slices, kUnpackSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* src = U.a + off;
    float* dst = U.b + off;
    __nv_bfloat16* sh = (kShadow && U.c) ? static_cast<__nv_bfloat16*>(U.c) + off : nullptr;
    run_unit<Hint::kStream, DEAR_UNPACK_UNROLL, kRealignLd2>(
        src, dst, n,
        [&](int64_t i) {
          const float v = src[i];
          dst[i] = v;
          if (kShadow && sh) sh[i] = __float2bfloat16_rn(v);
        },
        [&](int64_t head, int64_t q, float4 v) {
          HBM_ST4(reinterpret_cast<float4*>(dst + head) + q, v);
          if (kShadow && sh) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
            uint2 packed;
            packed.x = *reinterpret_cast<uint32_t*>(&lo);
            packed.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(sh + head)[q] = packed;
          }
        });
  });
}

// ------------------------------------------- fused peer RS+update --------
// Peer reduce-scatter streaming for a compile-time world size: per round each
// lane issues its KU parameter loads (realigned to the slot like warp_stream)
// and all KU x P slot loads from the P ranks' buffers before using any, so
// the NVLink round trips overlap (a runtime-P loop issues them one by one:
// the compiler cannot move a peer load above the previous vector's store).
// pg[j] is the slot vector base on rank (rank+1+j) % P: ring order.
template <int M, int P, int KU, typename Body>
__device__ __forceinline__ void warp_stream_rs(const float* w_floor, const float4* const* pg,
                                               int64_t n4, int64_t qmax, Body&& body) {
  const float4* s4 = reinterpret_cast<const float4*>(w_floor);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kThreads / 32;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = static_cast<int64_t>(warp) * 32 * KU; base < n4;
       base += static_cast<int64_t>(kWarps) * 32 * KU) {
    float4 a[KU];
    float4 v[KU][P];
#pragma unroll
    for (int k = 0; k < KU; ++k) {
      const int64_t q = base + k * 32 + lane;
      a[k] = q <= qmax ? __ldg(s4 + q) : zero;
#pragma unroll
      for (int j = 0; j < P; ++j) v[k][j] = q < n4 ? __ldcg(pg[j] + q) : zero;
    }
    float4 extra = zero;
    if constexpr (M != 0) {
      const int64_t qx = base + KU * 32;
      if (lane == 31 && qx <= qmax) extra = __ldg(s4 + qx);
    }
#pragma unroll
    for (int k = 0; k < KU; ++k) {
      const int64_t q = base + k * 32 + lane;
      float4 b = a[k];
      if constexpr (M != 0) {
        b = shfl_down4(a[k]);
        float4 nxt = extra;
        if (k + 1 < KU) {
          nxt.x = __shfl_sync(0xffffffffu, a[k + 1 < KU ? k + 1 : k].x, 0);
          nxt.y = __shfl_sync(0xffffffffu, a[k + 1 < KU ? k + 1 : k].y, 0);
          nxt.z = __shfl_sync(0xffffffffu, a[k + 1 < KU ? k + 1 : k].z, 0);
          nxt.w = __shfl_sync(0xffffffffu, a[k + 1 < KU ? k + 1 : k].w, 0);
        }
        if (lane == 31) b = nxt;
      }
      float4 acc = v[k][0];
#pragma unroll
      for (int j = 1; j < P; ++j) {
        acc.x = __fadd_rn(acc.x, v[k][j].x);
        acc.y = __fadd_rn(acc.y, v[k][j].y);
        acc.z = __fadd_rn(acc.z, v[k][j].z);
        acc.w = __fadd_rn(acc.w, v[k][j].w);
      }
      if (q < n4) body(q, realign<M>(a[k], b), acc);
    }
  }
}

// Ring-order sum (collective.cpp:70-90): chunk (rank+1)%P starts on rank
// rank+1 and picks up rank+2, ..., rank — the same fold as the local-group
// kernel, so the result is bit-exact with the fp32 restatement.
// One CTA per SM at most (kPeerSlices CTAs): registers for the in-flight
// peer loads instead of occupancy.
template <int PC, bool kMom, bool kWd>
__device__ __forceinline__ void rs_update_peer_body(const Unit* __restrict__ units,
                                                    const Slice* __restrict__ slices,
                                                    const HyperParams* __restrict__ hpp,
                                                    int has_buf, const PeerArgs& pa,
                                                    BucketFlags* flags, Blk blk) {
  cta_wait_peers(&flags->packed, &flags->packed, pa);  // every rank packed this bucket
  const HyperParams hp = *hpp;
  const int k0 = (pa.rank + 1) % pa.P;
  walk_slice(units, slices, kPeerSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* w = U.a + off;
    float* g = U.b + off;
    float* mom = kMom ? static_cast<float*>(U.c) + off : nullptr;
    auto sum1 = [&](const float* p) {
      int k = k0;
      float acc = __ldcg(at_peer(p, pa.delta[k]));
      for (int j = 1; j < pa.P; ++j) {
        k = k + 1 == pa.P ? 0 : k + 1;
        acc = __fadd_rn(acc, __ldcg(at_peer(p, pa.delta[k])));
      }
      return acc;
    };
    auto scalar = [&](int64_t i) {
      float m = kMom ? mom[i] : 0.f;
      g[i] = sgd_elem<kMom, kWd>(sum1(g + i), w[i], m, hp, has_buf);
      if (kMom) mom[i] = m;
    };
    if constexpr (PC > 0) {
      // Compile-time P: all peer loads of a round in flight (warp_stream_rs).
      constexpr int KU = PC <= 4 ? 4 : 2;
      int64_t head = ((16 - (reinterpret_cast<uintptr_t>(g) & 15)) & 15) >> 2;
      if (head > n) head = n;
      if (threadIdx.x < head) scalar(static_cast<int64_t>(threadIdx.x));
      const int64_t rest = n - head;
      const int64_t n4 = rest >> 2;
      if (n4 > 0) {
        const float4* pg[PC];
#pragma unroll
        for (int j = 0; j < PC; ++j) {
          const int r = (k0 + j) % PC;
          pg[j] = at_peer(reinterpret_cast<const float4*>(g + head), pa.delta[r]);
        }
        const float* ws = w + head;
        const int m = static_cast<int>((reinterpret_cast<uintptr_t>(ws) & 15) >> 2);
        const int64_t qmax = (m + rest - 1) >> 2;
        float4* g4 = reinterpret_cast<float4*>(g + head);
        float4* m4 = kMom ? reinterpret_cast<float4*>(mom + head) : nullptr;
        auto body = [&](int64_t q, float4 wv, float4 acc) {
          float4 mv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (kMom && has_buf) mv = m4[q];
          acc.x = sgd_elem<kMom, kWd>(acc.x, wv.x, mv.x, hp, has_buf);
          acc.y = sgd_elem<kMom, kWd>(acc.y, wv.y, mv.y, hp, has_buf);
          acc.z = sgd_elem<kMom, kWd>(acc.z, wv.z, mv.z, hp, has_buf);
          acc.w = sgd_elem<kMom, kWd>(acc.w, wv.w, mv.w, hp, has_buf);
          g4[q] = acc;
          if (kMom) m4[q] = mv;
        };
        switch (m) {
          case 0: warp_stream_rs<0, PC, KU>(ws - m, pg, n4, qmax, body); break;
          case 1: warp_stream_rs<1, PC, KU>(ws - m, pg, n4, qmax, body); break;
          case 2: warp_stream_rs<2, PC, KU>(ws - m, pg, n4, qmax, body); break;
          default: warp_stream_rs<3, PC, KU>(ws - m, pg, n4, qmax, body); break;
        }
      }
      for (int64_t i = head + n4 * 4 + threadIdx.x; i < n; i += kThreads) scalar(i);
      return;
    }
    run_unit<Hint::kKeep>(
        w, g, n,
        [&](int64_t i) {
          float m = kMom ? mom[i] : 0.f;
          g[i] = sgd_elem<kMom, kWd>(sum1(g + i), w[i], m, hp, has_buf);
          if (kMom) mom[i] = m;
        },
        [&](int64_t head, int64_t q, float4 wv) {
          const float4* g4 = reinterpret_cast<const float4*>(g + head) + q;
          int k = k0;
          float4 acc = __ldcg(at_peer(g4, pa.delta[k]));
          for (int j = 1; j < pa.P; ++j) {
            k = k + 1 == pa.P ? 0 : k + 1;
            const float4 v = __ldcg(at_peer(g4, pa.delta[k]));
            acc.x = __fadd_rn(acc.x, v.x);
            acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z);
            acc.w = __fadd_rn(acc.w, v.w);
          }
          float4 mv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (kMom && has_buf) mv = reinterpret_cast<float4*>(mom + head)[q];
          acc.x = sgd_elem<kMom, kWd>(acc.x, wv.x, mv.x, hp, has_buf);
          acc.y = sgd_elem<kMom, kWd>(acc.y, wv.y, mv.y, hp, has_buf);
          acc.z = sgd_elem<kMom, kWd>(acc.z, wv.z, mv.z, hp, has_buf);
          acc.w = sgd_elem<kMom, kWd>(acc.w, wv.w, mv.w, hp, has_buf);
          reinterpret_cast<float4*>(g + head)[q] = acc;
          if (kMom) reinterpret_cast<float4*>(mom + head)[q] = mv;
        });
  }, blk);
  signal_done(&flags->done[1], &flags->updated, blk);
}

template <int PC, bool kMom, bool kWd>
__global__ void __launch_bounds__(kThreads, 1)
    rs_update_peer_kernel(const Unit* __restrict__ units, const Slice* __restrict__ slices,
                          const HyperParams* __restrict__ hpp, int has_buf, PeerArgs pa,
                          BucketFlags* flags) {
  rs_update_peer_body<PC, kMom, kWd>(units, slices, hpp, has_buf, pa, flags, this_blk());
}

// ------------------------------------- zero-copy peer RS+update ----------
// The gradients and parameters themselves are IPC-mapped (one allocation
// each per rank, identical relative layout): no pack, no bucket buffer. The
// owner of chunk (rank+1)%P reads that chunk of every rank's GRADIENTS over
// NVLink, sums in the ring order of collective.cpp:70-90, applies 1/P and
// the SGD update (sgd_elem, same operation sequence as update_kernel with
// prescaled = 0) and writes w' straight into its own parameters and their
// bf16 copy. Peers then gather the owner's parameters (ag_unpack_peer_kernel
// with parameter deltas). Per element this moves 4 B of local gradient reads
// served to the ring + 10/P B of update traffic, where pack + slot RS moved
// 8 + 4 + 8/P.
//
// Cross-GPU protocol on the arena's per-bucket counters (graph-safe, no host
// epoch): the first CTA announces "my gradients of this bucket are complete"
// (packed += 1, release, system scope; the comm stream already waited on the
// producing streams' events); every CTA then waits until each peer's
// `packed` reached our `updated` + 1 — `updated` only moves when this kernel's
// last CTA finishes, after every CTA passed its wait, so it is this
// iteration's epoch on every rank.
__device__ __forceinline__ void cta_announce_and_wait(BucketFlags* flags, const PeerArgs& pa,
                                                      Blk b, bool announce = true) {
  if (threadIdx.x < 32) {
    if (announce && b.id == 0 && threadIdx.x == 0) {
      __threadfence_system();
      atomicAdd_system(&flags->packed, 1u);
    }
    const uint32_t target = ld_acquire_sys(&flags->updated) + 1u;
    const int k = threadIdx.x;
    if (k < pa.P && k != pa.rank) {
      const uint32_t* f = at_peer(&flags->packed, pa.delta[k]);
      const long long t0 = clock64();
      while (static_cast<int32_t>(ld_acquire_sys(f) - target) < 0) {
        __nanosleep(128);
        if (pa.spin_limit > 0 && clock64() - t0 > pa.spin_limit) __trap();
      }
    }
    __syncwarp();
  }
  __syncthreads();
}

__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* sh, int64_t q, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 packed;
  packed.x = *reinterpret_cast<uint32_t*>(&lo);
  packed.y = *reinterpret_cast<uint32_t*>(&hi);
#ifndef DEAR_ZC_NO_EVICT
  __stcs(reinterpret_cast<uint2*>(sh) + q, packed);
#else
  reinterpret_cast<uint2*>(sh)[q] = packed;
#endif
}

// Units: a = gradient (local address; rank k's copy at a + ga.delta[k]),
// b = parameter (in/out), c = bf16 copy or null. Momentum shard element i of
// the op lives at mom_base[i] (the op's elements are the owned chunk in
// order, so Unit::start + offset is the chunk position). Parameters and
// gradients share their 16 B phase (registration requires 16 B alignment),
// so after a scalar head every stream is float4-aligned.
// Vectors per lane per round (each with P gradient loads in flight). One:
// throttled for the same reason as DEAR_PEER_UNROLL — in the step, the
// reduce-scatter's NVLink / L2 pressure slows the concurrent backprop GEMMs
// more than a faster reduce-scatter saves. Measured in-step (comm_trace,
// profiles/r02v2_comm_throttle.log): BERT-L N = 4 8.95 -> 7.58 ms (KU 2 -> 1
// with unroll 4), N = 2 8.27 -> 7.46 ms (KU 4 -> 1).
#ifndef DEAR_ZC_KU2
#define DEAR_ZC_KU2 1
#endif
#ifndef DEAR_ZC_KU4
#define DEAR_ZC_KU4 1
#endif
#ifndef DEAR_ZC_KU8
#define DEAR_ZC_KU8 1
#endif
// Evict-first hints on every zero-copy stream so the comm traffic does not
// push the backprop GEMMs' operands out of L2 (in-step BERT-L, P = 4: 7.48 ->
// 7.33 ms, tools/micro/var_sweep2.sh); DEAR_ZC_NO_EVICT restores plain accesses.
#ifndef DEAR_ZC_NO_EVICT
#define ZC_LDR(p) __ldcs(p)
#define ZC_LDW(p) __ldcs(p)
#define ZC_ST(p, v) __stcs(p, v)
#else
#define ZC_LDR(p) __ldcg(p)
#define ZC_LDW(p) (*(p))
#define ZC_ST(p, v) (*(p) = (v))
#endif
template <int PC, bool kMom, bool kWd, bool kShadow>
__device__ __forceinline__ void rs_update_zc_body(const Unit* __restrict__ units,
                                                  const Slice* __restrict__ slices,
                                                  const HyperParams* __restrict__ hpp, int has_buf,
                                                  float* mom_base, const PeerArgs& pa,
                                                  const PeerArgs& ga, BucketFlags* flags, Blk blk,
                                                  bool announce = true) {
  trace_stamp(0);
  const uint32_t epoch = g_comm_trace ? *reinterpret_cast<volatile uint32_t*>(&flags->updated) : 0u;
  cta_announce_and_wait(flags, pa, blk, announce);
  trace_stamp(1);
  const HyperParams hp = *hpp;
  const int P = PC > 0 ? PC : pa.P;
  const int k0 = (pa.rank + 1) % P;
  walk_slice(units, slices, kZcSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* g = U.a + off;
    float* w = U.b + off;
    float* mom = kMom ? mom_base + U.start + off : nullptr;
    __nv_bfloat16* sh = (kShadow && U.c) ? static_cast<__nv_bfloat16*>(U.c) + off : nullptr;
    auto scalar = [&](int64_t i) {
      int k = k0;
      float acc = __ldcg(at_peer(g + i, ga.delta[k]));
      for (int j = 1; j < P; ++j) {
        k = k + 1 == P ? 0 : k + 1;
        acc = __fadd_rn(acc, __ldcg(at_peer(g + i, ga.delta[k])));
      }
      float m = kMom ? mom[i] : 0.f;
      const float v = sgd_elem<kMom, kWd>(acc, w[i], m, hp, has_buf);
      w[i] = v;
      if (kMom) mom[i] = m;
      if (kShadow && sh) sh[i] = __float2bfloat16_rn(v);
    };
    int64_t head = ((16 - (reinterpret_cast<uintptr_t>(w) & 15)) & 15) >> 2;
    if (head > n) head = n;
    if (threadIdx.x < head) scalar(static_cast<int64_t>(threadIdx.x));
    const int64_t n4 = (n - head) >> 2;
    if constexpr (PC > 0) {
      constexpr int KU = PC <= 2 ? DEAR_ZC_KU2 : (PC <= 4 ? DEAR_ZC_KU4 : DEAR_ZC_KU8);
      const float4* pg[PC];
#pragma unroll
      for (int j = 0; j < PC; ++j)
        pg[j] = at_peer(reinterpret_cast<const float4*>(g + head), ga.delta[(k0 + j) % PC]);
      float4* w4 = reinterpret_cast<float4*>(w + head);
      // The momentum shard is indexed by chunk position, which need not share
      // the parameters' 16 B phase: scalar (still coalesced) access then.
      float* mh = kMom ? mom + head : nullptr;
      const bool mvec = kMom && (reinterpret_cast<uintptr_t>(mh) & 15) == 0;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      constexpr int kWarps = kThreads / 32;
      const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t base = static_cast<int64_t>(warp) * 32 * KU; base < n4;
           base += static_cast<int64_t>(kWarps) * 32 * KU) {
        float4 wv[KU];
        float4 v[KU][PC];
#pragma unroll
        for (int k = 0; k < KU; ++k) {
          const int64_t q = base + k * 32 + lane;
          wv[k] = q < n4 ? ZC_LDW(w4 + q) : zero;
#pragma unroll
          for (int j = 0; j < PC; ++j) v[k][j] = q < n4 ? ZC_LDR(pg[j] + q) : zero;
        }
#pragma unroll
        for (int k = 0; k < KU; ++k) {
          const int64_t q = base + k * 32 + lane;
          if (q >= n4) continue;
          float4 acc = v[k][0];
#pragma unroll
          for (int j = 1; j < PC; ++j) {
            acc.x = __fadd_rn(acc.x, v[k][j].x);
            acc.y = __fadd_rn(acc.y, v[k][j].y);
            acc.z = __fadd_rn(acc.z, v[k][j].z);
            acc.w = __fadd_rn(acc.w, v[k][j].w);
          }
          float4 mv = zero;
          if (kMom && has_buf) {
            if (mvec) {
              mv = reinterpret_cast<const float4*>(mh)[q];
            } else {
              mv = make_float4(mh[4 * q], mh[4 * q + 1], mh[4 * q + 2], mh[4 * q + 3]);
            }
          }
          float4 o;
          o.x = sgd_elem<kMom, kWd>(acc.x, wv[k].x, mv.x, hp, has_buf);
          o.y = sgd_elem<kMom, kWd>(acc.y, wv[k].y, mv.y, hp, has_buf);
          o.z = sgd_elem<kMom, kWd>(acc.z, wv[k].z, mv.z, hp, has_buf);
          o.w = sgd_elem<kMom, kWd>(acc.w, wv[k].w, mv.w, hp, has_buf);
          ZC_ST(w4 + q, o);
          if (kMom) {
            if (mvec) {
              reinterpret_cast<float4*>(mh)[q] = mv;
            } else {
              mh[4 * q] = mv.x;
              mh[4 * q + 1] = mv.y;
              mh[4 * q + 2] = mv.z;
              mh[4 * q + 3] = mv.w;
            }
          }
          if (kShadow && sh) store_bf16x4(sh + head, q, o);
        }
      }
    } else {
      for (int64_t q = threadIdx.x; q < n4; q += kThreads)
        for (int e = 0; e < 4; ++e) scalar(head + 4 * q + e);
    }
    for (int64_t i = head + n4 * 4 + threadIdx.x; i < n; i += kThreads) scalar(i);
  }, blk);
  trace_finish(0, flags, epoch, blk.id);
  signal_done(&flags->done[1], &flags->updated, blk);
}

template <int PC, bool kMom, bool kWd, bool kShadow>
__global__ void DEAR_ZC_BOUNDS
    rs_update_zc_kernel(const Unit* __restrict__ units, const Slice* __restrict__ slices,
                        const HyperParams* __restrict__ hpp, int has_buf, float* mom_base,
                        PeerArgs pa, PeerArgs ga, BucketFlags* flags, int announce) {
  rs_update_zc_body<PC, kMom, kWd, kShadow>(units, slices, hpp, has_buf, mom_base, pa, ga, flags,
                                            this_blk(), announce != 0);
}

// ------------------------------------------- fused peer AG+unpack ---------
// Source element of a unit: U.a + off on rank U.peer, i.e. at sa.delta[U.peer]
// (sa = arena deltas for bucket slots, parameter deltas for zero-copy).
template <bool kShadow>
__device__ __forceinline__ void ag_unpack_peer_body(const Unit* __restrict__ units,
                                                    const Slice* __restrict__ slices,
                                                    const PeerArgs& pa, const PeerArgs& sa,
                                                    BucketFlags* flags, int n_slices, Blk blk) {
  trace_stamp(0);
  const uint32_t epoch = g_comm_trace ? *reinterpret_cast<volatile uint32_t*>(&flags->updated) : 0u;
  cta_wait_peers(&flags->updated, &flags->updated, pa);  // every owner updated its shard
  trace_stamp(1);
  walk_slice(units, slices, n_slices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* src = at_peer(U.a + off, sa.delta[U.peer]);
    float* dst = U.b + off;
    __nv_bfloat16* sh = (kShadow && U.c) ? static_cast<__nv_bfloat16*>(U.c) + off : nullptr;
    run_unit<Hint::kStream, kPeerUnroll>(
        src, dst, n,
        [&](int64_t i) {
          const float v = src[i];
          dst[i] = v;
          if (kShadow && sh) sh[i] = __float2bfloat16_rn(v);
        },
        [&](int64_t head, int64_t q, float4 v) {
          ZC_ST(reinterpret_cast<float4*>(dst + head) + q, v);
          if (kShadow && sh) store_bf16x4(sh + head, q, v);
        });
  }, blk);
  trace_finish(1, flags, epoch, blk.id);
  signal_done(&flags->done[2], &flags->gathered, blk);
}

template <bool kShadow>
__global__ void DEAR_ZC_BOUNDS
    ag_unpack_peer_kernel(const Unit* __restrict__ units, const Slice* __restrict__ slices,
                          PeerArgs pa, PeerArgs sa, BucketFlags* flags, int n_slices) {
  ag_unpack_peer_body<kShadow>(units, slices, pa, sa, flags, n_slices, this_blk());
}

// ------------------------------------------------ NVLS (multimem) --------
// NVLink SHARP: the gradients, parameters and bf16 copies live in a symmetric
// heap bound to one multicast object (nvls.cpp); address p + mc_delta is the
// multicast alias of local address p. multimem.ld_reduce makes the NVSwitch
// fetch the element from every rank and return the sum (LDGMC in SASS), and a
// store to a multicast address is replicated to every rank, so the owner of a
// chunk reduces it with ONE load per element and broadcasts its update with
// ONE posted store: the switch, not the SMs, does the P-way reduction and the
// fan-out. The switch's summation order is unspecified (exact at P = 2, where
// a + b = b + a; within 1e-5 of the fp64 oracle otherwise, like NCCL).
//
// Cross-rank protocol, all on per-bucket counters in the heap (NvlsFlags),
// bumped on EVERY rank at once by multimem.red and polled locally — no
// NVLink round trip in any spin: packed / updated / gathered grow by P per
// iteration; `epoch` is the local arena's flags->updated (this rank's RS
// count for the bucket).
__device__ __forceinline__ float4 mc_ld_reduce4(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float mc_ld_reduce1(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st4(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_st1(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// 4 bf16 (8 B) to a multicast address.
__device__ __forceinline__ void mc_st_bf16x4(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
  __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
  asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1,%2};" ::"l"(p),
               "f"(__uint_as_float(*reinterpret_cast<uint32_t*>(&lo))),
               "f"(__uint_as_float(*reinterpret_cast<uint32_t*>(&hi)))
               : "memory");
}
// One bf16: a plain strong store to the multicast alias is replicated too.
__device__ __forceinline__ void mc_st_bf16(__nv_bfloat16* p, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  asm volatile("st.relaxed.sys.global.b16 [%0], %1;" ::"l"(p),
               "h"(*reinterpret_cast<const unsigned short*>(&h))
               : "memory");
}
__device__ __forceinline__ void mc_red_add(uint32_t* p, uint32_t v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <typename T>
__device__ __forceinline__ T* mc(T* p, int64_t d) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + d);
}
template <typename T>
__device__ __forceinline__ const T* mc(const T* p, int64_t d) {
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(p) + d);
}

// Spin (one thread) until the local copy of a multicast counter reaches target.
__device__ __forceinline__ void spin_local(const uint32_t* f, uint32_t target,
                                           long long spin_limit) {
  const long long t0 = clock64();
  while (static_cast<int32_t>(ld_acquire_sys(f) - target) < 0) {
    __nanosleep(64);
    if (spin_limit > 0 && clock64() - t0 > spin_limit) __trap();
  }
}

// Last-CTA completion for the NVLS kernels: every CTA orders its (multicast)
// stores at system scope before counting itself done; the last one bumps the
// rank-local epoch (if any) and the multicast counter on every rank.
__device__ __forceinline__ bool nvls_signal(uint32_t* done, uint32_t* local_epoch,
                                            uint32_t* mc_counter) {
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) {
      *done = 0;
      if (local_epoch) *local_epoch += 1;
      __threadfence_system();
      mc_red_add(mc_counter, 1u);
    }
  }
  __syncthreads();
  return last;
}

#ifndef DEAR_NVLS_KU
#define DEAR_NVLS_KU 4
#endif

// Reduce-scatter + SGD update of the owned chunk (units: a = gradient, b =
// parameter, c = bf16 copy, all local heap addresses). The bf16 copy is NOT
// written here: the all-gather's multicast store refreshes it on every rank,
// the owner included.
template <bool kMom, bool kWd>
__global__ void DEAR_ZC_BOUNDS
    rs_update_nvls_kernel(const Unit* __restrict__ units, const Slice* __restrict__ slices,
                          const HyperParams* __restrict__ hpp, int has_buf, float* mom_base,
                          int64_t mc_delta, BucketFlags* flags, NvlsFlags* ucf, NvlsFlags* mcf,
                          int P, long long spin_limit) {
  if (threadIdx.x == 0) {
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(&flags->updated);
    if (blockIdx.x == 0) {
      // This rank's gradients of the bucket are complete (the comm stream
      // waited on the producers' events): announce it on every rank.
      __threadfence_system();
      mc_red_add(&mcf->packed, 1u);
    }
    spin_local(&ucf->packed, static_cast<uint32_t>(P) * (epoch + 1u), spin_limit);
  }
  __syncthreads();
  const HyperParams hp = *hpp;
  walk_slice(units, slices, kZcSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* g = U.a + off;
    float* w = U.b + off;
    float* mom = kMom ? mom_base + U.start + off : nullptr;
    auto scalar = [&](int64_t i) {
      const float acc = mc_ld_reduce1(mc(g + i, mc_delta));
      float m = kMom ? mom[i] : 0.f;
      w[i] = sgd_elem<kMom, kWd>(acc, w[i], m, hp, has_buf);
      if (kMom) mom[i] = m;
    };
    int64_t head = ((16 - (reinterpret_cast<uintptr_t>(w) & 15)) & 15) >> 2;
    if (head > n) head = n;
    if (threadIdx.x < head) scalar(static_cast<int64_t>(threadIdx.x));
    const int64_t n4 = (n - head) >> 2;
    const float4* gm4 = reinterpret_cast<const float4*>(mc(g + head, mc_delta));
    float4* w4 = reinterpret_cast<float4*>(w + head);
    float* mh = kMom ? mom + head : nullptr;
    const bool mvec = kMom && (reinterpret_cast<uintptr_t>(mh) & 15) == 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int KU = DEAR_NVLS_KU, kWarps = kThreads / 32;
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = static_cast<int64_t>(warp) * 32 * KU; base < n4;
         base += static_cast<int64_t>(kWarps) * 32 * KU) {
      float4 acc[KU], wv[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int64_t q = base + k * 32 + lane;
        acc[k] = q < n4 ? mc_ld_reduce4(reinterpret_cast<const float*>(gm4 + q)) : zero;
        wv[k] = q < n4 ? w4[q] : zero;
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int64_t q = base + k * 32 + lane;
        if (q >= n4) continue;
        float4 mv = zero;
        if (kMom && has_buf)
          mv = mvec ? reinterpret_cast<const float4*>(mh)[q]
                    : make_float4(mh[4 * q], mh[4 * q + 1], mh[4 * q + 2], mh[4 * q + 3]);
        float4 o;
        o.x = sgd_elem<kMom, kWd>(acc[k].x, wv[k].x, mv.x, hp, has_buf);
        o.y = sgd_elem<kMom, kWd>(acc[k].y, wv[k].y, mv.y, hp, has_buf);
        o.z = sgd_elem<kMom, kWd>(acc[k].z, wv[k].z, mv.z, hp, has_buf);
        o.w = sgd_elem<kMom, kWd>(acc[k].w, wv[k].w, mv.w, hp, has_buf);
        w4[q] = o;
        if (kMom) {
          if (mvec) {
            reinterpret_cast<float4*>(mh)[q] = mv;
          } else {
            mh[4 * q] = mv.x;
            mh[4 * q + 1] = mv.y;
            mh[4 * q + 2] = mv.z;
            mh[4 * q + 3] = mv.w;
          }
        }
      }
    }
    for (int64_t i = head + n4 * 4 + threadIdx.x; i < n; i += kThreads) scalar(i);
  });
  nvls_signal(&flags->done[1], &flags->updated, &mcf->updated);
}

// All-gather: the owner broadcasts its updated chunk (and its bf16 copy) with
// multicast stores into every rank's parameters; the last CTA then signals
// and waits until every owner's broadcast of this bucket has landed here.
template <bool kShadow>
__global__ void DEAR_ZC_BOUNDS ag_nvls_kernel(const Unit* __restrict__ units,
                                              const Slice* __restrict__ slices, int64_t mc_delta,
                                              BucketFlags* flags, NvlsFlags* ucf, NvlsFlags* mcf,
                                              int P, long long spin_limit) {
  walk_slice(units, slices, kZcSlices, [&](const Unit& U, int64_t off, int64_t n) {
    const float* w = U.b + off;
    float* wm = mc(U.b + off, mc_delta);
    __nv_bfloat16* shm =
        (kShadow && U.c) ? mc(static_cast<__nv_bfloat16*>(U.c) + off, mc_delta) : nullptr;
    auto scalar = [&](int64_t i) {
      const float v = w[i];
      mc_st1(wm + i, v);
      if (kShadow && shm) mc_st_bf16(shm + i, v);
    };
    int64_t head = ((16 - (reinterpret_cast<uintptr_t>(w) & 15)) & 15) >> 2;
    if (head > n) head = n;
    if (threadIdx.x < head) scalar(static_cast<int64_t>(threadIdx.x));
    const int64_t n4 = (n - head) >> 2;
    const float4* w4 = reinterpret_cast<const float4*>(w + head);
    constexpr int KU = DEAR_NVLS_KU;
    for (int64_t q0 = threadIdx.x; q0 < n4; q0 += static_cast<int64_t>(kThreads) * KU) {
      float4 v[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int64_t q = q0 + static_cast<int64_t>(k) * kThreads;
        if (q < n4) v[k] = __ldcs(w4 + q);
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int64_t q = q0 + static_cast<int64_t>(k) * kThreads;
        if (q < n4) {
          mc_st4(wm + head + 4 * q, v[k]);
          if (kShadow && shm) mc_st_bf16x4(shm + head + 4 * q, v[k]);
        }
      }
    }
    for (int64_t i = head + n4 * 4 + threadIdx.x; i < n; i += kThreads) scalar(i);
  });
  if (nvls_signal(&flags->done[2], nullptr, &mcf->gathered) && threadIdx.x == 0) {
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(&flags->updated);
    spin_local(&ucf->gathered, static_cast<uint32_t>(P) * epoch, spin_limit);
    __threadfence_system();
  }
}

// dear_step's "gradients consumed" fence on NVLS: every owner's reduce-scatter
// of the last bucket (hence of all, stream order) has read our gradients.
__global__ void nvls_wait_updated_kernel(const uint32_t* epoch, const NvlsFlags* ucf, int P,
                                         long long spin_limit) {
  if (threadIdx.x == 0)
    spin_local(&ucf->updated, static_cast<uint32_t>(P) * *reinterpret_cast<const volatile uint32_t*>(epoch),
               spin_limit);
}

// ------------------------------------- same-device group launches ---------
// All P ranks' CTAs of one peer kernel in ONE cooperative grid (rank =
// blockIdx.x / nb): the cross-rank counter waits inside are then between
// CTAs that are guaranteed co-resident, never between separate launches.
template <int PC, bool kMom, bool kWd, bool kShadow>
__global__ void DEAR_ZC_BOUNDS group_rs_zc_kernel(const GroupOp* __restrict__ ops, int nb,
                                                  int has_buf) {
  const GroupOp& o = ops[blockIdx.x / nb];
  rs_update_zc_body<PC, kMom, kWd, kShadow>(o.units, o.slices, o.hp, has_buf, o.mom, o.pa, o.sa,
                                            o.flags, Blk{static_cast<int>(blockIdx.x) % nb, nb});
}

template <int PC, bool kMom, bool kWd>
__global__ void __launch_bounds__(kThreads, 1) group_rs_peer_kernel(const GroupOp* __restrict__ ops,
                                                                    int nb, int has_buf) {
  const GroupOp& o = ops[blockIdx.x / nb];
  rs_update_peer_body<PC, kMom, kWd>(o.units, o.slices, o.hp, has_buf, o.pa, o.flags,
                                     Blk{static_cast<int>(blockIdx.x) % nb, nb});
}

template <bool kShadow>
__global__ void DEAR_ZC_BOUNDS group_ag_kernel(const GroupOp* __restrict__ ops, int nb) {
  const GroupOp& o = ops[blockIdx.x / nb];
  ag_unpack_peer_body<kShadow>(o.units, o.slices, o.pa, o.sa, o.flags, o.n_slices,
                               Blk{static_cast<int>(blockIdx.x) % nb, nb});
}

// ---------------------------------------------------- local collectives ----
__global__ void local_rs_kernel(float* const* __restrict__ bufs, int P, int64_t stride,
                                int64_t count) {
  const int64_t total = static_cast<int64_t>(P) * count;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(t / count);
    const int64_t off = static_cast<int64_t>(r) * stride + (t - static_cast<int64_t>(r) * count);
    int k = (r + 1) % P;
    float acc = bufs[k][off];
    for (int j = 1; j < P; ++j) {
      k = (k + 1) % P;
      acc = __fadd_rn(acc, bufs[k][off]);
    }
    bufs[r][off] = acc;
  }
}

__global__ void local_ag_kernel(float* const* __restrict__ bufs, int P, int64_t stride,
                                int64_t count) {
  const int64_t total = static_cast<int64_t>(P) * P * count;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pair = t / count;
    const int r = static_cast<int>(pair / P), s = static_cast<int>(pair % P);
    if (r == s) continue;
    const int64_t off = static_cast<int64_t>(s) * stride + (t - pair * count);
    bufs[r][off] = bufs[s][off];
  }
}

__global__ void set_lr_kernel(HyperParams* hp, float lr) { hp->lr = lr; }

// ---------------------------------------------------------------- hash ----
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void hash_kernel(const float* __restrict__ x, int64_t n, uint64_t salt,
                            unsigned long long* acc) {
  uint64_t h = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t bits = __float_as_uint(x[i]);
    h += mix64(bits ^ mix64(static_cast<uint64_t>(i) + salt));
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_down_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, static_cast<unsigned long long>(h));
}

// Grid of the bucket kernels: kSlices (one slice per CTA) unless
// DEAR_BUCKET_CTAS caps it (CTAs then walk several slices), which leaves SMs
// to concurrently running GEMMs.
bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("DEAR_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// <<<grid, kThreads, 0, s>>> with programmatic stream serialization.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), int grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

int bucket_grid(int n_slices, int want = 0) {
  static int cap = [] {
    const char* e = std::getenv("DEAR_BUCKET_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int g = cap > 0 ? cap : want;
  return g > 0 && g < n_slices ? g : n_slices;
}

}  // namespace

cudaError_t launch_pack(const Unit* units, const Slice* slices, int64_t total, float scale,
                        int grid, cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  return launch_pdl(pack_kernel<false>, bucket_grid(kPackSlices, grid), s, units, slices, scale,
                    static_cast<BucketFlags*>(nullptr), PeerArgs{}, kPackSlices);
}

cudaError_t launch_pack_signal(const Unit* units, const Slice* slices, int64_t total, float scale,
                               BucketFlags* flags, const PeerArgs& pa, cudaStream_t s) {
  (void)total;  // the signal must fire even for an empty bucket
  if (kPeerPackLight)
    pack_kernel<true><<<bucket_grid(kPackPeerSlices), kThreads, 0, s>>>(units, slices, scale, flags,
                                                                       pa, kPackPeerSlices);
  else
    pack_kernel<true><<<bucket_grid(kSlices), kThreads, 0, s>>>(units, slices, scale, flags, pa,
                                                                kSlices);
  return cudaGetLastError();
}

cudaError_t launch_pack_push(const Unit* units, const Slice* slices, float scale,
                             BucketFlags* flags, const PeerArgs& pa, cudaStream_t s) {
  pack_kernel<true, true><<<bucket_grid(kPackPeerSlices), kThreads, 0, s>>>(units, slices, scale,
                                                                           flags, pa, kPackPeerSlices);
  return cudaGetLastError();
}

cudaError_t launch_wait_peers(const uint32_t* mine, const uint32_t* watch, const PeerArgs& pa,
                              cudaStream_t s) {
  wait_peers_kernel<<<1, 32, 0, s>>>(mine, watch, pa);
  return cudaGetLastError();
}

template <int PC>
void launch_rs_update_peer_p(const Unit* units, const Slice* slices, const HyperParams* hp,
                             int has_momentum_buf, int use_momentum, int use_wd,
                             const PeerArgs& pa, BucketFlags* flags, cudaStream_t s) {
  const int grid = bucket_grid(kPeerSlices);
  if (use_momentum && use_wd)
    rs_update_peer_kernel<PC, true, true><<<grid, kThreads, 0, s>>>(units, slices, hp, has_momentum_buf, pa, flags);
  else if (use_momentum)
    rs_update_peer_kernel<PC, true, false><<<grid, kThreads, 0, s>>>(units, slices, hp, has_momentum_buf, pa, flags);
  else if (use_wd)
    rs_update_peer_kernel<PC, false, true><<<grid, kThreads, 0, s>>>(units, slices, hp, has_momentum_buf, pa, flags);
  else
    rs_update_peer_kernel<PC, false, false><<<grid, kThreads, 0, s>>>(units, slices, hp, has_momentum_buf, pa, flags);
}

cudaError_t launch_rs_update_peer(const Unit* units, const Slice* slices, int64_t total,
                                  const HyperParams* hp, int has_momentum_buf, int use_momentum,
                                  int use_wd, const PeerArgs& pa, BucketFlags* flags,
                                  cudaStream_t s) {
  (void)total;
  switch (pa.P) {
    case 2: launch_rs_update_peer_p<2>(units, slices, hp, has_momentum_buf, use_momentum, use_wd, pa, flags, s); break;
    case 4: launch_rs_update_peer_p<4>(units, slices, hp, has_momentum_buf, use_momentum, use_wd, pa, flags, s); break;
    case 8: launch_rs_update_peer_p<8>(units, slices, hp, has_momentum_buf, use_momentum, use_wd, pa, flags, s); break;
    default: launch_rs_update_peer_p<0>(units, slices, hp, has_momentum_buf, use_momentum, use_wd, pa, flags, s); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_ag_unpack_peer(const Unit* units, const Slice* slices, int64_t total,
                                  int with_shadow, const PeerArgs& pa, const PeerArgs& sa,
                                  BucketFlags* flags, int n_slices, cudaStream_t s) {
  (void)total;
  const size_t smem = 0;
  const int g = bucket_grid(n_slices);
  if (with_shadow)
    ag_unpack_peer_kernel<true><<<g, kThreads, smem, s>>>(units, slices, pa, sa, flags, n_slices);
  else
    ag_unpack_peer_kernel<false><<<g, kThreads, smem, s>>>(units, slices, pa, sa, flags, n_slices);
  return cudaGetLastError();
}

template <int PC, bool kMom, bool kWd>
void launch_rs_zc_p(const Unit* units, const Slice* slices, const HyperParams* hp, int has_buf,
                    float* mom_base, int with_shadow, const PeerArgs& pa, const PeerArgs& ga,
                    BucketFlags* flags, int announce, cudaStream_t s) {
  const int grid = bucket_grid(kZcSlices);
  const size_t smem = 0;
  if (with_shadow)
    rs_update_zc_kernel<PC, kMom, kWd, true><<<grid, kThreads, smem, s>>>(
        units, slices, hp, has_buf, mom_base, pa, ga, flags, announce);
  else
    rs_update_zc_kernel<PC, kMom, kWd, false><<<grid, kThreads, smem, s>>>(
        units, slices, hp, has_buf, mom_base, pa, ga, flags, announce);
}

template <int PC>
void launch_rs_zc_pc(const Unit* units, const Slice* slices, const HyperParams* hp, int has_buf,
                     float* mom_base, int use_momentum, int use_wd, int with_shadow,
                     const PeerArgs& pa, const PeerArgs& ga, BucketFlags* flags, int announce,
                     cudaStream_t s) {
  if (use_momentum && use_wd)
    launch_rs_zc_p<PC, true, true>(units, slices, hp, has_buf, mom_base, with_shadow, pa, ga, flags, announce, s);
  else if (use_momentum)
    launch_rs_zc_p<PC, true, false>(units, slices, hp, has_buf, mom_base, with_shadow, pa, ga, flags, announce, s);
  else if (use_wd)
    launch_rs_zc_p<PC, false, true>(units, slices, hp, has_buf, mom_base, with_shadow, pa, ga, flags, announce, s);
  else
    launch_rs_zc_p<PC, false, false>(units, slices, hp, has_buf, mom_base, with_shadow, pa, ga, flags, announce, s);
}

cudaError_t launch_rs_update_zc(const Unit* units, const Slice* slices, const HyperParams* hp,
                                int has_momentum_buf, float* mom_base, int use_momentum,
                                int use_wd, int with_shadow, const PeerArgs& pa,
                                const PeerArgs& ga, BucketFlags* flags, cudaStream_t s,
                                int announce) {
  switch (pa.P) {
    case 2: launch_rs_zc_pc<2>(units, slices, hp, has_momentum_buf, mom_base, use_momentum, use_wd, with_shadow, pa, ga, flags, announce, s); break;
    case 4: launch_rs_zc_pc<4>(units, slices, hp, has_momentum_buf, mom_base, use_momentum, use_wd, with_shadow, pa, ga, flags, announce, s); break;
    case 8: launch_rs_zc_pc<8>(units, slices, hp, has_momentum_buf, mom_base, use_momentum, use_wd, with_shadow, pa, ga, flags, announce, s); break;
    default: launch_rs_zc_pc<0>(units, slices, hp, has_momentum_buf, mom_base, use_momentum, use_wd, with_shadow, pa, ga, flags, announce, s); break;
  }
  return cudaGetLastError();
}

namespace {
template <typename... KArgs, typename... Args>
cudaError_t coop(void (*k)(KArgs...), int grid, cudaStream_t s, Args... args) {
  void* pv[] = {static_cast<void*>(&args)...};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(kThreads),
                                     pv, 0, s);
}

template <int PC, bool kMom, bool kWd>
cudaError_t group_rs_zc_p(const GroupOp* ops, int P, int nb, int has_buf, int shadow,
                          cudaStream_t s) {
  if (shadow) return coop(group_rs_zc_kernel<PC, kMom, kWd, true>, P * nb, s, ops, nb, has_buf);
  return coop(group_rs_zc_kernel<PC, kMom, kWd, false>, P * nb, s, ops, nb, has_buf);
}

template <int PC>
cudaError_t group_rs_zc_pc(const GroupOp* ops, int P, int nb, int has_buf, int mom, int wd,
                           int shadow, cudaStream_t s) {
  if (mom && wd) return group_rs_zc_p<PC, true, true>(ops, P, nb, has_buf, shadow, s);
  if (mom) return group_rs_zc_p<PC, true, false>(ops, P, nb, has_buf, shadow, s);
  if (wd) return group_rs_zc_p<PC, false, true>(ops, P, nb, has_buf, shadow, s);
  return group_rs_zc_p<PC, false, false>(ops, P, nb, has_buf, shadow, s);
}

template <int PC>
cudaError_t group_rs_peer_pc(const GroupOp* ops, int P, int nb, int has_buf, int mom, int wd,
                             cudaStream_t s) {
  if (mom && wd) return coop(group_rs_peer_kernel<PC, true, true>, P * nb, s, ops, nb, has_buf);
  if (mom) return coop(group_rs_peer_kernel<PC, true, false>, P * nb, s, ops, nb, has_buf);
  if (wd) return coop(group_rs_peer_kernel<PC, false, true>, P * nb, s, ops, nb, has_buf);
  return coop(group_rs_peer_kernel<PC, false, false>, P * nb, s, ops, nb, has_buf);
}
}  // namespace

cudaError_t launch_group_rs_zc(const GroupOp* ops, int P, int nb, int has_buf, int use_momentum,
                               int use_wd, int with_shadow, cudaStream_t s) {
  switch (P) {
    case 2: return group_rs_zc_pc<2>(ops, P, nb, has_buf, use_momentum, use_wd, with_shadow, s);
    case 4: return group_rs_zc_pc<4>(ops, P, nb, has_buf, use_momentum, use_wd, with_shadow, s);
    case 8: return group_rs_zc_pc<8>(ops, P, nb, has_buf, use_momentum, use_wd, with_shadow, s);
    default: return group_rs_zc_pc<0>(ops, P, nb, has_buf, use_momentum, use_wd, with_shadow, s);
  }
}

cudaError_t launch_group_rs_peer(const GroupOp* ops, int P, int nb, int has_buf,
                                 int use_momentum, int use_wd, cudaStream_t s) {
  switch (P) {
    case 2: return group_rs_peer_pc<2>(ops, P, nb, has_buf, use_momentum, use_wd, s);
    case 4: return group_rs_peer_pc<4>(ops, P, nb, has_buf, use_momentum, use_wd, s);
    case 8: return group_rs_peer_pc<8>(ops, P, nb, has_buf, use_momentum, use_wd, s);
    default: return group_rs_peer_pc<0>(ops, P, nb, has_buf, use_momentum, use_wd, s);
  }
}

cudaError_t launch_group_ag(const GroupOp* ops, int P, int nb, int with_shadow, cudaStream_t s) {
  if (with_shadow) return coop(group_ag_kernel<true>, P * nb, s, ops, nb);
  return coop(group_ag_kernel<false>, P * nb, s, ops, nb);
}

template <bool kMom, bool kWd>
void rs_nvls_launch(const Unit* units, const Slice* slices, const HyperParams* hp, int has_buf,
                    float* mom, const NvlsArgs& na, BucketFlags* flags, cudaStream_t s) {
  rs_update_nvls_kernel<kMom, kWd><<<bucket_grid(kZcSlices), kThreads, 0, s>>>(
      units, slices, hp, has_buf, mom, na.mc_delta, flags, na.ucf, na.mcf, na.P, na.spin_limit);
}

cudaError_t launch_rs_update_nvls(const Unit* units, const Slice* slices, const HyperParams* hp,
                                  int has_momentum_buf, float* mom_base, int use_momentum,
                                  int use_wd, const NvlsArgs& na, BucketFlags* flags,
                                  cudaStream_t s) {
  if (use_momentum && use_wd)
    rs_nvls_launch<true, true>(units, slices, hp, has_momentum_buf, mom_base, na, flags, s);
  else if (use_momentum)
    rs_nvls_launch<true, false>(units, slices, hp, has_momentum_buf, mom_base, na, flags, s);
  else if (use_wd)
    rs_nvls_launch<false, true>(units, slices, hp, has_momentum_buf, mom_base, na, flags, s);
  else
    rs_nvls_launch<false, false>(units, slices, hp, has_momentum_buf, mom_base, na, flags, s);
  return cudaGetLastError();
}

cudaError_t launch_ag_nvls(const Unit* units, const Slice* slices, int with_shadow,
                           const NvlsArgs& na, BucketFlags* flags, cudaStream_t s) {
  if (with_shadow)
    ag_nvls_kernel<true><<<bucket_grid(kZcSlices), kThreads, 0, s>>>(
        units, slices, na.mc_delta, flags, na.ucf, na.mcf, na.P, na.spin_limit);
  else
    ag_nvls_kernel<false><<<bucket_grid(kZcSlices), kThreads, 0, s>>>(
        units, slices, na.mc_delta, flags, na.ucf, na.mcf, na.P, na.spin_limit);
  return cudaGetLastError();
}

cudaError_t launch_nvls_wait_updated(const uint32_t* epoch, const NvlsArgs& na, cudaStream_t s) {
  nvls_wait_updated_kernel<<<1, 32, 0, s>>>(epoch, na.ucf, na.P, na.spin_limit);
  return cudaGetLastError();
}

cudaError_t launch_update(const Unit* units, const Slice* slices, int64_t total,
                          const HyperParams* hp, int has_momentum_buf, int use_momentum,
                          int use_wd, int grid, cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  const int ug = bucket_grid(kUpdSlices, grid);
  if (use_momentum && use_wd)
    return launch_pdl(update_kernel<true, true>, ug, s, units, slices, hp, has_momentum_buf);
  if (use_momentum)
    return launch_pdl(update_kernel<true, false>, ug, s, units, slices, hp, has_momentum_buf);
  if (use_wd)
    return launch_pdl(update_kernel<false, true>, ug, s, units, slices, hp, has_momentum_buf);
  return launch_pdl(update_kernel<false, false>, ug, s, units, slices, hp, has_momentum_buf);
}

cudaError_t launch_unpack(const Unit* units, const Slice* slices, int64_t total, int with_shadow,
                          int grid, cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  const int ug = bucket_grid(kUnpackSlices, grid);
  if (with_shadow) return launch_pdl(unpack_kernel<true>, ug, s, units, slices);
  return launch_pdl(unpack_kernel<false>, ug, s, units, slices);
}

cudaError_t launch_update_direct(const Unit* units, const Slice* slices, int64_t total,
                                 const HyperParams* hp, int use_wd, int with_shadow,
                                 cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  const int grid = bucket_grid(kDirSlices);
  if (use_wd && with_shadow)
    return launch_pdl(update_direct_kernel<true, true>, grid, s, units, slices, hp);
  if (use_wd) return launch_pdl(update_direct_kernel<true, false>, grid, s, units, slices, hp);
  if (with_shadow) return launch_pdl(update_direct_kernel<false, true>, grid, s, units, slices, hp);
  return launch_pdl(update_direct_kernel<false, false>, grid, s, units, slices, hp);
}

void make_slices(const Unit* units, int n_units, int64_t total, Slice* out, int n_slices,
                 int c_elem_bytes) {
  int64_t per = (total + n_slices - 1) / n_slices;
  per = (per + 3) / 4 * 4;
  int u = 0;
  int64_t base = 0;  // start of unit u
  for (int c = 0; c < n_slices; ++c) {
    const int64_t lo = static_cast<int64_t>(c) * per;
    const int64_t cnt = lo >= total ? 0 : (total - lo < per ? total - lo : per);
    Slice& sl = out[c];
    sl = Slice{};
    sl.count = cnt;
    if (cnt <= 0) continue;
    while (u < n_units && base + units[u].len <= lo) {
      base += units[u].len;
      ++u;
    }
    const int64_t off = lo - base;
    const Unit& U = units[u];
    sl.unit = u;
    sl.first = U;
    sl.first.a = U.a ? U.a + off : nullptr;
    sl.first.b = U.b ? U.b + off : nullptr;
    // c: momentum (fp32) for update units, bf16 shadow for unpack units.
    sl.first.c = U.c ? static_cast<void*>(static_cast<char*>(U.c) + off * c_elem_bytes) : nullptr;
    sl.first.len = U.len - off;
    sl.first.start = lo;
    sl.first.pad = static_cast<int32_t>(off & 0x7fffffff);
  }
}

cudaError_t launch_local_reduce_scatter(float* const* bufs_dev, int P, int64_t stride,
                                        int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  local_rs_kernel<<<kSms * 4, 256, 0, s>>>(bufs_dev, P, stride, count);
  return cudaGetLastError();
}

cudaError_t launch_local_all_gather(float* const* bufs_dev, int P, int64_t stride,
                                    int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  local_ag_kernel<<<kSms * 4, 256, 0, s>>>(bufs_dev, P, stride, count);
  return cudaGetLastError();
}

cudaError_t set_comm_trace(void* buf, uint32_t cap) {
  CommTraceRec* p = static_cast<CommTraceRec*>(buf);
  const uint32_t zero = 0;
  cudaError_t e = cudaMemcpyToSymbol(g_comm_trace, &p, sizeof p);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_comm_trace_cap, &cap, sizeof cap);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_comm_trace_n, &zero, sizeof zero);
  return e;
}

cudaError_t comm_trace_count(uint32_t* n) {
  return cudaMemcpyFromSymbol(n, g_comm_trace_n, sizeof *n);
}

cudaError_t launch_set_lr(HyperParams* hp, float lr, cudaStream_t s) {
  set_lr_kernel<<<1, 1, 0, s>>>(hp, lr);
  return cudaGetLastError();
}

cudaError_t launch_hash(const float* x, int64_t n, uint64_t salt, unsigned long long* acc,
                        cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  hash_kernel<<<kSms * 2, 256, 0, s>>>(x, n, salt, acc);
  return cudaGetLastError();
}

}  // namespace dear
