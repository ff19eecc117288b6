// Hand-written sm_100a GEMM for the synthetic layer compute.
//
//   TMA (cp.async.bulk.tensor.2d, 128B swizzle) -> 4..8-stage smem ring
//   (mbarrier full/empty) -> tcgen05.mma kind::f16 (bf16 in, fp32 accumulate
//   in TMEM, issued by one thread) -> tcgen05.ld epilogue -> global.
//
// Persistent: two CTAs per SM (102 KB smem ring, one 256-column TMEM
// accumulator each) walk a static round-robin list of output tiles (128 x BN,
// BN <= 256 a multiple of 16 chosen per problem). With two resident CTAs the
// epilogue of one overlaps the other's mainloop — and, across launches under
// programmatic dependent launch, the next GEMM's CTA streams its operands
// while the previous GEMM's CTA on the same SM drains its epilogue. (The
// earlier one-CTA-per-SM form, 192 KB ring and two accumulators, is
// DEAR_GEMM_RING_KB=192 DEAR_GEMM_ACCS=2 DEAR_GEMM_CTAS_PER_SM=1; the two-CTA
// form cut the BERT-L compute-only step from 8.80 to 6.42 ms,
// profiles/r01e_gemm_two_ctas.log.) A launch may carry up to two independent problems (the wgrad and
// dgrad of one layer's backprop), sharing the persistent grid. Launches use
// programmatic dependent launch: the next GEMM's CTAs run their prologue
// (barrier init, TMEM alloc, descriptor prefetch) while this one drains, and
// block in griddepcontrol.wait before touching memory.
//
// Warp roles per CTA (192 threads):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue; warp w reads TMEM lanes 32*(w%4) .. +31
// With `accumulate`, a problem's K range may be split across tiles and the
// partial tiles are reduced into fp32 D with red.global.add.v4.f32.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "dear_gemm.h"
#include "dear_internal.h"

namespace dear {
namespace gemm {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
#ifndef DEAR_GEMM_BN_MAX
#define DEAR_GEMM_BN_MAX 256
#endif
constexpr int kBNMax = DEAR_GEMM_BN_MAX;  // widest tile = TMEM accumulator columns
constexpr int kMaxStages = 8;
constexpr int kAStage = kBM * kBK * 2;     // 16 KB
constexpr int kBStage = kBNMax * kBK * 2;  // 32 KB (widest B stage)
// Ring size (and with it the CTAs an SM can hold): 102 KB + 9.5 KB of
// barriers / one epilogue staging buffer per warp fits two CTAs per SM
// (2 stages at BN = 256, 3 at BN = 128, up to 4). Measured against 94 KB with
// double-buffered staging (BN = 256 impossible there): ResNet-50 N = 1 16,621
// -> 20,326 samples/s (profiles/r01e_gemm_ring_epi.log).
#ifndef DEAR_GEMM_RING_KB
#define DEAR_GEMM_RING_KB 102
#endif
#ifndef DEAR_GEMM_ACCS
#define DEAR_GEMM_ACCS 1
#endif
#ifndef DEAR_GEMM_CTAS_PER_SM
#define DEAR_GEMM_CTAS_PER_SM 2
#endif
static_assert(DEAR_GEMM_ACCS * DEAR_GEMM_CTAS_PER_SM * DEAR_GEMM_BN_MAX <= 512,
              "TMEM has 512 columns per SM");
constexpr int kRingBytes = DEAR_GEMM_RING_KB * 1024;
constexpr int kThreads = 192;
constexpr int kAccCols = kBNMax;
constexpr int kNumAcc = DEAR_GEMM_ACCS;  // TMEM accumulators per CTA (1 or 2)
constexpr int kTmemCols = kNumAcc * kAccCols;
// Epilogue staging for TMA stores: per epilogue warp two 32x32 bf16 buffers.
constexpr int kEpiBufBytes = 32 * 32 * 2;
#ifndef DEAR_GEMM_EPI_BUFS
#define DEAR_GEMM_EPI_BUFS 1
#endif
constexpr int kEpiBufs = DEAR_GEMM_EPI_BUFS;  // staging buffers per epilogue warp
constexpr int kEpiBytes = 4 * kEpiBufs * kEpiBufBytes;  // 8 KB with one
constexpr int kEpiOffset = kRingBytes + 512;     // after the barriers, 512 B aligned
constexpr int kSmemBytes = kEpiOffset + kEpiBytes + 1024;
constexpr int kMaxProblems = 2;
constexpr int kSms = 148;

struct alignas(64) Problem {
  CUtensorMap tmA;
  CUtensorMap tmB;
  void* D;
  int64_t ldd;
  int64_t M, N;
  int64_t d_limit;
  int32_t num_kb;
  int32_t kb_per_split;
  int32_t splits;
  int32_t bn;
  int32_t m_tiles;
  int32_t n_tiles;
  int32_t tiles;
  int32_t b_mn_major;
  int32_t d_fp32;
  int32_t accumulate;
  int32_t b_boxes;
  uint32_t idesc;
  uint32_t tx_bytes;
  // Thread-block cluster of cm x cn CTAs sharing operands through TMA
  // multicast: CTA (i, j) computes tile (mg*cm + i, ng*cn + j); the A tile
  // of row i is fetched once, in cn pieces of a_rows rows, and multicast to
  // the cn CTAs of that row; B likewise to the cm CTAs of column j.
  int32_t cm, cn;
  int32_t mg_tiles, ng_tiles;  // cluster tiles along M / N
  int32_t a_rows;              // 128 / cn
  int32_t b_rows;              // K-major: bn / cm rows; MN-major: 64 / cm k-rows per box
  // CTA pair (cta_group::2): the two CTAs of a 2-CTA cluster compute one
  // 256 x bn tile with M=256 MMAs issued by the even CTA; each CTA fetches its
  // 128 rows of A and half (bn/2) of B, the MMA reads the other half from the
  // peer SM. Encoded as cm = 2, cn = 1 (CTA rank = row half), no multicast.
  int32_t pair;
  // Caller guarantees A and B are not written by kernels that can still be
  // running when this GEMM starts (dear_gemm_plan_set_flags): the producer
  // then streams operands before griddepcontrol.wait; only stores wait.
  int32_t early_operands;
  // bf16, non-accumulating D: the epilogue stages 32x32 chunks in smem and
  // writes them with TMA bulk stores (full lines, asynchronous; TMA clips rows
  // >= M and columns >= N). tmD: box 32x32, 64 B swizzle; tmD16: box 16x32 for
  // the last 16 columns of a tile whose bn is an odd multiple of 16.
  CUtensorMap tmD;
  CUtensorMap tmD16;
  int32_t d_tma;      // 1: bf16 TMA stores; 2: fp32 TMA reduce-add (accumulate)
  // d_tma == 2: tmD is fp32 with box 16x32 over the r_full complete rows of
  // D (flat limit); a partial last row (row r_full) goes through red.add.
  int64_t r_full;      // row added by red.add (partial under d_limit), or INT64_MAX
  int64_t d_lim_rows;  // rows covered by the TMA map
  int32_t tma_reduce_ok;  // fp32 TMA reduce-add possible (flag DEAR_GEMM_RED_ADD turns it off)
};

struct Launch {
  Problem p[kMaxProblems];
  int32_t n_problems;
  int32_t total_tiles;
  int32_t stages;       // smem ring depth (narrow B tiles -> deeper ring)
  int32_t stage_bytes;  // A (16 KB) + widest B of the problems, 1 KB aligned
  int32_t cm, cn;       // cluster shape shared by the problems of the launch
  int32_t pair;         // CTA-pair (cta_group::2) launch
  int32_t early;        // every problem has early_operands
  uint64_t* trace;      // optional per-CTA phase timestamps (profiling), or null
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  uint32_t polls = 0;
  do {
    // A pipeline bug must fail loudly (trap) rather than hang the GPU.
    if (++polls > (1u << 28)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}

// Profiling variant (-DDEAR_GEMM_WAITPROF): accumulate the cycles a role spends
// blocked in mbar_wait, to tell a data-starved MMA issuer from a full ring.
#ifdef DEAR_GEMM_WAITPROF
#define WAIT_T(acc, bar, ph)             \
  do {                                   \
    const long long t0_ = clock64();     \
    mbar_wait(bar, ph);                  \
    acc += clock64() - t0_;              \
  } while (0)
#else
#define WAIT_T(acc, bar, ph) mbar_wait(bar, ph)
#endif

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst,
                                               int32_t c0, int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src,
                                                  int32_t c0, int32_t c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_clusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// UMMA shared-memory matrix descriptor, SWIZZLE_128B, Blackwell version 1.
//   K-major  : rows of 128 B (64 bf16 along K); 8-row groups SBO = 1024 B apart.
//   MN-major : 64 MN-elements per 128 B row, one row per k; 8-k groups
//              SBO = 1024 B apart; 64-wide MN blocks LBO = 8192 B apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// Arrive on the barrier at the same smem offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---- CTA-pair (cta_group::2) variants -------------------------------------
// Shared::cluster address of `p`'s counterpart in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// TMA into this CTA's smem, completing on an mbarrier of either pair CTA.
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar_cluster,
                                                 void* dst, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t a, uint64_t b,
                                           uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// Arrive (when the issued MMAs complete) on the barrier at `bar`'s offset in
// both CTAs of the pair.
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// Stores 32 accumulator columns of one row; columns >= col_end (the end of
// this tile clipped to N) and flat offsets >= d_limit are not written.
__device__ __forceinline__ void store_row_chunk(const Problem& p, int64_t row, int64_t col0,
                                                int64_t col_end, const uint32_t (&v)[32]) {
  if (row >= p.M) return;
  const int64_t base = row * p.ldd;
  if (p.d_fp32) {
    float* D = static_cast<float*>(p.D);
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const int64_t col = col0 + j;
      const int64_t flat = base + col;
      const bool full = col + 3 < col_end && (p.d_limit < 0 || flat + 3 < p.d_limit) &&
                        (flat & 3) == 0;
      const float a = __uint_as_float(v[j]), b = __uint_as_float(v[j + 1]),
                  c = __uint_as_float(v[j + 2]), d = __uint_as_float(v[j + 3]);
      if (full) {
        if (p.accumulate)
          red_add_v4(D + flat, a, b, c, d);
        else
          *reinterpret_cast<float4*>(D + flat) = make_float4(a, b, c, d);
      } else {
        const float e[4] = {a, b, c, d};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (col + t < col_end && (p.d_limit < 0 || flat + t < p.d_limit)) {
            if (p.accumulate)
              atomicAdd(D + flat + t, e[t]);
            else
              D[flat + t] = e[t];
          }
        }
      }
    }
  } else {
    __nv_bfloat16* D = static_cast<__nv_bfloat16*>(p.D);
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t col = col0 + j;
      const int64_t flat = base + col;
      const bool full = col + 7 < col_end && (p.d_limit < 0 || flat + 7 < p.d_limit) &&
                        (flat & 7) == 0;
      if (full) {
        uint4 pk;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
        __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
        __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
        pk.x = *reinterpret_cast<uint32_t*>(&h0);
        pk.y = *reinterpret_cast<uint32_t*>(&h1);
        pk.z = *reinterpret_cast<uint32_t*>(&h2);
        pk.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(D + flat) = pk;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (col + t < col_end && (p.d_limit < 0 || flat + t < p.d_limit))
            D[flat + t] = __float2bfloat16_rn(__uint_as_float(v[j + t]));
        }
      }
    }
  }
}

struct TileCoord {
  int prob;
  int64_t m0, n0;
  int kb0, kb1;
};

// Cluster tile t of the launch: problems back to back; inside a problem
// (split, m group, n group) with n fastest. CTA (ci, cj) of the cluster takes
// tile (mg * cm + ci, ng * cn + cj); tiles past M / N compute on zero-filled
// operands (they still source their multicast pieces) and store nothing.
__device__ __forceinline__ TileCoord decode(const Launch& L, int t, int ci, int cj) {
  TileCoord c;
  c.prob = (L.n_problems > 1 && t >= L.p[0].tiles) ? 1 : 0;
  const Problem& P = L.p[c.prob];
  const int local = c.prob ? t - L.p[0].tiles : t;
  const int per = P.mg_tiles * P.ng_tiles;
  const int split = local / per;
  const int r = local - split * per;
  c.m0 = static_cast<int64_t>((r / P.ng_tiles) * P.cm + ci) * kBM;
  c.n0 = static_cast<int64_t>((r % P.ng_tiles) * P.cn + cj) * P.bn;
  c.kb0 = split * P.kb_per_split;
  c.kb1 = min(c.kb0 + P.kb_per_split, P.num_kb);
  return c;
}

// kPair: 2-CTA clusters issuing cta_group::2 MMAs (see Problem::pair); every
// tcgen05 instruction of a kernel must use the same cta_group, hence a
// separate instantiation.
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ Launch L) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int stages = L.stages;
  const int stage_bytes = L.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tmem_full = empty + kMaxStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int csize = kPair ? 2 : L.cm * L.cn;
  const int crank = csize > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int ci = kPair ? crank : crank / L.cn, cj = kPair ? 0 : crank % L.cn;
  const bool leader = !kPair || crank == 0;
  const int cid = csize > 1 ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int ncl = csize > 1 ? static_cast<int>(n_clusters_x()) : static_cast<int>(gridDim.x);
  // CTAs sharing this CTA's A tile (same row) and B tile (same column).
  uint16_t row_mask = 0, col_mask = 0;
  if (!kPair) {
    for (int j = 0; j < L.cn; ++j) row_mask |= static_cast<uint16_t>(1u << (ci * L.cn + j));
    for (int i = 0; i < L.cm; ++i) col_mask |= static_cast<uint16_t>(1u << (i * L.cn + cj));
  }

  uint64_t* tr = L.trace ? L.trace + blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = globaltimer();  // CTA start
  // Let the next kernel in the stream start its prologue as soon as SMs free.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      // pair: released by the leader's MMA commit; clusters: by every CTA this
      // CTA multicasts into (its row and column)
      mbar_init(&empty[s], kPair ? 1u : static_cast<uint32_t>(L.cm + L.cn - 1));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], kPair ? 8 : 4);  // pair: both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < L.n_problems; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&L.p[i].tmA))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&L.p[i].tmB))
                   : "memory");
      if (L.p[i].d_tma)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&L.p[i].tmD))
                     : "memory");
    }
  }
  if (warp == 1) {
    if (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (csize > 1)
    cluster_sync();  // peers' barriers are initialised before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr && threadIdx.x == 0) tr[1] = globaltimer();  // prologue done
  // Everything above overlaps the previous kernel. Global memory is touched
  // only after the dependency is released, except operand loads of `early`
  // launches; the MMA issuer touches no global memory.
  if (warp >= 2 || (warp == 0 && !L.early)) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tr && warp == 2 && lane == 0) tr[2] = globaltimer();  // dependency released

  long long w_acc = 0;  // cycles blocked (profiling variant only)
  if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = cid; t < L.total_tiles; t += ncl) {
        const TileCoord tc = decode(L, t, ci, cj);
        const Problem& P = L.p[tc.prob];
        const int nk = tc.kb1 - tc.kb0;
        for (int i = 0; i < nk; ++i, ++g) {
          const int kb = tc.kb0 + i;
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          WAIT_T(w_acc, &empty[s], ph ^ 1);
          const int kc = kb * kBK;
          uint8_t* sA = smem + s * stage_bytes;
          uint8_t* sB = sA + kAStage;
          if (kPair) {
            // Both CTAs' bytes land on the leader's full barrier.
            if (leader) mbar_expect_tx(&full[s], P.tx_bytes);
            const uint32_t fb = mapa_shared(&full[s], 0);
            tma_load_2d_pair(&P.tmA, fb, sA, kc, static_cast<int32_t>(tc.m0));
            const int32_t nh = static_cast<int32_t>(tc.n0) + crank * (P.bn / 2);
            if (!P.b_mn_major) {
              tma_load_2d_pair(&P.tmB, fb, sB, kc, nh);
            } else {
              for (int j = 0; j < P.b_boxes; ++j)
                tma_load_2d_pair(&P.tmB, fb, sB + j * 8192, nh + 64 * j, kc);
            }
            continue;
          }
          mbar_expect_tx(&full[s], P.tx_bytes);
          // A: this CTA's piece (rows cj*a_rows ..) of its row's tile.
          const int32_t am = static_cast<int32_t>(tc.m0) + cj * P.a_rows;
          uint8_t* dA = sA + cj * P.a_rows * 128;
          if (P.cn > 1)
            tma_load_2d_mc(&P.tmA, &full[s], dA, kc, am, row_mask);
          else
            tma_load_2d(&P.tmA, &full[s], dA, kc, am);
          if (!P.b_mn_major) {
            const int32_t bn0 = static_cast<int32_t>(tc.n0) + ci * P.b_rows;
            uint8_t* dB = sB + ci * P.b_rows * 128;
            if (P.cm > 1)
              tma_load_2d_mc(&P.tmB, &full[s], dB, kc, bn0, col_mask);
            else
              tma_load_2d(&P.tmB, &full[s], dB, kc, bn0);
          } else {
            for (int j = 0; j < P.b_boxes; ++j) {
              uint8_t* dB = sB + j * 8192 + ci * P.b_rows * 128;
              const int32_t c0 = static_cast<int32_t>(tc.n0 + 64 * j);
              const int32_t c1 = kc + ci * P.b_rows;
              if (P.cm > 1)
                tma_load_2d_mc(&P.tmB, &full[s], dB, c0, c1, col_mask);
              else
                tma_load_2d(&P.tmB, &full[s], dB, c0, c1);
            }
          }
        }
      }
#ifdef DEAR_GEMM_WAITPROF
      if (tr) tr[4] = w_acc;  // producer: cycles waiting for free stages
#endif
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
#ifdef DEAR_GEMM_WAITPROF
      const long long t_loop = clock64();
#endif
      uint32_t g = 0, j = 0;
      for (int t = cid; t < L.total_tiles; t += ncl, ++j) {
        const TileCoord tc = decode(L, t, ci, cj);
        const Problem& P = L.p[tc.prob];
        const uint32_t acc = j % kNumAcc, aph = (j / kNumAcc) & 1;
        long long w_tm = 0;
        WAIT_T(w_tm, &tmem_empty[acc], aph ^ 1);
        (void)w_tm;
#ifdef DEAR_GEMM_WAITPROF
        if (tr) tr[5] += w_tm;
#endif
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * kAccCols;
        const int nk = tc.kb1 - tc.kb0;
        for (int i = 0; i < nk; ++i, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          WAIT_T(w_acc, &full[s], ph);
          tc_fence_after();
#ifndef DEAR_GEMM_WAITPROF
          if (tr && g == 0) tr[3] = globaltimer();  // first stage landed
#endif
          const uint32_t a_base = smem_u32(smem + s * stage_bytes);
          const uint32_t b_base = a_base + kAStage;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = P.b_mn_major ? sdesc(b_base + k * 2048, 8192, 1024)
                                             : sdesc(b_base + k * 32, 16, 1024);
            if (kPair)
              umma2_bf16(d_tmem, ad, bd, P.idesc, (i != 0 || k != 0) ? 1u : 0u);
            else
              umma_bf16(d_tmem, ad, bd, P.idesc, (i != 0 || k != 0) ? 1u : 0u);
          }
          if (kPair)
            umma2_commit_both(&empty[s]);
          else if (csize > 1)
            umma_commit_mc(&empty[s], static_cast<uint16_t>(row_mask | col_mask));
          else
            umma_commit(&empty[s]);
        }
        if (kPair)
          umma2_commit_both(&tmem_full[acc]);
        else
          umma_commit(&tmem_full[acc]);
      }
#ifdef DEAR_GEMM_WAITPROF
      if (tr) tr[7] = clock64() - t_loop;  // MMA issuer: whole loop
      if (tr) tr[3] = w_acc;  // MMA issuer: cycles waiting for landed stages
#else
      if (tr) tr[4] = globaltimer();  // last MMA issued
#endif
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    uint32_t j = 0;
    uint32_t epi_chunk = 0;  // TMA-store staging buffer parity
    for (int t = cid; t < L.total_tiles; t += ncl, ++j) {
      const TileCoord tc = decode(L, t, ci, cj);
      const Problem& P = L.p[tc.prob];
      const uint32_t acc = j % kNumAcc, aph = (j / kNumAcc) & 1;
      mbar_wait(&tmem_full[acc], aph);
      tc_fence_after();
      const int64_t row = tc.m0 + 32 * q + lane;
      const int64_t col_end = min(P.N, tc.n0 + P.bn);
      const uint32_t base = tmem + acc * kAccCols + (static_cast<uint32_t>(32 * q) << 16);
      if (P.d_tma == 2) {
        // fp32 accumulate: two 16-column sub-chunks per TMEM load, each staged
        // (64 B per row, 64 B swizzle) and added into D by a TMA reduce; L2
        // performs the adds on full lines. Row r_full (partial under the flat
        // limit) is added by its lane directly.
        uint8_t* epi = smem + kEpiOffset + q * kEpiBufs * kEpiBufBytes;
        for (int c = 0; c < P.bn; c += 32) {
          uint32_t v[32];
          tmem_ld32(base + static_cast<uint32_t>(c), v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (c + 16 * h >= P.bn) break;
            uint8_t* buf = epi + (epi_chunk % kEpiBufs) * kEpiBufBytes;
            ++epi_chunk;
            if (lane == 0) bulk_wait_read<kEpiBufs - 1>();
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint4 w = make_uint4(v[16 * h + 4 * jj], v[16 * h + 4 * jj + 1],
                                         v[16 * h + 4 * jj + 2], v[16 * h + 4 * jj + 3]);
              const int phys = jj ^ ((lane >> 1) & 3);
              *reinterpret_cast<uint4*>(buf + lane * 64 + phys * 16) = w;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_2d(&P.tmD, buf, static_cast<int32_t>(tc.n0 + c + 16 * h),
                                static_cast<int32_t>(tc.m0 + 32 * q));
              bulk_commit();
            }
          }
          if (row == P.r_full) store_row_chunk(P, row, tc.n0 + c, col_end, v);
        }
      } else if (P.d_tma) {
        // 32 rows x 32 columns per chunk: lane = row; bf16 row of 64 B in four
        // 16 B pieces, piece j stored at j ^ ((row >> 1) & 3) (TMA 64 B swizzle;
        // conflict-free smem writes). kEpiBufs staging buffers per warp.
        uint8_t* epi = smem + kEpiOffset + q * kEpiBufs * kEpiBufBytes;
        for (int c = 0; c < P.bn; c += 32, ++epi_chunk) {
          uint32_t v[32];
          tmem_ld32(base + static_cast<uint32_t>(c), v);
          uint8_t* buf = epi + (epi_chunk % kEpiBufs) * kEpiBufBytes;
          if (lane == 0) bulk_wait_read<kEpiBufs - 1>();  // this buffer's previous store read it
          __syncwarp();
          const bool half = P.bn - c == 16;  // a tile's odd last 16 columns
          if (!half) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              uint4 w;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj]), __uint_as_float(v[8 * jj + 1]));
              __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 2]), __uint_as_float(v[8 * jj + 3]));
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 4]), __uint_as_float(v[8 * jj + 5]));
              __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 6]), __uint_as_float(v[8 * jj + 7]));
              w.x = *reinterpret_cast<uint32_t*>(&h0);
              w.y = *reinterpret_cast<uint32_t*>(&h1);
              w.z = *reinterpret_cast<uint32_t*>(&h2);
              w.w = *reinterpret_cast<uint32_t*>(&h3);
              const int phys = jj ^ ((lane >> 1) & 3);
              *reinterpret_cast<uint4*>(buf + lane * 64 + phys * 16) = w;
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              uint4 w;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj]), __uint_as_float(v[8 * jj + 1]));
              __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 2]), __uint_as_float(v[8 * jj + 3]));
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 4]), __uint_as_float(v[8 * jj + 5]));
              __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(v[8 * jj + 6]), __uint_as_float(v[8 * jj + 7]));
              w.x = *reinterpret_cast<uint32_t*>(&h0);
              w.y = *reinterpret_cast<uint32_t*>(&h1);
              w.z = *reinterpret_cast<uint32_t*>(&h2);
              w.w = *reinterpret_cast<uint32_t*>(&h3);
              *reinterpret_cast<uint4*>(buf + lane * 32 + jj * 16) = w;  // no swizzle
            }
          }
          fence_proxy_async_smem();  // generic-proxy writes -> TMA (async proxy)
          __syncwarp();
          if (lane == 0) {
            const int32_t c0 = static_cast<int32_t>(tc.n0 + c);
            const int32_t c1 = static_cast<int32_t>(tc.m0 + 32 * q);
            tma_store_2d(half ? &P.tmD16 : &P.tmD, buf, c0, c1);
            bulk_commit();
          }
        }
      } else {
        for (int c = 0; c < P.bn; c += 32) {
          uint32_t v[32];
          tmem_ld32(base + static_cast<uint32_t>(c), v);
          store_row_chunk(P, row, tc.n0 + c, col_end, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair)
          mbar_arrive_cluster(mapa_shared(&tmem_empty[acc], 0));
        else
          mbar_arrive(&tmem_empty[acc]);
      }
    }
    if (lane == 0) bulk_wait_all();  // TMA stores complete before the CTA retires
#ifndef DEAR_GEMM_WAITPROF
    if (tr && warp == 2 && lane == 0) tr[5] = globaltimer();  // epilogue done
#endif
  }
  tc_fence_before();
  if (csize > 1)
    cluster_sync();  // nobody exits while peers may still multicast into it
  else
    __syncthreads();
  if (tr && threadIdx.x == 0) tr[6] = globaltimer();  // CTA end
  if (warp == 1) {
    tc_fence_after();
    if (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
      throw Error(DEAR_EINTERNAL, "cuTensorMapEncodeTiled unavailable");
    }
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

void make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
              uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
              CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t esize = dt == CU_TENSOR_MAP_DATA_TYPE_FLOAT32 ? 4 : 2;
  const cuuint64_t strides[1] = {ld_elems * esize};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, dt, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw Error(DEAR_EINTERNAL, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  }
}

struct TileChoice {
  int bn, cm, cn, pair;
};

int max_active_clusters(int csize, bool pair = false);

// Joint choice of the tile width BN and the cluster shape (cm x cn) for one
// problem: estimated time = waves x k-blocks x max(MMA cycles, L2->SM operand
// cycles) + per-tile overhead, where a cluster fetches each A tile once per
// row (multicast to cn CTAs) and each B tile once per column (to cm CTAs),
// and a wave is every resident cluster running one cluster tile. Constraints:
// BN a multiple of 16 (of 8*cm for split B pieces), <= 256.
// modes: bit 0 single CTAs, bit 1 CTA pairs, bit 2 multicast clusters.
enum { kModeSingle = 1, kModePair = 2, kModeCluster = 4 };
TileChoice choose_tiles(int64_t M, int64_t N, int kb_per_tile, int splits, bool mn_major,
                        int modes) {
  // Operand bytes an SM can take in per cycle in the mainloop: measured k-block
  // cadence of 128 x bn tiles on B200 (~0.47 us for 32 KB, tools/gemm_cadence.py,
  // profiles/r01_gemm_trace.md), i.e. per-SM ingress, not the tensor pipe, bounds
  // the per-layer shapes.
  const double ingress = 36.0;
  TileChoice best{256, 1, 1, 0};
  double best_cost = 1e300;
  // {cm, cn, pair}: pair = 2-CTA cta_group::2 tiles of 256 x bn (each SM
  // fetches 128 rows of A and bn/2 rows of B); cm x cn = multicast clusters.
  const int shapes[5][3] = {{1, 1, 0}, {1, 1, 1}, {2, 1, 0}, {1, 2, 0}, {2, 2, 0}};
  for (const auto& sh : shapes) {
    const int cm = sh[0], cn = sh[1], pair = sh[2];
    if (pair && !(modes & kModePair)) continue;
    if (!pair && cm * cn > 1 && !(modes & kModeCluster)) continue;
    if (!pair && cm * cn == 1 && !(modes & kModeSingle)) continue;
    const int rows = pair ? 2 * kBM : kBM;  // M per (pair) tile
    const int64_t m_tiles = (M + rows - 1) / rows;
    if (cm > m_tiles) continue;
    const int active = pair ? max_active_clusters(2, true) : max_active_clusters(cm * cn);
    for (int bn = 256; bn >= 48; bn -= 16) {
      if (bn % (8 * cm)) continue;
      if (mn_major && 64 % cm) continue;
      if (pair && mn_major && bn != 128 && bn != 256) continue;  // 64-col boxes per half
      const int64_t n_tiles = (N + bn - 1) / bn;
      if (cn > n_tiles) continue;
      // too-wide tiles waste MMA columns on padding; skip if > 1 tile of slack
      if (n_tiles > 1 && (n_tiles - 1) * bn >= N) continue;
      const int64_t groups = ((m_tiles + cm - 1) / cm) * ((n_tiles + cn - 1) / cn) * splits;
      const int64_t waves = (groups + active - 1) / active;
      const double mma = 2.0 * bn;  // per SM: 4 x (128 x bn / 256) cycles per k-block
      const double mem = pair ? (16384.0 + 64.0 * bn) / ingress
                              : (16384.0 / cn + 128.0 * bn / cm) / ingress;
      const double cost = waves * (kb_per_tile * std::max(mma, mem) + 1500.0);
      if (cost < best_cost * 0.999) {
        best_cost = cost;
        best = {bn, cm, cn, pair};
      }
    }
  }
  return best;
}

}  // namespace gemm
}  // namespace dear

struct dear_gemm_plan {
  dear::gemm::Problem p;
  const void* A = nullptr;  // creation arguments the tile geometry depends on
  const void* B = nullptr;
  int64_t lda = 0, ldb = 0, K = 0;
};

namespace dear {
namespace gemm {

// Tile-dependent fields of a plan (BN, pair / cluster shape, TMA boxes).
void configure(dear_gemm_plan* plan, const TileChoice& tch) {
  Problem& p = plan->p;
  const int bn = tch.bn;
  const bool mn = p.b_mn_major != 0;
  p.bn = bn;
  p.n_tiles = static_cast<int32_t>((p.N + bn - 1) / bn);
  p.pair = tch.pair;
  const uint32_t mma_m = p.pair ? 2 * kBM : kBM;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(p.b_mn_major) << 16) |
            (static_cast<uint32_t>(bn >> 3) << 17) | ((mma_m >> 4) << 24);
  if (p.pair) {
    // Per CTA: 128 rows of A and half of B; the leader's barrier counts both.
    p.b_boxes = mn ? bn / 2 / 64 : 1;
    p.tx_bytes = 2u * (kAStage + (mn ? p.b_boxes * 8192u : static_cast<uint32_t>(bn / 2) * kBK * 2));
    p.cm = 2;
    p.cn = 1;
    p.a_rows = kBM;
    p.b_rows = mn ? 64 : bn / 2;
  } else {
    p.b_boxes = (bn + 63) / 64;
    p.tx_bytes = kAStage + (mn ? p.b_boxes * 8192 : static_cast<uint32_t>(bn) * kBK * 2);
    p.cm = tch.cm;
    p.cn = tch.cn;
    p.a_rows = kBM / p.cn;
    p.b_rows = mn ? 64 / p.cm : bn / p.cm;
  }
  p.mg_tiles = (p.m_tiles + p.cm - 1) / p.cm;
  p.ng_tiles = (p.n_tiles + p.cn - 1) / p.cn;
  p.tiles = p.mg_tiles * p.ng_tiles * p.splits;  // cluster tiles
  make_map(&p.tmA, plan->A, static_cast<uint64_t>(plan->K), static_cast<uint64_t>(p.M),
           static_cast<uint64_t>(plan->lda), kBK, static_cast<uint32_t>(p.a_rows));
  if (!mn)
    make_map(&p.tmB, plan->B, static_cast<uint64_t>(plan->K), static_cast<uint64_t>(p.N),
             static_cast<uint64_t>(plan->ldb), kBK, static_cast<uint32_t>(p.b_rows));
  else
    make_map(&p.tmB, plan->B, static_cast<uint64_t>(p.N), static_cast<uint64_t>(plan->K),
             static_cast<uint64_t>(plan->ldb), 64, static_cast<uint32_t>(p.b_rows));
}

}  // namespace gemm
}  // namespace dear

namespace {
uint64_t* g_trace = nullptr;  // device buffer: 8 timestamps per CTA (profiling only)
}

using dear::Error;

namespace {

}  // namespace

namespace dear {
namespace gemm {
void set_smem_attr() {
  static bool done = false;
  if (!done) {
    if (cudaFuncSetAttribute(gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes) != cudaSuccess ||
        cudaFuncSetAttribute(gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes) != cudaSuccess)
      throw Error(DEAR_EINTERNAL, "cudaFuncSetAttribute(gemm smem)");
    if (cudaFuncSetAttribute(gemm_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                             1) != cudaSuccess)
      (void)cudaGetLastError();
    done = true;
  }
}

int max_active_clusters(int csize, bool pair) {
  static int cache[2][17] = {{0}};
  if (csize <= 1) return kSms * DEAR_GEMM_CTAS_PER_SM;
  if (cache[pair][csize]) return cache[pair][csize];
  set_smem_attr();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(csize * (kSms / csize)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(csize);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, pair ? gemm_kernel<true> : gemm_kernel<false>, &cfg) !=
          cudaSuccess ||
      n < 1) {
    (void)cudaGetLastError();
    n = kSms / csize / 2;
  }
  cache[pair][csize] = n;
  return n;
}
}  // namespace gemm
}  // namespace dear

namespace {

void launch(const dear::gemm::Launch& L, cudaStream_t stream) {
  using namespace dear::gemm;
  set_smem_attr();
  const int csize = L.pair ? 2 : L.cm * L.cn;
  // DEAR_GEMM_MAX_CTAS caps the persistent grid (leaves SMs to comm kernels).
  static const int cap = [] {
    const char* e = std::getenv("DEAR_GEMM_MAX_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  int resident = dear::gemm::max_active_clusters(csize, L.pair != 0);
  if (cap > 0) resident = std::max(1, std::min(resident, cap / csize));
  const int clusters = std::min(L.total_tiles, resident);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * csize));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = static_cast<unsigned>(csize);
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = csize > 1 ? 2 : 1;
  const cudaError_t e = L.pair ? cudaLaunchKernelEx(&cfg, gemm_kernel<true>, L)
                               : cudaLaunchKernelEx(&cfg, gemm_kernel<false>, L);
  if (e != cudaSuccess) throw Error(DEAR_EINTERNAL, std::string("gemm launch: ") + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int dear_gemm_plan_create(const void* A, int64_t lda, const void* B, int64_t ldb,
                          int32_t b_mn_major, void* D, int64_t ldd, int32_t d_fp32, int64_t M,
                          int64_t N, int64_t K, int64_t d_limit, int32_t accumulate,
                          int32_t split_k, dear_gemm_plan** out) {
  DEAR_API_BEGIN
  using namespace dear::gemm;
  if (!A || !B || !D || !out) throw Error(DEAR_EINVAL, "dear_gemm: null pointer");
  if (M <= 0 || N <= 0 || K <= 0) throw Error(DEAR_EINVAL, "dear_gemm: M, N, K must be > 0");
  if (lda % 8 || ldb % 8 || lda < K || (!b_mn_major && ldb < K) || (b_mn_major && ldb < N))
    throw Error(DEAR_EINVAL, "dear_gemm: leading dimensions must be multiples of 8 and cover the matrix");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    throw Error(DEAR_EINVAL, "dear_gemm: A and B must be 16-byte aligned");
  if (ldd < N) throw Error(DEAR_EINVAL, "dear_gemm: ldd < N");
  if (accumulate && !d_fp32) throw Error(DEAR_EINVAL, "dear_gemm: accumulate needs fp32 D");
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    throw Error(DEAR_EINVAL, "dear_gemm: dimensions exceed 2^31");
  if (!accumulate && split_k > 1) throw Error(DEAR_EINVAL, "dear_gemm: split_k > 1 needs accumulate");
  auto* plan = new dear_gemm_plan();
  Problem& p = plan->p;
  const int num_kb = static_cast<int>((K + kBK - 1) / kBK);
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  int splits = 1;
  if (accumulate) {
    if (split_k > 0) {
      splits = split_k;
    } else {
      // Enough (split) tiles for the persistent grid, but keep >= 16 k-blocks
      // (K >= 1024) per split so the fp32 reductions stay a small fraction of
      // the operand traffic.
      const int64_t nt = (N + kBNMax - 1) / kBNMax;
      const int64_t tiles = m_tiles * nt;
      splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kSms / tiles, num_kb / 16)));
    }
    splits = std::max(1, std::min(splits, num_kb));
  }
  const int kb_per = (num_kb + splits - 1) / splits;
  splits = (num_kb + kb_per - 1) / kb_per;
  // Clusters are opt-in (DEAR_GEMM_CLUSTER=1): on the per-layer shapes they cut
  // L2->SM traffic but their scheduling spread costs more than they save
  // (profiles/r01_gemm_trace.md).
  const char* env = std::getenv("DEAR_GEMM_CLUSTER");
  const bool clusters = env && env[0] == '1';
  // CTA pairs are on by default (DEAR_GEMM_PAIR=0 disables, =2 forces them).
  const char* penv = std::getenv("DEAR_GEMM_PAIR");
  const bool pairs = !(penv && penv[0] == '0');
  const int modes = (penv && penv[0] == '2')
                        ? kModePair
                        : kModeSingle | (pairs ? kModePair : 0) | (clusters ? kModeCluster : 0);
  TileChoice tch = choose_tiles(M, N, kb_per, splits, b_mn_major != 0, modes);
  if (const char* fb = std::getenv("DEAR_GEMM_BN")) {  // tuning experiments only
    const int v = std::atoi(fb);
    if (v >= 16 && v <= 256 && v % 16 == 0 &&
        !(tch.pair && b_mn_major && v != 128 && v != 256))
      tch = {v, tch.pair ? 2 : 1, 1, tch.pair};
  }
  p.D = D;
  p.ldd = ldd;
  p.M = M;
  p.N = N;
  p.d_limit = d_limit;
  p.num_kb = num_kb;
  p.kb_per_split = kb_per;
  p.splits = splits;
  p.m_tiles = static_cast<int32_t>(m_tiles);
  p.b_mn_major = b_mn_major ? 1 : 0;
  p.d_fp32 = d_fp32 ? 1 : 0;
  p.accumulate = accumulate ? 1 : 0;
  plan->A = A;
  plan->B = B;
  plan->lda = lda;
  plan->ldb = ldb;
  plan->K = K;
  // TMA-store epilogue for bf16, non-accumulating D (16 B aligned rows).
  const char* tenv = std::getenv("DEAR_GEMM_TMA_STORE");
  p.d_tma = (!d_fp32 && !accumulate && ldd % 8 == 0 &&
             (reinterpret_cast<uintptr_t>(D) & 15) == 0 && !(tenv && tenv[0] == '0'))
                ? 1
                : 0;
  // fp32 accumulate: TMA reduce-add over the complete rows under the flat
  // limit (rows r with r*ldd + N <= d_limit); a partial row after them is
  // added by red.add in the epilogue.
  p.r_full = INT64_MAX;
  p.d_lim_rows = M;
  const char* renv = std::getenv("DEAR_GEMM_TMA_REDUCE");
  if (!p.d_tma && d_fp32 && accumulate && ldd % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(D) & 15) == 0 && !(tenv && tenv[0] == '0') &&
      !(renv && renv[0] == '0')) {
    int64_t full = M;
    if (d_limit >= 0) full = d_limit >= N ? std::min<int64_t>(M, (d_limit - N) / ldd + 1) : 0;
    if (full > 0) {
      p.d_tma = 2;
      p.tma_reduce_ok = 1;
      p.d_lim_rows = full;
      if (d_limit >= 0 && full < M && full * ldd < d_limit) p.r_full = full;
    }
  }
  try {
    if (p.d_tma == 2) {
      make_map(&p.tmD, D, static_cast<uint64_t>(N), static_cast<uint64_t>(p.d_lim_rows),
               static_cast<uint64_t>(ldd), 16, 32, CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
    } else if (p.d_tma) {
      make_map(&p.tmD, D, static_cast<uint64_t>(N), static_cast<uint64_t>(M),
               static_cast<uint64_t>(ldd), 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
      make_map(&p.tmD16, D, static_cast<uint64_t>(N), static_cast<uint64_t>(M),
               static_cast<uint64_t>(ldd), 16, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    }
    configure(plan, tch);
  } catch (...) {
    delete plan;
    throw;
  }
  *out = plan;
  DEAR_API_END
}

int dear_gemm_run_group(dear_gemm_plan* const* plans, int32_t n, void* stream) {
  DEAR_API_BEGIN
  using namespace dear::gemm;
  if (!plans || n < 1 || n > kMaxProblems) throw Error(DEAR_EINVAL, "dear_gemm_run_group: 1 or 2 plans");
  if (n == 2 && plans[0] && plans[1] &&
      (plans[0]->p.cm != plans[1]->p.cm || plans[0]->p.cn != plans[1]->p.cn ||
       plans[0]->p.pair != plans[1]->p.pair)) {
    // Different cluster shapes cannot share a launch.
    const int r0 = dear_gemm_run_group(plans, 1, stream);
    if (r0 != DEAR_OK) return r0;
    return dear_gemm_run_group(plans + 1, 1, stream);
  }
  Launch L;
  L.n_problems = n;
  L.total_tiles = 0;
  int b_stage = 0;
  for (int i = 0; i < n; ++i) {
    if (!plans[i]) throw Error(DEAR_EINVAL, "dear_gemm_run_group: null plan");
    L.p[i] = plans[i]->p;
    L.total_tiles += plans[i]->p.tiles;
    const Problem& P = plans[i]->p;
    const int b_rows = P.pair ? P.bn / 2 : P.bn;  // pair: this CTA's half of B
    const int bs = P.b_mn_major ? P.b_boxes * 8192 : (b_rows * kBK * 2 + 1023) / 1024 * 1024;
    b_stage = std::max(b_stage, bs);
  }
  L.stage_bytes = kAStage + b_stage;
#ifdef DEAR_GEMM_FIXED_STAGES
  L.stage_bytes = kAStage + kBStage;
  L.stages = DEAR_GEMM_FIXED_STAGES;
#else
  L.stages = std::min(kMaxStages, kRingBytes / L.stage_bytes);
#endif
  L.cm = plans[0]->p.cm;
  L.cn = plans[0]->p.cn;
  L.pair = plans[0]->p.pair;
  L.early = 1;
  for (int i = 0; i < n; ++i) L.early &= plans[i]->p.early_operands;
  L.trace = g_trace;
  launch(L, static_cast<cudaStream_t>(stream));
  DEAR_API_END
}

int dear_gemm_run(dear_gemm_plan* plan, void* stream) {
  return dear_gemm_run_group(&plan, 1, stream);
}

int dear_gemm_plan_info(dear_gemm_plan* plan, int32_t* bn, int32_t* n_tiles, int32_t* m_tiles,
                        int32_t* splits) {
  DEAR_API_BEGIN
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  if (bn) *bn = plan->p.bn;
  if (n_tiles) *n_tiles = plan->p.n_tiles;
  if (m_tiles) *m_tiles = plan->p.m_tiles;
  if (splits) *splits = plan->p.splits;
  DEAR_API_END
}

int dear_gemm_plan_cluster(dear_gemm_plan* plan, int32_t* cm, int32_t* cn, int32_t* resident) {
  DEAR_API_BEGIN
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  if (cm) *cm = plan->p.cm;
  if (cn) *cn = plan->p.cn;
  if (resident)
    *resident = plan->p.pair ? dear::gemm::max_active_clusters(2, true)
                             : dear::gemm::max_active_clusters(plan->p.cm * plan->p.cn);
  DEAR_API_END
}

int dear_gemm_plan_set_tile(dear_gemm_plan* plan, int32_t bn, int32_t pair) {
  DEAR_API_BEGIN
  using namespace dear::gemm;
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  if (bn < 16 || bn > kBNMax || bn % 16)
    throw Error(DEAR_EINVAL, "dear_gemm_plan_set_tile: bn must be a multiple of 16 in [16, 256]");
  if (pair && plan->p.b_mn_major && bn != 128 && bn != 256)
    throw Error(DEAR_EINVAL, "dear_gemm_plan_set_tile: MN-major B in CTA pairs needs bn 128 or 256");
  configure(plan, TileChoice{bn, 1, 1, pair ? 1 : 0});
  DEAR_API_END
}

int dear_gemm_plan_set_splits(dear_gemm_plan* plan, int32_t split_k) {
  DEAR_API_BEGIN
  using namespace dear::gemm;
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  Problem& p = plan->p;
  if (split_k < 1) throw Error(DEAR_EINVAL, "dear_gemm_plan_set_splits: split_k must be >= 1");
  if (split_k > 1 && !p.accumulate)
    throw Error(DEAR_EINVAL, "dear_gemm_plan_set_splits: split_k > 1 needs accumulate");
  const int splits = std::min<int>(split_k, p.num_kb);
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
  configure(plan, TileChoice{p.bn, p.pair ? 2 : p.cm, p.pair ? 1 : p.cn, p.pair});
  DEAR_API_END
}

int dear_gemm_plan_set_flags(dear_gemm_plan* plan, int32_t flags) {
  DEAR_API_BEGIN
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  if (flags & ~(DEAR_GEMM_EARLY_OPERANDS | DEAR_GEMM_RED_ADD))
    throw Error(DEAR_EINVAL, "dear_gemm_plan_set_flags: unknown flag");
  plan->p.early_operands = (flags & DEAR_GEMM_EARLY_OPERANDS) ? 1 : 0;
  if (plan->p.tma_reduce_ok) plan->p.d_tma = (flags & DEAR_GEMM_RED_ADD) ? 0 : 2;
  DEAR_API_END
}

int dear_gemm_plan_pair(dear_gemm_plan* plan, int32_t* pair) {
  DEAR_API_BEGIN
  if (!plan || !pair) throw Error(DEAR_EINVAL, "null plan");
  *pair = plan->p.pair;
  DEAR_API_END
}

int dear_gemm_set_trace(void* device_buffer) {
  DEAR_API_BEGIN
  g_trace = static_cast<uint64_t*>(device_buffer);
  DEAR_API_END
}

int dear_gemm_plan_destroy(dear_gemm_plan* plan) {
  DEAR_API_BEGIN
  delete plan;
  DEAR_API_END
}

}  // extern "C"
