// Hand-written sm_100a GEMM for the synthetic layer compute.
//
//   TMA (cp.async.bulk.tensor.2d, 128B swizzle) -> 4..8-stage smem ring
//   (mbarrier full/empty) -> tcgen05.mma kind::f16 (bf16 in, fp32 accumulate
//   in TMEM, issued by one thread) -> tcgen05.ld epilogue -> global.
//
// Persistent: one CTA per SM walks a static round-robin list of output tiles
// (128 x BN, BN <= 256 a multiple of 16 chosen per problem). TMEM holds two
// 256-column accumulators, so the epilogue of tile i overlaps the mainloop of
// tile i+1. A launch may carry up to two independent problems (the wgrad and
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
#include <string>

#include "dear_gemm.h"
#include "dear_internal.h"

namespace dear {
namespace gemm {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kBNMax = 256;
constexpr int kMaxStages = 8;
constexpr int kAStage = kBM * kBK * 2;     // 16 KB
constexpr int kBStage = kBNMax * kBK * 2;  // 32 KB (widest B stage)
constexpr int kRingBytes = 4 * (kAStage + kBStage);  // 192 KB: 4..8 stages by BN
constexpr int kThreads = 192;
constexpr int kAccCols = 256;
constexpr int kTmemCols = 2 * kAccCols;
constexpr int kSmemBytes = kRingBytes + 1024 + 256;
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
};

struct Launch {
  Problem p[kMaxProblems];
  int32_t n_problems;
  int32_t total_tiles;
  int32_t stages;       // smem ring depth (narrow B tiles -> deeper ring)
  int32_t stage_bytes;  // A (16 KB) + widest B of the problems, 1 KB aligned
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

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
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

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
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

// Tile t of the launch: problems back to back; inside a problem
// (split, m_tile, n_tile) with n fastest, so concurrently running CTAs share
// the same A rows.
__device__ __forceinline__ TileCoord decode(const Launch& L, int t) {
  TileCoord c;
  c.prob = (L.n_problems > 1 && t >= L.p[0].tiles) ? 1 : 0;
  const Problem& P = L.p[c.prob];
  const int local = c.prob ? t - L.p[0].tiles : t;
  const int per = P.m_tiles * P.n_tiles;
  const int split = local / per;
  const int r = local - split * per;
  c.m0 = static_cast<int64_t>(r / P.n_tiles) * kBM;
  c.n0 = static_cast<int64_t>(r % P.n_tiles) * P.bn;
  c.kb0 = split * P.kb_per_split;
  c.kb1 = min(c.kb0 + P.kb_per_split, P.num_kb);
  return c;
}

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

  // Let the next kernel in the stream start its prologue as soon as SMs free.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < L.n_problems; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&L.p[i].tmA))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&L.p[i].tmB))
                   : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Everything above overlaps the previous kernel; memory is touched only now.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < L.total_tiles; t += gridDim.x) {
        const TileCoord tc = decode(L, t);
        const Problem& P = L.p[tc.prob];
        for (int kb = tc.kb0; kb < tc.kb1; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], P.tx_bytes);
          const int kc = kb * kBK;
          uint8_t* sA = smem + s * stage_bytes;
          uint8_t* sB = sA + kAStage;
          tma_load_2d(&P.tmA, &full[s], sA, kc, static_cast<int32_t>(tc.m0));
          if (!P.b_mn_major) {
            tma_load_2d(&P.tmB, &full[s], sB, kc, static_cast<int32_t>(tc.n0));
          } else {
            for (int j = 0; j < P.b_boxes; ++j)
              tma_load_2d(&P.tmB, &full[s], sB + j * 8192, static_cast<int32_t>(tc.n0 + 64 * j),
                          kc);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      uint32_t g = 0, j = 0;
      for (int t = blockIdx.x; t < L.total_tiles; t += gridDim.x, ++j) {
        const TileCoord tc = decode(L, t);
        const Problem& P = L.p[tc.prob];
        const uint32_t acc = j & 1, aph = (j >> 1) & 1;
        mbar_wait(&tmem_empty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * kAccCols;
        for (int kb = tc.kb0; kb < tc.kb1; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * stage_bytes);
          const uint32_t b_base = a_base + kAStage;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = P.b_mn_major ? sdesc(b_base + k * 2048, 8192, 1024)
                                             : sdesc(b_base + k * 32, 16, 1024);
            umma_bf16(d_tmem, ad, bd, P.idesc, (kb != tc.kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[acc]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    uint32_t j = 0;
    for (int t = blockIdx.x; t < L.total_tiles; t += gridDim.x, ++j) {
      const TileCoord tc = decode(L, t);
      const Problem& P = L.p[tc.prob];
      const uint32_t acc = j & 1, aph = (j >> 1) & 1;
      mbar_wait(&tmem_full[acc], aph);
      tc_fence_after();
      const int64_t row = tc.m0 + 32 * q + lane;
      const int64_t col_end = min(P.N, tc.n0 + P.bn);
      const uint32_t base = tmem + acc * kAccCols + (static_cast<uint32_t>(32 * q) << 16);
      for (int c = 0; c < P.bn; c += 32) {
        uint32_t v[32];
        tmem_ld32(base + static_cast<uint32_t>(c), v);
        store_row_chunk(P, row, tc.n0 + c, col_end, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
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
              uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw Error(DEAR_EINTERNAL, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  }
}

// Tile width: the fewest N tiles (<= 256 wide) unless more, narrower tiles
// fill the persistent grid markedly better (fewer waves of work per SM).
int choose_bn(int64_t M, int64_t N, int splits) {
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  auto waves_cost = [&](int64_t bn) {
    const int64_t nt = (N + bn - 1) / bn;
    const int64_t tiles = m_tiles * nt * splits;
    const int64_t waves = (tiles + kSms - 1) / kSms;
    // per-tile mainloop cost ~ max(bn, 64) columns + fixed overhead
    return waves * (std::max<int64_t>(bn, 64) + 48);
  };
  const int64_t nt0 = (N + kBNMax - 1) / kBNMax;
  int64_t best_bn = ((N + nt0 - 1) / nt0 + 15) / 16 * 16;
  int64_t best = waves_cost(best_bn);
  for (int64_t nt = nt0 + 1; nt <= nt0 * 4; ++nt) {
    const int64_t bn = ((N + nt - 1) / nt + 15) / 16 * 16;
    if (bn < 64) break;
    const int64_t c = waves_cost(bn);
    if (c < best) {
      best = c;
      best_bn = bn;
    }
  }
  return static_cast<int>(best_bn);
}

}  // namespace gemm
}  // namespace dear

struct dear_gemm_plan {
  dear::gemm::Problem p;
};

using dear::Error;

namespace {

void launch(const dear::gemm::Launch& L, cudaStream_t stream) {
  using namespace dear::gemm;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes) != cudaSuccess)
      throw Error(DEAR_EINTERNAL, "cudaFuncSetAttribute(gemm smem)");
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min(L.total_tiles, kSms)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_kernel, L);
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
  const int bn = choose_bn(M, N, splits);
  p.D = D;
  p.ldd = ldd;
  p.M = M;
  p.N = N;
  p.d_limit = d_limit;
  p.num_kb = num_kb;
  p.kb_per_split = kb_per;
  p.splits = splits;
  p.bn = bn;
  p.m_tiles = static_cast<int32_t>(m_tiles);
  p.n_tiles = static_cast<int32_t>((N + bn - 1) / bn);
  p.tiles = p.m_tiles * p.n_tiles * splits;
  p.b_mn_major = b_mn_major ? 1 : 0;
  p.d_fp32 = d_fp32 ? 1 : 0;
  p.accumulate = accumulate ? 1 : 0;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(p.b_mn_major) << 16) |
            (static_cast<uint32_t>(bn >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
  p.b_boxes = (bn + 63) / 64;
  p.tx_bytes = kAStage + (b_mn_major ? p.b_boxes * 8192 : static_cast<uint32_t>(bn) * kBK * 2);
  try {
    make_map(&p.tmA, A, static_cast<uint64_t>(K), static_cast<uint64_t>(M),
             static_cast<uint64_t>(lda), kBK, kBM);
    if (!b_mn_major)
      make_map(&p.tmB, B, static_cast<uint64_t>(K), static_cast<uint64_t>(N),
               static_cast<uint64_t>(ldb), kBK, static_cast<uint32_t>(bn));
    else
      make_map(&p.tmB, B, static_cast<uint64_t>(N), static_cast<uint64_t>(K),
               static_cast<uint64_t>(ldb), 64, kBK);
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
  Launch L;
  L.n_problems = n;
  L.total_tiles = 0;
  int b_stage = 0;
  for (int i = 0; i < n; ++i) {
    if (!plans[i]) throw Error(DEAR_EINVAL, "dear_gemm_run_group: null plan");
    L.p[i] = plans[i]->p;
    L.total_tiles += plans[i]->p.tiles;
    const Problem& P = plans[i]->p;
    const int bs = P.b_mn_major ? P.b_boxes * 8192 : (P.bn * kBK * 2 + 1023) / 1024 * 1024;
    b_stage = std::max(b_stage, bs);
  }
  L.stage_bytes = kAStage + b_stage;
  L.stages = std::min(kMaxStages, kRingBytes / L.stage_bytes);
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

int dear_gemm_plan_destroy(dear_gemm_plan* plan) {
  DEAR_API_BEGIN
  delete plan;
  DEAR_API_END
}

}  // extern "C"
