// Hand-written sm_100a GEMM: TMA (cp.async.bulk.tensor, 128B swizzle) ->
// 4-stage smem ring (mbarrier full/empty) -> tcgen05.mma (kind::f16, bf16 in,
// fp32 accumulate in TMEM, issued by one thread) -> tcgen05.ld epilogue.
//
// Warp roles per CTA (192 threads):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..5  epilogue: warp w reads TMEM lanes 32*(w%4) .. +31
// One CTA computes one 128 x BN output tile (BN <= 256, a multiple of 16
// chosen on the host to minimise N padding) over a K range; with
// `accumulate` the K range may be split across CTAs (grid.z) and partial
// tiles are reduced into fp32 D with red.global.add.v4.f32.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "dear_gemm.h"
#include "dear_internal.h"

namespace dear {
namespace gemm {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kBNMax = 256;
constexpr int kStages = 4;
constexpr int kAStage = kBM * kBK * 2;     // 16 KB
constexpr int kBStage = kBNMax * kBK * 2;  // 32 KB
constexpr int kThreads = 192;
constexpr int kTmemCols = 256;
constexpr int kSmemBytes = kStages * (kAStage + kBStage) + 1024 + 256;

struct Params {
  void* D;
  int64_t ldd;
  int64_t M, N;
  int64_t d_limit;
  int32_t num_kb;
  int32_t kb_per_split;
  int32_t bn;
  int32_t b_mn_major;
  int32_t d_fp32;
  int32_t accumulate;
  uint32_t idesc;
  int32_t b_boxes;
  uint32_t tx_bytes;
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  uint32_t polls = 0;
  do {
    // A pipeline bug must fail loudly (trap) rather than hang the GPU.
    if (++polls > (1u << 27)) __trap();
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
// this CTA's tile clipped to N) are not written.
__device__ __forceinline__ void store_row_chunk(const Params& p, int64_t row, int64_t col0,
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

__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBStage);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * p.bn;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kBM;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int kb1 = min(kb0 + p.kb_per_split, p.num_kb);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
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

  if (nkb > 0) {
    if (warp == 0) {
      if (lane == 0) {
        for (int i = 0; i < nkb; ++i) {
          const int s = i % kStages;
          const uint32_t ph = (i / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], p.tx_bytes);
          const int kc = (kb0 + i) * kBK;
          tma_load_2d(&tmA, &full[s], sA + s * kAStage, kc, static_cast<int32_t>(m0));
          if (!p.b_mn_major) {
            tma_load_2d(&tmB, &full[s], sB + s * kBStage, kc, static_cast<int32_t>(n0));
          } else {
            for (int j = 0; j < p.b_boxes; ++j)
              tma_load_2d(&tmB, &full[s], sB + s * kBStage + j * 8192,
                          static_cast<int32_t>(n0 + 64 * j), kc);
          }
        }
      }
    } else if (warp == 1) {
      if (lane == 0) {
        for (int i = 0; i < nkb; ++i) {
          const int s = i % kStages;
          const uint32_t ph = (i / kStages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * kAStage);
          const uint32_t b_base = smem_u32(sB + s * kBStage);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = sdesc(a_base + k * 32, 16, 1024);
            const uint64_t bd = p.b_mn_major ? sdesc(b_base + k * 2048, 8192, 1024)
                                             : sdesc(b_base + k * 32, 16, 1024);
            umma_bf16(tmem, ad, bd, p.idesc, (i | k) != 0);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(tmem_full);
      }
      __syncwarp();
    } else {
      mbar_wait(tmem_full, 0);
      tc_fence_after();
      const int q = warp & 3;
      const int64_t row = m0 + 32 * q + lane;
      const int64_t col_end = min(p.N, n0 + p.bn);
      for (int c = 0; c < p.bn; c += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(c), v);
        store_row_chunk(p, row, n0 + c, col_end, v);
      }
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

}  // namespace gemm
}  // namespace dear

struct dear_gemm_plan {
  alignas(64) CUtensorMap a;
  alignas(64) CUtensorMap b;
  dear::gemm::Params p;
  dim3 grid;
};

using dear::Error;

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
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes) != cudaSuccess)
      throw Error(DEAR_EINTERNAL, "cudaFuncSetAttribute(gemm smem)");
    attr = true;
  }
  auto* plan = new dear_gemm_plan();
  Params& p = plan->p;
  const int64_t n_tiles = (N + kBNMax - 1) / kBNMax;
  int64_t bn = (N + n_tiles - 1) / n_tiles;
  bn = (bn + 15) / 16 * 16;
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  const int num_kb = static_cast<int>((K + kBK - 1) / kBK);
  int splits = 1;
  if (accumulate) {
    const int64_t tiles = n_tiles * m_tiles;
    splits = split_k > 0 ? split_k : static_cast<int>(tiles < 148 ? 148 / tiles : 1);
    if (splits < 1) splits = 1;
    if (splits > num_kb) splits = num_kb;
  } else if (split_k > 1) {
    delete plan;
    throw Error(DEAR_EINVAL, "dear_gemm: split_k > 1 needs accumulate");
  }
  int kb_per = (num_kb + splits - 1) / splits;
  splits = (num_kb + kb_per - 1) / kb_per;
  p.D = D;
  p.ldd = ldd;
  p.M = M;
  p.N = N;
  p.d_limit = d_limit;
  p.num_kb = num_kb;
  p.kb_per_split = kb_per;
  p.bn = static_cast<int32_t>(bn);
  p.b_mn_major = b_mn_major ? 1 : 0;
  p.d_fp32 = d_fp32 ? 1 : 0;
  p.accumulate = accumulate ? 1 : 0;
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(p.b_mn_major) << 16) |
            (static_cast<uint32_t>(bn >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
  p.b_boxes = static_cast<int32_t>((bn + 63) / 64);
  p.tx_bytes = kAStage + (b_mn_major ? p.b_boxes * 8192 : static_cast<uint32_t>(bn) * kBK * 2);
  try {
    make_map(&plan->a, A, static_cast<uint64_t>(K), static_cast<uint64_t>(M),
             static_cast<uint64_t>(lda), kBK, kBM);
    if (!b_mn_major)
      make_map(&plan->b, B, static_cast<uint64_t>(K), static_cast<uint64_t>(N),
               static_cast<uint64_t>(ldb), kBK, static_cast<uint32_t>(bn));
    else
      make_map(&plan->b, B, static_cast<uint64_t>(N), static_cast<uint64_t>(K),
               static_cast<uint64_t>(ldb), 64, kBK);
  } catch (...) {
    delete plan;
    throw;
  }
  plan->grid = dim3(static_cast<unsigned>(n_tiles), static_cast<unsigned>(m_tiles),
                    static_cast<unsigned>(splits));
  *out = plan;
  DEAR_API_END
}

int dear_gemm_run(dear_gemm_plan* plan, void* stream) {
  DEAR_API_BEGIN
  using namespace dear::gemm;
  if (!plan) throw Error(DEAR_EINVAL, "dear_gemm_run: null plan");
  gemm_kernel<<<plan->grid, kThreads, kSmemBytes, static_cast<cudaStream_t>(stream)>>>(
      plan->a, plan->b, plan->p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(DEAR_EINTERNAL, std::string("gemm launch: ") + cudaGetErrorString(e));
  DEAR_API_END
}

int dear_gemm_plan_info(dear_gemm_plan* plan, int32_t* bn, int32_t* n_tiles, int32_t* m_tiles,
                        int32_t* splits) {
  DEAR_API_BEGIN
  if (!plan) throw Error(DEAR_EINVAL, "null plan");
  if (bn) *bn = plan->p.bn;
  if (n_tiles) *n_tiles = static_cast<int32_t>(plan->grid.x);
  if (m_tiles) *m_tiles = static_cast<int32_t>(plan->grid.y);
  if (splits) *splits = static_cast<int32_t>(plan->grid.z);
  DEAR_API_END
}

int dear_gemm_plan_destroy(dear_gemm_plan* plan) {
  DEAR_API_BEGIN
  delete plan;
  DEAR_API_END
}

}  // extern "C"
