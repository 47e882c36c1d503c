// TF32 tensor-core contractions for sm_100a (the "tf32" precision mode).
//
// Activations, weights and gradients stay float32 in HBM (the verification
// mode's layout); the contractions run on the 5th-generation tensor cores with
// tcgen05.mma kind::tf32 (10-bit mantissa operands, fp32 accumulation in TMEM).
// One warp-specialised persistent kernel (one CTA per SM, cta_group::1):
//   warp 0      TMA producer: A and B k-blocks of 32 fp32 (128-byte rows,
//               128B swizzle) into a STAGES-deep mbarrier ring
//   warp 1      TMEM allocator + elected-lane MMA issuer (4 x K=8 MMAs per stage)
//   warps 2-5   epilogue: tcgen05.ld 32 lanes x 32 columns, bias / ReLU /
//               ReLU-mask / channel-blocked fp32 store, or split-K partials
// Two TMEM accumulators (2 x BN columns) double-buffer the epilogue against
// the next tile's main loop.
//
// Operand modes (all K-blocks are 32 elements = 128 B; K-major tiles use the 128B
// swizzle, MN-major ones the 128B swizzle with 32-byte atoms that tf32 requires):
//   A_K    [M][K] K-major tile (FC x / gy, the explicit-im2col input layer)
//   A_MN   [K][M] MN-major 32-element chunks (weight gradients: gy^T)
//   A_I2C  TMA im2col of an NHWC (channel-blocked) activation, K = (tap, 32-ch chunk):
//          conv forward, and the data gradient as a stride-1 forward conv of gy
//          with the rotated filters
//   B_K    [N][K] K-major (weights)
//   B_MN   [K][N] MN-major (FC data / weight gradients)
//   B_I2C  TMA im2col, MN-major 32-channel chunks: the conv weight gradient
//          gw[n][(i, j, c)] = sum_pixels gy[p][n] x_im2col[p][(i, j, c)], written
//          straight into the device filter layout [N][kh][kw][C]
// Reductions over split-K slices are summed in slice order (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm_ops.cuh"
#include "tf32.cuh"

namespace pc {
namespace tf32 {

constexpr int BM = 128, BK = 32;           // BK fp32 = 128 B rows
constexpr int A_STAGE = BM * BK * 4;        // 16 KB
enum { A_K = 0, A_MN = 1, A_I2C = 2 };
enum { B_K = 0, B_MN = 1, B_I2C = 2 };
enum { E_STORE = 0, E_PART = 1 };

struct Params {
  CUtensorMap ta, tb;
  int M, N, num_kb, kps, splits, tiles_m, tiles_n, tiles;
  // A_I2C: k-block kb = (tap, chunk): tap = kb / cpt
  int a_k, a_cpt, a_cs, a_s, a_lo, a_Ho, a_Wo;
  // B_I2C: column n = tap * C + c
  int b_C, b_cs, b_k, b_s, b_lo, b_Ho, b_Wo;
  // tiled K-major operands over a channel-blocked K dimension (cb: block width)
  int a_cb, b_cb;
  // epilogue
  float* out;
  long long o_ld, o_cb, o_bstride;
  const float* bias;
  const float* mask;
  int relu;
  float* part;
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* m, uint64_t* bar, uint32_t dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_3d(const CUtensorMap* m, uint64_t* bar, uint32_t dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_i2c(const CUtensorMap* m, uint64_t* bar, uint32_t dst, int c, int w, int h,
                                        int n, int blk, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], {%8, %9, %10};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(blk), "h"(ow),
      "h"(oh), "h"((uint16_t)0)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// Shared-memory descriptor (sm100: version bit 46; layout type at bits 61-63):
//   K-major operands: 128B swizzle (type 2), SBO = 1024 B per 8-row group;
//   MN-major tf32 operands: "128B swizzle, 32-byte atoms" (type 1, TMA
//   SWIZZLE_128B_ATOM_32B) — the only MN-major layout the tf32 MMA accepts:
//   4-row (512 B) groups (SBO), LBO = stride of the 32-element MN chunks.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t type = 2) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (type << 61);
}
// D f32 (bits 4-5 = 1), A / B tf32 (format 2 at bits 7-9 / 10-12), majorness (bits 15 / 16), N >> 3, M >> 4
template <int BN, bool AMN, bool BMN>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) | ((BMN ? 1u : 0u) << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
  return 1024 + STAGES * (A_STAGE + BN * BK * 4) + (2 * STAGES + 4) * 8 + 16;
}

// ------------------------------------------------------------------ kernel
template <int AM, int BMODE, int EPI, int BN, int STAGES>
__global__ void __launch_bounds__(192, 1) tf32_gemm_k(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int B_STAGE = BN * BK * 4;
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 4);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tb)) : "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    int git = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int tm = t % p.tiles_m, r = t / p.tiles_m, tn = r % p.tiles_n, z = r / p.tiles_n;
      const int m0 = tm * BM, n0 = tn * BN;
      const int kb0 = z * p.kps, kb1 = min(p.num_kb, kb0 + p.kps);
      int a_b = 0, a_oy = 0, a_ox = 0;
      if constexpr (AM == A_I2C) {
        a_ox = m0 % p.a_Wo;
        const int q = m0 / p.a_Wo;
        a_oy = q % p.a_Ho;
        a_b = q / p.a_Ho;
      }
      int nvalid = BN / 32;
      if constexpr (BMODE == B_I2C) nvalid = min(BN / 32, (p.N - n0 + 31) / 32);
      for (int kb = kb0; kb < kb1; ++kb, ++git) {
        const int s = git % STAGES;
        mbar_wait(&empty[s], ((git / STAGES) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&full[s], A_STAGE + nvalid * 32 * BK * 4);
          const uint32_t dA = smem_u32(sA + s * A_STAGE), dB = smem_u32(sB + s * B_STAGE);
          const int k0 = kb * BK;
          if constexpr (AM == A_K) {
            tma_3d(&p.ta, &full[s], dA, k0 % p.a_cb, m0, k0 / p.a_cb);
          } else if constexpr (AM == A_MN) {
#pragma unroll
            for (int q = 0; q < BM / 32; ++q) tma_2d(&p.ta, &full[s], dA + q * (32 * BK * 4), m0 + 32 * q, k0);
          } else {
            const int tap = kb / p.a_cpt, c = (kb - tap * p.a_cpt) * BK;
            const int ki = tap / p.a_k, kj = tap - ki * p.a_k;
            tma_i2c(&p.ta, &full[s], dA, c % p.a_cs, a_ox * p.a_s + p.a_lo, a_oy * p.a_s + p.a_lo, a_b, c / p.a_cs,
                    (uint16_t)kj, (uint16_t)ki);
          }
          if constexpr (BMODE == B_K) {
            tma_3d(&p.tb, &full[s], dB, k0 % p.b_cb, n0, k0 / p.b_cb);
          } else if constexpr (BMODE == B_MN) {
#pragma unroll
            for (int q = 0; q < BN / 32; ++q) tma_3d(&p.tb, &full[s], dB + q * (32 * BK * 4), (n0 + 32 * q) % p.b_cb,
                                                    k0, (n0 + 32 * q) / p.b_cb);
          } else {
            const int hw = p.b_Ho * p.b_Wo;
            const int pb = k0 / hw, rem = k0 - pb * hw, poy = rem / p.b_Wo, pox = rem - poy * p.b_Wo;
            for (int q = 0; q < nvalid; ++q) {
              const int col = n0 + 32 * q, tap = col / p.b_C, c = col - tap * p.b_C;
              const int ki = tap / p.b_k, kj = tap - ki * p.b_k;
              tma_i2c(&p.tb, &full[s], dB + q * (32 * BK * 4), c % p.b_cs, pox * p.b_s + p.b_lo,
                      poy * p.b_s + p.b_lo, pb, c / p.b_cs, (uint16_t)kj, (uint16_t)ki);
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr bool AMN = AM == A_MN, BMN = BMODE != B_K;
    constexpr uint32_t IDESC = idesc_tf32<BN, AMN, BMN>();
    // K-major: +32 B per K=8 step inside the 128-byte row; MN-major: +8 rows (1024 B)
    constexpr uint32_t A_KSTEP = (AMN ? 1024 : 32) >> 4, B_KSTEP = (BMN ? 1024 : 32) >> 4;
    const uint64_t a0 = AMN ? sdesc(smem_u32(sA), 32 * BK * 4, 512, 1) : sdesc(smem_u32(sA), 16, 1024);
    const uint64_t b0 = BMN ? sdesc(smem_u32(sB), 32 * BK * 4, 512, 1) : sdesc(smem_u32(sB), 16, 1024);
    int git = 0, lt = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++lt) {
      const int z = t / p.tiles_m / p.tiles_n;
      const int kb0 = z * p.kps, kb1 = min(p.num_kb, kb0 + p.kps);
      const int acc = lt & 1;
      mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
      fence_after();
      const uint32_t tacc = tmem + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb, ++git) {
        const int s = git % STAGES;
        mbar_wait(&full[s], (git / STAGES) & 1);
        fence_after();
        if (elect_one()) {
          const uint64_t ad = a0 + (uint64_t)((s * A_STAGE) >> 4), bd = b0 + (uint64_t)((s * B_STAGE) >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            mma_tf32(tacc, ad + kk * A_KSTEP, bd + kk * B_KSTEP, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    int lt = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++lt) {
      const int tm = t % p.tiles_m, r = t / p.tiles_m, tn = r % p.tiles_n, z = r / p.tiles_n;
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      fence_after();
      const long long m = (long long)tm * BM + quad * 32 + lane;
      const uint32_t tb = tmem + acc * BN + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tb + c0, v);
        const int n0 = tn * BN + c0;
        if (m >= p.M || n0 >= p.N) continue;
        const int nc = min(32, p.N - n0);
        if constexpr (EPI == E_PART) {
          float* o = p.part + ((long long)z * p.M + m) * p.N + n0;
          if (nc == 32 && (p.N & 3) == 0) {   // 128 contiguous bytes per lane: 8 x 16-byte stores
#pragma unroll
            for (int i = 0; i < 8; ++i)
              reinterpret_cast<float4*>(o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
            for (int i = 0; i < nc; ++i) o[i] = v[i];
          }
        } else if (nc == 32 && (p.o_cb & 31) == 0 && (n0 % p.o_cb) + 32 <= p.o_cb &&
                   ((p.o_ld | p.o_bstride) & 3) == 0) {
          // the 32 columns lie in one channel block: bias + ReLU + ReLU mask (16-byte mask
          // loads of the same layout), 8 x 16-byte stores
          const long long blk = n0 / p.o_cb;
          const long long off = blk * p.o_bstride + m * p.o_ld + (n0 - blk * p.o_cb);
          float* o = p.out + off;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float val = p.bias ? v[i] + p.bias[n0 + i] : v[i];
            v[i] = p.relu ? (val > 0.f ? val : 0.f) : val;
          }
          if (p.mask) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 mk = __ldg(reinterpret_cast<const float4*>(p.mask + off) + i);
              v[4 * i] = mk.x > 0.f ? v[4 * i] : 0.f;
              v[4 * i + 1] = mk.y > 0.f ? v[4 * i + 1] : 0.f;
              v[4 * i + 2] = mk.z > 0.f ? v[4 * i + 2] : 0.f;
              v[4 * i + 3] = mk.w > 0.f ? v[4 * i + 3] : 0.f;
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          for (int i = 0; i < nc; ++i) {
            const long long n = n0 + i;
            float val = p.bias ? v[i] + p.bias[n] : v[i];
            if (p.relu) val = val > 0.f ? val : 0.f;
            const long long blk = n / p.o_cb;
            const long long idx = blk * p.o_bstride + m * p.o_ld + (n - blk * p.o_cb);
            if (p.mask && !(p.mask[idx] > 0.f)) val = 0.f;
            p.out[idx] = val;
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 g_tiled = nullptr;
static PFN_cuTensorMapEncodeIm2col_v12000 g_i2c = nullptr;
static std::once_flag g_once;

static bool encoders() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_i2c = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  });
  return g_tiled && g_i2c;
}

// fp32 view {inner, rows, blocks} (strides ld, bstride elements), box {32, box_rows, 1}; 128B swizzle
// for K-major operands, 128B swizzle with 32-byte atoms for MN-major ones (mn = true)
static CUtensorMapSwizzle swz(bool mn) { return mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B; }
static bool map3(CUtensorMap* m, const void* ptr, long long inner, long long rows, long long blocks, long long ld,
                 long long bstride, int box_rows, bool mn = false) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ld % 4 || (blocks > 1 && bstride % 4) || box_rows > 256) return false;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(blocks > 1 ? bstride : ld * rows) * 4};
  cuuint32_t box[3] = {32u, (cuuint32_t)box_rows, 1u}, estr[3] = {1u, 1u, 1u};
  return g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz(mn), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool map2(CUtensorMap* m, const void* ptr, long long inner, long long rows, long long ld, int box_rows,
                 bool mn = false) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ld % 4) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows}, estr[2] = {1u, 1u};
  return g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz(mn), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// im2col view of a channel-blocked NHWC fp32 activation [nblk][B][H][W][cs]: each load
// walks `pixels` output positions x 32 channels.
static bool map_i2c(CUtensorMap* m, const void* ptr, int cs, int W, int H, int B, int nblk, long long cstride,
                    int pixels, int k, int s, int pad, bool mn = false) {
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || cs % 32 || (nblk > 1 && cstride % 4)) return false;
  cuuint64_t dims[5] = {(cuuint64_t)cs, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)nblk};
  cuuint64_t strides[4] = {(cuuint64_t)cs * 4, (cuuint64_t)W * cs * 4, (cuuint64_t)H * W * cs * 4,
                           (cuuint64_t)(nblk > 1 ? cstride : (long long)B * H * W * cs) * 4};
  int lower[3] = {-pad, -pad, 0}, upper[3] = {pad - (k - 1), pad - (k - 1), 0};
  cuuint32_t estr[5] = {1u, (cuuint32_t)s, (cuuint32_t)s, 1u, 1u};
  return g_i2c(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<void*>(ptr), dims, strides, lower, upper, 32u,
               (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz(mn),
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static std::atomic<unsigned long long> g_tf32_launches{0};

static int num_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}

template <int AM, int BMODE, int EPI, int BN>
static int launch_bn(Params& p, cudaStream_t st) {
  constexpr int STAGES = BN == 64 ? 8 : BN == 128 ? 6 : 4;
  constexpr int smem = smem_bytes<BN, STAGES>();
  static_assert(smem <= 227 * 1024, "tf32 stage ring exceeds shared memory");
  auto kern = tf32_gemm_k<AM, BMODE, EPI, BN, STAGES>;
  static bool init = false;
  if (!init) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "tf32 cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    init = true;
  }
  p.tiles_m = ceil_div(p.M, BM);
  p.tiles_n = ceil_div(p.N, BN);
  p.tiles = p.tiles_m * p.tiles_n * p.splits;
  const int grid = std::min(p.tiles, num_sms());
  kern<<<grid, 192, smem, st>>>(p);
  g_tf32_launches.fetch_add(1, std::memory_order_relaxed);
  PC_CUDA_CHECK_LAUNCH("tf32_gemm");
  return PC_OK;
}

// widest tile that still gives every SM a tile (N = 96 -> one 128-wide tile)
static int pick_bn(long long M, long long N, long long splits = 1) {
  const long long tm = ceil_div(M, BM) * splits;
  if (N > 128 && tm * ceil_div(N, 256) >= num_sms()) return 256;
  if (N > 64 || tm * ceil_div(N, 64) < num_sms() / 2) return 128;
  return 64;
}

template <int AM, int BMODE, int EPI>
static int dispatch(Params& p, int bn, cudaStream_t st) {
  if (bn == 256) return launch_bn<AM, BMODE, EPI, 256>(p, st);
  if (bn == 128) return launch_bn<AM, BMODE, EPI, 128>(p, st);
  return launch_bn<AM, BMODE, EPI, 64>(p, st);
}

static Params base(int M, int N, int K) {
  Params p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.num_kb = ceil_div(K, BK);
  p.kps = p.num_kb;
  p.splits = 1;
  p.a_cb = p.b_cb = 1 << 30;
  return p;
}

static void set_store(Params& p, float* out, long long ld, long long cb, long long bstride, const float* bias,
                      const float* mask, bool relu) {
  p.out = out;
  p.o_ld = ld;
  p.o_cb = cb;
  p.o_bstride = bstride;
  p.bias = bias;
  p.mask = mask;
  p.relu = relu ? 1 : 0;
}

// split-K for long reductions over few tiles (weight gradients): ~2 tiles per SM
static void set_splits(Params& p, int bn_guess) {
  const long long tiles = (long long)ceil_div(p.M, BM) * ceil_div(p.N, bn_guess);
  long long s = (2LL * num_sms() + tiles - 1) / tiles;
  s = std::min<long long>(s, std::max(1, p.num_kb / 8));
  s = std::max<long long>(1, std::min<long long>(s, 64));
  p.kps = ceil_div(p.num_kb, s);
  p.splits = ceil_div(p.num_kb, p.kps);
}

}  // namespace tf32

using namespace tf32;

bool tf32_conv_ok(const pc_conv_geom& g) {
  return encoders() && g.C % 32 == 0 && g.cs % 32 == 0 && g.N % 4 == 0 && (g.C == g.cs || g.cstride % 4 == 0);
}

int tf32_conv_forward(const pc_conv_geom& g, const float* x, const float* w, const float* bias, float* y, int flags,
                      cudaStream_t st) {
  const int M = g.B * g.Ho * g.Wo, K = g.k * g.k * g.C;
  Params p = base(M, g.N, K);
  const int bn = pick_bn(M, g.N);
  PC_REQUIRE(map_i2c(&p.ta, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, BM, g.k, g.stride, g.pad) &&
                 map3(&p.tb, w, K, g.N, 1, K, 0, bn),
             PC_ECUDA, "tf32 conv forward: tensor maps");
  p.a_k = g.k, p.a_cpt = g.C / BK, p.a_cs = g.cs, p.a_s = g.stride, p.a_lo = -g.pad, p.a_Ho = g.Ho, p.a_Wo = g.Wo;
  set_store(p, y, g.N, g.N, 0, bias, nullptr, (flags & PC_RELU) != 0);
  return dispatch<A_I2C, B_K, E_STORE>(p, bn, st);
}

// wt[c][i][j][n] = w[n][k-1-i][k-1-j][c]: the filters of the data gradient, per tap
// a 32 x 32 shared-memory tile transpose of [N][C] (coalesced on both sides)
__global__ void __launch_bounds__(256) tf32_dgrad_w_k(const float* __restrict__ w, float* __restrict__ wt, int N,
                                                      int KK, int C) {
  __shared__ float tile[32][33];
  const int ij = blockIdx.z, src = KK - 1 - ij;
  const int c0 = blockIdx.x * 32, n0 = blockIdx.y * 32, tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int n = n0 + r, c = c0 + tx;
    tile[r][tx] = (n < N && c < C) ? w[((long long)n * KK + src) * C + c] : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r, n = n0 + tx;
    if (c < C && n < N) wt[((long long)c * KK + ij) * N + n] = tile[tx][r];
  }
}

size_t tf32_dgrad_ws(const pc_conv_geom& g) { return ((size_t)g.N * g.k * g.k * g.C + 64) * sizeof(float); }

int tf32_conv_dgrad(const pc_conv_geom& g, const float* w, const float* gy, float* gx, const float* mask,
                    float* wt, cudaStream_t st) {
  PC_REQUIRE(g.stride == 1 && g.N % 32 == 0, PC_EVALUE, "tf32 data gradient: stride-1 conv, N %% 32 == 0");
  const int KK = g.k * g.k;
  tf32_dgrad_w_k<<<dim3((unsigned)ceil_div(g.C, 32), (unsigned)ceil_div(g.N, 32), (unsigned)KK), 256, 0, st>>>(
      w, wt, g.N, KK, g.C);
  PC_CUDA_CHECK_LAUNCH("tf32_dgrad_w");
  // forward conv of gy [B][Ho][Wo][N] (stride 1, pad k-1-p) with wt [C][k][k][N] -> gx [B][H][W][C]
  const int M = g.B * g.H * g.W, K = KK * g.N, pad = g.k - 1 - g.pad;
  Params p = base(M, g.C, K);
  const int bn = pick_bn(M, g.C);
  PC_REQUIRE(map_i2c(&p.ta, gy, g.N, g.Wo, g.Ho, g.B, 1, 0, BM, g.k, 1, pad) &&
                 map3(&p.tb, wt, K, g.C, 1, K, 0, bn),
             PC_ECUDA, "tf32 conv dgrad: tensor maps");
  p.a_k = g.k, p.a_cpt = g.N / BK, p.a_cs = g.N, p.a_s = 1, p.a_lo = -pad, p.a_Ho = g.H, p.a_Wo = g.W;
  set_store(p, gx, g.cs, g.cs, g.cstride, nullptr, mask, false);
  return dispatch<A_I2C, B_K, E_STORE>(p, bn, st);
}

long long tf32_wgrad_splits(const pc_conv_geom& g) {
  Params p = base(g.N, g.k * g.k * g.C, g.B * g.Ho * g.Wo);
  set_splits(p, g.k * g.k * g.C >= 256 ? 256 : 128);
  return p.splits;
}

int tf32_conv_wgrad(const pc_conv_geom& g, const float* x, const float* gy, float* gw, float* part, cudaStream_t st) {
  // gw[n][(i, j, c)] = sum_p gy[p][n] x_im2col[p][(i, j, c)]: A = gy (MN-major), B = im2col(x) (MN-major)
  const int P = g.B * g.Ho * g.Wo, NN = g.k * g.k * g.C;
  Params p = base(g.N, NN, P);
  set_splits(p, NN >= 256 ? 256 : 128);
  PC_REQUIRE(map2(&p.ta, gy, g.N, P, g.N, BK, true) &&
                 map_i2c(&p.tb, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, BK, g.k, g.stride, g.pad, true),
             PC_ECUDA, "tf32 conv wgrad: tensor maps");
  p.b_C = g.C, p.b_cs = g.cs, p.b_k = g.k, p.b_s = g.stride, p.b_lo = -g.pad, p.b_Ho = g.Ho, p.b_Wo = g.Wo;
  // 256-wide N tiles: 48 KB of operands per 128 x 256 x 32 MMA step instead of 32 KB per
  // 128 x 128 x 32 (the weight gradients are TMA-bound with 4-byte operands)
  const bool wide = NN >= 256;
  if (p.splits == 1) {
    set_store(p, gw, NN, NN, 0, nullptr, nullptr, false);
    return wide ? launch_bn<A_MN, B_I2C, E_STORE, 256>(p, st) : launch_bn<A_MN, B_I2C, E_STORE, 128>(p, st);
  }
  p.part = part;
  int rc = wide ? launch_bn<A_MN, B_I2C, E_PART, 256>(p, st) : launch_bn<A_MN, B_I2C, E_PART, 128>(p, st);
  if (rc) return rc;
  return reduce_partials(part, p.splits, (long long)g.N * NN, gw, st);
}

// ---------------------------------------------------------------- FC (and the explicit-im2col input layer)
bool tf32_fc_ok(int D, int U, const pc_mat& x) {
  return encoders() && D % 4 == 0 && U % 4 == 0 && x.ld % 4 == 0 && (x.cb >= D || x.cb % 32 == 0) &&
         (x.cb >= D || x.bstride % 4 == 0);
}

int tf32_fc_forward(int B, int D, int U, const pc_mat& x, const float* w, const float* bias, float* y, int flags,
                    cudaStream_t st) {
  // y[b][u] = x[b][:] . w[u][:]: A = x (K-major, channel-blocked K), B = w (K-major)
  Params p = base(B, U, D);
  const long long cb = x.cb >= D ? D : x.cb, nblk = (D + cb - 1) / cb;
  const int bn = pick_bn(B, U);
  PC_REQUIRE(map3(&p.ta, x.ptr, cb, B, nblk, x.ld, x.bstride, BM) && map3(&p.tb, w, D, U, 1, D, 0, bn), PC_ECUDA,
             "tf32 fc forward: tensor maps");
  p.a_cb = (int)cb;
  set_store(p, y, U, U, 0, bias, nullptr, (flags & PC_RELU) != 0);
  return dispatch<A_K, B_K, E_STORE>(p, bn, st);
}

int tf32_fc_dgrad(int B, int D, int U, const float* w, const float* gy, const pc_mat& gx, const float* mask,
                  cudaStream_t st) {
  // gx[b][d] = sum_u gy[b][u] w[u][d]: A = gy (K-major), B = w (MN-major: d contiguous)
  Params p = base(B, D, U);
  PC_REQUIRE(map3(&p.ta, gy, U, B, 1, U, 0, BM) && map3(&p.tb, w, D, U, 1, D, 0, BK, true), PC_ECUDA,
             "tf32 fc dgrad: tensor maps");
  p.b_cb = 1 << 30;
  const long long cb = gx.cb >= D ? D : gx.cb;
  set_store(p, static_cast<float*>(gx.ptr), gx.ld, cb, gx.bstride, nullptr, mask, false);
  return dispatch<A_K, B_MN, E_STORE>(p, pick_bn(B, D), st);
}

long long tf32_fc_wgrad_splits(int B, int D, int U) {
  Params p = base(U, D, B);
  set_splits(p, D >= 256 ? 256 : 128);
  return p.splits;
}

int tf32_fc_wgrad(int B, int D, int U, const pc_mat& x, const float* gy, float* gw, float* part, cudaStream_t st) {
  // gw[u][d] = sum_b gy[b][u] x[b][d]: A = gy (MN-major), B = x (MN-major, channel-blocked d)
  Params p = base(U, D, B);
  set_splits(p, D >= 256 ? 256 : 128);
  const long long cb = x.cb >= D ? D : x.cb, nblk = (D + cb - 1) / cb;
  PC_REQUIRE(map2(&p.ta, gy, U, B, U, BK, true) && map3(&p.tb, x.ptr, cb, B, nblk, x.ld, x.bstride, BK, true),
             PC_ECUDA,
             "tf32 fc wgrad: tensor maps");
  p.b_cb = (int)cb;
  const bool wide = D >= 256;
  if (p.splits == 1) {
    set_store(p, gw, D, D, 0, nullptr, nullptr, false);
    return wide ? launch_bn<A_MN, B_MN, E_STORE, 256>(p, st) : launch_bn<A_MN, B_MN, E_STORE, 128>(p, st);
  }
  p.part = part;
  int rc = wide ? launch_bn<A_MN, B_MN, E_PART, 256>(p, st) : launch_bn<A_MN, B_MN, E_PART, 128>(p, st);
  if (rc) return rc;
  return reduce_partials(part, p.splits, (long long)U * D, gw, st);
}

}  // namespace pc

extern "C" PC_API unsigned long long pc_tf32_contractions(void) { return pc::tf32::g_tf32_launches.load(); }
