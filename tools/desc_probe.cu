// Probe (B200, sm_100a): can a tcgen05.mma SMEM descriptor start at an arbitrary
// 128-byte row inside a 128B-swizzled, TMA-written K-major tile?  This decides
// whether a stride-1 convolution can reuse one resident input halo for every
// filter tap (A operand for tap (i, j) = the halo shifted by i*W + j rows).
//
// For each row shift r and each value of the descriptor's base-offset field,
// D = A[r : r+128, 0:64] * B[0:64, 0:64]^T is computed on the tensor core and
// compared with the host result.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -o tools/desc_probe tools/desc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe_k(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int shift,
                        int base_mode, float* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;                // 256 rows x 128 B
  uint8_t* sB = sm + 256 * 128;    // 64 rows x 128 B
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(256 * 128 + 64 * 128)
                 : "memory");
    for (int h = 0; h < 2; ++h)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              smem_u32(sA + h * 128 * 128)),
          "l"((uint64_t)&ta), "r"(smem_u32(&bar)), "r"(0), "r"(h * 128)
          : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(sB)),
        "l"((uint64_t)&tb), "r"(smem_u32(&bar)), "r"(0), "r"(0)
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.b32 %0, 1, 0, p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar))
                   : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t aaddr = smem_u32(sA) + shift * 128;
    const uint32_t base_off = base_mode == 0 ? 0u : base_mode == 1 ? ((aaddr >> 7) & 7u) : ((8u - ((aaddr >> 7) & 7u)) & 7u);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = (uint64_t)(((aaddr + kk * 32) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
                          ((uint64_t)1 << 46) | ((uint64_t)base_off << 49) | ((uint64_t)2 << 61);
      const uint64_t bd = (uint64_t)(((smem_u32(sB) + kk * 32) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) |
                          ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
      asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(kk)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  __syncthreads();
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.b32 %0, 1, 0, p;}"
                   : "=r"(ok)
                   : "r"(smem_u32(&mbar))
                   : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 8; ++q) out[row * 64 + c0 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  const int RA = 256;
  std::vector<__nv_bfloat16> ha(RA * 64), hb(64 * 64);
  std::vector<float> fa(RA * 64), fb(64 * 64);
  for (int i = 0; i < RA * 64; ++i) {
    fa[i] = (float)((i * 37 + 11) % 17 - 8) / 8.f;
    ha[i] = __float2bfloat16(fa[i]);
  }
  for (int i = 0; i < 64 * 64; ++i) {
    fb[i] = (float)((i * 13 + 5) % 11 - 5) / 4.f;
    hb[i] = __float2bfloat16(fb[i]);
  }
  __nv_bfloat16 *da, *db;
  float* dout;
  cudaMalloc(&da, ha.size() * 2);
  cudaMalloc(&db, hb.size() * 2);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap ta, tb;
  cuuint64_t dA[2] = {64, (cuuint64_t)RA}, dB[2] = {64, 64}, st[1] = {128};
  cuuint32_t boxA[2] = {64, 128}, boxB[2] = {64, 64}, es[2] = {1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, da, dA, st, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, db, dB, st, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(probe_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> got(128 * 64);
  const int shifts[] = {0, 1, 2, 3, 5, 7, 8, 13, 31, 57, 100};
  const char* modes[] = {"base_offset=0", "base_offset=(addr>>7)&7", "base_offset=(8-(addr>>7))&7"};
  for (int shift : shifts) {
    printf("shift %3d:", shift);
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(dout, 0, 128 * 64 * 4);
      probe_k<<<1, 128, 64 * 1024>>>(ta, tb, shift, mode, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("  [%s: CUDA error %s]\n", modes[mode], cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 64; ++k)
            ref += (double)__bfloat162float(ha[(m + shift) * 64 + k]) * __bfloat162float(hb[n * 64 + k]);
          maxerr = fmax(maxerr, fabs(ref - got[m * 64 + n]));
        }
      printf("  [%s: %s %.3g]", modes[mode], maxerr < 1e-3 ? "OK " : "BAD", maxerr);
    }
    printf("\n");
  }
  return 0;
}
