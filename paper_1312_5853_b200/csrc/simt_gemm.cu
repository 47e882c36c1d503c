// fp32 verification path: exact-fp32 FFMA implicit GEMMs for conv and FC.
//
// This is the "fp32 mode" of the parity contract (<= 1e-5 relative against
// the float64 reference): plain fp32 fused multiply-adds in smem-tiled SIMT
// tiles. Plain TF32/bf16 tensor-core math cannot meet that bound,
// so this path deliberately stays off the tensor pipe. The bf16 production
// path is umma_gemm.cu.
//
// One generic kernel C[M,N] = sum_k A(m,k) B(n,k): the operand loaders are
// functors (im2col gather, transposed-conv gather, dense/blocked views) and
// the epilogue is a functor (bias/ReLU/mask store or split-K partial store).
#include "common.cuh"
#include "gemm_ops.cuh"

namespace pc {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16, S_NT = 256;

// ACC = double for the weight gradients: their reductions run over every pixel of
// the batch (AlexNet conv1 at B = 256: 774,400 terms, ~30k dependent adds per
// split-K slice); products of two floats are exact in double, so only the fp32
// operands' own rounding remains in the verification mode.
template <class AL, class BL, class EP, typename ACC = float>
__global__ void __launch_bounds__(S_NT) simt_gemm_k(int M, int N, int K, int kps, AL a, BL b, EP ep) {
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;
  const int kbeg = blockIdx.z * kps, kend = min(K, kbeg + kps);
  ACC acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += SB_K) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = t + S_NT * i, r = e / SB_K, kk = e % SB_K;
      int gk = k0 + kk;
      As[kk][r] = (m0 + r < M && gk < kend) ? a(m0 + r, gk) : 0.f;
      Bs[kk][r] = (n0 + r < N && gk < kend) ? b(n0 + r, gk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { av[i] = As[kk][ty * 4 + i]; bv[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (sizeof(ACC) == 8)
            acc[i][j] = fma((double)av[i], (double)bv[j], acc[i][j]);
          else
            acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) ep(m, n, blockIdx.z, (float)acc[i][j]);
    }
}

template <typename ACC = float, class AL, class BL, class EP>
int simt_gemm(int M, int N, int K, int splits, const AL& a, const BL& b, const EP& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0) return PC_OK;
  int kps = ceil_div(K, splits);
  kps = ceil_div(kps, SB_K) * SB_K;
  splits = ceil_div(K, kps);
  dim3 grid(ceil_div(N, SB_N), ceil_div(M, SB_M), splits > 0 ? splits : 1);
  simt_gemm_k<AL, BL, EP, ACC><<<grid, S_NT, 0, st>>>(M, N, K, kps, a, b, ep);
  PC_CUDA_CHECK_LAUNCH("simt_gemm");
  return PC_OK;
}

// Split-K count for a long reduction over K with few output tiles.
int simt_splits(int M, int N, long long K) {
  long long tiles = (long long)ceil_div(M, SB_M) * ceil_div(N, SB_N);
  long long want = (2 * 148 + tiles - 1) / tiles;
  long long cap = K / 1024;
  if (want > cap) want = cap;
  if (want > 64) want = 64;
  return (int)(want < 1 ? 1 : want);
}

#define SIMT_DISPATCH(prec, T, ...)                                         \
  do {                                                                      \
    if ((prec) == PC_FP32) { using T = float; __VA_ARGS__; }                \
    else if ((prec) == PC_BF16) { using T = __nv_bfloat16; __VA_ARGS__; }   \
    else { set_error("unknown precision"); return PC_EVALUE; }              \
  } while (0)

int simt_conv_forward(const pc_conv_geom& g, const void* x, const void* w, const float* bias, void* y,
                      int prec, int flags, cudaStream_t st) {
  int M = g.B * g.Ho * g.Wo, K = g.k * g.k * g.C;
  SIMT_DISPATCH(prec, T, {
    ImColLoader<T> a{static_cast<const T*>(x), g};
    DenseLoader<T> b{static_cast<const T*>(w), Blocked{K, kNoBlock, 0}};
    StoreEpi<T> ep{static_cast<T*>(y), Blocked{g.N, kNoBlock, 0}, bias, nullptr,
                   (flags & PC_RELU) != 0};
    return simt_gemm(M, g.N, K, 1, a, b, ep, st);
  });
}

int simt_conv_dgrad(const pc_conv_geom& g, const void* w, const void* gy, void* gx, const void* mask,
                    cudaStream_t st, int prec) {
  int M = g.B * g.H * g.W, K = g.k * g.k * g.N;
  SIMT_DISPATCH(prec, T, {
    DgradColLoader<T> a{static_cast<const T*>(gy), g};
    DgradWeightLoader<T> b{static_cast<const T*>(w), g};
    StoreEpi<T> ep{static_cast<T*>(gx), Blocked{g.cs, g.cs, g.cstride}, nullptr,
                   static_cast<const T*>(mask), false};
    return simt_gemm(M, g.C, K, 1, a, b, ep, st);
  });
}

int simt_conv_wgrad(const pc_conv_geom& g, const void* x, const void* gy, float* gw, float* ws,
                    int splits, cudaStream_t st, int prec) {
  int M = g.N, N = g.k * g.k * g.C, K = g.B * g.Ho * g.Wo;
  SIMT_DISPATCH(prec, T, {
    DenseMNLoader<T> a{static_cast<const T*>(gy), Blocked{g.N, kNoBlock, 0}};
    ImColLoaderT<T> b{ImColLoader<T>{static_cast<const T*>(x), g}};
    if (splits <= 1) {
      PartialEpi ep{gw, 0, N};
      return simt_gemm<double>(M, N, K, 1, a, b, ep, st);
    }
    PartialEpi ep{ws, (long long)M * N, N};
    int rc = simt_gemm<double>(M, N, K, splits, a, b, ep, st);
    if (rc) return rc;
    return reduce_partials(ws, splits, (long long)M * N, gw, st);
  });
}

int simt_fc_forward(int B, int D, int U, const pc_mat& x, const void* w, const float* bias, void* y,
                    int prec, int flags, cudaStream_t st) {
  SIMT_DISPATCH(prec, T, {
    DenseLoader<T> a{static_cast<const T*>(x.ptr), Blocked{x.ld, x.cb, x.bstride}};
    DenseLoader<T> b{static_cast<const T*>(w), Blocked{D, kNoBlock, 0}};
    StoreEpi<T> ep{static_cast<T*>(y), Blocked{U, kNoBlock, 0}, bias, nullptr,
                   (flags & PC_RELU) != 0};
    return simt_gemm(B, U, D, 1, a, b, ep, st);
  });
}

int simt_fc_dgrad(int B, int D, int U, const void* w, const void* gy, const pc_mat& gx, const void* mask,
                  cudaStream_t st, int prec) {
  SIMT_DISPATCH(prec, T, {
    DenseLoader<T> a{static_cast<const T*>(gy), Blocked{U, kNoBlock, 0}};
    DenseMNLoader<T> b{static_cast<const T*>(w), Blocked{D, kNoBlock, 0}};
    StoreEpi<T> ep{static_cast<T*>(gx.ptr), Blocked{gx.ld, gx.cb, gx.bstride}, nullptr,
                   static_cast<const T*>(mask), false};
    return simt_gemm(B, D, U, 1, a, b, ep, st);
  });
}

int simt_fc_wgrad(int B, int D, int U, const pc_mat& x, const void* gy, float* gw, cudaStream_t st,
                  int prec) {
  SIMT_DISPATCH(prec, T, {
    DenseMNLoader<T> a{static_cast<const T*>(gy), Blocked{U, kNoBlock, 0}};
    DenseMNLoader<T> b{static_cast<const T*>(x.ptr), Blocked{x.ld, x.cb, x.bstride}};
    PartialEpi ep{gw, 0, D};
    return simt_gemm<double>(U, D, B, 1, a, b, ep, st);
  });
}

}  // namespace pc
