// Operand loaders and epilogues of the implicit GEMMs (fp32 verification path),
// plus the deterministic split-K / bias-gradient reductions shared by all paths.
#pragma once
#include "common.cuh"

namespace pc {

constexpr long long kNoBlock = 1LL << 62;

// A(r, k) with k contiguous in a (possibly channel-blocked) row-major matrix.
template <typename T> struct DenseLoader {
  const T* p;
  Blocked v;
  __device__ __forceinline__ float operator()(long long r, long long k) const { return ld(p + v.at(r, k)); }
};
// A(r, k) = stored[k][r]: the operand is MN-major in memory.
template <typename T> struct DenseMNLoader {
  const T* p;
  Blocked v;
  __device__ __forceinline__ float operator()(long long r, long long k) const { return ld(p + v.at(k, r)); }
};

// im2col of an NHWC (channel-blocked) input: row = output pixel, col = (i, j, c).
template <typename T> struct ImColLoader {
  const T* x;
  pc_conv_geom g;
  __device__ __forceinline__ float operator()(long long m, long long k) const {
    int ox = (int)(m % g.Wo);
    long long t = m / g.Wo;
    int oy = (int)(t % g.Ho);
    long long b = t / g.Ho;
    int c = (int)(k % g.C);
    int t2 = (int)(k / g.C);
    int j = t2 % g.k, i = t2 / g.k;
    int iy = oy * g.stride + i - g.pad, ix = ox * g.stride + j - g.pad;
    if (iy < 0 || ix < 0 || iy >= g.H || ix >= g.W) return 0.f;
    long long pix = (b * g.H + iy) * g.W + ix;
    int blk = c / g.cs;
    return ld(x + blk * g.cstride + pix * g.cs + (c - blk * g.cs));
  }
};
template <typename T> struct ImColLoaderT {  // B(kc, pixel) = im2col(pixel, kc)
  ImColLoader<T> f;
  __device__ __forceinline__ float operator()(long long r, long long k) const { return f(k, r); }
};

// Transposed-conv gather for dgrad: row = input pixel (b, y, x), col = (i, j, n).
template <typename T> struct DgradColLoader {
  const T* gy;
  pc_conv_geom g;
  __device__ __forceinline__ float operator()(long long m, long long k) const {
    int x = (int)(m % g.W);
    long long t = m / g.W;
    int y = (int)(t % g.H);
    long long b = t / g.H;
    int n = (int)(k % g.N);
    int t2 = (int)(k / g.N);
    int j = t2 % g.k, i = t2 / g.k;
    int ny = y + g.pad - i, nx = x + g.pad - j;
    if (ny < 0 || nx < 0 || ny % g.stride || nx % g.stride) return 0.f;
    int oy = ny / g.stride, ox = nx / g.stride;
    if (oy >= g.Ho || ox >= g.Wo) return 0.f;
    return ld(gy + ((b * g.Ho + oy) * g.Wo + ox) * g.N + n);
  }
};
template <typename T> struct DgradWeightLoader {  // B(c, (i, j, n)) = w[n][i][j][c]
  const T* w;
  pc_conv_geom g;
  __device__ __forceinline__ float operator()(long long c, long long k) const {
    int n = (int)(k % g.N);
    int ij = (int)(k / g.N);
    return ld(w + ((long long)n * g.k * g.k + ij) * g.C + c);
  }
};

template <typename T> struct StoreEpi {
  T* out;
  Blocked v;
  const float* bias;
  const T* mask;
  bool relu;
  __device__ __forceinline__ void operator()(long long m, long long n, int, float acc) const {
    float val = bias ? acc + bias[n] : acc;
    if (relu) val = val > 0.f ? val : 0.f;
    long long idx = v.at(m, n);
    if (mask && !(ld(mask + idx) > 0.f)) val = 0.f;
    out[idx] = cvt<T>(val);
  }
};

struct PartialEpi {
  float* out;
  long long zstride;
  long long ldo;
  __device__ __forceinline__ void operator()(long long m, long long n, int z, float acc) const {
    out[z * zstride + m * ldo + n] = acc;
  }
};

// out[i] = sum_{z < splits} ws[z * n + i], ascending z (deterministic split-K).
int reduce_partials(const float* ws, int splits, long long n, float* out, cudaStream_t st,
                    const pc_sgd_fuse* upd = nullptr);

int apply_sgd(const float* g, long long n, const pc_sgd_fuse* upd, cudaStream_t st);

// Momentum-SGD update of 4 consecutive elements (i % 4 == 0; 16-byte aligned rows).
__device__ __forceinline__ void sgd_apply4(const pc_sgd_fuse& u, long long i, float4 g) {
  float4 p = *reinterpret_cast<float4*>(u.p + i), v = *reinterpret_cast<float4*>(u.v + i);
  v.x = u.momentum * v.x - u.lr * (g.x + u.weight_decay * p.x);
  v.y = u.momentum * v.y - u.lr * (g.y + u.weight_decay * p.y);
  v.z = u.momentum * v.z - u.lr * (g.z + u.weight_decay * p.z);
  v.w = u.momentum * v.w - u.lr * (g.w + u.weight_decay * p.w);
  p.x += v.x; p.y += v.y; p.z += v.z; p.w += v.w;
  *reinterpret_cast<float4*>(u.v + i) = v;
  *reinterpret_cast<float4*>(u.p + i) = p;
  if (u.p_lowp) {
    __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(u.p_lowp) + i);
    q[0] = __floats2bfloat162_rn(p.x, p.y);
    q[1] = __floats2bfloat162_rn(p.z, p.w);
  }
}

// Momentum-SGD update of one element (kernels.sgd_step arithmetic).
__device__ __forceinline__ void sgd_apply(const pc_sgd_fuse& u, long long i, float g) {
  float p = u.p[i], v = u.v[i];
  v = u.momentum * v - u.lr * (g + u.weight_decay * p);
  p += v;
  u.v[i] = v;
  u.p[i] = p;
  if (u.p_lowp) static_cast<__nv_bfloat16*>(u.p_lowp)[i] = __float2bfloat16_rn(p);
}
// Bias gradient: out[c] = sum_r g[r * N + c] (two-pass, fixed order). ws >= colsum_ws(P, N) floats.
long long colsum_ws(long long P, int N);
int colsum(const void* g, long long P, int N, int prec, float* out, float* ws, cudaStream_t st);

int simt_splits(int M, int N, long long K);

// fp32 verification GEMMs (simt_gemm.cu)
int simt_conv_forward(const pc_conv_geom& g, const void* x, const void* w, const float* bias, void* y,
                      int prec, int flags, cudaStream_t st);
int simt_conv_dgrad(const pc_conv_geom& g, const void* w, const void* gy, void* gx, const void* mask,
                    cudaStream_t st, int prec);
int simt_conv_wgrad(const pc_conv_geom& g, const void* x, const void* gy, float* gw, float* ws,
                    int splits, cudaStream_t st, int prec);
int simt_fc_forward(int B, int D, int U, const pc_mat& x, const void* w, const float* bias, void* y,
                    int prec, int flags, cudaStream_t st);
int simt_fc_dgrad(int B, int D, int U, const void* w, const void* gy, const pc_mat& gx, const void* mask,
                  cudaStream_t st, int prec);
int simt_fc_wgrad(int B, int D, int U, const pc_mat& x, const void* gy, float* gw, cudaStream_t st,
                  int prec);

}  // namespace pc
