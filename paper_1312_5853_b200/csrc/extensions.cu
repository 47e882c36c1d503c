// Layers beyond the reference: Krizhevsky's local response
// normalisation across channels and dropout with a counter-based SplitMix64
// mask. Definitions: oracle/ref_kernels.py (lrn_*, dropout_*) and
// paper_1312_5853_b200/rng.py (dropout_state / dropout_keep).
//
// LRN (NHWC, channels contiguous): one thread per (pixel, channel); the window
// sum re-reads the pixel's <= size neighbouring channels (L1 hits).
// Dropout: the keep decision of an element is recomputed from its dense index
// in both passes (no mask tensor), so the forward and backward agree bit for
// bit with each other and with rng.dropout_keep on the host.
#include "common.cuh"

namespace pc {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr unsigned long long GOLDEN = 0x9E3779B97F4A7C15ull;

// rng.derive(seed, DOMAIN_DROPOUT = 6, (step << 16) | layer).state
__device__ __forceinline__ unsigned long long dropout_state(unsigned long long seed, unsigned long long step,
                                                            int layer) {
  const unsigned long long s = mix64(seed ^ (6ull * GOLDEN));
  return mix64(s ^ (((step & 0xFFFFFFFFFFFFull) << 16) | (unsigned long long)(layer & 0xFFFF)));
}

template <typename T>
__global__ void lrn_fwd_k(long long P, int C, int h, float k, float alpha, float beta, const T* __restrict__ x,
                          T* __restrict__ y) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P * C) return;
  const long long pix = t / C;
  const int c = (int)(t - pix * C);
  const T* xp = x + pix * C;
  float s = 0.f;
  const int lo = c - h < 0 ? 0 : c - h, hi = c + h >= C ? C - 1 : c + h;
  for (int q = lo; q <= hi; ++q) {
    const float a = ld(xp + q);
    s += a * a;
  }
  const float a = ld(xp + c);
  y[t] = cvt<T>(a * powf(k + alpha * s, -beta));
}

template <typename T>
__global__ void lrn_bwd_k(long long P, int C, int h, float k, float alpha, float beta, const T* __restrict__ x,
                          const T* __restrict__ gy, T* __restrict__ gx) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P * C) return;
  const long long pix = t / C;
  const int c = (int)(t - pix * C);
  const T* xp = x + pix * C;
  const T* gp = gy + pix * C;
  auto scale = [&](int cc) {
    float s = 0.f;
    const int lo = cc - h < 0 ? 0 : cc - h, hi = cc + h >= C ? C - 1 : cc + h;
    for (int q = lo; q <= hi; ++q) {
      const float a = ld(xp + q);
      s += a * a;
    }
    return k + alpha * s;
  };
  // gx_c = g_c S_c^-b - 2 a b x_c sum_{|c'-c| <= h} g_c' x_c' S_c'^(-b-1)
  float win = 0.f;
  const int lo = c - h < 0 ? 0 : c - h, hi = c + h >= C ? C - 1 : c + h;
  for (int q = lo; q <= hi; ++q) win += ld(gp + q) * ld(xp + q) * powf(scale(q), -beta - 1.f);
  const float xc = ld(xp + c);
  gx[t] = cvt<T>(ld(gp + c) * powf(scale(c), -beta) - 2.f * alpha * beta * xc * win);
}

// NHWC slice [B][H][W][C] of a dense NCHW activation [.][C_dense][H][W]: column
// channel offset c_off, global first row row0. keep iff (u >> 11) >= thresh.
template <typename T>
__global__ void dropout_k(int B, int H, int W, int C, int C_dense, int c_off, long long row0,
                          unsigned long long seed, const unsigned long long* __restrict__ step, int layer,
                          unsigned long long thresh, float scale, const T* __restrict__ x, T* __restrict__ y) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)B * H * W * C;
  if (t >= n) return;
  const int c = (int)(t % C);
  const long long r1 = t / C;
  const int xx = (int)(r1 % W);
  const long long r2 = r1 / W;
  const int yy = (int)(r2 % H);
  const long long b = r2 / H;
  const unsigned long long idx =
      (unsigned long long)(row0 + b) * ((unsigned long long)C_dense * H * W) +
      ((unsigned long long)(c_off + c) * H + yy) * W + xx;
  const unsigned long long u = mix64(dropout_state(seed, *step, layer) + (idx + 1ull) * GOLDEN);
  y[t] = cvt<T>((u >> 11) >= thresh ? ld(x + t) * scale : 0.f);
}

__global__ void counter_add_k(unsigned long long* c, long long d) { *c += (unsigned long long)d; }

#define EXT_DISPATCH(prec, T, ...)                                                  \
  do {                                                                              \
    if ((prec) == PC_FP32) {                                                        \
      using T = float;                                                              \
      __VA_ARGS__;                                                                  \
    } else if ((prec) == PC_BF16) {                                                 \
      using T = __nv_bfloat16;                                                      \
      __VA_ARGS__;                                                                  \
    } else {                                                                        \
      PC_REQUIRE(false, PC_EVALUE, "unknown precision %d", (int)(prec));            \
    }                                                                               \
  } while (0)

static int grid256(long long n) { return (int)((n + 255) / 256); }

}  // namespace pc

using namespace pc;

extern "C" int pc_lrn_forward(long long P, int C, int size, float k, float alpha, float beta, const void* x,
                              void* y, int prec, pc_stream_t st) {
  PC_REQUIRE(P >= 0 && C > 0 && size >= 1 && size % 2 == 1 && k > 0.f, PC_EVALUE, "lrn: bad arguments");
  if (P == 0) return PC_OK;
  EXT_DISPATCH(prec, T, lrn_fwd_k<T><<<grid256(P * C), 256, 0, S(st)>>>(P, C, size / 2, k, alpha, beta,
                                                                           static_cast<const T*>(x),
                                                                           static_cast<T*>(y)));
  PC_CUDA_CHECK_LAUNCH("lrn_forward");
  return PC_OK;
}

extern "C" int pc_lrn_backward(long long P, int C, int size, float k, float alpha, float beta, const void* x,
                               const void* gy, void* gx, int prec, pc_stream_t st) {
  PC_REQUIRE(P >= 0 && C > 0 && size >= 1 && size % 2 == 1 && k > 0.f, PC_EVALUE, "lrn: bad arguments");
  if (P == 0) return PC_OK;
  EXT_DISPATCH(prec, T, lrn_bwd_k<T><<<grid256(P * C), 256, 0, S(st)>>>(
                            P, C, size / 2, k, alpha, beta, static_cast<const T*>(x), static_cast<const T*>(gy),
                            static_cast<T*>(gx)));
  PC_CUDA_CHECK_LAUNCH("lrn_backward");
  return PC_OK;
}

extern "C" int pc_dropout(int B, int H, int W, int C, int C_dense, int c_off, long long row0,
                          unsigned long long seed, const unsigned long long* step, int layer,
                          unsigned long long thresh, float p, const void* x, void* y, int prec, pc_stream_t st) {
  PC_REQUIRE(B >= 0 && H > 0 && W > 0 && C > 0 && C_dense >= C && c_off >= 0 && c_off + C <= C_dense && row0 >= 0 &&
                 p >= 0.f && p < 1.f && step != nullptr,
             PC_EVALUE, "dropout: bad arguments");
  const long long n = (long long)B * H * W * C;
  if (n == 0) return PC_OK;
  const float scale = 1.f / (1.f - p);
  EXT_DISPATCH(prec, T, dropout_k<T><<<grid256(n), 256, 0, S(st)>>>(B, H, W, C, C_dense, c_off, row0, seed, step,
                                                                      layer, thresh, scale, static_cast<const T*>(x),
                                                                      static_cast<T*>(y)));
  PC_CUDA_CHECK_LAUNCH("dropout");
  return PC_OK;
}

extern "C" int pc_counter_add(unsigned long long* counter, long long delta, pc_stream_t st) {
  PC_REQUIRE(counter != nullptr, PC_EVALUE, "counter_add: null counter");
  counter_add_k<<<1, 1, 0, S(st)>>>(counter, delta);
  PC_CUDA_CHECK_LAUNCH("counter_add");
  return PC_OK;
}
