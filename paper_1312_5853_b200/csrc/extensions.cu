// Layers beyond the reference: Krizhevsky's local response
// normalisation across channels and dropout with a counter-based SplitMix64
// mask. Definitions: oracle/ref_kernels.py (lrn_*, dropout_*) and
// paper_1312_5853_b200/rng.py (dropout_state / dropout_keep).
//
// LRN (NHWC, channels contiguous): a thread per (pixel, 8-channel group) with
// 16-byte loads; the channel-window sums slide through registers (forward:
// sum of squares; backward: S and the windowed g x S^(-b-1) sum), one powf per
// output channel. The scalar kernels remain for C % 8 != 0 / size > 9.
// Dropout: the keep decision of an element is recomputed from its dense index
// in both passes (no mask tensor), so the forward and backward agree bit for
// bit with each other and with rng.dropout_keep on the host.
#include <cstdlib>

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

// 8 consecutive channels of one pixel as floats (16-byte load for bf16, 2 x 16 B for fp32).
template <typename T> struct Vec8;
template <> struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* v) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float* v) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

// Channels [c0 - 8, c0 + 16) of one pixel (zero outside [0, C)): the thread's own
// 8-channel group and both neighbour groups, each one vector load (the neighbours'
// loads of the same bytes hit L1). HALF <= 8 channels of window on either side.
template <typename T>
__device__ __forceinline__ void load_window24(const T* px, int c0, int C, float* w) {
  if (c0 >= 8) Vec8<T>::load(px + c0 - 8, w); else
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0.f;
  Vec8<T>::load(px + c0, w + 8);
  if (c0 + 8 < C) Vec8<T>::load(px + c0 + 8, w + 16); else
#pragma unroll
    for (int i = 0; i < 8; ++i) w[16 + i] = 0.f;
}

// LRN forward, NHWC: a thread per (pixel, 8-channel group). Squares of the 24-channel
// window in registers; the size-wide channel window sum slides across the group
// (one add + one subtract per output channel); y = x * (k + alpha * S)^-beta.
// Zero channels outside [0, C) reproduce the clipped window of the definition.
template <typename T, int H>
__global__ void __launch_bounds__(256) lrn_fwd_v8_k(long long P, int C, float k, float alpha, float beta,
                                                    const T* __restrict__ x, T* __restrict__ y) {
  PC_PDL_TRIGGER();
  const int G = C >> 3;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P * G) return;
  const long long pix = t / G;
  const int c0 = (int)(t - pix * G) * 8;
  const T* px = x + pix * C;
  float w[24];
  load_window24(px, c0, C, w);
  float q[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) q[i] = w[i] * w[i];
  float s = 0.f;
#pragma unroll
  for (int i = 8 - H; i <= 8 + H; ++i) s += q[i];
  float out[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i > 0) s += q[8 + i + H] - q[8 + i - 1 - H];
    out[i] = w[8 + i] * __powf(k + alpha * s, -beta);
  }
  Vec8<T>::store(y + pix * C + c0, out);
}

// LRN backward: gx_c = g_c S_c^-b - 2ab x_c sum_{|c'-c|<=h} g_c' x_c' S_c'^(-b-1).
// The thread needs S over channels [c0 - h, c0 + 8 + h) (window sums of x^2 over
// [c0 - 2h, c0 + 8 + 2h), inside the 24-channel window for h <= 4), then the
// windowed sum of t = g x S^(-b-1) over its 8 channels — all in registers.
template <typename T, int H>
__global__ void __launch_bounds__(256) lrn_bwd_v8_k(long long P, int C, float k, float alpha, float beta,
                                                    const T* __restrict__ x, const T* __restrict__ gy,
                                                    T* __restrict__ gx) {
  PC_PDL_TRIGGER();
  const int G = C >> 3;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= P * G) return;
  const long long pix = t / G;
  const int c0 = (int)(t - pix * G) * 8;
  float w[24], g[24];
  load_window24(x + pix * C, c0, C, w);
  load_window24(gy + pix * C, c0, C, g);
  float q[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) q[i] = w[i] * w[i];
  // S at window positions [8 - H, 16 + H): sliding sum of q over +-H
  constexpr int NS = 8 + 2 * H;
  float sp[NS], tt[NS];
  float s = 0.f;
#pragma unroll
  for (int i = 8 - 2 * H; i <= 8; ++i) s += q[i];
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const int pos = 8 - H + j;
    if (j > 0) s += q[pos + H] - q[pos - 1 - H];
    const float S = k + alpha * s;
    const float sb = __powf(S, -beta);
    sp[j] = sb;                            // S^-b
    tt[j] = g[pos] * w[pos] * __fdividef(sb, S);   // g x S^(-b-1); zero outside [0, C) (g = x = 0)
  }
  float win = 0.f;
#pragma unroll
  for (int j = 0; j <= 2 * H; ++j) win += tt[j];
  float out[8];
  const float c2 = 2.f * alpha * beta;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i > 0) win += tt[i + 2 * H] - tt[i - 1];
    out[i] = g[8 + i] * sp[H + i] - c2 * w[8 + i] * win;
  }
  Vec8<T>::store(gx + pix * C + c0, out);
}

// Scalar fallback (C % 8 != 0 or size > 9): one thread per (pixel, channel).
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

// PC_LRN_VEC=0: the scalar kernels (A/B and a cross-check of the vector path)
static bool lrn_vec_enabled() {
  static const int on = [] {
    const char* e = getenv("PC_LRN_VEC");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

}  // namespace pc

using namespace pc;

extern "C" int pc_lrn_forward(long long P, int C, int size, float k, float alpha, float beta, const void* x,
                              void* y, int prec, pc_stream_t st) {
  PC_REQUIRE(P >= 0 && C > 0 && size >= 1 && size % 2 == 1 && k > 0.f, PC_EVALUE, "lrn: bad arguments");
  if (P == 0) return PC_OK;
  const int h = size / 2;
  if (C % 8 == 0 && h <= 4 && lrn_vec_enabled()) {
    EXT_DISPATCH(prec, T, {
      const T* xx = static_cast<const T*>(x);
      T* yy = static_cast<T*>(y);
      const int g = grid256(P * (C / 8));
      switch (h) {
        case 0: lrn_fwd_v8_k<T, 0><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, yy); break;
        case 1: lrn_fwd_v8_k<T, 1><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, yy); break;
        case 2: lrn_fwd_v8_k<T, 2><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, yy); break;
        case 3: lrn_fwd_v8_k<T, 3><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, yy); break;
        default: lrn_fwd_v8_k<T, 4><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, yy); break;
      }
    });
  } else {
    EXT_DISPATCH(prec, T, lrn_fwd_k<T><<<grid256(P * C), 256, 0, S(st)>>>(P, C, h, k, alpha, beta,
                                                                             static_cast<const T*>(x),
                                                                             static_cast<T*>(y)));
  }
  PC_CUDA_CHECK_LAUNCH("lrn_forward");
  return PC_OK;
}

extern "C" int pc_lrn_backward(long long P, int C, int size, float k, float alpha, float beta, const void* x,
                               const void* gy, void* gx, int prec, pc_stream_t st) {
  PC_REQUIRE(P >= 0 && C > 0 && size >= 1 && size % 2 == 1 && k > 0.f, PC_EVALUE, "lrn: bad arguments");
  if (P == 0) return PC_OK;
  const int h = size / 2;
  if (C % 8 == 0 && h <= 4 && lrn_vec_enabled()) {
    EXT_DISPATCH(prec, T, {
      const T* xx = static_cast<const T*>(x);
      const T* gg = static_cast<const T*>(gy);
      T* oo = static_cast<T*>(gx);
      const int g = grid256(P * (C / 8));
      switch (h) {
        case 0: lrn_bwd_v8_k<T, 0><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, gg, oo); break;
        case 1: lrn_bwd_v8_k<T, 1><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, gg, oo); break;
        case 2: lrn_bwd_v8_k<T, 2><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, gg, oo); break;
        case 3: lrn_bwd_v8_k<T, 3><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, gg, oo); break;
        default: lrn_bwd_v8_k<T, 4><<<g, 256, 0, S(st)>>>(P, C, k, alpha, beta, xx, gg, oo); break;
      }
    });
  } else {
    EXT_DISPATCH(prec, T, lrn_bwd_k<T><<<grid256(P * C), 256, 0, S(st)>>>(
                              P, C, h, k, alpha, beta, static_cast<const T*>(x), static_cast<const T*>(gy),
                              static_cast<T*>(gx)));
  }
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
