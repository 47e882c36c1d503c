// Bandwidth-bound layers of the step: ReLU, max-pool (u8 argmax, gather
// backward), softmax cross-entropy, multi-tensor momentum SGD and the layout
// helpers. Every kernel moves 8 elements (16 B of bf16 / 32 B of fp32) per
// thread where the extents allow, so loads and stores are 128-bit.
#include "common.cuh"

namespace pc {

// 8-element vector load/store ------------------------------------------------
template <typename T> struct Vec8;
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* v) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
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

static inline int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  return (int)(g < 1 ? 1 : (g > (1LL << 30) ? (1LL << 30) : g));
}

// ReLU -------------------------------------------------------------------------
template <typename T>
__global__ void relu_fwd_k(long long n, const T* __restrict__ x, T* __restrict__ y) {
  long long i8 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 8;
  if (i8 + 8 <= n && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 31) == 0) {
    float v[8];
    Vec8<T>::load(x + i8, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = v[j] > 0.f ? v[j] : (v[j] != v[j] ? v[j] : 0.f);
    Vec8<T>::store(y + i8, v);
  } else {
    for (long long i = i8; i < n && i < i8 + 8; ++i) {
      float a = ld(x + i);
      y[i] = cvt<T>(a > 0.f ? a : (a != a ? a : 0.f));
    }
  }
}

template <typename T>
__global__ void relu_bwd_k(long long n, const T* __restrict__ x, const T* __restrict__ g,
                           T* __restrict__ gx) {
  long long i8 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 8;
  if (i8 + 8 <= n &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gx)) & 31) == 0) {
    float a[8], b[8];
    Vec8<T>::load(x + i8, a);
    Vec8<T>::load(g + i8, b);
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = a[j] > 0.f ? b[j] : 0.f;
    Vec8<T>::store(gx + i8, b);
  } else {
    for (long long i = i8; i < n && i < i8 + 8; ++i) gx[i] = cvt<T>(ld(x + i) > 0.f ? ld(g + i) : 0.f);
  }
}

// Max-pool ---------------------------------------------------------------------
// One thread per (b, oy, ox, 8-channel group) when C % 8 == 0, else per channel.
// bf16 3x3 / stride-2 max-pool forward (8 channels per thread). Fast path for
// windows whose 9 x 8 values are all non-negative and not NaN (the network's
// ReLU outputs): raw bf16 bit patterns are then order-preserving, so one 32-bit
// integer max over (bits << 16 | 15 - index) gives the maximum and, among equal
// values, the first window position — np.argmax's rule, bit-exact. Any negative
// value or NaN in the window falls back to the exact float comparison (first NaN
// wins, -0 == +0). The kernel was integer-ALU bound (ncu: ALU pipe 80%, 372
// instructions per thread); the key build is one PRMT and the max tree DPX
// three-input maxes.
// Index math in 32 bits with precomputed divisors (the host guarantees every
// offset < 2^31): the runtime divisions were a third of the instructions.
__global__ void maxpool_fwd_bf16_k3s2_k(int B, int H, int W, int C, int Ho, int Wo, FastDiv fcg, FastDiv fwo,
                                        FastDiv fho, const __nv_bfloat16* __restrict__ x,
                                        __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ arg) {
  PC_PDL_TRIGGER();
  const unsigned cg = (unsigned)(C >> 3);
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (unsigned)B * Ho * Wo * cg) return;
  const unsigned pix = fcg.div(t);
  const unsigned c0 = (t - pix * cg) * 8;
  const unsigned row = fwo.div(pix);
  const unsigned ox = pix - row * (unsigned)Wo;
  const unsigned b = fho.div(row);
  const unsigned oy = row - b * (unsigned)Ho;
  // keys: (bf16 bits << 16) | (15 - window index), built with one PRMT per channel
  // and element; the 9-way max per channel is 4 three-input DPX maxes (VIMNMX3):
  // the largest value and, among equal values, the first index. The window's 36
  // words stay in registers (the rare fallback reuses them).
  const __nv_bfloat16* x0 = x + (((b * (unsigned)H + oy * 2) * (unsigned)W + ox * 2) * (unsigned)C + c0);
  const unsigned WC = (unsigned)W * C;
  uint4 r[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) r[e] = __ldg(reinterpret_cast<const uint4*>(x0 + ((e / 3) * WC + (e % 3) * (unsigned)C)));
  uint32_t mk[8];
  uint32_t sign = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t lo[9], hi[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) {
      const uint32_t w = q == 0 ? r[e].x : q == 1 ? r[e].y : q == 2 ? r[e].z : r[e].w;
      sign |= w;
      lo[e] = __byte_perm(w, 15u - e, 0x1054);  // (low channel bits << 16) | (15 - e)
      hi[e] = __byte_perm(w, 15u - e, 0x3254);  // (high channel bits << 16) | (15 - e)
    }
    mk[2 * q] = __vimax3_u32(__vimax3_u32(lo[0], lo[1], lo[2]), __vimax3_u32(lo[3], lo[4], lo[5]),
                             __vimax3_u32(lo[6], lo[7], lo[8]));
    mk[2 * q + 1] = __vimax3_u32(__vimax3_u32(hi[0], hi[1], hi[2]), __vimax3_u32(hi[3], hi[4], hi[5]),
                                 __vimax3_u32(hi[6], hi[7], hi[8]));
  }
  bool nan = false;
#pragma unroll
  for (int v = 0; v < 8; ++v) nan |= (mk[v] >> 16) > 0x7F80u;
  const unsigned o = pix * (unsigned)C + c0;
  if ((sign & 0x80008000u) == 0u && !nan) {
    uint4 outv;
    outv.x = __byte_perm(mk[0], mk[1], 0x7632);
    outv.y = __byte_perm(mk[2], mk[3], 0x7632);
    outv.z = __byte_perm(mk[4], mk[5], 0x7632);
    outv.w = __byte_perm(mk[6], mk[7], 0x7632);
    *reinterpret_cast<uint4*>(y + o) = outv;
    // index byte of channel v = 15 - (key & 15): bytes 0 of the keys, packed, then 0x0F - b
    const uint32_t i0 = __byte_perm(__byte_perm(mk[0], mk[1], 0x0040), __byte_perm(mk[2], mk[3], 0x0040), 0x5410);
    const uint32_t i1 = __byte_perm(__byte_perm(mk[4], mk[5], 0x0040), __byte_perm(mk[6], mk[7], 0x0040), 0x5410);
    uint2 packed;
    packed.x = 0x0F0F0F0Fu - (i0 & 0x0F0F0F0Fu);
    packed.y = 0x0F0F0F0Fu - (i1 & 0x0F0F0F0Fu);
    *reinterpret_cast<uint2*>(arg + o) = packed;
    return;
  }
  float best[8];
  int bi[8];
  unsigned short bits[8];  // the winner's original bits (NaN payload kept)
#pragma unroll
  for (int v = 0; v < 8; ++v) { best[v] = 0.f; bi[v] = -1; bits[v] = 0; }
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const uint32_t w[4] = {r[e].x, r[e].y, r[e].z, r[e].w};
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const unsigned short hb = (unsigned short)(w[v >> 1] >> (16 * (v & 1)));
      const float val = __uint_as_float((uint32_t)hb << 16);
      const bool nan_v = val != val, nan_b = best[v] != best[v];
      if (bi[v] < 0 || (!nan_b && (val > best[v] || nan_v))) { best[v] = val; bi[v] = e; bits[v] = hb; }
    }
  }
  uint4 outv;
  outv.x = bits[0] | ((uint32_t)bits[1] << 16);
  outv.y = bits[2] | ((uint32_t)bits[3] << 16);
  outv.z = bits[4] | ((uint32_t)bits[5] << 16);
  outv.w = bits[6] | ((uint32_t)bits[7] << 16);
  uint2 packed;
  packed.x = (uint32_t)bi[0] | ((uint32_t)bi[1] << 8) | ((uint32_t)bi[2] << 16) | ((uint32_t)bi[3] << 24);
  packed.y = (uint32_t)bi[4] | ((uint32_t)bi[5] << 8) | ((uint32_t)bi[6] << 16) | ((uint32_t)bi[7] << 24);
  *reinterpret_cast<uint4*>(y + o) = outv;
  *reinterpret_cast<uint2*>(arg + o) = packed;
}

template <typename T, int V, int KS = 0, int SS = 0>
__global__ void maxpool_fwd_k(int B, int H, int W, int C, int k_, int s_, int Ho, int Wo,
                              const T* __restrict__ x, T* __restrict__ y, uint8_t* __restrict__ arg) {
  // KS > 0: compile-time k x k / stride s (AlexNet 3/2): the window loop unrolls and
  // all k*k loads are in flight at once
  const int k = KS > 0 ? KS : k_, s = KS > 0 ? SS : s_;
  // 32-bit index math (the host guarantees < 2^31 work items): 64-bit division is emulated
  const unsigned cg = (unsigned)(C / V);
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned total = (unsigned)B * Ho * Wo * cg;
  if (t >= total) return;
  const unsigned pix = t / cg;
  const int c0 = (int)(t - pix * cg) * V;
  const unsigned row = pix / (unsigned)Wo;
  const int ox = (int)(pix - row * Wo);
  const int b = (int)(row / (unsigned)Ho);
  const int oy = (int)(row - (unsigned)b * Ho);
  float best[V];
  int bi[V];
#pragma unroll
  for (int v = 0; v < V; ++v) { best[v] = 0.f; bi[v] = -1; }
#pragma unroll
  for (int i = 0; i < (KS > 0 ? KS : 16); ++i) {
    if (KS == 0 && i >= k) break;
    const T* xr = x + (((long long)b * H + oy * s + i) * W + ox * s) * C + c0;
#pragma unroll
    for (int j = 0; j < (KS > 0 ? KS : 16); ++j) {
      if (KS == 0 && j >= k) break;
      float val[V];
      if constexpr (V == 8) {
        Vec8<T>::load(xr + (long long)j * C, val);
      } else {
        val[0] = ld(xr + (long long)j * C);
      }
      int idx = i * k + j;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        bool nan_v = val[v] != val[v], nan_b = best[v] != best[v];
        // np.argmax: first maximum wins, the first NaN wins over everything
        if (bi[v] < 0 || (!nan_b && (val[v] > best[v] || nan_v))) { best[v] = val[v]; bi[v] = idx; }
      }
    }
  }
  long long o = (long long)pix * C + c0;
  if constexpr (V == 8) {
    Vec8<T>::store(y + o, best);
    uint2 packed;
    uint8_t* pb = reinterpret_cast<uint8_t*>(&packed);
#pragma unroll
    for (int v = 0; v < 8; ++v) pb[v] = (uint8_t)bi[v];
    *reinterpret_cast<uint2*>(arg + o) = packed;
  } else {
    y[o] = cvt<T>(best[0]);
    arg[o] = (uint8_t)bi[0];
  }
}

template <typename T, int V>
__global__ void maxpool_bwd_k(int B, int H, int W, int C, int k, int s, int Ho, int Wo,
                              const T* __restrict__ gy, const uint8_t* __restrict__ arg,
                              const T* __restrict__ mask, T* __restrict__ gx) {
  const unsigned cg = (unsigned)(C / V);
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned total = (unsigned)B * H * W * cg;
  if (t >= total) return;
  const unsigned pix = t / cg;
  const int c0 = (int)(t - pix * cg) * V;
  const unsigned row = pix / (unsigned)W;
  const int x = (int)(pix - row * W);
  const int b = (int)(row / (unsigned)H);
  const int y = (int)(row - (unsigned)b * H);
  // windows oy with oy*s <= y <= oy*s + k - 1
  int oy_lo = y - k + 1 <= 0 ? 0 : (y - k + 1 + s - 1) / s;
  int oy_hi = min(y / s, Ho - 1);
  int ox_lo = x - k + 1 <= 0 ? 0 : (x - k + 1 + s - 1) / s;
  int ox_hi = min(x / s, Wo - 1);
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  for (int oy = oy_lo; oy <= oy_hi; ++oy) {
    for (int ox = ox_lo; ox <= ox_hi; ++ox) {
      int want = (y - oy * s) * k + (x - ox * s);
      long long o = (((long long)b * Ho + oy) * Wo + ox) * C + c0;
      if constexpr (V == 8) {
        uint2 packed = __ldg(reinterpret_cast<const uint2*>(arg + o));
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(&packed);
        float g[8];
        Vec8<T>::load(gy + o, g);
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[v] += (pb[v] == want) ? g[v] : 0.f;
      } else {
        if (arg[o] == want) acc[0] += ld(gy + o);
      }
    }
  }
  long long o = (long long)pix * C + c0;
  if (mask) {
    float mk[V];
    if constexpr (V == 8) Vec8<T>::load(mask + o, mk); else mk[0] = ld(mask + o);
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = mk[v] > 0.f ? acc[v] : 0.f;
  }
  if constexpr (V == 8) Vec8<T>::store(gx + o, acc); else gx[o] = cvt<T>(acc[0]);
}

// acc[0..7] += the 8 bf16 values packed in s0..s3 (low half first), two lanes per
// packed fp32x2 add (FADD2): the same per-element IEEE adds in the same order.
__device__ __forceinline__ void bf16x8_accumulate(float* acc, uint32_t s0, uint32_t s1, uint32_t s2, uint32_t s3) {
  const uint32_t w[4] = {s0, s1, s2, s3};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 a = make_float2(acc[2 * i], acc[2 * i + 1]);
    a = __fadd2_rn(a, make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u)));
    acc[2 * i] = a.x;
    acc[2 * i + 1] = a.y;
  }
}

// bf16 k=3, s=2 backward with byte-SIMD routing: for each covering window and
// each of its (at most 4) window positions inside this 2x2 block, one __vcmpeq4
// per 4 channels selects the channels whose argmax is that position, the byte
// masks are widened to 16-bit lanes (prmt) and AND the packed bf16 gradient, so
// a contribution costs two integer ops and an fp32 add per channel instead of a
// compare/select/add per (pixel, window, channel). Same fixed order (ascending
// (oy, ox) per pixel) and fp32 accumulation as maxpool_bwd_k3s2_k.
__global__ void __launch_bounds__(256) maxpool_bwd_bf16_k3s2_k(int B, int H, int W, int C, int Ho, int Wo,
                                                               FastDiv fcg, FastDiv fw2, FastDiv fh2,
                                                               const __nv_bfloat16* __restrict__ gy,
                                                               const uint8_t* __restrict__ arg,
                                                               const __nv_bfloat16* __restrict__ mask,
                                                               __nv_bfloat16* __restrict__ gx) {
  PC_PDL_TRIGGER();
  const int H2 = (H + 1) >> 1, W2 = (W + 1) >> 1;
  const unsigned cg = (unsigned)(C >> 3);
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (unsigned)B * H2 * W2 * cg) return;
  const unsigned blk = fcg.div(t);
  const int c0 = (int)(t - blk * cg) * 8;
  const unsigned r = fw2.div(blk);
  const int X = (int)(blk - r * W2);
  const int b = (int)fh2.div(r);
  const int Y = (int)(r - (unsigned)b * H2);
  float acc[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[q][v] = 0.f;
#pragma unroll
  for (int dy = -1; dy <= 0; ++dy) {
    const int oy = Y + dy;
    if (oy < 0 || oy >= Ho) continue;
#pragma unroll
    for (int dx = -1; dx <= 0; ++dx) {
      const int ox = X + dx;
      if (ox < 0 || ox >= Wo) continue;
      const unsigned o = (((unsigned)b * Ho + oy) * Wo + ox) * (unsigned)C + c0;
      const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o));
      const uint4 g = __ldg(reinterpret_cast<const uint4*>(gy + o));
#pragma unroll
      for (int qy = 0; qy < 2; ++qy) {
        const int li = qy - 2 * dy;  // row of pixel (2Y + qy) inside window oy
        if (li > 2) continue;
#pragma unroll
        for (int qx = 0; qx < 2; ++qx) {
          const int lj = qx - 2 * dx;
          if (lj > 2) continue;
          const unsigned want = 0x01010101u * (unsigned)(li * 3 + lj);
          const unsigned m0 = __vcmpeq4(a.x, want), m1 = __vcmpeq4(a.y, want);
          const unsigned s0 = g.x & __byte_perm(m0, 0, 0x1100), s1 = g.y & __byte_perm(m0, 0, 0x3322);
          const unsigned s2 = g.z & __byte_perm(m1, 0, 0x1100), s3 = g.w & __byte_perm(m1, 0, 0x3322);
          bf16x8_accumulate(acc[qy * 2 + qx], s0, s1, s2, s3);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int y = 2 * Y + (q >> 1), x = 2 * X + (q & 1);
    if (y >= H || x >= W) continue;
    const unsigned o = (((unsigned)b * H + y) * W + x) * (unsigned)C + c0;
    if (mask) {
      float mk[8];
      Vec8<__nv_bfloat16>::load(mask + o, mk);
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[q][v] = mk[v] > 0.f ? acc[q][v] : 0.f;
    }
    Vec8<__nv_bfloat16>::store(gx + o, acc[q]);
  }
}

// bf16 3x3/s2 backward that also reduces the bias gradient of the layer whose
// upstream gradient it writes (conv -> ReLU -> pool: gx IS that conv's gy): a
// fixed grid walks the 2x2 blocks grid-stride (the thread's 8-channel group is
// constant because 256 % (C / 8) == 0), each thread sums the bf16 values it
// stores, the CTA combines its row lanes in a fixed order into part[block][C],
// and pool_bias_rows_k sums the CTA rows (a CTA per 8 channels, fixed tree).
// Deterministic; saves the separate two-pass reduction that re-read gx.
__global__ void __launch_bounds__(256) maxpool_bwd_bf16_k3s2_bias_k(int B, int H, int W, int C, int Ho, int Wo,
                                                                    FastDiv fcg, FastDiv fw2, FastDiv fh2,
                                                                    const __nv_bfloat16* __restrict__ gy,
                                                                    const uint8_t* __restrict__ arg,
                                                                    const __nv_bfloat16* __restrict__ mask,
                                                                    __nv_bfloat16* __restrict__ gx,
                                                                    float* __restrict__ part) {
  PC_PDL_TRIGGER();
  __shared__ float red[256][9];
  const int H2 = (H + 1) >> 1, W2 = (W + 1) >> 1;
  const unsigned cg = (unsigned)(C >> 3);
  const unsigned total = (unsigned)B * H2 * W2 * cg;
  float bsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned blk = fcg.div(t);
    const int c0 = (int)(t - blk * cg) * 8;
    const unsigned r = fw2.div(blk);
    const int X = (int)(blk - r * W2);
    const int b = (int)fh2.div(r);
    const int Y = (int)(r - (unsigned)b * H2);
    float acc[4][8];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[q][v] = 0.f;
#pragma unroll
    for (int dy = -1; dy <= 0; ++dy) {
      const int oy = Y + dy;
      if (oy < 0 || oy >= Ho) continue;
#pragma unroll
      for (int dx = -1; dx <= 0; ++dx) {
        const int ox = X + dx;
        if (ox < 0 || ox >= Wo) continue;
        const unsigned o = (((unsigned)b * Ho + oy) * Wo + ox) * (unsigned)C + c0;
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o));
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(gy + o));
#pragma unroll
        for (int qy = 0; qy < 2; ++qy) {
          const int li = qy - 2 * dy;
          if (li > 2) continue;
#pragma unroll
          for (int qx = 0; qx < 2; ++qx) {
            const int lj = qx - 2 * dx;
            if (lj > 2) continue;
            const unsigned want = 0x01010101u * (unsigned)(li * 3 + lj);
            const unsigned m0 = __vcmpeq4(a.x, want), m1 = __vcmpeq4(a.y, want);
            const unsigned s0 = g.x & __byte_perm(m0, 0, 0x1100), s1 = g.y & __byte_perm(m0, 0, 0x3322);
            const unsigned s2 = g.z & __byte_perm(m1, 0, 0x1100), s3 = g.w & __byte_perm(m1, 0, 0x3322);
            bf16x8_accumulate(acc[qy * 2 + qx], s0, s1, s2, s3);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * Y + (q >> 1), x = 2 * X + (q & 1);
      if (y >= H || x >= W) continue;
      const unsigned o = (((unsigned)b * H + y) * W + x) * (unsigned)C + c0;
      if (mask) {
        float mk[8];
        Vec8<__nv_bfloat16>::load(mask + o, mk);
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[q][v] = mk[v] > 0.f ? acc[q][v] : 0.f;
      }
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        h[e] = __floats2bfloat162_rn(acc[q][2 * e], acc[q][2 * e + 1]);
        const float2 f = __bfloat1622float2(h[e]);  // the stored values: what a reduction of gx would read
        bsum[2 * e] += f.x;
        bsum[2 * e + 1] += f.y;
      }
      *reinterpret_cast<uint4*>(gx + o) = u;
    }
  }
#pragma unroll
  for (int v = 0; v < 8; ++v) red[threadIdx.x][v] = bsum[v];
  __syncthreads();
  // thread -> (channel group q = tid % cg, lane = tid / cg); lanes combine in order
  const int lanes = 256 / (int)cg;
  if (threadIdx.x < cg * 8) {
    const int q = threadIdx.x >> 3, v = threadIdx.x & 7;
    float sum = 0.f;
    for (int l = 0; l < lanes; ++l) sum += red[l * cg + q][v];
    part[(long long)blockIdx.x * C + q * 8 + v] = sum;
  }
}

// Column sums of the per-CTA partial rows: a CTA per 8 columns, thread r summing
// rows r, r + 256, ... (float4 pairs), then a fixed shared-memory tree over the 256
// threads. Deterministic.
__global__ void __launch_bounds__(256) pool_bias_rows_k(const float* __restrict__ part, int R, int N,
                                                        float* __restrict__ out) {
  PC_PDL_TRIGGER();
  __shared__ float sh[256][9];
  const int grp = blockIdx.x;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int r = threadIdx.x; r < R; r += 256) {
    const float4* p = reinterpret_cast<const float4*>(part + (long long)r * N + grp * 8);
    const float4 x = __ldg(p), y = __ldg(p + 1);
    a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w; a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sh[threadIdx.x][i] = a[i];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
#pragma unroll
      for (int i = 0; i < 8; ++i) sh[threadIdx.x][i] += sh[threadIdx.x + w][i];
    __syncthreads();
  }
  if (threadIdx.x < 8) out[grp * 8 + threadIdx.x] = sh[0][threadIdx.x];
}

// k=3, s=2 (every AlexNet pool): one thread per 2x2 input block (Y, X) and 8
// channels. The block is covered exactly by windows {Y-1, Y} x {X-1, X}, so the
// thread reads those <= 4 windows' gradient + argmax once and writes 4 pixels
// (a 4x cut in loads per output vs the per-pixel gather). Contributions are
// still added in ascending (oy, ox) order per pixel, as in pc_maxpool_backward.
template <typename T>
__global__ void maxpool_bwd_k3s2_k(int B, int H, int W, int C, int Ho, int Wo, const T* __restrict__ gy,
                                   const uint8_t* __restrict__ arg, const T* __restrict__ mask,
                                   T* __restrict__ gx) {
  const int H2 = (H + 1) >> 1, W2 = (W + 1) >> 1;
  const unsigned cg = (unsigned)(C >> 3);
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (unsigned)B * H2 * W2 * cg) return;
  const unsigned blk = t / cg;
  const int c0 = (int)(t - blk * cg) * 8;
  const unsigned r = blk / (unsigned)W2;
  const int X = (int)(blk - r * W2);
  const int b = (int)(r / (unsigned)H2);
  const int Y = (int)(r - (unsigned)b * H2);
  float acc[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[q][v] = 0.f;
#pragma unroll
  for (int dy = -1; dy <= 0; ++dy) {
    const int oy = Y + dy;
    if (oy < 0 || oy >= Ho) continue;
#pragma unroll
    for (int dx = -1; dx <= 0; ++dx) {
      const int ox = X + dx;
      if (ox < 0 || ox >= Wo) continue;
      const long long o = (((long long)b * Ho + oy) * Wo + ox) * C + c0;
      uint2 packed = __ldg(reinterpret_cast<const uint2*>(arg + o));
      const uint8_t* pb = reinterpret_cast<const uint8_t*>(&packed);
      float g[8];
      Vec8<T>::load(gy + o, g);
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // pixel (2Y + q/2, 2X + q%2): local index in window (oy, ox)
        const int li = 2 * Y + (q >> 1) - 2 * oy, lj = 2 * X + (q & 1) - 2 * ox;
        const int want = (li <= 2 && lj <= 2) ? li * 3 + lj : 255;  // 255: pixel outside this window
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[q][v] += (pb[v] == want) ? g[v] : 0.f;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int y = 2 * Y + (q >> 1), x = 2 * X + (q & 1);
    if (y >= H || x >= W) continue;
    const unsigned o = (((unsigned)b * H + y) * W + x) * (unsigned)C + c0;
    if (mask) {
      float mk[8];
      Vec8<T>::load(mask + o, mk);
#pragma unroll
      for (int v = 0; v < 8; ++v) acc[q][v] = mk[v] > 0.f ? acc[q][v] : 0.f;
    }
    Vec8<T>::store(gx + o, acc[q]);
  }
}

// Softmax cross-entropy: one CTA per row ------------------------------------------
template <int NT>
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float w = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, w) : v + w;
  }
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  v = sh[0];
  for (int i = 1; i < NT / 32; ++i) v = is_max ? fmaxf(v, sh[i]) : v + sh[i];
  return v;
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT) softmax_xent_k(int K, const T* __restrict__ logits,
                                                     const int32_t* __restrict__ labels, double scale,
                                                     T* __restrict__ grad, double* __restrict__ row_loss,
                                                     int* __restrict__ bad) {
  __shared__ float sh[NT / 32];
  int row = blockIdx.x;
  const T* z = logits + (long long)row * K;
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < K; i += NT) mx = fmaxf(mx, ld(z + i));
  mx = block_reduce<NT>(mx, true, sh);
  float sum = 0.f;
  for (int i = threadIdx.x; i < K; i += NT) sum += expf(ld(z + i) - mx);
  sum = block_reduce<NT>(sum, false, sh);
  int lab = labels[row];
  bool ok = lab >= 0 && lab < K;
  float inv = 1.f / sum, sc = (float)scale;
  for (int i = threadIdx.x; i < K; i += NT) {
    float p = expf(ld(z + i) - mx) * inv;
    grad[(long long)row * K + i] = cvt<T>((p - (i == lab ? 1.f : 0.f)) * sc);
  }
  if (threadIdx.x == 0) {
    if (!ok) { *bad = 1; row_loss[row] = 0.0; return; }
    double logp = (double)(ld(z + lab) - mx) - log((double)sum);
    row_loss[row] = -logp * scale;
  }
}

// Warp per row (K <= 32 * KPL): the row stays in registers (lane l holds classes
// l, l + 32, ...), max and sum-of-exp are warp-shuffle reductions, one pass of
// loads and one of stores; 8 rows per 256-thread CTA. Same arithmetic as
// softmax_xent_k (fp32 exp / sums, fp64 log-probability of the label).
template <typename T, int KPL>
__global__ void __launch_bounds__(256) softmax_xent_warp_k(int B, int K, const T* __restrict__ logits,
                                                          const int32_t* __restrict__ labels, double scale,
                                                          T* __restrict__ grad, double* __restrict__ row_loss,
                                                          int* __restrict__ bad, double* __restrict__ loss_out,
                                                          unsigned* __restrict__ ticket) {
  PC_PDL_TRIGGER();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row < B) {
    const T* z = logits + (long long)row * K;
    float x[KPL];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int i = lane + 32 * j;
      x[j] = i < K ? ld(z + i) : -INFINITY;
      mx = fmaxf(mx, x[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      x[j] = lane + 32 * j < K ? expf(x[j] - mx) : 0.f;
      sum += x[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int lab = labels[row];
    const bool ok = lab >= 0 && lab < K;
    const float inv = 1.f / sum, sc = (float)scale;
    T* g = grad + (long long)row * K;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const int i = lane + 32 * j;
      if (i < K) g[i] = cvt<T>((x[j] * inv - (i == lab ? 1.f : 0.f)) * sc);
    }
    if (lane == 0) {
      if (!ok) {
        *bad = 1;
        row_loss[row] = 0.0;
      } else {
        const double logp = (double)(ld(z + lab) - mx) - log((double)sum);
        row_loss[row] = -logp * scale;
      }
    }
  }
  if (loss_out == nullptr) return;
  // the step loss in the last block to finish (ticket): sum_f64_k's order exactly
  __shared__ unsigned last;
  __shared__ double sh[8];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int i = threadIdx.x; i < B; i += 256) acc += __ldcg(row_loss + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sh[0];
    for (int w = 1; w < 8; ++w) t += sh[w];
    loss_out[0] = t;
    *ticket = 0u;   // ready for the next step (graph replay)
  }
}

// Step loss: 256 threads, thread t summing v[t], v[t + 256], ... in order, then a
// fixed tree (warp xor-shuffles, then the 8 warp sums in order): deterministic,
// and the row losses load in parallel instead of one dependent chain.
__global__ void __launch_bounds__(256) sum_f64_k(int n, const double* __restrict__ v, double* __restrict__ out) {
  PC_PDL_TRIGGER();
  __shared__ double sh[8];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) acc += v[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = sh[0];
    for (int w = 1; w < 8; ++w) t += sh[w];
    out[0] = t;
  }
}

// Multi-tensor momentum SGD: blockIdx.y = tensor --------------------------------------
__global__ void sgd_k(const pc_sgd_tensor* __restrict__ tab, float lr, float mom, float wd) {
  PC_PDL_TRIGGER();
  pc_sgd_tensor t = tab[blockIdx.y];
  long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < t.n; i += stride) {
    if (i + 4 <= t.n && ((reinterpret_cast<uintptr_t>(t.p) | reinterpret_cast<uintptr_t>(t.v) |
                          reinterpret_cast<uintptr_t>(t.g)) & 15) == 0) {
      float4 p = *reinterpret_cast<float4*>(t.p + i);
      float4 v = *reinterpret_cast<float4*>(t.v + i);
      float4 g = __ldg(reinterpret_cast<const float4*>(t.g + i));
      v.x = mom * v.x - lr * (g.x + wd * p.x);
      v.y = mom * v.y - lr * (g.y + wd * p.y);
      v.z = mom * v.z - lr * (g.z + wd * p.z);
      v.w = mom * v.w - lr * (g.w + wd * p.w);
      p.x += v.x; p.y += v.y; p.z += v.z; p.w += v.w;
      *reinterpret_cast<float4*>(t.v + i) = v;
      *reinterpret_cast<float4*>(t.p + i) = p;
      if (t.p_lowp) {
        __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(t.p_lowp) + i);
        q[0] = __floats2bfloat162_rn(p.x, p.y);
        q[1] = __floats2bfloat162_rn(p.z, p.w);
      }
    } else {
      for (long long j = i; j < t.n && j < i + 4; ++j) {
        float p = t.p[j], v = t.v[j], g = t.g[j];
        v = mom * v - lr * (g + wd * p);
        p += v;
        t.v[j] = v;
        t.p[j] = p;
        if (t.p_lowp) static_cast<__nv_bfloat16*>(t.p_lowp)[j] = __float2bfloat16_rn(p);
      }
    }
  }
}

// Background variant (a few CTAs per SM beside a running GEMM): grid-stride with
// two float4 groups in flight per thread, same arithmetic as sgd_k.
__global__ void __launch_bounds__(256) sgd_bg_k(const pc_sgd_tensor* __restrict__ tab, float lr, float mom,
                                                float wd) {
  const pc_sgd_tensor t = tab[blockIdx.y];
  const bool vec = ((reinterpret_cast<uintptr_t>(t.p) | reinterpret_cast<uintptr_t>(t.v) |
                     reinterpret_cast<uintptr_t>(t.g)) & 15) == 0 &&
                   (t.p_lowp == nullptr || (reinterpret_cast<uintptr_t>(t.p_lowp) & 7) == 0);
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  const long long n4 = vec ? t.n / 4 * 4 : 0;
  long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4;
  for (; i + stride < n4; i += 2 * stride) {
    float4 p[2], v[2], g[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      p[u] = *reinterpret_cast<const float4*>(t.p + i + u * stride);
      v[u] = *reinterpret_cast<const float4*>(t.v + i + u * stride);
      g[u] = __ldg(reinterpret_cast<const float4*>(t.g + i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      v[u].x = mom * v[u].x - lr * (g[u].x + wd * p[u].x);
      v[u].y = mom * v[u].y - lr * (g[u].y + wd * p[u].y);
      v[u].z = mom * v[u].z - lr * (g[u].z + wd * p[u].z);
      v[u].w = mom * v[u].w - lr * (g[u].w + wd * p[u].w);
      p[u].x += v[u].x; p[u].y += v[u].y; p[u].z += v[u].z; p[u].w += v[u].w;
      *reinterpret_cast<float4*>(t.v + i + u * stride) = v[u];
      *reinterpret_cast<float4*>(t.p + i + u * stride) = p[u];
      if (t.p_lowp) {
        __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(t.p_lowp) + i + u * stride);
        q[0] = __floats2bfloat162_rn(p[u].x, p[u].y);
        q[1] = __floats2bfloat162_rn(p[u].z, p[u].w);
      }
    }
  }
  for (; i < t.n; i += stride) {
    for (long long j = i; j < t.n && j < i + 4; ++j) {
      float p = t.p[j], v = t.v[j], g = t.g[j];
      v = mom * v - lr * (g + wd * p);
      p += v;
      t.v[j] = v;
      t.p[j] = p;
      if (t.p_lowp) static_cast<__nv_bfloat16*>(t.p_lowp)[j] = __float2bfloat16_rn(p);
    }
  }
}

// Layout helpers ---------------------------------------------------------------------
template <typename T>
__global__ void nchw_to_nhwc_k(int B, int C, int H, int W, int Cp, const float* __restrict__ src,
                               T* __restrict__ dst) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = (long long)B * H * W * Cp;
  if (t >= total) return;
  int c = (int)(t % Cp);
  long long pix = t / Cp;
  int x = (int)(pix % W);
  int y = (int)((pix / W) % H);
  int b = (int)(pix / ((long long)W * H));
  float v = c < C ? src[(((long long)b * C + c) * H + y) * W + x] : 0.f;
  dst[t] = cvt<T>(v);
}

// Explicit im2col for the network's input layer: col[pixel][(c*k + i)*k + j]
// (the reference's K order, kernels.py:94-100) = x[b][c][oy*s+i-p][ox*s+j-p],
// zero-padded to Kp columns, straight from the float32 NCHW batch. One CTA per
// output row (b, oy): the C*k input rows it needs are staged in shared memory,
// then the Wo x Kp output rows are written with 16-byte stores.
template <typename TS, typename TD>
__global__ void im2col_rows_k(int C, int H, int W, int k, int s, int p, int Ho, int Wo, int Kp,
                              const TS* __restrict__ x, TD* __restrict__ col) {
  extern __shared__ float rows[];  // [C][k][W]
  const int bo = blockIdx.x;
  const int b = bo / Ho, oy = bo - b * Ho;
  for (int t = threadIdx.x; t < C * k * W; t += blockDim.x) {
    int xw = t % W, r = t / W;
    int i = r % k, c = r / k;
    int iy = oy * s + i - p;
    rows[t] = (iy >= 0 && iy < H) ? ld(x + (((long long)b * C + c) * H + iy) * W + xw) : 0.f;
  }
  __syncthreads();
  const int K = C * k * k, chunks = Kp / 8;
  TD* out = col + (long long)bo * Wo * Kp;
  for (int t = threadIdx.x; t < Wo * chunks; t += blockDim.x) {
    int ox = t / chunks, q = t - ox * chunks;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int kk = q * 8 + e;
      float val = 0.f;
      if (kk < K) {
        int j = kk % k, r = kk / k;  // r = c*k + i
        int ix = ox * s + j - p;
        if (ix >= 0 && ix < W) val = rows[r * W + ix];
      }
      v[e] = val;
    }
    Vec8<TD>::store(out + (long long)ox * Kp + q * 8, v);
  }
}

// Space-to-depth of the network input for a strided input conv: one thread per
// output block (b, Y, X) reads its s x s x C input values (consecutive threads =
// consecutive X, so each (c, row) read is coalesced across the warp) and writes
// the Cs-channel row, ch = (dy*s + dx)*C + c, with 16-byte stores (zero for
// padding and ch >= s*s*C). Each input element is read exactly once.
// read-only (non-coherent) scalar load of an input written by an earlier kernel
__device__ __forceinline__ float ldg_ro(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ldg_ro(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
// float64 source (a parconv caller's images): rounded to float first, exactly the value
// the float32 host path uploads (the reference's images are float32-quantised)
__device__ __forceinline__ float ldg_ro(const double* p) { return __double2float_rn(__ldg(p)); }

template <typename TS, int CS, int SS, int CC, typename TD = __nv_bfloat16>  // SS, CC > 0: compile-time stride / channels
__global__ void __launch_bounds__(256) s2d_k(int B, int C_, int H, int W, int s_, int p, int Hs, int Ws,
                                             const TS* __restrict__ x, TD* __restrict__ dst, int ones) {
  const int s = SS > 0 ? SS : s_, C = CC > 0 ? CC : C_;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)B * Hs * Ws) return;
  const int X = (int)(t % Ws);
  const long long r = t / Ws;
  const int Y = (int)(r % Hs), b = (int)(r / Hs);
  float v[CS];
#pragma unroll
  for (int i = 0; i < CS; ++i) v[i] = i == ones ? 1.f : 0.f;
  if constexpr (SS > 0 && CC > 0) {
#pragma unroll
    for (int dy = 0; dy < SS; ++dy) {
      const int iy = Y * SS + dy - p;
#pragma unroll
      for (int dx = 0; dx < SS; ++dx) {
        const int ix = X * SS + dx - p;
        const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
#pragma unroll
        for (int c = 0; c < CC; ++c)
          v[(dy * SS + dx) * CC + c] = ok ? ldg_ro(x + (((long long)b * CC + c) * H + iy) * W + ix) : 0.f;
      }
    }
  } else {
    int ch = 0;
    for (int dy = 0; dy < s; ++dy) {
      const int iy = Y * s + dy - p;
      for (int dx = 0; dx < s; ++dx) {
        const int ix = X * s + dx - p;
        const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
        for (int c = 0; c < C; ++c, ++ch) {
          const float val = ok ? ld(x + (((long long)b * C + c) * H + iy) * W + ix) : 0.f;
#pragma unroll
          for (int i = 0; i < CS; ++i)
            if (i == ch) v[i] = val;
        }
      }
    }
  }
  TD* out = dst + t * CS;
#pragma unroll
  for (int q = 0; q < CS / 8; ++q) Vec8<TD>::store(out + q * 8, v + q * 8);
}

// bf16 source, one CTA per output block row (b, Y): for each channel the SS input
// rows of that block row are one contiguous span of the NCHW plane; it is staged
// into SMEM with 16-byte loads (aligned down, the tail clamped to the tensor),
// then each thread assembles one SS x SS block and writes its CS channels as
// 16-byte stores. Rows/columns outside the image are zero.
__device__ __forceinline__ float s2d_f(float v) { return v; }
__device__ __forceinline__ float s2d_f(double v) { return __double2float_rn(v); }
__device__ __forceinline__ float s2d_f(__nv_bfloat16 v) { return __bfloat162float(v); }

template <int CS, int SS, int CC>
__global__ void __launch_bounds__(64) s2d_rows_k(int H, int W, int p, int Hs, int Ws, long long total,
                                                 const __nv_bfloat16* __restrict__ x,
                                                 __nv_bfloat16* __restrict__ dst, int ones) {
  PC_PDL_TRIGGER();
  extern __shared__ __align__(16) uint8_t s2d_sm[];
  const int span = SS * W;                    // elements of SS consecutive rows
  const int slot = ((span + 7) / 8 + 1) * 8;  // per-channel staging (aligned-down start)
  __nv_bfloat16* lin = reinterpret_cast<__nv_bfloat16*>(s2d_sm);
  __nv_bfloat16* lout = lin + CC * slot;  // [Ws][CS] staged output row (16-byte aligned: slot % 8 == 0)
  const int b = blockIdx.x / Hs, Y = blockIdx.x - b * Hs;
  const int iy0 = Y * SS - p;
  int sh[CC];
#pragma unroll
  for (int c = 0; c < CC; ++c) {
    // rows iy0 .. iy0+SS-1 of plane (b, c), clipped to the image
    const int r0 = iy0 < 0 ? 0 : iy0, r1 = iy0 + SS > H ? H : iy0 + SS;
    const long long e0 = (((long long)b * CC + c) * H + iy0) * W;  // may precede the plane (top padding)
    const long long a0 = e0 & ~7LL;
    sh[c] = (int)(e0 - a0);
    if (r1 <= r0) continue;
    const long long lo = (((long long)b * CC + c) * H + r0) * W, hi = (((long long)b * CC + c) * H + r1) * W;
    const int k0 = (int)((lo - a0) >> 3), k1 = (int)((hi - a0 + 7) >> 3);
    for (int k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
      const long long e = a0 + 8LL * k;
      uint4 u;
      if (e + 8 <= total) {
        u = __ldg(reinterpret_cast<const uint4*>(x + e));
      } else {
        __nv_bfloat16* ub = reinterpret_cast<__nv_bfloat16*>(&u);
        for (int q = 0; q < 8; ++q) ub[q] = e + q < total ? x[e + q] : __float2bfloat16(0.f);
      }
      *reinterpret_cast<uint4*>(lin + c * slot + 8 * k) = u;
    }
  }
  __syncthreads();
  for (int X = threadIdx.x; X < Ws; X += blockDim.x) {
    float v[CS];
#pragma unroll
    for (int i = 0; i < CS; ++i) v[i] = i == ones ? 1.f : 0.f;
#pragma unroll
    for (int dy = 0; dy < SS; ++dy) {
      const int iy = iy0 + dy;
#pragma unroll
      for (int dx = 0; dx < SS; ++dx) {
        const int ix = X * SS + dx - p;
        const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
#pragma unroll
        for (int c = 0; c < CC; ++c)
          v[(dy * SS + dx) * CC + c] = ok ? __bfloat162float(lin[c * slot + sh[c] + dy * W + ix]) : 0.f;
      }
    }
    // stage the block row in SMEM; 16-byte chunk q of block X at slot q ^ (X % 8)
    // (XOR swizzle: conflict-free writes, static register indices)
#pragma unroll
    for (int q = 0; q < CS / 8; ++q) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
      *reinterpret_cast<uint4*>(lout + (X * CS + ((q ^ (X & 7)) % (CS / 8)) * 8)) = u;
    }
  }
  __syncthreads();
  // the (b, Y) block row is contiguous in dst: coalesced 16-byte stores
  static_assert(CS / 8 == 8 || CS / 8 == 4, "swizzle over 8 (or 4) chunks per block");
  uint4* out = reinterpret_cast<uint4*>(dst + (long long)blockIdx.x * Ws * CS);
  const uint4* src = reinterpret_cast<const uint4*>(lout);
  for (int c = threadIdx.x; c < Ws * CS / 8; c += blockDim.x) {
    const int X = c / (CS / 8), q = c % (CS / 8);
    out[c] = src[X * (CS / 8) + ((q ^ (X & 7)) % (CS / 8))];
  }
}

// float / float64 source (the float32 device-resident batch, a caller's float64
// images), one CTA of 64 threads per output block row (b, Y): each of the SS*CC
// input rows of the block row is staged, converted to float and shifted so that
// block X's SS values are one aligned float4 in SMEM (scalar loads, coalesced
// across the warp, 48 independent loads per lane in flight); each thread then
// assembles its block from conflict-free float4 reads and the block row leaves as
// coalesced 16-byte stores through a swizzled SMEM row (as s2d_rows_k).
template <typename TS, int SS, int CC, int IT>
__global__ void __launch_bounds__(64) s2d_rows_f_k(int H, int W, int p, int Hs, int Ws,
                                                   const TS* __restrict__ x, __nv_bfloat16* __restrict__ dst,
                                                   int ones) {
  PC_PDL_TRIGGER();
  constexpr int CS = 64, ROWS = SS * CC, RS = 32 * IT;  // staged row: RS >= SS * Ws values
  static_assert(SS == 4 && ROWS % 2 == 0, "4 values per block, rows split over two warps");
  // staged already rounded to bf16 (the output's rounding of the same float value)
  __shared__ __align__(16) __nv_bfloat16 lin[ROWS * RS];
  __shared__ __align__(16) __nv_bfloat16 lout[RS / SS * CS];
  const int b = blockIdx.x / Hs, Y = blockIdx.x - b * Hs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float val[ROWS / 2][IT];
#pragma unroll
  for (int rr = 0; rr < ROWS / 2; ++rr) {
    const int r = warp * (ROWS / 2) + rr, c = r / SS, dy = r - c * SS;  // row r = (c, dy)
    const int iy = Y * SS + dy - p;
    const bool rok = iy >= 0 && iy < H;
    const TS* src = x + (((long long)b * CC + c) * H + (rok ? iy : 0)) * W;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int ix = lane + 32 * k - p;
      val[rr][k] = rok && ix >= 0 && ix < W ? s2d_f(__ldg(src + ix)) : 0.f;
    }
  }
#pragma unroll
  for (int rr = 0; rr < ROWS / 2; ++rr)
#pragma unroll
    for (int k = 0; k < IT; ++k) lin[(warp * (ROWS / 2) + rr) * RS + lane + 32 * k] = __float2bfloat16_rn(val[rr][k]);
  __syncthreads();
  for (int X = threadIdx.x; X < Ws; X += blockDim.x) {
    float v[CS];
#pragma unroll
    for (int i = 0; i < CS; ++i) v[i] = i == ones ? 1.f : 0.f;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int c = r / SS, dy = r - c * SS;
      const uint2 f = *reinterpret_cast<const uint2*>(lin + r * RS + SS * X);
      v[(dy * SS + 0) * CC + c] = __uint_as_float(f.x << 16);
      v[(dy * SS + 1) * CC + c] = __uint_as_float(f.x & 0xFFFF0000u);
      v[(dy * SS + 2) * CC + c] = __uint_as_float(f.y << 16);
      v[(dy * SS + 3) * CC + c] = __uint_as_float(f.y & 0xFFFF0000u);
    }
#pragma unroll
    for (int q = 0; q < CS / 8; ++q) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
      *reinterpret_cast<uint4*>(lout + (X * CS + (q ^ (X & 7)) * 8)) = u;
    }
  }
  __syncthreads();
  uint4* out = reinterpret_cast<uint4*>(dst + (long long)blockIdx.x * Ws * CS);
  const uint4* sm = reinterpret_cast<const uint4*>(lout);
  for (int c = threadIdx.x; c < Ws * CS / 8; c += blockDim.x) {
    const int X = c / (CS / 8), q = c % (CS / 8);
    out[c] = sm[X * (CS / 8) + (q ^ (X & 7))];
  }
}

__global__ void mask_f32_k(long long n, const uint8_t* __restrict__ keep, float* __restrict__ buf) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!keep[i]) buf[i] = 0.f;
}

// One CTA per image row (b, y): coalesced read of the C planes of that row into
// shared memory, coalesced write of the W x Cp channels-last row.
template <typename T>
__global__ void nchw_to_nhwc_row_k(int C, int H, int W, int Cp, const float* __restrict__ src,
                                   T* __restrict__ dst) {
  extern __shared__ float row[];  // [C][W]
  const int by = blockIdx.x;
  const int b = by / H, y = by - b * H;
  for (int t = threadIdx.x; t < C * W; t += blockDim.x) {
    int c = t / W, x = t - c * W;
    row[t] = src[(((long long)b * C + c) * H + y) * W + x];
  }
  __syncthreads();
  T* out = dst + (long long)by * W * Cp;
  for (int t = threadIdx.x; t < W * Cp; t += blockDim.x) {
    int x = t / Cp, c = t - x * Cp;
    out[t] = cvt<T>(c < C ? row[c * W + x] : 0.f);
  }
}

template <typename T>
__global__ void sum_buffers_k(int k, long long n, const void* const* __restrict__ src,
                              T* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float acc = ld(static_cast<const T*>(src[0]) + i);
    for (int j = 1; j < k; ++j) acc += ld(static_cast<const T*>(src[j]) + i);
    dst[i] = cvt<T>(acc);
  }
}

template <typename S, typename D>
__global__ void cast_k(long long n, const S* __restrict__ src, D* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = cvt<D>(ld(src + i));
}

template <typename T>
__global__ void scale_k(long long n, const T* __restrict__ src, T* __restrict__ dst, float a) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = cvt<T>(ld(src + i) * a);
}

}  // namespace pc

using namespace pc;

#define DISPATCH_PREC(prec, T, ...)                                    \
  do {                                                                 \
    if ((prec) == PC_FP32) { using T = float; __VA_ARGS__; }           \
    else if ((prec) == PC_BF16) { using T = __nv_bfloat16; __VA_ARGS__; } \
    else { pc::set_error("unknown precision"); return PC_EVALUE; }     \
  } while (0)

extern "C" int pc_relu_forward(long long n, const void* x, void* y, int prec, pc_stream_t st) {
  PC_REQUIRE(n >= 0, PC_ESHAPE, "relu: negative size");
  if (n == 0) return PC_OK;
  DISPATCH_PREC(prec, T, relu_fwd_k<T><<<grid_for((n + 7) / 8, 256), 256, 0, S(st)>>>(
      n, static_cast<const T*>(x), static_cast<T*>(y)));
  PC_CUDA_CHECK_LAUNCH("relu_forward");
  return PC_OK;
}

extern "C" int pc_relu_backward(long long n, const void* x, const void* g, void* gx, int prec,
                                pc_stream_t st) {
  PC_REQUIRE(n >= 0, PC_ESHAPE, "relu: negative size");
  if (n == 0) return PC_OK;
  DISPATCH_PREC(prec, T, relu_bwd_k<T><<<grid_for((n + 7) / 8, 256), 256, 0, S(st)>>>(
      n, static_cast<const T*>(x), static_cast<const T*>(g), static_cast<T*>(gx)));
  PC_CUDA_CHECK_LAUNCH("relu_backward");
  return PC_OK;
}

static int pool_geom(int H, int W, int k, int s, int* Ho, int* Wo) {
  PC_REQUIRE(k >= 1 && s >= 1 && k <= 16, PC_EVALUE, "maxpool: bad kernel/stride %d/%d", k, s);
  PC_REQUIRE(H >= k && W >= k && (H - k) % s == 0 && (W - k) % s == 0, PC_EVALUE,
             "maxpool geometry does not tile: %dx%d k%d s%d", H, W, k, s);
  *Ho = (H - k) / s + 1;
  *Wo = (W - k) / s + 1;
  return PC_OK;
}

static bool aligned(const void* p, int a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

extern "C" int pc_maxpool_forward(int B, int H, int W, int C, int k, int s, const void* x, void* y,
                                  uint8_t* argmax, int prec, pc_stream_t st) {
  int Ho, Wo, rc = pool_geom(H, W, k, s, &Ho, &Wo);
  if (rc) return rc;
  if ((long long)B * C == 0) return PC_OK;
  bool vec = C % 8 == 0 && aligned(x, 32) && aligned(y, 32) && aligned(argmax, 8);
  long long work = (long long)B * Ho * Wo * (vec ? C / 8 : C);
  PC_REQUIRE(work < (1LL << 31), PC_EVALUE, "maxpool: too many elements for one launch");
  DISPATCH_PREC(prec, T, {
    if (vec && k == 3 && s == 2 && prec == PC_BF16 && aligned(x, 16) && (long long)B * H * W * C < (1LL << 31))
      maxpool_fwd_bf16_k3s2_k<<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, Ho, Wo, FastDiv(C / 8), FastDiv(Wo), FastDiv(Ho), static_cast<const __nv_bfloat16*>(x),
          static_cast<__nv_bfloat16*>(y), argmax);
    else if (vec && k == 3 && s == 2)
      maxpool_fwd_k<T, 8, 3, 2><<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, k, s, Ho, Wo, static_cast<const T*>(x), static_cast<T*>(y), argmax);
    else if (vec)
      maxpool_fwd_k<T, 8><<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, k, s, Ho, Wo, static_cast<const T*>(x), static_cast<T*>(y), argmax);
    else
      maxpool_fwd_k<T, 1><<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, k, s, Ho, Wo, static_cast<const T*>(x), static_cast<T*>(y), argmax);
  });
  PC_CUDA_CHECK_LAUNCH("maxpool_forward");
  return PC_OK;
}

// enough CTAs that each thread walks only ~1-2 blocks (the gather's load latency is
// hidden by parallelism, as in the plain backward), few enough partial rows to sum
static int pool_bias_ctas() {
  static const int n = [] {
    const char* e = getenv("PC_POOL_BIAS_CTAS");
    return e ? atoi(e) : 148 * 8;
  }();
  return n;
}

extern "C" size_t pc_maxpool_backward_bias_workspace(int C) { return (size_t)pool_bias_ctas() * C * sizeof(float); }

extern "C" int pc_maxpool_backward_bias(int B, int H, int W, int C, int k, int s, const void* gy,
                                        const uint8_t* argmax, const void* mask, void* gx, int prec, float* gb,
                                        void* ws, size_t ws_bytes, pc_stream_t st) {
  if (!gb) return pc_maxpool_backward(B, H, W, C, k, s, gy, argmax, mask, gx, prec, st);
  int Ho, Wo, rc = pool_geom(H, W, k, s, &Ho, &Wo);
  if (rc) return rc;
  PC_REQUIRE(prec == PC_BF16 && k == 3 && s == 2 && C % 8 == 0 && 256 % (C / 8) == 0 && aligned(gy, 32) &&
                 aligned(gx, 32) && aligned(argmax, 8) && (!mask || aligned(mask, 32)) && aligned(ws, 16) &&
                 (long long)B * H * W * C < (1LL << 31),
             PC_EVALUE, "maxpool_backward_bias: bf16 3x3/s2, C/8 dividing 256, aligned buffers, < 2^31 elements");
  PC_REQUIRE(ws_bytes >= pc_maxpool_backward_bias_workspace(C), PC_EVALUE, "maxpool_backward_bias: workspace");
  if ((long long)B * C == 0) {
    cudaMemsetAsync(gb, 0, sizeof(float) * C, S(st));
    return PC_OK;
  }
  float* part = static_cast<float*>(ws);
  maxpool_bwd_bf16_k3s2_bias_k<<<pool_bias_ctas(), 256, 0, S(st)>>>(
      B, H, W, C, Ho, Wo, FastDiv(C / 8), FastDiv((W + 1) / 2), FastDiv((H + 1) / 2),
      static_cast<const __nv_bfloat16*>(gy), argmax, static_cast<const __nv_bfloat16*>(mask),
      static_cast<__nv_bfloat16*>(gx), part);
  pool_bias_rows_k<<<C / 8, 256, 0, S(st)>>>(part, pool_bias_ctas(), C, gb);
  count_launches(1);
  PC_CUDA_CHECK_LAUNCH("maxpool_backward_bias");
  return PC_OK;
}

extern "C" int pc_maxpool_backward(int B, int H, int W, int C, int k, int s, const void* gy,
                                   const uint8_t* argmax, const void* mask, void* gx, int prec,
                                   pc_stream_t st) {
  int Ho, Wo, rc = pool_geom(H, W, k, s, &Ho, &Wo);
  if (rc) return rc;
  if ((long long)B * C == 0) return PC_OK;
  bool vec = C % 8 == 0 && aligned(gy, 32) && aligned(gx, 32) && aligned(argmax, 8) &&
             (!mask || aligned(mask, 32));
  long long work = (long long)B * H * W * (vec ? C / 8 : C);
  PC_REQUIRE(work < (1LL << 31), PC_EVALUE, "maxpool: too many elements for one launch");
  const long long work22 = (long long)B * ((H + 1) / 2) * ((W + 1) / 2) * (C / 8);
  DISPATCH_PREC(prec, T, {
    if (vec && k == 3 && s == 2 && prec == PC_BF16 && (long long)B * H * W * C < (1LL << 31))
      maxpool_bwd_bf16_k3s2_k<<<grid_for(work22, 256), 256, 0, S(st)>>>(
          B, H, W, C, Ho, Wo, FastDiv(C / 8), FastDiv((W + 1) / 2), FastDiv((H + 1) / 2),
          static_cast<const __nv_bfloat16*>(gy), argmax,
          static_cast<const __nv_bfloat16*>(mask), static_cast<__nv_bfloat16*>(gx));
    else if (vec && k == 3 && s == 2)
      maxpool_bwd_k3s2_k<T><<<grid_for(work22, 256), 256, 0, S(st)>>>(
          B, H, W, C, Ho, Wo, static_cast<const T*>(gy), argmax, static_cast<const T*>(mask),
          static_cast<T*>(gx));
    else if (vec)
      maxpool_bwd_k<T, 8><<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, k, s, Ho, Wo, static_cast<const T*>(gy), argmax,
          static_cast<const T*>(mask), static_cast<T*>(gx));
    else
      maxpool_bwd_k<T, 1><<<grid_for(work, 256), 256, 0, S(st)>>>(
          B, H, W, C, k, s, Ho, Wo, static_cast<const T*>(gy), argmax,
          static_cast<const T*>(mask), static_cast<T*>(gx));
  });
  PC_CUDA_CHECK_LAUNCH("maxpool_backward");
  return PC_OK;
}

extern "C" int pc_softmax_xent(int B, int K, const void* logits, const int32_t* labels, double scale,
                               void* grad, double* row_loss, int* bad_label, int prec, pc_stream_t st) {
  PC_REQUIRE(B >= 0 && K >= 2, PC_ESHAPE, "softmax_xent: bad extents B=%d K=%d", B, K);
  if (B == 0) return PC_OK;
  if (K <= 32 * 32) {
    DISPATCH_PREC(prec, T, softmax_xent_warp_k<T, 32><<<(B + 7) / 8, 256, 0, S(st)>>>(
        B, K, static_cast<const T*>(logits), labels, scale, static_cast<T*>(grad), row_loss, bad_label, nullptr,
        nullptr));
  } else {
    DISPATCH_PREC(prec, T, softmax_xent_k<T, 256><<<B, 256, 0, S(st)>>>(
        K, static_cast<const T*>(logits), labels, scale, static_cast<T*>(grad), row_loss, bad_label));
  }
  PC_CUDA_CHECK_LAUNCH("softmax_xent");
  return PC_OK;
}

extern "C" int pc_sum_f64(int n, const double* v, double* out, pc_stream_t st) {
  sum_f64_k<<<1, 256, 0, S(st)>>>(n, v, out);
  PC_CUDA_CHECK_LAUNCH("sum_f64");
  return PC_OK;
}

extern "C" int pc_softmax_xent_loss(int B, int K, const void* logits, const int32_t* labels, double scale, void* grad,
                                    double* row_loss, int* bad_label, double* loss, unsigned* ticket, int prec,
                                    pc_stream_t st) {
  PC_REQUIRE(B >= 0 && K >= 2, PC_ESHAPE, "softmax_xent: bad extents B=%d K=%d", B, K);
  if (B == 0) return pc_sum_f64(0, row_loss, loss, st);
  if (K > 32 * 32 || ticket == nullptr) {
    int rc = pc_softmax_xent(B, K, logits, labels, scale, grad, row_loss, bad_label, prec, st);
    return rc ? rc : pc_sum_f64(B, row_loss, loss, st);
  }
  DISPATCH_PREC(prec, T, softmax_xent_warp_k<T, 32><<<(B + 7) / 8, 256, 0, S(st)>>>(
      B, K, static_cast<const T*>(logits), labels, scale, static_cast<T*>(grad), row_loss, bad_label, loss,
      ticket));
  PC_CUDA_CHECK_LAUNCH("softmax_xent_loss");
  return PC_OK;
}

extern "C" int pc_sgd_step(int n_tensors, const pc_sgd_tensor* table, long long max_numel, float lr,
                           float momentum, float weight_decay, pc_stream_t st) {
  PC_REQUIRE(n_tensors >= 0 && n_tensors <= 65535, PC_EVALUE, "sgd: bad tensor count %d", n_tensors);
  if (n_tensors == 0 || max_numel <= 0) return PC_OK;
  int gx = grid_for((max_numel + 3) / 4, 256);
  if (gx > 1184) gx = 1184;  // 8 CTAs per SM on 148 SMs; grid-stride beyond that
  sgd_k<<<dim3(gx, n_tensors), 256, 0, S(st)>>>(table, lr, momentum, weight_decay);
  PC_CUDA_CHECK_LAUNCH("sgd_step");
  return PC_OK;
}

extern "C" int pc_sgd_step_ex(int n_tensors, const pc_sgd_tensor* table, long long max_numel, float lr,
                              float momentum, float weight_decay, int ctas_per_sm, pc_stream_t st) {
  if (ctas_per_sm <= 0) return pc_sgd_step(n_tensors, table, max_numel, lr, momentum, weight_decay, st);
  PC_REQUIRE(n_tensors >= 0 && n_tensors <= 65535, PC_EVALUE, "sgd: bad tensor count %d", n_tensors);
  if (n_tensors == 0 || max_numel <= 0) return PC_OK;
  static int sms = [] {
    int d = 0, n = 148;
    if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  int gx = sms * ctas_per_sm / n_tensors;
  const int need = grid_for((max_numel + 3) / 4, 256);
  if (gx > need) gx = need;
  if (gx < 1) gx = 1;
  sgd_bg_k<<<dim3(gx, n_tensors), 256, 0, S(st)>>>(table, lr, momentum, weight_decay);
  PC_CUDA_CHECK_LAUNCH("sgd_step_ex");
  return PC_OK;
}

extern "C" int pc_nchw_to_nhwc(int B, int C, int H, int W, int Cp, const float* src, void* dst,
                               int prec, pc_stream_t st) {
  PC_REQUIRE(Cp >= C, PC_ESHAPE, "nchw_to_nhwc: Cp < C");
  long long n = (long long)B * H * W * Cp;
  if (n == 0) return PC_OK;
  size_t row_bytes = sizeof(float) * (size_t)C * W;
  if (row_bytes <= 48 * 1024) {
    DISPATCH_PREC(prec, T, nchw_to_nhwc_row_k<T><<<B * H, 256, row_bytes, S(st)>>>(
        C, H, W, Cp, src, static_cast<T*>(dst)));
  } else {
    DISPATCH_PREC(prec, T, nchw_to_nhwc_k<T><<<grid_for(n, 256), 256, 0, S(st)>>>(
        B, C, H, W, Cp, src, static_cast<T*>(dst)));
  }
  PC_CUDA_CHECK_LAUNCH("nchw_to_nhwc");
  return PC_OK;
}

extern "C" int pc_im2col(int B, int C, int H, int W, int k, int s, int p, int Kp, const void* src, int src_prec,
                         void* dst, pc_stream_t st) {
  return pc_im2col_ex(B, C, H, W, k, s, p, Kp, src, src_prec, dst, PC_BF16, st);
}

extern "C" int pc_im2col_ex(int B, int C, int H, int W, int k, int s, int p, int Kp, const void* src, int src_prec,
                            void* dst, int dst_prec, pc_stream_t st) {
  PC_REQUIRE(B >= 0 && C > 0 && k > 0 && s > 0 && p >= 0 && Kp % 8 == 0 && Kp >= C * k * k, PC_EVALUE,
             "im2col: bad arguments (Kp must be a multiple of 8 and >= C*k*k)");
  int sh = H + 2 * p - k, sw = W + 2 * p - k;
  PC_REQUIRE(sh >= 0 && sw >= 0 && sh % s == 0 && sw % s == 0, PC_EVALUE, "im2col: geometry does not tile");
  int Ho = sh / s + 1, Wo = sw / s + 1;
  size_t smem = sizeof(float) * (size_t)C * k * W;
  PC_REQUIRE(smem <= 200 * 1024, PC_EVALUE, "im2col: input rows do not fit shared memory");
  if (B == 0) return PC_OK;
  DISPATCH_PREC(src_prec, TS, {
    DISPATCH_PREC(dst_prec, TD, {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(im2col_rows_k<TS, TD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      im2col_rows_k<TS, TD><<<B * Ho, 256, smem, S(st)>>>(C, H, W, k, s, p, Ho, Wo, Kp, static_cast<const TS*>(src),
                                                          static_cast<TD*>(dst));
    });
  });
  PC_CUDA_CHECK_LAUNCH("im2col");
  return PC_OK;
}

extern "C" int pc_space_to_depth(int B, int C, int H, int W, int s, int p, int Cs, const void* src, int src_prec,
                                 void* dst, pc_stream_t st) {
  return pc_space_to_depth_ex(B, C, H, W, s, p, Cs, src, src_prec, -1, dst, st);
}

// Float32 output (the tf32 mode's input layer runs the same space-to-depth 3x3 conv).
extern "C" int pc_space_to_depth_f32(int B, int C, int H, int W, int s, int p, int Cs, const void* src,
                                     int src_prec, int ones, float* dst, pc_stream_t st) {
  PC_REQUIRE(B >= 0 && C > 0 && H > 0 && W > 0 && s > 0 && p >= 0 && Cs >= s * s * C && (Cs == 64 || Cs == 32),
             PC_EVALUE, "space_to_depth: bad arguments (Cs must be 32 or 64 and >= s*s*C)");
  PC_REQUIRE(ones < 0 || (ones >= s * s * C && ones < Cs), PC_EVALUE,
             "space_to_depth: the ones channel must be a padding channel");
  const int Hs = (H + 2 * p + s - 1) / s, Ws = (W + 2 * p + s - 1) / s;
  const long long n = (long long)B * Hs * Ws;
  if (n == 0) return PC_OK;
  const int g = grid_for(n, 256);
  if (src_prec == PC_FP64) {
    const double* x = static_cast<const double*>(src);
    PC_REQUIRE(Cs == 64 && C == 3 && (s == 4 || s == 2), PC_EVALUE, "space_to_depth: float64 source needs C=3, s=2|4");
    if (s == 4) s2d_k<double, 64, 4, 3, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
    else s2d_k<double, 64, 2, 3, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
    PC_CUDA_CHECK_LAUNCH("space_to_depth");
    return PC_OK;
  }
  DISPATCH_PREC(src_prec, TS, {
    const TS* x = static_cast<const TS*>(src);
    if (Cs == 64 && s == 4 && C == 3)
      s2d_k<TS, 64, 4, 3, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
    else if (Cs == 64 && s == 2 && C == 3)
      s2d_k<TS, 64, 2, 3, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
    else if (Cs == 64)
      s2d_k<TS, 64, 0, 0, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
    else
      s2d_k<TS, 32, 0, 0, float><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, dst, ones);
  });
  PC_CUDA_CHECK_LAUNCH("space_to_depth");
  return PC_OK;
}

extern "C" int pc_space_to_depth_ex(int B, int C, int H, int W, int s, int p, int Cs, const void* src,
                                    int src_prec, int ones, void* dst, pc_stream_t st) {
  PC_REQUIRE(B >= 0 && C > 0 && H > 0 && W > 0 && s > 0 && p >= 0 && Cs >= s * s * C && (Cs == 64 || Cs == 32),
             PC_EVALUE, "space_to_depth: bad arguments (Cs must be 32 or 64 and >= s*s*C)");
  PC_REQUIRE(ones < 0 || (ones >= s * s * C && ones < Cs), PC_EVALUE,
             "space_to_depth: the ones channel must be a padding channel");
  const int Hs = (H + 2 * p + s - 1) / s, Ws = (W + 2 * p + s - 1) / s;
  const long long n = (long long)B * Hs * Ws;
  if (n == 0) return PC_OK;
  const int g = grid_for(n, 256);
  auto* d = static_cast<__nv_bfloat16*>(dst);
  static const int rows_f = [] {   // PC_S2D_ROWS=0: the per-block kernel for float / float64 sources
    const char* e = getenv("PC_S2D_ROWS");
    return e ? atoi(e) : 1;
  }();
  if (rows_f && Cs == 64 && s == 4 && C == 3 && Ws * 4 <= 256 &&
      (src_prec == PC_FP32 || src_prec == PC_FP64 || (rows_f == 2 && src_prec == PC_BF16))) {
    if (src_prec == PC_BF16)
      s2d_rows_f_k<__nv_bfloat16, 4, 3, 8><<<B * Hs, 64, 0, S(st)>>>(H, W, p, Hs, Ws,
                                                                     static_cast<const __nv_bfloat16*>(src), d, ones);
    else if (src_prec == PC_FP32)
      s2d_rows_f_k<float, 4, 3, 8><<<B * Hs, 64, 0, S(st)>>>(H, W, p, Hs, Ws, static_cast<const float*>(src), d, ones);
    else
      s2d_rows_f_k<double, 4, 3, 8><<<B * Hs, 64, 0, S(st)>>>(H, W, p, Hs, Ws, static_cast<const double*>(src), d,
                                                             ones);
    PC_CUDA_CHECK_LAUNCH("space_to_depth");
    return PC_OK;
  }
  if (src_prec == PC_BF16 && Cs == 64 && s == 4 && C == 3 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const size_t smem = (size_t)C * (((size_t)s * W + 7) / 8 + 1) * 8 * 2 + (size_t)Ws * 64 * 2;
    if (smem <= 48 * 1024) {  // AlexNet conv1: row-staged
      s2d_rows_k<64, 4, 3><<<B * Hs, 64, smem, S(st)>>>(H, W, p, Hs, Ws, (long long)B * C * H * W,
                                                         static_cast<const __nv_bfloat16*>(src), d, ones);
      PC_CUDA_CHECK_LAUNCH("space_to_depth");
      return PC_OK;
    }
  }
  if (src_prec == PC_FP64) {   // float64 images straight from the caller (fixed-geometry kernels only)
    const double* x = static_cast<const double*>(src);
    PC_REQUIRE(Cs == 64 && C == 3 && (s == 4 || s == 2), PC_EVALUE, "space_to_depth: float64 source needs C=3, s=2|4");
    if (s == 4) s2d_k<double, 64, 4, 3><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
    else s2d_k<double, 64, 2, 3><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
    PC_CUDA_CHECK_LAUNCH("space_to_depth");
    return PC_OK;
  }
  DISPATCH_PREC(src_prec, TS, {
    const TS* x = static_cast<const TS*>(src);
    if (Cs == 64 && s == 4 && C == 3)        // AlexNet conv1 (11x11/s4)
      s2d_k<TS, 64, 4, 3><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
    else if (Cs == 64 && s == 2 && C == 3)   // small64 conv1 (6x6/s2)
      s2d_k<TS, 64, 2, 3><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
    else if (Cs == 64)
      s2d_k<TS, 64, 0, 0><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
    else
      s2d_k<TS, 32, 0, 0><<<g, 256, 0, S(st)>>>(B, C, H, W, s, p, Hs, Ws, x, d, ones);
  });
  PC_CUDA_CHECK_LAUNCH("space_to_depth");
  return PC_OK;
}

// Input-layer weight gradient finish: gb[n] = gw[n][ones] (the weight gradient
// of the all-ones padding channel at tap (0, 0) IS the bias gradient: sum over
// pixels of gy * 1), then the structural zeros are pinned (keep mask).
__global__ void s2d_wgrad_finish_k(int N, int K, int ones, const uint8_t* __restrict__ keep,
                                   float* __restrict__ gw, float* __restrict__ gb) {
  PC_PDL_TRIGGER();
  const long long n = (long long)N * K;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / K), c = (int)(i - (long long)r * K);
    if (c == ones) gb[r] = gw[i];
    if (!keep[i]) gw[i] = 0.f;
  }
}

extern "C" int pc_s2d_wgrad_finish(int N, int K, int ones, const uint8_t* keep, float* gw, float* gb,
                                   pc_stream_t st) {
  PC_REQUIRE(N > 0 && K > 0 && ones >= 0 && ones < K && keep && gw && gb, PC_EVALUE, "s2d_wgrad_finish: bad arguments");
  int g = grid_for((long long)N * K, 256);
  if (g > 148 * 8) g = 148 * 8;
  s2d_wgrad_finish_k<<<g, 256, 0, S(st)>>>(N, K, ones, keep, gw, gb);
  PC_CUDA_CHECK_LAUNCH("s2d_wgrad_finish");
  return PC_OK;
}

extern "C" int pc_mask_f32(long long n, const uint8_t* keep, float* buf, pc_stream_t st) {
  if (n == 0) return PC_OK;
  int g = grid_for(n, 256);
  if (g > 148 * 8) g = 148 * 8;
  mask_f32_k<<<g, 256, 0, S(st)>>>(n, keep, buf);
  PC_CUDA_CHECK_LAUNCH("mask_f32");
  return PC_OK;
}

extern "C" int pc_sum_buffers(int k, long long n, const void* const* src, void* dst, int prec,
                              pc_stream_t st) {
  PC_REQUIRE(k >= 1, PC_EVALUE, "sum_buffers: k < 1");
  if (n == 0) return PC_OK;
  int g = grid_for(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  DISPATCH_PREC(prec, T, sum_buffers_k<T><<<g, 256, 0, S(st)>>>(k, n, src, static_cast<T*>(dst)));
  PC_CUDA_CHECK_LAUNCH("sum_buffers");
  return PC_OK;
}

extern "C" int pc_cast(long long n, const void* src, int sp, void* dst, int dp, pc_stream_t st) {
  if (n == 0) return PC_OK;
  int g = grid_for(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  DISPATCH_PREC(sp, TS, DISPATCH_PREC(dp, TD, cast_k<TS, TD><<<g, 256, 0, S(st)>>>(
      n, static_cast<const TS*>(src), static_cast<TD*>(dst))));
  PC_CUDA_CHECK_LAUNCH("cast");
  return PC_OK;
}

extern "C" int pc_scale(long long n, const void* src, void* dst, float a, int prec, pc_stream_t st) {
  if (n == 0) return PC_OK;
  int g = grid_for(n, 256);
  if (g > 148 * 16) g = 148 * 16;
  DISPATCH_PREC(prec, T, scale_k<T><<<g, 256, 0, S(st)>>>(n, static_cast<const T*>(src),
                                                           static_cast<T*>(dst), a));
  PC_CUDA_CHECK_LAUNCH("scale");
  return PC_OK;
}
