// extern "C" entry points for the contractions (conv / FC) and the shared
// reductions; dispatches PC_FP32 to the exact-fp32 SIMT path and PC_BF16 to
// the tcgen05 tensor-core path (umma_gemm.cu).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "gemm_ops.cuh"
#include "tf32.cuh"
#include "umma.cuh"

namespace pc {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
static std::atomic<unsigned long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

__global__ void reduce_partials_k(const float* __restrict__ ws, int splits, long long n,
                                  float* __restrict__ out, pc_sgd_fuse upd, int fused) {
  PC_PDL_TRIGGER();
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < n;
       i += (long long)gridDim.x * blockDim.x * 4) {
    if (i + 4 <= n && (n & 3) == 0) {
      float4 a = __ldg(reinterpret_cast<const float4*>(ws + i));
      for (int z = 1; z < splits; ++z) {
        float4 b = __ldg(reinterpret_cast<const float4*>(ws + z * n + i));
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      if (fused) {
        sgd_apply4(upd, i, a);
      } else {
        *reinterpret_cast<float4*>(out + i) = a;
      }
    } else {
      for (long long j = i; j < n && j < i + 4; ++j) {
        float a = ws[j];
        for (int z = 1; z < splits; ++z) a += ws[z * n + j];
        if (fused) sgd_apply(upd, j, a);
        else out[j] = a;
      }
    }
  }
}

// Many slices of a short output (the input layer: 148 slices of 55 K weights):
// 8 lanes per float4, lane l summing slices l, l + 8, ... (unrolled, loads in
// flight), then a fixed xor-shuffle tree — deterministic, and 8x the parallelism
// of one thread walking all slices.
__global__ void __launch_bounds__(256) reduce_partials_wide_k(const float* __restrict__ ws, int splits, long long n,
                                                              float* __restrict__ out, pc_sgd_fuse upd, int fused) {
  PC_PDL_TRIGGER();
  const long long i = ((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 3) * 4;
  const int lane = threadIdx.x & 7;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n) {
#pragma unroll 4
    for (int z = lane; z < splits; z += 8) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(ws + z * n + i));
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
    a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
    a.z += __shfl_xor_sync(0xffffffffu, a.z, o);
    a.w += __shfl_xor_sync(0xffffffffu, a.w, o);
  }
  if (lane == 0 && i < n) {
    if (fused) sgd_apply4(upd, i, a);
    else *reinterpret_cast<float4*>(out + i) = a;
  }
}

int reduce_partials(const float* ws, int splits, long long n, float* out, cudaStream_t st, const pc_sgd_fuse* upd) {
  if (n == 0) return PC_OK;
  if (splits >= 32 && (n & 3) == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 &&
      (upd || (reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
    pc_sgd_fuse u;
    memset(&u, 0, sizeof(u));
    if (upd) u = *upd;
    const long long threads = (n / 4) * 8;
    reduce_partials_wide_k<<<(int)((threads + 255) / 256), 256, 0, st>>>(ws, splits, n, out, u, upd != nullptr);
    PC_CUDA_CHECK_LAUNCH("reduce_partials");
    return PC_OK;
  }
  long long g = (n / 4 + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  pc_sgd_fuse u;
  memset(&u, 0, sizeof(u));
  if (upd) u = *upd;
  reduce_partials_k<<<(int)g, 256, 0, st>>>(ws, splits, n, out, u, upd != nullptr);
  PC_CUDA_CHECK_LAUNCH("reduce_partials");
  return PC_OK;
}

__global__ void sgd_region_k(const float* __restrict__ g, long long n, pc_sgd_fuse upd) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    sgd_apply(upd, i, g[i]);
}

// Update from a materialised gradient (paths without a fused epilogue).
int apply_sgd(const float* g, long long n, const pc_sgd_fuse* upd, cudaStream_t st) {
  if (n == 0) return PC_OK;
  long long b = (n + 255) / 256;
  sgd_region_k<<<(int)(b > 1184 ? 1184 : b), 256, 0, st>>>(g, n, *upd);
  PC_CUDA_CHECK_LAUNCH("apply_sgd");
  return PC_OK;
}

// Bias gradients: pass 1 sums rows [r*RB, (r+1)*RB) per column block; pass 2
// sums the row-block partials in ascending order. Fixed order => deterministic.
// Row blocks are sized so pass 1 keeps ~8 CTAs per SM in flight; pass 2 gives
// each column a warp (fixed-order strided sums, then a fixed shuffle tree).
// Rows per pass-1 block: each of the CTA's row lanes (256 threads / 8-column groups)
// sums ~24 rows, so pass 1 has many CTAs with many 16-byte loads in flight.
// Rows per pass-1 block: enough blocks for ~8 resident CTAs on each of 148 SMs
// (the conv3-5 upstream gradients, 22-33 MB, ran at ~3 TB/s with 2.4 CTAs per SM),
// at least 4 rows per lane.
static long long cs_rb(long long P, int N) {
  const int groups = N % 8 == 0 ? N / 8 : 0;
  if (!groups) return 512;
  const long long lanes = 256 / (groups < 256 ? groups : 256);
  static const int occ = [] {  // target pass-1 CTAs per SM (PC_CS_OCC; 0 = 24 rows per lane)
    const char* e = getenv("PC_CS_OCC");
    return e ? atoi(e) : 8;
  }();
  if (occ <= 0) return lanes * 24;
  const long long want = (P + 148LL * occ - 1) / (148LL * occ);
  const long long rb = (want + lanes - 1) / lanes * lanes;
  return rb > lanes * 4 ? rb : lanes * 4;
}
long long colsum_ws(long long P, int N) { return ((P + cs_rb(P, N) - 1) / cs_rb(P, N)) * (long long)N; }

template <typename T>
__global__ void colsum1_k(const T* __restrict__ g, long long P, int N, int RB, float* __restrict__ part) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  long long r0 = (long long)blockIdx.y * RB, r1 = min(P, r0 + RB);
  float acc = 0.f;
  for (long long r = r0; r < r1; ++r) acc += ld(g + r * N + c);
  part[(long long)blockIdx.y * N + c] = acc;
}

template <typename T> struct V8;
template <> struct V8<__nv_bfloat16> {
  static __device__ __forceinline__ void add(const __nv_bfloat16* p, float* a) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      a[2 * i] += f.x;
      a[2 * i + 1] += f.y;
    }
  }
};
template <> struct V8<float> {
  static __device__ __forceinline__ void add(const float* p, float* a) {
    float4 x = __ldg(reinterpret_cast<const float4*>(p)), y = __ldg(reinterpret_cast<const float4*>(p) + 1);
    a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w; a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
  }
};

// Vectorised pass 1 (N % 8 == 0, 16-byte rows): a CTA owns CB 8-column groups of
// one row block; its 256 threads are CB column groups x (256 / CB) row lanes, each
// lane accumulating 8 columns with 16-byte loads; lanes combine in a fixed order.
template <typename T>
__global__ void __launch_bounds__(256) colsum1_v8_k(const T* __restrict__ g, long long P, int N, int RB,
                                                    float* __restrict__ part) {
  PC_PDL_TRIGGER();
  __shared__ float sh[256 * 8];
  const int groups = N / 8;
  const int CB = min(groups, 256), lanes = 256 / CB;
  const int q = threadIdx.x % CB, lane = threadIdx.x / CB;
  const int grp = blockIdx.x * CB + q;
  const long long r0 = (long long)blockIdx.y * RB, r1 = min(P, r0 + RB);
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (lane < lanes && grp < groups) {
    const T* col = g + (long long)grp * 8;
#pragma unroll 4
    for (long long r = r0 + lane; r < r1; r += lanes) V8<T>::add(col + r * N, a);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sh[threadIdx.x * 8 + i] = a[i];
  __syncthreads();
  for (int t = threadIdx.x; t < CB * 8; t += 256) {
    const int qq = t / 8, i = t % 8;
    if (blockIdx.x * CB + qq >= groups) continue;
    float s = 0.f;
    for (int l = 0; l < lanes; ++l) s += sh[(l * CB + qq) * 8 + i];
    part[(long long)blockIdx.y * N + (long long)(blockIdx.x * CB + qq) * 8 + i] = s;
  }
}

// Pass 2: a CTA per 8 columns, 128 row lanes each (a warp reads 4 rows x 32 B);
// lane partials are combined in a fixed order (deterministic). Wide lanes keep
// each lane's chain of dependent L2 loads short (R is ~1000-1500 row blocks).
constexpr int CS2_LANES = 128;
__global__ void __launch_bounds__(8 * CS2_LANES) colsum2_k(const float* __restrict__ part, int R, int N,
                                                           float* __restrict__ out) {
  PC_PDL_TRIGGER();
  __shared__ float sh[CS2_LANES][9];
  __shared__ float sh2[8][9];
  const int cx = threadIdx.x & 7, ry = threadIdx.x >> 3;
  const int c = blockIdx.x * 8 + cx;
  float acc = 0.f;
  if (c < N)
#pragma unroll 4
    for (int r = ry; r < R; r += CS2_LANES) acc += part[(long long)r * N + c];
  sh[ry][cx] = acc;
  __syncthreads();
  if (ry < 8) {  // 8 x 8 threads: each sums 16 lanes of one column, then lane ry == 0 combines
    float t = 0.f;
    for (int k = 0; k < CS2_LANES / 8; ++k) t += sh[ry * (CS2_LANES / 8) + k][cx];
    sh2[ry][cx] = t;
  }
  __syncthreads();
  if (ry == 0 && c < N) {
    float t = sh2[0][cx];
    for (int k = 1; k < 8; ++k) t += sh2[k][cx];
    out[c] = t;
  }
}

// Short reductions (FC: P = batch): one pass, a CTA per 64 columns (8 groups of
// 8) x 32 row lanes; the lanes are combined in a fixed order.
template <typename T>
__global__ void __launch_bounds__(256) colsum_short_k(const T* __restrict__ g, int P, int N, float* __restrict__ out) {
  PC_PDL_TRIGGER();
  __shared__ float sh[32][64 + 1];
  const int q = threadIdx.x & 7, lane = threadIdx.x >> 3;
  const int grp = blockIdx.x * 8 + q;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (grp < N / 8) {
    const T* col = g + (long long)grp * 8;
#pragma unroll 4
    for (int r = lane; r < P; r += 32) V8<T>::add(col + (long long)r * N, a);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sh[lane][q * 8 + i] = a[i];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = blockIdx.x * 64 + threadIdx.x;
    float t = sh[0][threadIdx.x];
    for (int l = 1; l < 32; ++l) t += sh[l][threadIdx.x];
    if (c < N) out[c] = t;
  }
}

int colsum(const void* g, long long P, int N, int prec, float* out, float* ws, cudaStream_t st) {
  if (N == 0) return PC_OK;
  if (P > 0 && P <= 4096 && N % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
    const int blocks = (N + 63) / 64;
    if (prec == PC_FP32)
      colsum_short_k<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(g), (int)P, N, out);
    else
      colsum_short_k<__nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(g), (int)P, N, out);
    PC_CUDA_CHECK_LAUNCH("colsum");
    return PC_OK;
  }
  const int RB = (int)cs_rb(P, N);
  int R = (int)((P + RB - 1) / RB);
  if (R == 0) {
    cudaMemsetAsync(out, 0, sizeof(float) * N, st);
    return PC_OK;
  }
  const bool vec = N % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  if (vec) {
    const int groups = N / 8, CB = groups < 256 ? groups : 256;
    dim3 g1((groups + CB - 1) / CB, R);
    if (prec == PC_FP32)
      colsum1_v8_k<float><<<g1, 256, 0, st>>>(static_cast<const float*>(g), P, N, RB, ws);
    else
      colsum1_v8_k<__nv_bfloat16><<<g1, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(g), P, N, RB, ws);
  } else {
    dim3 g1((N + 127) / 128, R);
    if (prec == PC_FP32)
      colsum1_k<float><<<g1, 128, 0, st>>>(static_cast<const float*>(g), P, N, RB, ws);
    else
      colsum1_k<__nv_bfloat16><<<g1, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(g), P, N, RB, ws);
  }
  colsum2_k<<<(N + 7) / 8, 8 * CS2_LANES, 0, st>>>(ws, R, N, out);
  count_launches(1);
  PC_CUDA_CHECK_LAUNCH("colsum");
  return PC_OK;
}

static int check_prec(int prec);

// Background bias gradient (side stream, beside the data/weight-gradient GEMMs,
// whose persistent CTAs hold nearly all shared memory): no shared memory, a
// fixed grid of `ctas` CTAs. Pass 1: thread t owns 8-column group t % G and row
// lane t / G of L = threads / G lanes, summing rows lane, lane + L, ... into
// part[lane][.]; pass 2: a warp per 8-column group, lane l summing partial rows
// l, l + 32, ... then a fixed xor-shuffle tree. Fixed order => deterministic.
template <typename T>
__global__ void __launch_bounds__(256) bias_bg1_k(const T* __restrict__ g, long long P, int N, int L,
                                                  float* __restrict__ part) {
  const int groups = N / 8;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = t % groups, lane = t / groups;
  if (lane >= L) return;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const T* col = g + (long long)grp * 8;
#pragma unroll 4
  for (long long r = lane; r < P; r += L) V8<T>::add(col + r * N, a);
  float4* o = reinterpret_cast<float4*>(part + (long long)lane * N + grp * 8);
  o[0] = make_float4(a[0], a[1], a[2], a[3]);
  o[1] = make_float4(a[4], a[5], a[6], a[7]);
}

__global__ void __launch_bounds__(128) bias_bg2_k(const float* __restrict__ part, int L, int N,
                                                  float* __restrict__ out) {
  const int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (grp >= N / 8) return;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int r = lane; r < L; r += 32) V8<float>::add(part + (long long)r * N + grp * 8, a);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] += __shfl_xor_sync(0xffffffffu, a[i], o);
  if (lane < 8) {
    float v = a[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) v = lane == i ? a[i] : v;
    out[grp * 8 + lane] = v;
  }
}

static int bias_bg_lanes(int N, int ctas) { return (ctas * 256) / (N / 8); }

extern "C" PC_API size_t pc_bias_grad_workspace(long long P, int N, int ctas) {
  if (N <= 0 || N % 8 || ctas <= 0) return 0;
  return (size_t)bias_bg_lanes(N, ctas) * N * sizeof(float);
}

extern "C" PC_API int pc_bias_grad(long long P, int N, const void* gy, int prec, float* gb, float* ws, size_t ws_bytes,
                            int ctas, pc_stream_t st) {
  PC_REQUIRE(N > 0 && N % 8 == 0 && P >= 0 && ctas > 0 && (reinterpret_cast<uintptr_t>(gy) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(ws) & 15) == 0,
             PC_EVALUE, "bias_grad: N %% 8 == 0, 16-byte aligned buffers required");
  PC_REQUIRE(ws_bytes >= pc_bias_grad_workspace(P, N, ctas), PC_EVALUE, "bias_grad: workspace too small");
  int rc = check_prec(prec);
  if (rc) return rc;
  const int L = bias_bg_lanes(N, ctas);
  PC_REQUIRE(L >= 1, PC_EVALUE, "bias_grad: too few CTAs for %d columns", N);
  const int blocks = (int)(((long long)L * (N / 8) + 255) / 256);
  if (prec == PC_FP32)
    bias_bg1_k<float><<<blocks, 256, 0, S(st)>>>(static_cast<const float*>(gy), P, N, L, ws);
  else
    bias_bg1_k<__nv_bfloat16><<<blocks, 256, 0, S(st)>>>(static_cast<const __nv_bfloat16*>(gy), P, N, L, ws);
  bias_bg2_k<<<(N / 8 + 3) / 4, 128, 0, S(st)>>>(ws, L, N, gb);
  count_launches(1);
  PC_CUDA_CHECK_LAUNCH("bias_grad");
  return PC_OK;
}

static int check_geom(const pc_conv_geom* g) {
  PC_REQUIRE(g != nullptr, PC_EVALUE, "null conv geometry");
  PC_REQUIRE(g->B >= 0 && g->H > 0 && g->W > 0 && g->C > 0 && g->N > 0 && g->k > 0 && g->stride > 0 &&
                 g->pad >= 0, PC_ESHAPE, "conv: non-positive extent");
  int sh = g->H + 2 * g->pad - g->k, sw = g->W + 2 * g->pad - g->k;
  PC_REQUIRE(sh >= 0 && sw >= 0 && sh % g->stride == 0 && sw % g->stride == 0, PC_EVALUE,
             "conv geometry does not produce an integer output extent: input %dx%d, kernel %d, "
             "stride %d, pad %d", g->H, g->W, g->k, g->stride, g->pad);
  PC_REQUIRE(g->Ho == sh / g->stride + 1 && g->Wo == sw / g->stride + 1, PC_ESHAPE,
             "conv: output extents %dx%d do not match geometry", g->Ho, g->Wo);
  PC_REQUIRE(g->cs > 0 && g->C % g->cs == 0, PC_ESHAPE, "conv: channel block %d does not divide %d",
             g->cs, g->C);
  PC_REQUIRE(g->k * g->k <= 255, PC_EVALUE, "conv: kernel too large");
  return PC_OK;
}

static int check_prec(int prec) {
  PC_REQUIRE(prec == PC_FP32 || prec == PC_BF16, PC_EVALUE, "unknown precision %d", prec);
  return PC_OK;
}
// contraction entry points also take PC_TF32: float storage, tf32 tensor-core math
static int check_cprec(int prec) {
  PC_REQUIRE(prec == PC_FP32 || prec == PC_BF16 || prec == PC_TF32, PC_EVALUE, "unknown precision %d", prec);
  return PC_OK;
}
static int storage(int prec) { return prec == PC_TF32 ? PC_FP32 : prec; }

}  // namespace pc

using namespace pc;

extern "C" const char* pc_last_error(void) { return g_err.c_str(); }
extern "C" int pc_version(void) { return 1; }
extern "C" PC_API int pc_set_grid_cap(int ctas) {
  PC_REQUIRE(ctas >= 0, PC_EVALUE, "grid cap must be >= 0");
  set_grid_cap(ctas);
  return PC_OK;
}
extern "C" unsigned long long pc_launch_count(void) { return g_launches.load(); }

// Single-process multi-GPU fabric: the calling thread's current device may read
// `peer`'s memory directly (pc_sum_buffers over peer pointers, peer copies over NVLink).
extern "C" PC_API int pc_enable_peer_access(int peer) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "enable_peer_access: %s", cudaGetErrorString(e));
  if (peer == dev) return PC_OK;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, dev, peer);
  PC_REQUIRE(can, PC_ECUDA, "device %d cannot access device %d's memory (no P2P path)", dev, peer);
  e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return PC_OK;
  }
  PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "cudaDeviceEnablePeerAccess(%d): %s", peer, cudaGetErrorString(e));
  return PC_OK;
}

// dst <- src (bytes), either device (unified addressing; a peer copy between GPUs), on `stream`.
extern "C" PC_API int pc_copy_async(void* dst, const void* src, size_t bytes, pc_stream_t st) {
  if (bytes == 0) return PC_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(st));
  PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "copy_async: %s", cudaGetErrorString(e));
  return PC_OK;
}
extern "C" int pc_has_tcgen05(void) { return umma_available() ? 1 : 0; }

extern "C" int pc_conv2d_forward(const pc_conv_geom* g, const void* x, const void* w, const float* bias,
                                 void* y, int prec, int flags, pc_stream_t st) {
  int rc = check_geom(g);
  if (rc || (rc = check_cprec(prec))) return rc;
  if (g->B == 0) return PC_OK;
  if (prec == PC_BF16) return umma_conv_forward(*g, x, w, bias, y, flags, S(st));
  if (prec == PC_TF32 && tf32_conv_ok(*g))
    return tf32_conv_forward(*g, static_cast<const float*>(x), static_cast<const float*>(w), bias,
                             static_cast<float*>(y), flags, S(st));
  return simt_conv_forward(*g, x, w, bias, y, storage(prec), flags, S(st));
}

static bool tf32_conv_dgrad_ok(const pc_conv_geom& g) { return tf32_conv_ok(g) && g.stride == 1 && g.N % 32 == 0; }

extern "C" size_t pc_conv2d_backward_workspace(const pc_conv_geom* g, int prec) {
  if (check_geom(g)) return 0;
  long long P = (long long)g->B * g->Ho * g->Wo;
  long long MN = (long long)g->N * g->k * g->k * g->C;
  const bool tc32 = prec == PC_TF32 && tf32_conv_ok(*g);
  long long splits = prec == PC_BF16 ? umma_wgrad_splits(*g)
                     : tc32 ? tf32_wgrad_splits(*g) : simt_splits(g->N, g->k * g->k * g->C, P);
  long long floats = (splits > 1 ? splits * MN : 0) + colsum_ws(P, g->N);
  size_t extra = prec == PC_BF16 ? umma_conv_extra_ws(*g, prec)
                 : (prec == PC_TF32 && tf32_conv_dgrad_ok(*g)) ? tf32_dgrad_ws(*g) : 0;
  return (size_t)floats * sizeof(float) + extra;
}

extern "C" int pc_conv2d_backward(const pc_conv_geom* g, const void* x, const void* w, const void* gy,
                                  void* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                                  void* workspace, size_t ws_bytes, pc_stream_t st) {
  return pc_conv2d_backward_ex(g, x, w, gy, gx, mask, gw, gb, prec, flags, workspace, ws_bytes, nullptr, st);
}

extern "C" int pc_conv2d_backward_ex(const pc_conv_geom* g, const void* x, const void* w, const void* gy,
                                     void* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                                     void* workspace, size_t ws_bytes, const pc_sgd_fuse* upd, pc_stream_t st) {
  int rc = check_geom(g);
  if (rc || (rc = check_cprec(prec))) return rc;
  size_t need = pc_conv2d_backward_workspace(g, prec);
  PC_REQUIRE(!(flags & PC_WANT_DW) || ws_bytes >= need, PC_EVALUE,
             "conv2d_backward: workspace %zu B < required %zu B", ws_bytes, need);
  long long P = (long long)g->B * g->Ho * g->Wo;
  if (flags & PC_WANT_DX) {
    if (g->B == 0) return PC_OK;
    const void* mk = (flags & PC_MASK_DX) ? mask : nullptr;
    PC_REQUIRE(!(flags & PC_WT_PRESET) || prec == PC_BF16, PC_EVALUE, "PC_WT_PRESET: bf16 path only");
    if (prec == PC_TF32 && tf32_conv_dgrad_ok(*g)) {
      // the rotated filters live at the end of the workspace (after the colsum / split-K regions)
      PC_REQUIRE(workspace != nullptr && ws_bytes >= need, PC_EVALUE, "conv2d_backward: tf32 needs the workspace");
      float* wt = reinterpret_cast<float*>(static_cast<char*>(workspace) + need - tf32_dgrad_ws(*g));
      rc = tf32_conv_dgrad(*g, static_cast<const float*>(w), static_cast<const float*>(gy), static_cast<float*>(gx),
                           static_cast<const float*>(mk), wt, S(st));
    } else {
      rc = prec == PC_BF16 ? umma_conv_dgrad(*g, w, gy, gx, mk, S(st), workspace, ws_bytes, (flags & PC_WT_PRESET) != 0)
                           : simt_conv_dgrad(*g, w, gy, gx, mk, S(st), storage(prec));
    }
    if (rc) return rc;
  }
  if (flags & PC_WANT_DW) {
    float* ws = static_cast<float*>(workspace);
    if (g->B == 0) {
      cudaMemsetAsync(gw, 0, sizeof(float) * g->N * g->k * g->k * g->C, S(st));
      if (gb) cudaMemsetAsync(gb, 0, sizeof(float) * g->N, S(st));
      return PC_OK;
    }
    if (gb) {  // null: the caller derives the bias gradient otherwise (pc_s2d_wgrad_finish)
      rc = colsum(gy, P, g->N, storage(prec), gb, ws, S(st));
      if (rc) return rc;
    }
    float* part = ws + colsum_ws(P, g->N);
    if (prec == PC_BF16) {
      rc = umma_conv_wgrad(*g, x, gy, gw, part, S(st), upd);
    } else if (prec == PC_TF32 && tf32_conv_ok(*g)) {
      PC_REQUIRE(upd == nullptr, PC_EVALUE, "fused SGD update: bf16 tensor-core path only");
      rc = tf32_conv_wgrad(*g, static_cast<const float*>(x), static_cast<const float*>(gy), gw, part, S(st));
    } else {
      PC_REQUIRE(upd == nullptr, PC_EVALUE, "fused SGD update: bf16 tensor-core path only");
      rc = simt_conv_wgrad(*g, x, gy, gw, part, simt_splits(g->N, g->k * g->k * g->C, P), S(st), storage(prec));
    }
    if (rc) return rc;
  }
  return PC_OK;
}

extern "C" PC_API int pc_conv2d_dgrad_weights(const pc_conv_geom* g, const void* w, void* wt, int prec, pc_stream_t st) {
  int rc = check_geom(g);
  if (rc || (rc = check_prec(prec))) return rc;
  PC_REQUIRE(prec == PC_BF16 && w && wt, PC_EVALUE, "conv2d_dgrad_weights: bf16 weights required");
  return umma_conv_dgrad_weights(*g, w, wt, S(st));
}

static int check_mat(const pc_mat* m, const char* what) {
  PC_REQUIRE(m && m->ptr && m->ld > 0 && m->cb > 0, PC_EVALUE, "%s: bad matrix view", what);
  return PC_OK;
}

extern "C" size_t pc_fc_forward_workspace(int B, int D, int U, int prec) {
  return prec == PC_BF16 && B > 0 && D > 0 && U > 0 ? umma_fc_forward_ws(B, D, U) : 0;
}

extern "C" int pc_fc_forward_ex(int B, int D, int U, const pc_mat* x, const void* w, const float* bias, void* y,
                                int prec, int flags, void* workspace, size_t ws_bytes, pc_stream_t st) {
  int rc = check_cprec(prec);
  if (rc) return rc;
  PC_REQUIRE(B >= 0 && D > 0 && U > 0, PC_ESHAPE, "fc: bad extents B=%d D=%d U=%d", B, D, U);
  if (B == 0) return PC_OK;
  if ((rc = check_mat(x, "fc_forward x"))) return rc;
  if (prec == PC_BF16) return umma_fc_forward(B, D, U, *x, w, bias, y, flags, S(st), workspace, ws_bytes);
  if (prec == PC_TF32 && tf32_fc_ok(D, U, *x))
    return tf32_fc_forward(B, D, U, *x, static_cast<const float*>(w), bias, static_cast<float*>(y), flags, S(st));
  return simt_fc_forward(B, D, U, *x, w, bias, y, storage(prec), flags, S(st));
}

extern "C" int pc_fc_forward(int B, int D, int U, const pc_mat* x, const void* w, const float* bias,
                             void* y, int prec, int flags, pc_stream_t st) {
  return pc_fc_forward_ex(B, D, U, x, w, bias, y, prec, flags, nullptr, 0, st);
}

extern "C" size_t pc_fc_backward_workspace(int B, int D, int U, int prec) {
  // the data gradient's split-K partials run first and reuse the weight gradient's region
  size_t dg = prec == PC_BF16 && B > 0 ? umma_fc_dgrad_ws(B, D, U) : 0;
  if (prec == PC_TF32) {  // split-K partials of the tf32 weight gradient
    const long long sp = B > 0 ? tf32_fc_wgrad_splits(B, D, U) : 1;
    return (size_t)colsum_ws(B, U) * sizeof(float) + (sp > 1 ? (size_t)sp * U * D * sizeof(float) : 0);
  }
  return (size_t)colsum_ws(B, U) * sizeof(float) + std::max(umma_fc_extra_ws(B, D, U, prec), dg);
}

extern "C" int pc_fc_backward(int B, int D, int U, const pc_mat* x, const void* w, const void* gy,
                              const pc_mat* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                              void* workspace, size_t ws_bytes, pc_stream_t st) {
  return pc_fc_backward_ex(B, D, U, x, w, gy, gx, mask, gw, gb, prec, flags, workspace, ws_bytes, nullptr, st);
}

extern "C" int pc_fc_backward_ex(int B, int D, int U, const pc_mat* x, const void* w, const void* gy,
                                 const pc_mat* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                                 void* workspace, size_t ws_bytes, const pc_sgd_fuse* upd, pc_stream_t st) {
  int rc = check_cprec(prec);
  if (rc) return rc;
  PC_REQUIRE(B >= 0 && D > 0 && U > 0, PC_ESHAPE, "fc: bad extents B=%d D=%d U=%d", B, D, U);
  size_t need = pc_fc_backward_workspace(B, D, U, prec);
  PC_REQUIRE(ws_bytes >= need, PC_EVALUE, "fc_backward: workspace %zu B < required %zu B", ws_bytes, need);
  if (flags & PC_WANT_DX) {
    if ((rc = check_mat(gx, "fc_backward gx"))) return rc;
    if (B > 0) {
      const void* mk = (flags & PC_MASK_DX) ? mask : nullptr;
      if (prec == PC_TF32 && tf32_fc_ok(D, U, *gx))
        rc = tf32_fc_dgrad(B, D, U, static_cast<const float*>(w), static_cast<const float*>(gy), *gx,
                           static_cast<const float*>(mk), S(st));
      else
        rc = prec == PC_BF16 ? umma_fc_dgrad(B, D, U, w, gy, *gx, mk, S(st), workspace, ws_bytes)
                             : simt_fc_dgrad(B, D, U, w, gy, *gx, mk, S(st), storage(prec));
      if (rc) return rc;
    }
  }
  if (flags & PC_WANT_DW) {
    if ((rc = check_mat(x, "fc_backward x"))) return rc;
    if (B == 0) {
      cudaMemsetAsync(gw, 0, sizeof(float) * (size_t)U * D, S(st));
      if (gb) cudaMemsetAsync(gb, 0, sizeof(float) * U, S(st));
      return PC_OK;
    }
    float* ws = static_cast<float*>(workspace);
    if (gb) {  // null: the caller derives the bias gradient otherwise (pc_bias_grad)
      rc = colsum(gy, B, U, storage(prec), gb, ws, S(st));
      if (rc) return rc;
    }
    PC_REQUIRE(upd == nullptr || prec == PC_BF16, PC_EVALUE, "fused SGD update: bf16 tensor-core path only");
    if (prec == PC_TF32 && tf32_fc_ok(D, U, *x))
      rc = tf32_fc_wgrad(B, D, U, *x, static_cast<const float*>(gy), gw, ws + colsum_ws(B, U), S(st));
    else
      rc = prec == PC_BF16 ? umma_fc_wgrad(B, D, U, *x, gy, gw, ws + colsum_ws(B, U), S(st), upd)
                           : simt_fc_wgrad(B, D, U, *x, gy, gw, S(st), storage(prec));
    if (rc) return rc;
  }
  return PC_OK;
}
