// Trainer feed on the device: the synthetic ImageNet-shaped data
// of the reference (`pkg/src/parconv/data.py:52-96`, `rng.py:63-106`) generated
// directly in HBM, and the batch gather by sample index.
//
// Row r of the split = sample idx[r] = class k * per_class + q:
//   template[k][e] = uniform(-1, 1) draw e of derive(seed, DOMAIN_TEMPLATE = 3, k)
//   noise[k][q][e] = gauss draw (q * dim + e) of derive(seed, domain, k), std 0.5:
//                    Box-Muller on the stream's (2p+1, 2p+2)-th outputs, p = draw / 2,
//                    u1 = (top53 + 1) 2^-53, u2 = top53 2^-53, r = sqrt(-2 ln u1),
//                    even draw: r cos(2 pi u2), odd draw: r sin(2 pi u2)
//   image = float32(template + 0.5 * noise)   (the reference quantises to float32)
// SplitMix64 is counter based (output i = mix64(state + i * GOLDEN)), so every
// element is computed independently: one thread per output element, coalesced
// stores, no host round trip. The double-precision log / sin / cos are CUDA's
// (<= 1-2 ulp); the host uses numpy's — they can differ in the last bit of the
// double, which changes the float32 image only when the double lies within an
// ulp of a float32 rounding boundary (~1e-8 of the elements, tested).
#include <cstdint>

#include "common.cuh"

namespace pc {

__device__ __forceinline__ unsigned long long dmix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;

// rng.derive(seed, domain, index).state
__device__ __forceinline__ unsigned long long derive_state(unsigned long long seed, unsigned long long domain,
                                                           unsigned long long index) {
  return dmix64(dmix64(seed ^ (domain * kGolden)) ^ index);
}

template <typename T>
__global__ void __launch_bounds__(256) synthetic_rows_k(int per_class, long long dim, unsigned long long seed,
                                                        int domain, const long long* __restrict__ idx, int n,
                                                        float std_, T* __restrict__ out) {
  PC_PDL_TRIGGER();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * dim) return;
  const long long r = t / dim, e = t - r * dim;
  const long long sample = idx[r];
  const long long k = sample / per_class, q = sample - k * per_class;
  // template: uniform draw e (counter e + 1) of the class's template stream
  const unsigned long long ts = derive_state(seed, 3ull, (unsigned long long)k);
  const double u = (double)(dmix64(ts + (unsigned long long)(e + 1) * kGolden) >> 11) * 0x1p-53;
  const double tmpl = __dadd_rn(__dmul_rn(u, 2.0), -1.0);
  // noise: draw f of the class's noise stream, pair p = f / 2 -> counters 2p + 1, 2p + 2
  const unsigned long long ns = derive_state(seed, (unsigned long long)domain, (unsigned long long)k);
  const unsigned long long f = (unsigned long long)(q * dim + e), p = f >> 1;
  const unsigned long long a = dmix64(ns + (2 * p + 1) * kGolden), b = dmix64(ns + (2 * p + 2) * kGolden);
  const double u1 = __dmul_rn((double)(a >> 11) + 1.0, 0x1p-53);
  const double u2 = __dmul_rn((double)(b >> 11), 0x1p-53);
  const double radius = sqrt(__dmul_rn(-2.0, log(u1)));
  const double angle = __dmul_rn(6.283185307179586, u2);  // (2.0 * np.pi) * u2
  const double z = __dmul_rn(radius, (f & 1) ? sin(angle) : cos(angle));
  const double v = __dadd_rn(tmpl, __dmul_rn(z, (double)std_));
  out[t] = cvt<T>((float)v);  // float32 quantisation (round to nearest), then the storage type
}

// dst[r] = src[idx[r]] for rows of row_bytes: the batch gather of the device-resident
// training split by the epoch permutation. 16-byte words when the rows allow it
// (AlexNet's 3x227x227 float32 rows are 618,348 B: 4-byte words).
template <typename W>
__global__ void __launch_bounds__(256) gather_rows_k(const W* __restrict__ src, const long long* __restrict__ idx,
                                                     int n, long long row_w, W* __restrict__ dst) {
  PC_PDL_TRIGGER();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * row_w) return;
  const long long r = t / row_w, c = t - r * row_w;
  dst[t] = __ldg(src + idx[r] * row_w + c);
}

}  // namespace pc

using namespace pc;

extern "C" int pc_synthetic_rows(int classes, int per_class, long long dim, unsigned long long seed, int domain,
                                 const long long* idx, int n, float std_, void* out, int out_prec, pc_stream_t st) {
  PC_REQUIRE(classes >= 2 && per_class >= 1 && dim >= 1 && n >= 0 && (n == 0 || (idx && out)), PC_EVALUE,
             "synthetic_rows: bad arguments");
  if (n == 0) return PC_OK;
  const long long total = (long long)n * dim;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (out_prec == PC_FP32) {
    synthetic_rows_k<float><<<blocks, 256, 0, S(st)>>>(per_class, dim, seed, domain, idx, n, std_,
                                                        static_cast<float*>(out));
  } else if (out_prec == PC_BF16) {
    synthetic_rows_k<__nv_bfloat16><<<blocks, 256, 0, S(st)>>>(per_class, dim, seed, domain, idx, n, std_,
                                                                static_cast<__nv_bfloat16*>(out));
  } else {
    PC_REQUIRE(false, PC_EVALUE, "synthetic_rows: unknown precision %d", out_prec);
  }
  PC_CUDA_CHECK_LAUNCH("synthetic_rows");
  return PC_OK;
}

extern "C" int pc_gather_rows(int n, long long row_bytes, const void* src, const long long* idx, void* dst,
                              pc_stream_t st) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
  PC_REQUIRE(n >= 0 && row_bytes > 0 && row_bytes % 4 == 0 && (n == 0 || (src && idx && dst)) && (al & 3) == 0,
             PC_EVALUE, "gather_rows: rows must be 4-byte multiples on 4-byte aligned buffers");
  if (n == 0) return PC_OK;
  if (row_bytes % 16 == 0 && (al & 15) == 0) {
    const long long w = row_bytes / 16, total = (long long)n * w;
    gather_rows_k<uint4><<<(unsigned)((total + 255) / 256), 256, 0, S(st)>>>(
        static_cast<const uint4*>(src), idx, n, w, static_cast<uint4*>(dst));
  } else {
    const long long w = row_bytes / 4, total = (long long)n * w;
    gather_rows_k<uint32_t><<<(unsigned)((total + 255) / 256), 256, 0, S(st)>>>(
        static_cast<const uint32_t*>(src), idx, n, w, static_cast<uint32_t*>(dst));
  }
  PC_CUDA_CHECK_LAUNCH("gather_rows");
  return PC_OK;
}
