// bf16 tensor-core contractions for sm_100a: tcgen05.mma with the fp32
// accumulator in TMEM, operands staged in 128B-swizzled shared memory by TMA
// (dense / channel-blocked views, K-major or MN-major) or by an im2col gather
// (cp.async, 16 B = 8 channels per request, zero-fill for padding) for the
// convolution operand, and a fused epilogue (bias, ReLU, ReLU-mask of the
// producer, bf16 / fp32 / transposed-fp32 stores, split-K partials).
//
// Persistent CTAs (or CTA pairs, cta_group::2) walk a static tile schedule:
//   warps 0-3 (+6-9)  epilogue: 2 warps per TMEM lane quadrant (1 in the GATHER modes),
//                     tcgen05.ld 32 lanes x 16/32 columns
//   warp  4           TMEM allocator + elected-lane MMA issuer
//   warp  5           TMA producer
//   warps 6-21        cp.async gather producers (GATHER modes only)
// A STAGES-deep full/empty mbarrier ring connects producers and the MMA
// issuer; tcgen05.commit frees a stage and finally signals the epilogue.
//
// GEMM shapes per pass (M x N x K):
//   conv fwd   pixels x Cout x (kh*kw*Cin)      A = im2col(x)   B = w [Cout][K]     (K-major)
//   conv dgrad pixels x Cin  x (kh*kw*Cout)     A = im2col(gy)  B = w^T [Cin][K]    (K-major)
//   conv wgrad (kh*kw*Cin) x Cout x pixels      A = im2col(x)^T (MN)  B = gy (MN)   -> gw^T store
//   fc fwd     B x U x D     A = x (K)   B = W [U][D] (K)
//   fc dgrad   B x D x U     A = gy (K)  B = W (MN)
//   fc wgrad   U x D x B     A = gy (MN) B = x (MN)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_ops.cuh"
#include "umma.cuh"

namespace pc {
namespace umma {

// A operand sources: TMA tiled views, TMA im2col-mode loads (the hardware
// walks output pixels across rows / images and zero-fills the padding), or the
// cp.async gather kept for geometries the im2col box cannot express.
enum AMode {
  A_TMA_K = 0, A_TMA_MN = 1, A_GATHER_FWD = 2, A_GATHER_DGRAD = 3, A_GATHER_WGRAD = 4,
  A_IM2COL_K = 5, A_IM2COL_MN = 6, A_HALO_K = 7,
  // weight gradient with M <= 640 and N <= 128 (the input layer: 9 taps x 64
  // channels x 96 filters): one CTA holds MACC = 5 accumulators (all of M) x N in
  // TMEM, so each split-K slice streams the upstream gradient (B) exactly once
  A_IM2COL_MN5 = 8,
  // halo A with the whole B operand resident in shared memory (loaded once per
  // CTA): a narrow layer whose filters fit (the space-to-depth input layer: 9 taps
  // x 64 channels x 96 filters = 54 KB per SM of a CTA pair); stages carry only
  // the input window
  A_HALO_KR = 9,
  // weight gradient on a CTA pair with two M accumulators per CTA (M = 512 rows per
  // pair tile, N = 256 filters, TMEM 2 x 256 columns): the B tile (upstream
  // gradient) each SM loads feeds twice the MMA work — 25% fewer operand bytes per
  // FLOP than one 256 x 256 accumulator per pair, for the operand-bound N = 256
  // weight gradients (conv2, conv5); the epilogue is not overlapped (512 columns)
  A_IM2COL_MN2 = 10,
  // A_IM2COL_MN2 over 32-channel chunks (64B swizzle, MN-major): M rows = (tap,
  // 32-channel group) units with no padding for a channel count that is a multiple
  // of 32 but not of 64 (conv2's 96: 2400 rows instead of 25 x 128 = 3200)
  A_IM2COL_MN2_32 = 11,
  // K-major TMA im2col A (one 16 KB box per stage) with the whole B operand resident
  // (as A_HALO_KR): deep stage ring, no per-stage filter traffic, coalesced epilogue
  A_IM2COL_KR = 12,
  // A_HALO_KR with TWO vertically adjacent halo sub-tiles per CTA (two accumulators of
  // 128 TMEM columns, still double-buffered): one window per stage covers both, and
  // every tile boundary (accumulator handoff) is amortised over twice the MMAs
  A_HALO_KR2 = 13,
  // A_IM2COL_MN5 on a CTA pair: three M accumulators per CTA (768 rows per pair tile,
  // N <= 96 packed at p.N columns), the pair sharing the upstream-gradient tile; chunks
  // of rows past M are not loaded. Input layer weight gradient: 576 x 96.
  A_IM2COL_MN3P = 14,
  // A_IM2COL_K with TWO M accumulators per CTA (a CTA pair covers 512 output pixels,
  // TMEM 2 x BN columns, not double-buffered): each stage brings two 16 KB im2col
  // boxes and the CTA's one B half, so every B byte feeds twice the MMA work —
  // 48 KB per 1024 MMA cycles instead of 32 KB per 512 (the forward / data
  // gradient GEMMs are operand-delivery bound); the epilogue is not overlapped.
  // Chosen when the 512-row tiles quantise onto the 74 pairs as well as 256-row
  // ones (AlexNet conv2 forward: 365 tiles)
  A_IM2COL_K2 = 15
};
enum BMode { B_TMA_K = 0, B_TMA_MN = 1 };
enum EpiMode { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_T = 2, EPI_SGD = 3 };

constexpr int BM = 128, BK = 64;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB

struct alignas(64) Params {
  CUtensorMap tma_a;
  CUtensorMap tma_b;
  int M, N, K;
  int num_kb;        // k-blocks in total
  int kb_per_split;  // k-blocks per split-K slice
  int tiles;         // split slices x M tiles x N tiles (persistent walk)
  int a_cb, b_cb;  // channel-block width of a blocked TMA view (idx -> (idx % cb, idx / cb)); 0 = unblocked
  const __nv_bfloat16* gsrc;
  pc_conv_geom g;
  void* out;
  long long o_ld, o_cb, o_bstride;
  long long split_stride;
  const float* bias;
  const __nv_bfloat16* mask;
  int relu;
  int b_chunked;  // MN-major B encoded as a chunked 4-D view: one TMA op per stage
  // im2col-mode A: K index = (i, j, c) over i2c_C channels in blocks of i2c_cs,
  // output-pixel walk over (i2c_Ho, i2c_Wo) with stride i2c_s from corner (lw, lh)
  int i2c_C, i2c_cs, i2c_k, i2c_s, i2c_lw, i2c_lh, i2c_Wo, i2c_Ho;
  // K-major im2col: K walks (tap, 64-channel chunk); i2c_cpt = chunks per tap = ceil(C / 64).
  // A channel count that is not a multiple of 64 (AlexNet conv2: 96) loads its last
  // chunk past the channel extent — TMA zero-fills it — and the MMA issues only the
  // k16 steps that hold real channels.
  int i2c_cpt;
  // Halo (shifted-window) A for stride-1 convs: a tile is halo_R output rows x Wv
  // virtual columns of one image (Wv = Wo rounded up to 8). For each 64-channel
  // chunk and filter column j, one TMA box brings the tile's input window
  // (halo_R + k - 1 rows x Wv columns starting at column j + lo, zero outside the
  // image) into shared memory; the A operand of tap (i, j) is that buffer shifted by
  // i * Wv rows (a multiple of 8 rows: the tensor core reads such shifted 128B-swizzled
  // tiles at full rate; odd row shifts work but run ~3x slower, tools/desc_probe.cu).
  // Columns x >= Wo are discarded.
  int halo_R, halo_tpi, halo_Wv, halo_lo, halo_bytes;
  int macc_chunks;  // A_IM2COL_MN5: 64-row A chunks with real rows (<= 10)
  // A_IM2COL_MN with C % 64 != 0 (conv2's 96 channels): M rows walk (tap, m_cp
  // padded channels); the last 64-channel chunk of a tap is zero-filled by TMA
  // and the epilogue maps row (tap, c < C) to tap * C + c, dropping c >= C.
  int m_cp;
  int mt_rows;      // rows per M tile: 128 * CTA-group size * accumulators (set at launch)
  unsigned long long* trace;  // debug: per-CTA per-tile clock64 stamps (tools/trace_gemm.py), normally null
  // EPI_F32 through TMA stores: fp32 view {N, M, split slices} of p.out, box {32, 32, 1}, 128B swizzle
  int out_tma;
  CUtensorMap tma_out;
  // EPI_SGD: the weight gradient never leaves the SM — fp32 p and v {N, M} and
  // the bf16 shadow of p, updated in place (v = mom v - lr (g + wd p); p += v)
  CUtensorMap tma_p, tma_v, tma_pl;
  float lr, mom, wd;
  // A_IM2COL_K with a last channel chunk of <= 32 channels (conv2: 96 = 64 + 32):
  // that k-block loads 32-channel boxes (64-byte rows, 64B swizzle) of A and B
  // instead of zero-filled / unused 64-channel ones — a quarter fewer operand
  // bytes for the layer, whose GEMMs are limited by operand delivery
  int half_chunk;
  // half_chunk with one full chunk per tap (64 < C <= 96): k-blocks 0..taps-1 are the
  // taps' full 64-channel chunks, then each k-block pairs the 32-channel remainders
  // of two taps (two SW64 A/B halves in one stage): 38 k-blocks for conv2, not 50
  CUtensorMap tma_a32, tma_b32;
  // A_IM2COL_MN2_32: 32-channel groups per tap (M row m -> tap (m/32)/m_grp, group (m/32)%m_grp)
  int m_grp;
  int dbg_nostore;  // debug (PC_DEBUG_NOSTORE): the staged bf16 epilogue skips its global stores
  int dbg_noload;   // debug (PC_DEBUG_NOLOAD): halo producers skip the window loads
  int epi_direct;   // staged bf16 epilogue: per-row direct stores instead (PC_KR_DIRECT)
  int zero_tail16;  // halo forward: skip the k16 step of the last 16 channels (PC_ZERO_TAIL16 flag)
};

// Debug timeline: slot s of tile lt of CTA b (first TRACE_TILES tiles).
constexpr int TRACE_TILES = 64;
constexpr int TRACE_SLOTS = 16;
__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ void trace_put(const Params& p, int lt, int slot, long long v) {
  if (p.trace != nullptr && lt < TRACE_TILES)
    p.trace[((size_t)blockIdx.x * TRACE_TILES + lt) * TRACE_SLOTS + slot] = (unsigned long long)v;
}
__device__ __forceinline__ void trace_stamp(const Params& p, int lt, int slot) {
  if (p.trace != nullptr) trace_put(p, lt, slot, clk());
}

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Bounded wait: a pipeline bug traps (a launch error the host reports) instead
// of hanging the device forever.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins == (1u << 28)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t.reg .b32 r;\n\t"
      "elect.sync r|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Cluster (CTA pair) helpers -------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on the barrier at the same smem offset in CTA `rank` of the cluster.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

// TMA loads. CG == 2: the 2-SM form — both CTAs of the pair load their own half
// into their own shared memory, and the transaction bytes complete on the
// LEADER's (rank 0) barrier at the same offset (peer bit cleared).
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;
template <int CG>
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, uint32_t dst, int c0, int c1,
                                            int c2) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, uint32_t dst, int c0, int c1,
                                            int c2, int c3) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
  }
}
// im2col mode: {c, w, h, d, n} = (channel offset, pixel-walk start, batch, block),
// im2col offsets {w, h, d} = filter tap (j, i, 0).
template <int CG>
__device__ __forceinline__ void tma_im2col_5d(const CUtensorMap* map, uint64_t* bar, uint32_t dst, int c, int w,
                                              int h, int d, int n, uint16_t ow, uint16_t oh) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], {%8, %9, %10};" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(d), "r"(n),
        "h"(ow), "h"(oh), "h"((uint16_t)0)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.5d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], {%8, %9, %10};" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(c), "r"(w), "r"(h), "r"(d),
        "r"(n), "h"(ow), "h"(oh), "h"((uint16_t)0)
        : "memory");
  }
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// MMA completion -> mbarrier; CG == 2 signals the barrier in BOTH CTAs of the pair.
template <int CG>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  }
}
template <int CG>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 columns in one tcgen05.ld (one wait per 32 columns instead of per 16)
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

__device__ __forceinline__ int blk_off(int idx, int cb) { return cb ? (int)((unsigned)idx % (unsigned)cb) : idx; }
__device__ __forceinline__ int blk_idx(int idx, int cb) { return cb ? (int)((unsigned)idx / (unsigned)cb) : 0; }

// Shared-memory matrix descriptor, 128B swizzle (sm100 version bit 46 = 1).
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// Same with 64B swizzle (layout type 4): K-major rows of 32 bf16, 8-row atoms of 512 B.
__device__ __forceinline__ uint64_t make_desc_sw64(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (4ull << 61);
}

// Instruction descriptor: D f32, A/B bf16, majorness, N (pair tile width), M = 128 * CG.
template <int BN, bool A_MN, bool B_MN, int CG>
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4)                  // D = f32
         | (1u << 7) | (1u << 10)   // A, B = bf16
         | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16)
         | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
}

template <int BN>
constexpr int tmem_cols() {
  return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

// Halo stage: the input window for (channel chunk, filter column j) (<= 256 rows of
// 64 channels) plus the B tiles of that column's k filter rows (k <= HALO_KMAX).
constexpr int HALO_SLOT_BYTES = 256 * 128, HALO_KMAX = 5;
// A_HALO_KR: window slots of <= 224 rows and <= 56 KB of resident B tiles
constexpr int HALO_R_SLOT_BYTES = 224 * 128, RES_B_BYTES = 56 * 1024;
constexpr int HALO_R2_SLOT_BYTES = 336 * 128;  // A_HALO_KR2: (2 R + k - 1) x Wv <= 336 rows
template <int AM> constexpr bool a_is_gather() { return AM >= A_GATHER_FWD && AM <= A_GATHER_WGRAD; }
// cp.async gather producers (warps 6..): 8 warps, each thread 16 B per row for
// 1024 / GATHER_THREADS rows of the 128 x 64 stage.
constexpr int GATHER_THREADS = 512;
constexpr int GR = 1024 / GATHER_THREADS;  // rows (fwd/dgrad) or pixel rows (wgrad) per gather thread
template <int AM> constexpr bool a_is_mn() {
  return AM == A_TMA_MN || AM == A_GATHER_WGRAD || AM == A_IM2COL_MN || AM == A_IM2COL_MN5 || AM == A_IM2COL_MN2 ||
         AM == A_IM2COL_MN2_32 || AM == A_IM2COL_MN3P;
}
template <int AM> constexpr int macc_of() {
  return AM == A_IM2COL_MN5 ? 5 : AM == A_IM2COL_MN3P ? 3
         : (AM == A_IM2COL_MN2 || AM == A_IM2COL_MN2_32 || AM == A_HALO_KR2 || AM == A_IM2COL_K2) ? 2 : 1;
}

// Per-CTA shared memory: STAGES x (A 128 rows + B BN/CG rows) x 64 bf16, barriers.
template <int BN, int CG>
constexpr int halo_stage_bytes() { return HALO_SLOT_BYTES + HALO_KMAX * (BN / CG) * BK * 2; }
// B rows a CTA stages per k-block: an MN-major B is loaded in whole 64-column
// chunks (a pair tile of N = 192 stages 128 columns per CTA and the MMA reads 96)
template <int BN, int CG, bool BMN>
constexpr int b_rows() { return BMN ? (BN / CG + 63) / 64 * 64 : BN / CG; }
template <int BN, int STAGES, int CG, bool HALO = false, int MACC = 1, bool BMN = false>
constexpr int smem_bytes() {
  return 1024 /*align slack*/ + (HALO ? STAGES * halo_stage_bytes<BN, CG>()
                                      : STAGES * (MACC * A_STAGE_BYTES + b_rows<BN, CG, BMN>() * BK * 2)) +
         (2 * STAGES + 4) * 8 + 16;
}


// ------------------------------------------------------------------- kernel
// Persistent: each CTA (CG == 1) or CTA pair (CG == 2, a 2-SM cluster issuing
// tcgen05.mma.cta_group::2 with M = 256) walks tiles t = unit, unit + units, ...
// (tile order: split-K slice, then M, then N fastest). The smem stage ring runs
// continuously across tiles, and with two TMEM accumulators the epilogue of
// tile t overlaps the mainloop of tile t+1.
// CTA pair: each CTA loads its own 128 A rows and half of the B tile (BN/2
// rows) into its own smem; the leader (rank 0) waits on its full barrier for
// both halves' bytes, issues the MMAs, and its commits arrive on both CTAs'
// empty / accumulator-full barriers. Each CTA's epilogue drains its own TMEM
// (its 128 rows x BN) and arrives on the leader's accumulator-empty barrier.
template <int BN>
constexpr int acc_count() { return 2 * tmem_cols<BN>() <= 512 ? 2 : 1; }

struct TileCoord {
  int m0, n0, z, kb_begin, nkb;
};

template <int CG>
__device__ __forceinline__ TileCoord tile_coord(const Params& p, int t, int bn) {
  const int bmt = p.mt_rows;
  const int tn = (p.N + bn - 1) / bn, tm = (p.M + bmt - 1) / bmt;
  TileCoord c;
  c.z = t / (tm * tn);
  const int r = t - c.z * (tm * tn);
  c.m0 = (r / tn) * bmt;
  c.n0 = (r - (r / tn) * tn) * bn;
  c.kb_begin = c.z * p.kb_per_split;
  c.nkb = max(min(p.num_kb, c.kb_begin + p.kb_per_split) - c.kb_begin, 0);
  return c;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Accumulator-empty arrivals: relaxed — the MMA warp needs only the TMEM reads
// ordered (tcgen05.fence::before_thread_sync), not this thread's outstanding
// global stores, which a release arrive would wait for.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

// Epilogue: drain one accumulator (this CTA's 128 rows x BN fp32 in TMEM) per
// tile. EPW warps per TMEM lane quadrant split the 16-column chunks. Output
// addressing keeps (channel block, offset) incrementally — no divisions.
template <int EPI, int BN, int CG, int EPW, bool HALO, int MACC = 1>
__device__ __forceinline__ void epilogue(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty, int unit,
                                         int units, uint32_t rank, int quad, int grp, int lane) {
  constexpr int TCOLS = MACC > 1 ? 512 : tmem_cols<BN>();
  constexpr int ACC = MACC > 1 ? 1 : acc_count<BN>();
  const int row = quad * 32 + lane;
  int lt = 0;
  for (int t = unit; t < p.tiles; t += units, ++lt) {
    const TileCoord tc = tile_coord<CG>(p, t, BN);
    const int acc = lt % ACC;
    mbar_wait(&tfull[acc], (lt / ACC) & 1);
    tc_fence_after();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 5);
    for (int a = 0; a < MACC; ++a) {  // MACC > 1: accumulator a = rows [128 a, 128 a + 128), TMEM column a * N
    // accumulator a of CTA `rank`: rows [a * 128 * CG + rank * 128, ... + 128) of the tile
    long long m = (long long)tc.m0 + (long long)a * BM * CG + (long long)rank * BM + row;
    bool mrow = m < p.M;
    if (p.m_cp) {
      const long long tap = m / p.m_cp, c = m - tap * p.m_cp;
      mrow = mrow && c < p.i2c_C;
      m = tap * p.i2c_C + c;
    }
    if (p.m_grp) {  // A_IM2COL_MN2_32: row (unit = (tap, 32-channel group), c) -> tap * C + group * 32 + c
      const long long unit = m >> 5, tap = unit / p.m_grp;
      m = tap * p.i2c_C + (unit - tap * p.m_grp) * 32 + (m & 31);
    }
    if constexpr (HALO) {  // TMEM row -> (image, output row, column) of this CTA's halo tile
      const int tile = (tc.m0 + (int)rank * BM) / BM;
      const int hb = tile / p.halo_tpi, yy = row / p.halo_Wv, xx = row - yy * p.halo_Wv;
      const int y = (tile - hb * p.halo_tpi) * p.halo_R + yy;
      mrow = mrow && yy < p.halo_R && y < p.i2c_Ho && xx < p.i2c_Wo;
      m = ((long long)hb * p.i2c_Ho + y) * p.i2c_Wo + xx;
    }
    // accumulator stride: A_IM2COL_MN5 packs its 5 accumulators at p.N columns (N <= 96);
    // A_IM2COL_MN2 (MACC == 2) gives each a BN-wide (tmem_cols) slot
    const uint32_t tbase = tmem + acc * TCOLS + (MACC == 2 ? a * tmem_cols<BN>() : MACC > 1 ? a * p.N : 0) +
                           ((uint32_t)(quad * 32) << 16);
    const long long rowoff = m * p.o_ld;
    // (blk, rem) of output column n = n0 + c0 in a channel-blocked view (o_cb % 8 == 0)
    long long n = (long long)tc.n0 + grp * 16;
    long long blk = 0, rem = n;
    if constexpr (EPI == EPI_BF16) {
      blk = n / p.o_cb;
      rem = n - blk * p.o_cb;
    }
#pragma unroll 1
    for (int c0 = grp * 16; c0 < BN; c0 += 16 * EPW) {
      float v[16];
      if (tc.nkb > 0) {
        tmem_ld16(tbase + c0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0.f;
      }
      if (mrow && n < p.N) {
        if constexpr (EPI == EPI_BF16) {
          long long b = blk, r = rem;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long nn = n + 8 * h;
            if (nn >= p.N) break;
            float o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float val = v[8 * h + q];
              if (p.bias) val += __ldg(p.bias + nn + q);
              if (p.relu) val = val > 0.f ? val : 0.f;
              o[q] = val;
            }
            const long long idx = b * p.o_bstride + rowoff + r;
            if (p.mask) {
              uint4 mk = *reinterpret_cast<const uint4*>(p.mask + idx);
              const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mk);
#pragma unroll
              for (int q = 0; q < 8; ++q) o[q] = __bfloat162float(mb[q]) > 0.f ? o[q] : 0.f;
            }
            uint4 u;
            __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int q = 0; q < 4; ++q) hh[q] = __floats2bfloat162_rn(o[2 * q], o[2 * q + 1]);
            *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + idx) = u;
            r += 8;
            if (r >= p.o_cb) { r -= p.o_cb; ++b; }
          }
        } else if constexpr (EPI == EPI_F32) {
          float* o = static_cast<float*>(p.out) + tc.z * p.split_stride + rowoff + n;
          if (n + 16 <= p.N) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else {
            for (int q = 0; q < 16 && n + q < p.N; ++q) o[q] = v[q];
          }
        } else {
          float* o = static_cast<float*>(p.out) + tc.z * p.split_stride + m;
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (n + q < p.N) o[(n + q) * p.o_ld] = v[q];
        }
      }
      n += 16 * EPW;
      if constexpr (EPI == EPI_BF16) {
        rem += 16 * EPW;
        while (rem >= p.o_cb) { rem -= p.o_cb; ++blk; }
      }
    }
    }  // accumulators
    // accumulator drained: let the (leader's) MMA warp reuse it
    tc_fence_before();
    __syncwarp();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 6);
    if (lane == 0) {
      if constexpr (CG == 1) {
        mbar_arrive_relaxed(&tempty[acc]);
      } else {
        mbar_arrive_cluster_relaxed(&tempty[acc], 0);
      }
    }
  }
}

// fp32 epilogue by TMA store: each epilogue warp drains 32 accumulator columns
// of its 32 TMEM lanes into a 4 KB 128B-swizzled box in SMEM (conflict-free: lane
// r writes 16 B chunk j at r * 128 + ((j ^ r % 8) << 4)) and one lane issues a
// bulk tensor store of the box; the TMA engine writes whole 128-byte lines. The
// direct path (each lane storing its own row, 32 rows per warp instruction)
// reaches ~2 TB/s on the 151 MB fc6 weight gradient.
constexpr int F32_BOX_BYTES = 32 * 128;
constexpr int F32_STAGE_BYTES = 8 * F32_BOX_BYTES;  // one box per epilogue warp
template <int EPI, int BN, int STAGES, int CG, int AM, bool BMN = false>
constexpr bool f32_tma_epi() {
  return EPI == EPI_F32 && !a_is_gather<AM>() && macc_of<AM>() == 1 && AM != A_HALO_K && AM != A_HALO_KR &&
         AM != A_HALO_KR2 &&
         AM != A_IM2COL_KR &&
         BN % 32 == 0 &&
         smem_bytes<BN, STAGES, CG, false, 1, BMN>() + 1024 + F32_STAGE_BYTES <= 227 * 1024;
}
// bf16 TMA-store epilogue (epilogue_bf16_tma): the two-accumulator im2col GEMM;
// per epilogue warp two 32-row x 64-channel boxes
constexpr int BF16_BOX_BYTES = 32 * 128;
constexpr int BF16_WARP_BYTES = 2 * BF16_BOX_BYTES;
template <int EPI, int AM>
constexpr bool bf16_tma_epi() { return EPI == EPI_BF16 && AM == A_IM2COL_K2; }
// EPI_SGD boxes per epilogue warp: p (fp32 32x32, 128B swizzle), v (same), bf16
// shadow (32x32, 64B swizzle); then one transaction barrier per warp.
constexpr int SGD_WARP_BYTES = 4096 + 4096 + 2048;
constexpr int SGD_STAGE_BYTES = 8 * SGD_WARP_BYTES + 8 * 8;
template <int EPI, int BN, int STAGES, int CG, int AM, bool BMN = false>
constexpr int kernel_smem() {
  if constexpr (AM == A_HALO_KR2)
    return 1024 + STAGES * HALO_R2_SLOT_BYTES + RES_B_BYTES + (2 * STAGES + 5) * 8 + 16 + 1024 + 4 * 64 * BN + 4 * BN;
  if constexpr (AM == A_IM2COL_KR)
    return 1024 + STAGES * A_STAGE_BYTES + RES_B_BYTES + (2 * STAGES + 5) * 8 + 16 + 1024 + 4 * 64 * BN + 4 * BN;
  if constexpr (AM == A_HALO_KR)
    return 1024 + STAGES * HALO_R_SLOT_BYTES + RES_B_BYTES + (2 * STAGES + 5) * 8 + 16 + 1024 + 4 * 64 * BN + 4 * BN;
  return smem_bytes<BN, STAGES, CG, AM == A_HALO_K, macc_of<AM>(), BMN>() +
         (f32_tma_epi<EPI, BN, STAGES, CG, AM, BMN>() ? 1024 + F32_STAGE_BYTES : 0) +
         (EPI == EPI_SGD ? 1024 + SGD_STAGE_BYTES : 0) +
         (bf16_tma_epi<EPI, AM>() ? 1024 + 8 * BF16_WARP_BYTES : 0);
}

// Fused momentum-SGD epilogue: per 32-column group a warp TMA-loads the p and v
// boxes of its 32 rows (issued before its TMEM reads, so the load overlaps
// them), applies the update with the fp32 gradient straight from TMEM, and
// TMA-stores p, v and the bf16 shadow. Per parameter: 8 B read + 10 B written,
// against 4 B gradient store + 12 B read + 10 B written for a separate pass.
template <int BN, int CG, int EPW>
__device__ __forceinline__ void epilogue_sgd_tma(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                                 int unit, int units, uint32_t rank, int quad, int grp, int lane,
                                                 uint8_t* area, uint64_t* lbar) {
  constexpr int TCOLS = tmem_cols<BN>();
  constexpr int ACC = acc_count<BN>();
  const uint32_t sp = smem_u32(area), sv = sp + 4096, sl = sp + 8192;
  uint32_t phase = 0;
  int lt = 0;
  for (int t = unit; t < p.tiles; t += units, ++lt) {
    const TileCoord tc = tile_coord<CG>(p, t, BN);
    const int acc = lt % ACC;
    mbar_wait(&tfull[acc], (lt / ACC) & 1);
    tc_fence_after();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 5);
    const uint32_t tbase = tmem + acc * TCOLS + ((uint32_t)(quad * 32) << 16);
    const int row0 = tc.m0 + (int)rank * BM + quad * 32;
#pragma unroll 1
    for (int c0 = grp * 32; c0 < BN; c0 += 32 * EPW) {
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // previous stores have read the boxes
        mbar_arrive_expect_tx(lbar, 8192);
        tma_load_3d<1>(&p.tma_p, lbar, sp, tc.n0 + c0, row0, 0);
        tma_load_3d<1>(&p.tma_v, lbar, sv, tc.n0 + c0, row0, 0);
        // L2 prefetch of this warp's next group (next tile's first group at the
        // end of a tile): its loads then wait on L2, not HBM
        int nn = tc.n0 + c0 + 32 * EPW, nr = row0;
        if (c0 + 32 * EPW >= BN) {
          if (t + units < p.tiles) {
            const TileCoord nx = tile_coord<CG>(p, t + units, BN);
            nn = nx.n0 + grp * 32;
            nr = nx.m0 + (int)rank * BM + quad * 32;
          } else {
            nn = -1;
          }
        }
        if (nn >= 0) {
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                           reinterpret_cast<uint64_t>(&p.tma_p)),
                       "r"(nn), "r"(nr), "r"(0)
                       : "memory");
          asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                           reinterpret_cast<uint64_t>(&p.tma_v)),
                       "r"(nn), "r"(nr), "r"(0)
                       : "memory");
        }
      }
      float g[32];
      if (tc.nkb > 0) {
        tmem_ld32(tbase + c0, g);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) g[q] = 0.f;
      }
      mbar_wait(lbar, phase);
      phase ^= 1;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t off = lane * 128 + ((j ^ (lane & 7)) << 4);
        float4 pp, vv;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(pp.x), "=f"(pp.y), "=f"(pp.z), "=f"(pp.w)
                     : "r"(sp + off)
                     : "memory");
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(vv.x), "=f"(vv.y), "=f"(vv.z), "=f"(vv.w)
                     : "r"(sv + off)
                     : "memory");
        vv.x = p.mom * vv.x - p.lr * (g[4 * j] + p.wd * pp.x);
        vv.y = p.mom * vv.y - p.lr * (g[4 * j + 1] + p.wd * pp.y);
        vv.z = p.mom * vv.z - p.lr * (g[4 * j + 2] + p.wd * pp.z);
        vv.w = p.mom * vv.w - p.lr * (g[4 * j + 3] + p.wd * pp.w);
        pp.x += vv.x; pp.y += vv.y; pp.z += vv.z; pp.w += vv.w;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sp + off), "f"(pp.x), "f"(pp.y), "f"(pp.z),
                     "f"(pp.w)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sv + off), "f"(vv.x), "f"(vv.y), "f"(vv.z),
                     "f"(vv.w)
                     : "memory");
        __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y), hi = __floats2bfloat162_rn(pp.z, pp.w);
        const uint32_t loff = lane * 64 + (((j >> 1) ^ ((lane >> 1) & 3)) << 4) + (j & 1) * 8;
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(sl + loff), "r"(*reinterpret_cast<uint32_t*>(&lo)),
                     "r"(*reinterpret_cast<uint32_t*>(&hi))
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        const uint64_t mp = reinterpret_cast<uint64_t>(&p.tma_p), mv = reinterpret_cast<uint64_t>(&p.tma_v),
                       ml = reinterpret_cast<uint64_t>(&p.tma_pl);
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(mp),
                     "r"(tc.n0 + c0), "r"(row0), "r"(0), "r"(sp)
                     : "memory");
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(mv),
                     "r"(tc.n0 + c0), "r"(row0), "r"(0), "r"(sv)
                     : "memory");
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(ml),
                     "r"(tc.n0 + c0), "r"(row0), "r"(0), "r"(sl)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    tc_fence_before();
    __syncwarp();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 6);
    if (lane == 0) {
      if constexpr (CG == 1) {
        mbar_arrive_relaxed(&tempty[acc]);
      } else {
        mbar_arrive_cluster_relaxed(&tempty[acc], 0);
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

template <int BN, int CG, int EPW>
__device__ __forceinline__ void epilogue_f32_tma(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                                 int unit, int units, uint32_t rank, int quad, int grp, int lane,
                                                 uint8_t* box) {
  constexpr int TCOLS = tmem_cols<BN>();
  constexpr int ACC = acc_count<BN>();
  const uint32_t sbox = smem_u32(box);
  int lt = 0;
  for (int t = unit; t < p.tiles; t += units, ++lt) {
    const TileCoord tc = tile_coord<CG>(p, t, BN);
    const int acc = lt % ACC;
    mbar_wait(&tfull[acc], (lt / ACC) & 1);
    tc_fence_after();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 5);
    const uint32_t tbase = tmem + acc * TCOLS + ((uint32_t)(quad * 32) << 16);
    const int row0 = tc.m0 + (int)rank * BM + quad * 32;
#pragma unroll 1
    for (int c0 = grp * 32; c0 < BN; c0 += 32 * EPW) {
      float v[32];
      if (tc.nkb > 0) {
        tmem_ld32(tbase + c0, v);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = 0.f;
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // box free again
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sbox + lane * 128 + ((j ^ (lane & 7)) << 4)),
                     "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile(
            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                reinterpret_cast<uint64_t>(&p.tma_out)),
            "r"(tc.n0 + c0), "r"(row0), "r"(tc.z), "r"(sbox)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    // accumulator drained (the stores read SMEM, not TMEM): release it
    tc_fence_before();
    __syncwarp();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 6);
    if (lane == 0) {
      if constexpr (CG == 1) {
        mbar_arrive_relaxed(&tempty[acc]);
      } else {
        mbar_arrive_cluster_relaxed(&tempty[acc], 0);
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

// bf16 epilogue by TMA store (plain NHWC output, no ReLU mask): each epilogue warp
// drains 64 accumulator columns of its 32 TMEM lanes at a time (bias, ReLU, bf16)
// into a 4 KB 128B-swizzled box (conflict-free 16-byte writes), double-buffered,
// and one lane issues a bulk tensor store of the 32 x 64 box — whole 128-byte lines
// instead of 32 rows touched per warp store. Bias by broadcast float4 loads. Used
// by A_IM2COL_K2, whose two accumulators are drained between tiles (not overlapped):
// the per-row epilogue took 19.5k cycles per 512-row tile there.
template <int BN, int CG, int EPW, int MACC>
__device__ __forceinline__ void epilogue_bf16_tma(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                                  int unit, int units, uint32_t rank, int quad, int grp, int lane,
                                                  uint8_t* box) {
  constexpr int TCOLS = MACC > 1 ? 512 : tmem_cols<BN>();
  constexpr int ACC = MACC > 1 ? 1 : acc_count<BN>();
  static_assert(BN % 64 == 0, "bf16 TMA epilogue: 64-column boxes");
  const uint32_t sbox = smem_u32(box);
  int lt = 0, nb = 0;
  for (int t = unit; t < p.tiles; t += units, ++lt) {
    const TileCoord tc = tile_coord<CG>(p, t, BN);
    const int acc = lt % ACC;
    mbar_wait(&tfull[acc], (lt / ACC) & 1);
    tc_fence_after();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 5);
#pragma unroll 1
    for (int a = 0; a < MACC; ++a) {
      const uint32_t tbase = tmem + acc * TCOLS + (MACC == 2 ? a * tmem_cols<BN>() : 0) + ((uint32_t)(quad * 32) << 16);
      const int row0 = tc.m0 + a * BM * CG + (int)rank * BM + quad * 32;
#pragma unroll 1
      for (int c0 = grp * 64; c0 < BN; c0 += 64 * EPW) {
        const int n = tc.n0 + c0;
        if (n >= p.N) break;
        float v[64];
        if (tc.nkb > 0) {
          tmem_ld32(tbase + c0, v);
          tmem_ld32(tbase + c0 + 32, v + 32);
        } else {
#pragma unroll
          for (int q = 0; q < 64; ++q) v[q] = 0.f;
        }
        uint32_t w[32];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p.bias && n + 4 * q < p.N) b = __ldg(reinterpret_cast<const float4*>(p.bias + n) + q);
          float x0 = v[4 * q] + b.x, x1 = v[4 * q + 1] + b.y, x2 = v[4 * q + 2] + b.z, x3 = v[4 * q + 3] + b.w;
          if (p.relu) {
            x0 = x0 > 0.f ? x0 : 0.f;
            x1 = x1 > 0.f ? x1 : 0.f;
            x2 = x2 > 0.f ? x2 : 0.f;
            x3 = x3 > 0.f ? x3 : 0.f;
          }
          const __nv_bfloat162 h0 = __floats2bfloat162_rn(x0, x1), h1 = __floats2bfloat162_rn(x2, x3);
          w[2 * q] = *reinterpret_cast<const uint32_t*>(&h0);
          w[2 * q + 1] = *reinterpret_cast<const uint32_t*>(&h1);
        }
        const uint32_t buf = sbox + (uint32_t)(nb & 1) * BF16_BOX_BYTES;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // this buffer is free
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 128 + ((j ^ (lane & 7)) << 4)),
                       "r"(w[4 * j]), "r"(w[4 * j + 1]), "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                       : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&p.tma_out)),
              "r"(n), "r"(row0), "r"(buf)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        ++nb;
      }
    }
    // both accumulators read (the stores read SMEM, not TMEM): release them
    tc_fence_before();
    __syncwarp();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 6);
    if (lane == 0) {
      if constexpr (CG == 1) {
        mbar_arrive_relaxed(&tempty[acc]);
      } else {
        mbar_arrive_cluster_relaxed(&tempty[acc], 0);
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

// bf16 epilogue for A_HALO_KR with coalesced stores: the two warps of a TMEM lane
// quadrant each drain one half of the BN columns of their 32 rows (bias, ReLU)
// into a shared [32][BN] bf16 box (16-byte writes); after a
// 64-thread named barrier each warp stores two 8-row groups, lanes covering
// consecutive 16-byte chunks, so every warp store is 512 contiguous bytes. An
// 8-row group never straddles an output row (Wv % 8 == 0) and is contiguous in
// the NHWC output; virtual columns x >= Wo are skipped. The accumulator is
// released as soon as it is read. (Each lane storing its own 192-byte row kept
// this 96-column layer epilogue-bound.)
template <int BN, int CG, bool LINEAR = false, int HSUB = 1>
__device__ __forceinline__ void epilogue_bf16_halo(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                                   int unit, int units, uint32_t rank, int quad, int grp, int lane,
                                                   uint8_t* box) {
  constexpr int TCOLS = tmem_cols<BN>() * HSUB;  // one buffer: HSUB sub-tile accumulators
  constexpr int ACC = HSUB > 1 ? 2 : acc_count<BN>();
  constexpr int HALF = BN / 2, ROWB = BN * 2, CH = HALF * 2 / 16, RCH = ROWB / 16;
  static_assert(HALF % 16 == 0, "16-column TMEM loads");
  const uint32_t sbox = smem_u32(box);
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
  // bias of the (single) N tile staged in shared memory once: the per-tile loop reads it
  // with broadcast LDS instead of 48 dependent-latency global loads per thread
  float* sbias = reinterpret_cast<float*>(box + (4 - quad) * (64 * BN));  // after the 4 quadrant boxes
  {
    const int et = (grp * 4 + quad) * 32 + lane;  // 0..255 over the 8 epilogue warps
    for (int c = et; c < BN; c += 256) sbias[c] = (p.bias && c < p.N) ? __ldg(p.bias + c) : 0.f;
    asm volatile("bar.sync 5, 256;" ::: "memory");
  }
  int lt = 0;
  for (int t = unit; t < p.tiles; t += units, ++lt) {
    const TileCoord tc = tile_coord<CG>(p, t, BN);
    const int acc = lt % ACC;
    mbar_wait(&tfull[acc], (lt / ACC) & 1);
    tc_fence_after();
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 5);
#pragma unroll 1
    for (int sub = 0; sub < HSUB; ++sub) {
    const uint32_t tbase = tmem + acc * TCOLS + sub * tmem_cols<BN>() + grp * HALF + ((uint32_t)(quad * 32) << 16);
    float v[HALF];
#pragma unroll
    for (int c = 0; c < HALF / 32; ++c) tmem_ld32(tbase + 32 * c, v + 32 * c);
    if constexpr (HALF % 32 != 0) tmem_ld16(tbase + HALF - 16, v + HALF - 16);
    if (sub == HSUB - 1) {  // every sub-tile read: release the buffer to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 6);
      if (lane == 0) {
        if constexpr (CG == 1) {
          mbar_arrive_relaxed(&tempty[acc]);
        } else {
          mbar_arrive_cluster_relaxed(&tempty[acc], 0);
        }
      }
    }
    const int n0 = tc.n0 + grp * HALF;
#pragma unroll
    for (int q = 0; q < HALF; ++q) {
      float val = v[q] + sbias[n0 - tc.n0 + q];
      if (p.relu) val = val > 0.f ? val : 0.f;
      v[q] = val;
    }
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 12);
    if (p.epi_direct) {  // experiment (PC_KR_DIRECT): each lane stores its own row's 16-byte chunks
      const int row = quad * 32 + lane;
      long long m = -1;
      if constexpr (LINEAR) {
        const long long mm = (long long)tc.m0 + (long long)rank * BM + row;
        if (mm < p.M) m = mm;
      } else {
        const int tile = (tc.m0 + (int)rank * HSUB * BM) / (HSUB * BM);
        const int hb = tile / p.halo_tpi, yy = row / p.halo_Wv, xx = row - yy * p.halo_Wv;
        const int y = (tile - hb * p.halo_tpi) * p.halo_R * HSUB + sub * p.halo_R + yy;
        if (yy < p.halo_R && y < p.i2c_Ho && xx < p.i2c_Wo) m = ((long long)hb * p.i2c_Ho + y) * p.i2c_Wo + xx;
      }
      if (m >= 0) {
        __nv_bfloat16* dst = out + m * BN + grp * HALF;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          uint4 u;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
          *reinterpret_cast<uint4*>(dst + 8 * j) = u;
        }
      }
      continue;
    }
    // the previous tile's stores have read the box (64 threads: this quadrant's two warps)
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 13);
    #pragma unroll
    for (int s = 0; s < CH; ++s) {
      const int j = s;  // (a lane-rotated order would index v[] dynamically: local memory)
      uint32_t w[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * j + 2 * h], v[8 * j + 2 * h + 1]);
        w[h] = *reinterpret_cast<uint32_t*>(&b2);
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sbox + lane * ROWB + grp * HALF * 2 + 16 * j),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                   : "memory");
    }
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 14);
    const int tile = (tc.m0 + (int)rank * HSUB * BM) / (HSUB * BM);
    const int hb = LINEAR ? 0 : tile / p.halo_tpi;
    const int y0 = LINEAR ? 0 : (tile - hb * p.halo_tpi) * p.halo_R * HSUB + sub * p.halo_R;
#pragma unroll
    for (int g8 = 0; g8 < 2; ++g8) {
      const int r0 = 16 * grp + 8 * g8;  // first of this group's 8 rows within the quadrant
      int nrow;
      __nv_bfloat16* dst;
      if constexpr (LINEAR) {  // rows = consecutive output pixels
        const long long m = (long long)tc.m0 + (long long)rank * BM + quad * 32 + r0;
        if (m >= p.M) continue;
        nrow = (int)min(8LL, (long long)p.M - m);
        dst = out + m * BN;
      } else {
        const int row = quad * 32 + r0, yy = row / p.halo_Wv, xx = row - yy * p.halo_Wv, y = y0 + yy;
        if (yy >= p.halo_R || y >= p.i2c_Ho) continue;
        nrow = min(8, p.i2c_Wo - xx);
        dst = out + (((long long)hb * p.i2c_Ho + y) * p.i2c_Wo + xx) * BN;
      }
#pragma unroll
      for (int i = 0; i < (8 * RCH + 31) / 32; ++i) {
        const int c = i * 32 + lane, r = c / RCH, part = c - r * RCH;
        if (r < nrow && !p.dbg_nostore) {
          uint4 u;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                       : "r"(sbox + (r0 + r) * ROWB + 16 * part)
                       : "memory");
          *reinterpret_cast<uint4*>(dst + r * BN + part * 8) = u;
        }
      }
    }
    if (quad == 0 && grp == 0 && lane == 0) trace_stamp(p, lt, 15);
    }  // sub-tiles
  }
}

// Stage count for a (BN, CG) ring: one stage fewer for an fp32 output when that
// makes room for the TMA-store boxes.
template <int EPI, int BN, int S, int CG, bool BMN = false>
constexpr int fst() {
  const int extra = EPI == EPI_SGD ? 1024 + SGD_STAGE_BYTES : EPI == EPI_F32 && BN % 32 == 0 ? 1024 + F32_STAGE_BYTES : 0;
  int s = S;
  while (s > 2 && smem_bytes<BN, S, CG, false, 1, BMN>() - (S - s) * (BM * BK * 2 + b_rows<BN, CG, BMN>() * BK * 2) +
                         extra > 227 * 1024)
    --s;
  return s;
}

template <int AM> constexpr int kernel_threads() { return a_is_gather<AM>() ? 192 + GATHER_THREADS : 320; }

template <int AM, int BMODE, int EPI, int BN, int STAGES, int CG>
__global__ void __launch_bounds__(kernel_threads<AM>(), 1) umma_gemm_k(const __grid_constant__ Params p) {
  constexpr bool GATHER = a_is_gather<AM>();
  constexpr int EPW = GATHER ? 1 : 2;  // epilogue warps per TMEM lane quadrant (warps 0-3, and 6-9 unless gathering)
  // CTA-pair gather: each CTA gathers its own 128 A rows; the peer's gather
  // completions are relayed to the leader's full barrier by the peer's (idle) MMA warp.
  constexpr bool A_MN = a_is_mn<AM>();
  constexpr bool B_MN = BMODE == B_TMA_MN;
  constexpr int BNC = BN / CG;  // B rows (N) this CTA loads
  static_assert(!B_MN || BNC % 16 == 0, "MN-major B is loaded in 64-column chunks");
  constexpr int B_STAGE_BYTES = b_rows<BN, CG, B_MN>() * BK * 2;
  constexpr int MACC = macc_of<AM>();
  // MACC > 1: MMA N = p.N (<= BN, the B load width), accumulator a at TMEM column a * p.N
  const uint32_t IDESC = MACC > 2 ? ((make_idesc<BN, A_MN, B_MN, CG>() & ~(0x3Fu << 17)) | ((uint32_t)(p.N >> 3) << 17))
                                  : make_idesc<BN, A_MN, B_MN, CG>();
  constexpr bool KR2 = AM == A_HALO_KR2;
  // A_HALO_KR2: per buffer 2 sub-tile accumulators of tmem_cols<BN> columns, double-buffered
  constexpr int TCOLS = KR2 ? 2 * tmem_cols<BN>() : MACC > 1 ? 512 : tmem_cols<BN>();
  constexpr int ACC = KR2 ? 2 : MACC > 1 ? 1 : acc_count<BN>();
  constexpr int A_STAGE = MACC * A_STAGE_BYTES;  // this kernel's A bytes per stage (allocated)

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr bool IKR = AM == A_IM2COL_KR;
  constexpr bool BRES = AM == A_HALO_KR || IKR || AM == A_HALO_KR2;
  constexpr bool HALO = AM == A_HALO_K || AM == A_HALO_KR || AM == A_HALO_KR2;
  constexpr int RSLOT = AM == A_HALO_KR2 ? HALO_R2_SLOT_BYTES : HALO_R_SLOT_BYTES;
  // stage s: A at sA + s * A_STRIDE, B at sB + s * B_STRIDE (a halo stage holds its
  // window and its k B tiles contiguously; BRES: stages hold windows only, the B
  // tiles of every (k-block, filter row) sit after the ring)
  constexpr int A_STRIDE = IKR ? A_STAGE_BYTES : BRES ? RSLOT : HALO ? halo_stage_bytes<BN, CG>() : A_STAGE;
  constexpr int B_STRIDE = BRES ? 0 : HALO ? halo_stage_bytes<BN, CG>() : B_STAGE_BYTES;
  uint8_t* sA = smem;
  uint8_t* sB = IKR ? smem + STAGES * A_STAGE_BYTES
               : BRES ? smem + STAGES * RSLOT : HALO ? smem + HALO_SLOT_BYTES : smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(BRES ? sB + RES_B_BYTES
                                                    : smem + STAGES * (HALO ? halo_stage_bytes<BN, CG>()
                                                                            : A_STAGE + B_STAGE_BYTES));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [ACC]
  uint64_t* tempty = tfull + 2;      // [ACC]
  uint64_t* bres = tempty + 2;       // BRES: resident B loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2 + (BRES ? 1 : 0));
  constexpr bool F32TMA = f32_tma_epi<EPI, BN, STAGES, CG, AM, B_MN>();
  uint8_t* f32_boxes = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tmem_slot) + 4 + 1023) & ~uintptr_t(1023));
  uint64_t* sgd_bars = reinterpret_cast<uint64_t*>(f32_boxes + 8 * SGD_WARP_BYTES);  // EPI_SGD

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = p.tiles;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int units = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 4) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], !GATHER ? 1 : leader ? 1 + GATHER_THREADS + (CG - 1) : GATHER_THREADS);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < ACC; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], 4 * EPW * CG);
      }

      if constexpr (EPI == EPI_SGD)
        for (int w = 0; w < 8; ++w) mbar_init(&sgd_bars[w], 1);
      if constexpr (BRES) mbar_init(bres, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TCOLS * ACC));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TCOLS * ACC));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  if (warp == 5 && lane == 0) {
    prefetch_tmap(&p.tma_b);
    if constexpr (!GATHER) prefetch_tmap(&p.tma_a);
  }
  tc_fence_before();
  if constexpr (CG == 1) {
    __syncthreads();
  } else {
    cluster_sync();  // barrier inits and TMEM allocation visible to the peer before any remote arrive
  }
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, descriptor prefetch) may overlap the previous kernel's tail;
  // no global memory is touched before the previous grid has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 5) {
    // ------------------------------------------------------------ TMA producer
    // Warp-uniform loop (coordinates live in uniform registers); one elected
    // lane issues. im2col coordinates advance incrementally: the divisions run
    // once per tile, not once per k-block.
    int git = 0, plt = 0;
    if constexpr (BRES) {
      // resident B: tile r = kb * k + i (k-block kb = (chunk, filter column j), filter
      // row i) holds this CTA's BNC filters at K offset ((i k + j) C + 64 chunk)
      if (elect_one()) {
        const int nt = IKR ? p.num_kb : p.num_kb * p.i2c_k;
        if (leader) mbar_arrive_expect_tx(bres, CG * nt * B_STAGE_BYTES);
        for (int r = 0; r < nt; ++r) {
          int kcoord;
          if constexpr (IKR) {  // k-block r = (tap, 64-channel chunk)
            const int tap = r / p.i2c_cpt;
            kcoord = tap * p.i2c_C + (r - tap * p.i2c_cpt) * BK;
          } else {              // (k-block (chunk, column j), filter row i)
            const int kb = r / p.i2c_k, i = r - kb * p.i2c_k;
            const int ch = kb / p.i2c_k, j = kb - ch * p.i2c_k;
            kcoord = (i * p.i2c_k + j) * p.i2c_C + ch * BK;
          }
          tma_load_3d<CG>(&p.tma_b, bres, smem_u32(sB + r * B_STAGE_BYTES), kcoord, (int)rank * BNC, 0);
        }
      }
      __syncwarp();
    }
    for (int t = unit; t < total; t += units, ++plt) {
      if (lane == 0) trace_stamp(p, plt, 0);
      long long tr_wait = 0, tr_issue = 0;
      const TileCoord tc = tile_coord<CG>(p, t, BN);
      const int m0 = tc.m0 + (int)rank * BM;     // this CTA's A rows
      // this CTA's B rows (A_IM2COL_MN3P: the pair MMA has N = p.N <= BN, split in halves)
      const int n0 = tc.n0 + (int)rank * (AM == A_IM2COL_MN3P ? p.N / 2 : BNC);
      // A_IM2COL_K: tile's first output pixel (fixed) and the K position (c, i, j) of kb
      int t_b = 0, t_oy = 0, t_ox = 0, kc = 0, ki = 0, kj = 0, kblk = 0, kcoff = 0, ktap = 0;
      int t_b1 = 0, t_oy1 = 0, t_ox1 = 0;  // A_IM2COL_K2: the second accumulator's first pixel
      // A_IM2COL_MN: per-chunk (i, j, blk, coff) of the tile's M rows (fixed) and kb's pixel (b, oy, ox)
      constexpr bool A32 = AM == A_IM2COL_MN2_32;
      constexpr int ACH = A32 ? MACC * BM / 32 : MACC * BM / 64;  // A chunks per stage
      int ci[ACH], cj[ACH], cblk[ACH], ccoff[ACH];
      bool cvalid[ACH];  // A_IM2COL_MN3P: the chunk holds rows < M (others are not loaded)
      int pb = 0, poy = 0, pox = 0;
      // A_HALO_K: this CTA's tile (image hb, first output row hy0); K walks chunk-major
      int hb = 0, hy0 = 0;
      if constexpr (HALO) {  // k-block = (channel chunk, filter column j), j fastest
        // KR2: this CTA's tile = 2 sub-tiles (rows [tc.m0 + rank 256, +256)); halo_tpi counts them
        const int tile = KR2 ? (tc.m0 + (int)rank * 2 * BM) / (2 * BM) : m0 / BM;
        hb = tile / p.halo_tpi;
        hy0 = (tile - hb * p.halo_tpi) * p.halo_R * (KR2 ? 2 : 1);
        kc = (tc.kb_begin / p.i2c_k) * BK;
        kj = tc.kb_begin - (tc.kb_begin / p.i2c_k) * p.i2c_k;
      }
      if constexpr (AM == A_IM2COL_K || IKR || AM == A_IM2COL_K2) {
        // a CTA whose rows all lie past M (second half of a partial pair tile) loads
        // the first pixels instead (its rows are discarded by the epilogue): an
        // im2col start pixel outside the tensor faults the TMA unit
        const int mv = m0 < p.M ? m0 : 0;
        t_ox = mv % p.i2c_Wo;
        const int q = mv / p.i2c_Wo;
        t_oy = q % p.i2c_Ho;
        t_b = q / p.i2c_Ho;
        if constexpr (AM == A_IM2COL_K2) {  // accumulator 1: rows [m0 + 128 CG, +128)
          const int m1 = m0 + BM * CG, mv1 = m1 < p.M ? m1 : 0;
          t_ox1 = mv1 % p.i2c_Wo;
          const int q1 = mv1 / p.i2c_Wo;
          t_oy1 = q1 % p.i2c_Ho;
          t_b1 = q1 / p.i2c_Ho;
        }
        ktap = tc.kb_begin / p.i2c_cpt;
        kc = (tc.kb_begin - ktap * p.i2c_cpt) * BK;
        ki = ktap / p.i2c_k;
        kj = ktap - ki * p.i2c_k;
        kblk = kc / p.i2c_cs;
        kcoff = kc - kblk * p.i2c_cs;
      } else if constexpr (AM == A_IM2COL_MN || AM == A_IM2COL_MN5 || AM == A_IM2COL_MN2 || A32 ||
                           AM == A_IM2COL_MN3P) {
#pragma unroll
        for (int cch = 0; cch < ACH; ++cch) {
          // chunk cch = rows of accumulator cch / 2 (A32: cch / 4) (CTA pair: interleaved with the peer's)
          int kk = A32 ? tc.m0 + (cch >> 2) * (BM * CG) + (int)rank * BM + (cch & 3) * 32
                   : CG == 2 && MACC > 1 ? tc.m0 + (cch >> 1) * (BM * CG) + (int)rank * BM + (cch & 1) * 64
                                         : m0 + 64 * cch;
          cvalid[cch] = kk < p.M;
          if (kk >= p.M) kk = 0;  // rows past M are discarded by the epilogue
          int c, ij;
          if constexpr (A32) {
            const int unit = kk >> 5;
            ij = unit / p.m_grp;
            c = (unit - ij * p.m_grp) * 32;
          } else {
            const int cpt = p.m_cp ? p.m_cp : p.i2c_C;  // M rows per tap
            c = kk % cpt;
            ij = kk / cpt;
          }
          ci[cch] = ij / p.i2c_k;
          cj[cch] = ij - ci[cch] * p.i2c_k;
          cblk[cch] = c / p.i2c_cs;
          ccoff[cch] = c - cblk[cch] * p.i2c_cs;
        }
        const int pix0 = tc.kb_begin * BK, hw = p.i2c_Ho * p.i2c_Wo;
        pb = pix0 / hw;
        const int rem = pix0 - pb * hw;
        poy = rem / p.i2c_Wo;
        pox = rem - poy * p.i2c_Wo;
      }
      for (int it = 0; it < tc.nkb; ++it, ++git) {
        const int s = git % STAGES;
        const uint32_t ph = (git / STAGES) & 1;
        const long long c0 = p.trace ? clk() : 0;
        mbar_wait(&empty[s], ph ^ 1);
        const long long c1 = p.trace ? clk() : 0;
        const int kb = tc.kb_begin + it;
        if (HALO && p.dbg_noload) {  // debug: MMA + pipeline cost without operand traffic
          if (leader && elect_one()) mbar_arrive(&full[s]);
        } else if (HALO && elect_one()) {
          // the window for (chunk, column j) and the B tiles of taps (0..k-1, j)
          if (leader) mbar_arrive_expect_tx(&full[s], CG * (p.halo_bytes + (BRES ? 0 : p.i2c_k * B_STAGE_BYTES)));
          const uint32_t st0 = smem_u32(sA + s * A_STRIDE);
          tma_load_4d<CG>(&p.tma_a, &full[s], st0, kc, p.halo_lo + kj, hy0 + p.halo_lo, hb);
          if constexpr (!BRES)
            for (int i = 0; i < p.i2c_k; ++i)
              tma_load_3d<CG>(&p.tma_b, &full[s], st0 + HALO_SLOT_BYTES + i * B_STAGE_BYTES,
                              (i * p.i2c_k + kj) * p.i2c_C + kc, n0, 0);
        } else if (!HALO && elect_one()) {
          // A_IM2COL_K: the k-block of a last chunk with <= 32 channels moves 32-channel boxes
          const bool half = (AM == A_IM2COL_K || AM == A_IM2COL_K2) && p.half_chunk && kc + 32 >= p.i2c_C;
          if (leader)
            mbar_arrive_expect_tx(&full[s], IKR ? CG * A_STAGE_BYTES
                                  : AM == A_IM2COL_K2 ? CG * (B_STAGE_BYTES + 2 * A_STAGE_BYTES) / (half ? 2 : 1)
                                  : half ? CG * (B_STAGE_BYTES + A_STAGE_BYTES) / 2
                                  : AM == A_IM2COL_MN3P ? CG * B_STAGE_BYTES + p.macc_chunks * 64 * BK * 2
                                                 : CG * (B_STAGE_BYTES + (GATHER ? 0 : MACC > 1 ? p.macc_chunks * 64 * BK * 2
                                                                                       : A_STAGE_BYTES)));
          const uint32_t dB = smem_u32(sB + s * B_STAGE_BYTES);
          if constexpr (IKR) {
            // B resident
          } else if constexpr (B_MN) {
            if (p.b_chunked) {  // one op: {64 cols, BK rows, BNC/64 chunks} of the chunked view
              tma_load_4d<CG>(&p.tma_b, &full[s], dB, 0, kb * BK, blk_off(n0, p.b_cb) >> 6, blk_idx(n0, p.b_cb));
            } else {
#pragma unroll
              for (int c = 0; c < (BNC + 63) / 64; ++c) {
                int n = n0 + 64 * c;
                tma_load_3d<CG>(&p.tma_b, &full[s], dB + c * (64 * BK * 2), blk_off(n, p.b_cb), kb * BK,
                                blk_idx(n, p.b_cb));
              }
            }
          } else {
            const int k = (AM == A_IM2COL_K || AM == A_IM2COL_K2) ? ktap * p.i2c_C + kc : kb * BK;
            tma_load_3d<CG>(half ? &p.tma_b32 : &p.tma_b, &full[s], dB, blk_off(k, p.b_cb), n0, blk_idx(k, p.b_cb));
          }
          if constexpr (AM == A_IM2COL_K || IKR) {
            // 128 output pixels from the tile's first pixel; K block = 64 (or 32) channels of tap (i, j)
            tma_im2col_5d<CG>(half ? &p.tma_a32 : &p.tma_a, &full[s], smem_u32(sA + s * A_STAGE_BYTES), kcoff,
                              t_ox * p.i2c_s + p.i2c_lw, t_oy * p.i2c_s + p.i2c_lh, t_b, kblk, (uint16_t)kj,
                              (uint16_t)ki);
          } else if constexpr (AM == A_IM2COL_K2) {  // one box per accumulator, 16 KB apart
            const uint32_t dA = smem_u32(sA + s * A_STRIDE);
            tma_im2col_5d<CG>(half ? &p.tma_a32 : &p.tma_a, &full[s], dA, kcoff, t_ox * p.i2c_s + p.i2c_lw,
                              t_oy * p.i2c_s + p.i2c_lh, t_b, kblk, (uint16_t)kj, (uint16_t)ki);
            tma_im2col_5d<CG>(half ? &p.tma_a32 : &p.tma_a, &full[s], dA + A_STAGE_BYTES, kcoff,
                              t_ox1 * p.i2c_s + p.i2c_lw, t_oy1 * p.i2c_s + p.i2c_lh, t_b1, kblk, (uint16_t)kj,
                              (uint16_t)ki);
          } else if constexpr (AM == A_IM2COL_MN || AM == A_IM2COL_MN5 || AM == A_IM2COL_MN2 || A32 ||
                               AM == A_IM2COL_MN3P) {
            // K block = 64 consecutive pixels; M = (i, j, c): 64-channel chunks (A32: 32-channel)
#pragma unroll
            for (int cch = 0; cch < ACH; ++cch)
              if (MACC == 1 || A32 || (AM == A_IM2COL_MN3P ? cvalid[cch] : cch < p.macc_chunks))
              tma_im2col_5d<CG>(A32 ? &p.tma_a32 : &p.tma_a, &full[s],
                                smem_u32(sA + s * A_STAGE) + cch * ((A32 ? 32 : 64) * BK * 2),
                                ccoff[cch], pox * p.i2c_s + p.i2c_lw, poy * p.i2c_s + p.i2c_lh, pb, cblk[cch],
                                (uint16_t)cj[cch], (uint16_t)ci[cch]);
          } else if constexpr (!GATHER) {
            const uint32_t dA = smem_u32(sA + s * A_STAGE_BYTES);
            if constexpr (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c) {
                int m = m0 + 64 * c;
                tma_load_3d<CG>(&p.tma_a, &full[s], dA + c * (64 * BK * 2), blk_off(m, p.a_cb), kb * BK,
                                blk_idx(m, p.a_cb));
              }
            } else {
              int k = kb * BK;
              tma_load_3d<CG>(&p.tma_a, &full[s], dA, blk_off(k, p.a_cb), m0, blk_idx(k, p.a_cb));
            }
          }
        }
        __syncwarp();
        // advance the im2col K position / pixel walk to the next k-block
        if constexpr (AM == A_IM2COL_K || IKR || AM == A_IM2COL_K2) {
          kc += BK;
          kcoff += BK;
          if (kcoff >= p.i2c_cs) { kcoff = 0; ++kblk; }
          if (kc >= p.i2c_C) {
            kc = kcoff = kblk = 0;
            ++ktap;
            if (++kj == p.i2c_k) { kj = 0; ++ki; }
          }
        } else if constexpr (HALO) {
          if (++kj == p.i2c_k) { kj = 0; kc += BK; }
        } else if constexpr (AM == A_IM2COL_MN || AM == A_IM2COL_MN5 || AM == A_IM2COL_MN2 || A32 ||
                             AM == A_IM2COL_MN3P) {
          pox += BK;
          while (pox >= p.i2c_Wo) {
            pox -= p.i2c_Wo;
            if (++poy == p.i2c_Ho) { poy = 0; ++pb; }
          }
        }
        if (p.trace) {
          const long long c2 = clk();
          tr_wait += c1 - c0;
          tr_issue += c2 - c1;
        }
      }
      if (lane == 0) {
        trace_stamp(p, plt, 1);
        trace_put(p, plt, 8, tr_wait);
        trace_put(p, plt, 9, tr_issue);
      }
    }
  } else if (warp >= 6 && GATHER) {
    // ----------------------------------------------------- im2col gather producer
    if constexpr (GATHER) {
      const int gt = threadIdx.x - 192;
      const pc_conv_geom& g = p.g;
      int git = 0;
      for (int t = unit; t < total; t += units) {
        const TileCoord tc = tile_coord<CG>(p, t, BN);
        const int m0 = tc.m0 + (int)rank * BM;
        if constexpr (AM == A_GATHER_FWD || AM == A_GATHER_DGRAD) {
          // K-major rows = pixels; thread owns 16B chunk q of rows rb + 16*r8
          constexpr int RS = GATHER_THREADS / 8;  // row stride between a thread's rows
          const int q = gt & 7, rb = gt >> 3;
          int rb_b[GR], ry[GR], rx[GR];
#pragma unroll
          for (int r8 = 0; r8 < GR; ++r8) {
            int m = m0 + rb + RS * r8;
            int W_ = AM == A_GATHER_FWD ? g.Wo : g.W, H_ = AM == A_GATHER_FWD ? g.Ho : g.H;
            if (m < p.M) {
              int x = m % W_, q2 = m / W_;
              int y = q2 % H_;
              rb_b[r8] = q2 / H_;
              if constexpr (AM == A_GATHER_FWD) {
                ry[r8] = y * g.stride - g.pad;
                rx[r8] = x * g.stride - g.pad;
              } else {
                ry[r8] = y + g.pad;
                rx[r8] = x + g.pad;
              }
            } else {
              rb_b[r8] = 0;
              ry[r8] = -(1 << 28);
              rx[r8] = -(1 << 28);
            }
          }
          for (int it = 0; it < tc.nkb; ++it, ++git) {
            const int s = git % STAGES;
            const uint32_t ph = (git / STAGES) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            // 32-bit index math: 64-bit integer division is emulated (~100 instructions)
            const int k = (tc.kb_begin + it) * BK + q * 8;
            const bool kvalid = k < p.K;
            const uint32_t base = smem_u32(sA + s * A_STAGE_BYTES);
            if constexpr (AM == A_GATHER_FWD) {
              int c = kvalid ? (int)((unsigned)k % (unsigned)g.C) : 0;
              int ij = kvalid ? (int)((unsigned)k / (unsigned)g.C) : 0;
              int i = ij / g.k, j = ij - (ij / g.k) * g.k;
              int blk = c / g.cs, coff = c - blk * g.cs;
              const __nv_bfloat16* src0 = p.gsrc + blk * g.cstride + coff;
#pragma unroll
              for (int r8 = 0; r8 < GR; ++r8) {
                int r = rb + RS * r8;
                int iy = ry[r8] + i, ix = rx[r8] + j;
                bool ok = kvalid && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
                const __nv_bfloat16* src =
                    ok ? src0 + ((long long)(rb_b[r8] * g.H + iy) * g.W + ix) * g.cs : p.gsrc;
                cp_async16(base + r * 128 + ((q ^ (r & 7)) << 4), src, ok);
              }
            } else {
              int n = kvalid ? (int)((unsigned)k % (unsigned)g.N) : 0;
              int ij = kvalid ? (int)((unsigned)k / (unsigned)g.N) : 0;
              int i = ij / g.k, j = ij - (ij / g.k) * g.k;
              const __nv_bfloat16* src0 = p.gsrc + n;
#pragma unroll
              for (int r8 = 0; r8 < GR; ++r8) {
                int r = rb + RS * r8;
                int ny = ry[r8] - i, nx = rx[r8] - j;
                bool ok = kvalid && ny >= 0 && nx >= 0;
                int oy = 0, ox = 0;
                if (g.stride == 1) {
                  oy = ny; ox = nx;
                } else {
                  ok = ok && (ny % g.stride == 0) && (nx % g.stride == 0);
                  oy = ny / g.stride; ox = nx / g.stride;
                }
                ok = ok && oy < g.Ho && ox < g.Wo;
                const __nv_bfloat16* src =
                    ok ? src0 + ((long long)(rb_b[r8] * g.Ho + oy) * g.Wo + ox) * g.N : p.gsrc;
                cp_async16(base + r * 128 + ((q ^ (r & 7)) << 4), src, ok);
              }
            }
            cp_async_arrive_noinc(&full[s]);
          }
        } else {
          // A_GATHER_WGRAD: MN-major rows = pixels (K), chunk q = 8 consecutive (i,j,c) of this M tile
          constexpr int PS = GATHER_THREADS / 16;  // pixel stride between a thread's rows
          const int q = gt & 15, rb = gt >> 4;
          const int kc = m0 + q * 8;
          const bool mvalid = kc < p.M;
          int c = mvalid ? (int)((unsigned)kc % (unsigned)g.C) : 0;
          int ij = mvalid ? (int)((unsigned)kc / (unsigned)g.C) : 0;
          int i = ij / g.k, j = ij - (ij / g.k) * g.k;
          int blk = c / g.cs, coff = c - blk * g.cs;
          const __nv_bfloat16* src0 = p.gsrc + blk * g.cstride + coff;
          const unsigned hw = (unsigned)(g.Ho * g.Wo);
          const uint32_t cofs = (q >> 3) * (64 * BK * 2);
          for (int it = 0; it < tc.nkb; ++it, ++git) {
            const int s = git % STAGES;
            const uint32_t ph = (git / STAGES) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t base = smem_u32(sA + s * A_STAGE_BYTES) + cofs;
            // pixel of row rb (32-bit divides once per k-block), then step 8 pixels per row
            const unsigned pix0 = (unsigned)((tc.kb_begin + it) * BK + rb);
            int b = (int)(pix0 / hw);
            int rem = (int)(pix0 - (unsigned)b * hw);
            int oy = rem / g.Wo;
            int ox = rem - oy * g.Wo;
#pragma unroll
            for (int r8 = 0; r8 < GR; ++r8) {
              int r = rb + PS * r8;
              bool ok = mvalid && (int)pix0 + PS * r8 < p.K;
              int iy = oy * g.stride + i - g.pad, ix = ox * g.stride + j - g.pad;
              ok = ok && (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
              const __nv_bfloat16* src = ok ? src0 + ((long long)(b * g.H + iy) * g.W + ix) * g.cs : p.gsrc;
              cp_async16(base + r * 128 + (((q & 7) ^ (r & 7)) << 4), src, ok);
              ox += PS;
              while (ox >= g.Wo) {
                ox -= g.Wo;
                if (++oy == g.Ho) { oy = 0; ++b; }
              }
            }
            cp_async_arrive_noinc(&full[s]);
          }
        }
      }
    }
  } else if (warp == 4) {
    // --------------------------------------------------------------- MMA issuer
    // Warp-uniform loop; one elected lane issues the tcgen05.mma / commit.
    // Descriptors: the stage-0 descriptor plus (byte offset >> 4) of stage / k step.
    if (leader) {
      // A_IM2COL_MN2_32: MN-major 64B swizzle, 32-element MN groups of 64 K rows (4 KB apart)
      const uint64_t a0 = AM == A_IM2COL_MN2_32 ? make_desc_sw64(smem_u32(sA), 32 * BK * 2, 512)
                          : A_MN ? make_desc(smem_u32(sA), 64 * BK * 2, 1024) : make_desc(smem_u32(sA), 16, 1024);
      const uint64_t b0 = B_MN ? make_desc(smem_u32(sB), 64 * BK * 2, 1024) : make_desc(smem_u32(sB), 16, 1024);
      const uint64_t a0h = make_desc_sw64(smem_u32(sA), 16, 512), b0h = make_desc_sw64(smem_u32(sB), 16, 512);
      constexpr uint32_t A_KSTEP = (AM == A_IM2COL_MN2_32 ? 1024 : A_MN ? 2048 : 32) >> 4,
                         B_KSTEP = (B_MN ? 2048 : 32) >> 4;
      int git = 0, lt = 0;
      // halo: descriptor offset (16-byte units) of one filter row (Wv window rows of 128 B)
      // and of one KR2 sub-tile (R filter rows)
      const uint32_t hrstep = HALO ? (uint32_t)((p.halo_Wv * 128) >> 4) : 0u;
      const uint32_t hastep = HALO ? (uint32_t)p.halo_R * hrstep : 0u;
      if constexpr (BRES) {
        mbar_wait(bres, 0);
        tc_fence_after();
      }
      for (int t = unit; t < total; t += units, ++lt) {
        const TileCoord tc = tile_coord<CG>(p, t, BN);
        const int acc = lt % ACC;
        const uint32_t aph = (lt / ACC) & 1;
        if (lane == 0) trace_stamp(p, lt, 2);
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        if (lane == 0) trace_stamp(p, lt, 3);
        const uint32_t tacc = tmem + acc * TCOLS;
        long long tr_wait = 0, tr_issue = 0;
        // K-major im2col with a partial last channel chunk: k16 steps with real channels
        const bool partial = (AM == A_IM2COL_K || AM == A_IM2COL_K2) && (p.i2c_C % BK) != 0;
        int mchunk = partial ? tc.kb_begin % p.i2c_cpt : 0;
        // halo: k-block = (channel chunk, filter column j): k filter rows per stage
        int hj = HALO ? tc.kb_begin % p.i2c_k : 0, hch = HALO ? tc.kb_begin / p.i2c_k : 0;
        for (int it = 0; it < tc.nkb; ++it, ++git) {
          int nk16 = BK / 16;
          bool half = false;
          if (partial) {
            const int left = p.i2c_C - mchunk * BK;
            if (left < BK) nk16 = (left + 15) / 16;
            half = p.half_chunk && left <= 32;
            if (++mchunk == p.i2c_cpt) mchunk = 0;
          }
          if constexpr (HALO) {
            // zero_tail16: the last 16 input channels carry structural-zero filter weights
            const int left = p.i2c_C - (p.zero_tail16 ? 16 : 0) - hch * BK;
            if (left < BK) nk16 = (left + 15) / 16;
          }
          const int s = git % STAGES;
          const uint32_t ph = (git / STAGES) & 1;
          const long long c0 = p.trace ? clk() : 0;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const long long c1 = p.trace ? clk() : 0;
          if (it == 0 && lane == 0) trace_stamp(p, lt, 7);
          if constexpr (GATHER) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (elect_one()) {
            const uint64_t ad = (half ? a0h : a0) + (uint64_t)((s * A_STRIDE) >> 4);
            const uint64_t bd = BRES ? b0 + (uint64_t)(((tc.kb_begin + it) * (IKR ? 1 : p.i2c_k) * B_STAGE_BYTES) >> 4)
                                     : (half ? b0h : b0) + (uint64_t)((s * B_STRIDE) >> 4);
            if constexpr (HALO) {
              // filter row i: the window shifted by i * Wv rows (multiple of 8), B tile i;
              // KR2 sub-tile a: further shifted by a * R * Wv rows, accumulator a
              const int k = p.i2c_k;
#pragma unroll
              for (int a = 0; a < (KR2 ? 2 : 1); ++a)
              for (int i = 0; i < k; ++i) {
                const uint64_t ai = ad + (uint64_t)(a * hastep + i * hrstep);
                const uint64_t bi = bd + (uint64_t)((i * B_STAGE_BYTES) >> 4);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  if (kk < nk16)
                    tc_mma<CG>(tacc + a * tmem_cols<BN>(), ai + kk * A_KSTEP, bi + kk * B_KSTEP, IDESC,
                               (it > 0 || i > 0 || kk > 0) ? 1u : 0u);
              }
            } else if constexpr (MACC > 1) {
              // accumulator a: A rows [128 a, 128 a + 128) of the stage (two 64-row chunks)
              for (int a = 0; a < MACC; ++a) {
                if (AM == A_IM2COL_MN5 && 2 * a >= p.macc_chunks) break;
                const uint64_t aa = ad + (uint64_t)((a * A_STAGE_BYTES) >> 4);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                  if (kk < nk16)   // A_IM2COL_K2: the remainder chunk's real k16 steps
                    tc_mma<CG>(tacc + (MACC == 2 ? a * tmem_cols<BN>() : a * p.N), aa + kk * A_KSTEP,
                               bd + kk * B_KSTEP, IDESC, (it > 0 || kk > 0) ? 1u : 0u);
              }
            } else {
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk)
                if (kk < nk16)
                  tc_mma<CG>(tacc, ad + kk * A_KSTEP, bd + kk * B_KSTEP, IDESC, (it > 0 || kk > 0) ? 1u : 0u);
            }
            tc_commit<CG>(&empty[s]);
          }
          __syncwarp();
          if constexpr (HALO) {
            if (++hj == p.i2c_k) { hj = 0; ++hch; }
          }
          if (p.trace) {
            const long long c2 = clk();
            tr_wait += c1 - c0;
            tr_issue += c2 - c1;
          }
        }
        if (elect_one()) tc_commit<CG>(&tfull[acc]);
        __syncwarp();
        if (lane == 0) {
          trace_stamp(p, lt, 4);
          trace_put(p, lt, 10, tr_wait);
          trace_put(p, lt, 11, tr_issue);
        }
      }
    } else if constexpr (GATHER && CG == 2) {
      // peer CTA: relay each stage's gather completion to the leader's full barrier
      if (lane == 0) {
        int git = 0;
        for (int t = unit; t < total; t += units) {
          const TileCoord tc = tile_coord<CG>(p, t, BN);
          for (int it = 0; it < tc.nkb; ++it, ++git) {
            const int s = git % STAGES;
            mbar_wait(&full[s], (git / STAGES) & 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_cluster(&full[s], 0);
          }
        }
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3, grp = warp >= 6 ? 1 : 0;
    if constexpr (BRES && EPI == EPI_BF16) {
      epilogue_bf16_halo<BN, CG, IKR, KR2 ? 2 : 1>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane,
                                                   f32_boxes + quad * (64 * BN));
    } else if constexpr (EPI == EPI_SGD) {
      static_assert(EPW == 2 && BN % 32 == 0, "fused SGD epilogue: 8 epilogue warps, 32-column groups");
      epilogue_sgd_tma<BN, CG, EPW>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane,
                                    f32_boxes + (grp * 4 + quad) * SGD_WARP_BYTES, &sgd_bars[grp * 4 + quad]);
    } else if constexpr (bf16_tma_epi<EPI, AM>()) {
      if (p.out_tma) {
        epilogue_bf16_tma<BN, CG, EPW, MACC>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane,
                                             f32_boxes + (grp * 4 + quad) * BF16_WARP_BYTES);
      } else {
        epilogue<EPI, BN, CG, EPW, HALO, MACC>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane);
      }
    } else if constexpr (F32TMA) {
      if (p.out_tma) {
        epilogue_f32_tma<BN, CG, EPW>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane,
                                      f32_boxes + (grp * 4 + quad) * F32_BOX_BYTES);
      } else {
        epilogue<EPI, BN, CG, EPW, HALO, MACC>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane);
      }
    } else {
      epilogue<EPI, BN, CG, EPW, HALO, MACC>(p, tmem, tfull, tempty, unit, units, rank, quad, grp, lane);
    }
  }

  tc_fence_before();
  if constexpr (CG == 1) {
    __syncthreads();
  } else {
    cluster_sync();  // the leader's MMAs read this CTA's smem until the last tile drains
  }
  if (warp == 4) {
    tc_fence_after();
    if constexpr (CG == 1) {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS * ACC));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS * ACC));
    }
  }
}

// --------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 3-D bf16 view {inner, rows, blocks} with strides (ld, bstride) elements; box {64, box_rows, 1}.
static int make_map(CUtensorMap* map, const void* ptr, long long inner, long long rows, long long blocks,
                    long long ld, long long bstride, int box_rows, int box_inner = 64) {
  PC_REQUIRE(get_encode(), PC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  PC_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && ld % 8 == 0 && (blocks == 1 || bstride % 8 == 0),
             PC_EVALUE, "TMA view not 16-byte aligned (ld=%lld bstride=%lld)", ld, bstride);
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)blocks};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)(blocks > 1 ? bstride : ld * rows) * 2};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_inner == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PC_REQUIRE(r == CUDA_SUCCESS, PC_ECUDA, "cuTensorMapEncodeTiled failed (%d): inner=%lld rows=%lld blocks=%lld",
             (int)r, inner, rows, blocks);
  return PC_OK;
}

// MN-major operand as a chunked view {64 cols, rows, cols/64 chunks, blocks}: a
// box {64, 64, n_chunks, 1} lands as [chunk][row][128 B], the MN-major UMMA layout,
// so a whole BN-wide stage is one TMA op. Returns false when not expressible.
static bool make_mn_chunked_map(CUtensorMap* map, const void* ptr, long long cb, long long rows, long long blocks,
                                long long ld, long long bstride, int n_chunks) {
  if (!get_encode() || cb % 64 || ld % 8 || (reinterpret_cast<uintptr_t>(ptr) & 15) ||
      (blocks > 1 && bstride % 8) || n_chunks < 1 || n_chunks > 4)
    return false;
  cuuint64_t dims[4] = {64u, (cuuint64_t)rows, (cuuint64_t)(cb / 64), (cuuint64_t)blocks};
  cuuint64_t strides[3] = {(cuuint64_t)ld * 2, 128u, (cuuint64_t)(blocks > 1 ? bstride : ld * rows) * 2};
  cuuint32_t box[4] = {64u, (cuuint32_t)BK, (cuuint32_t)n_chunks, 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  return g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static PFN_cuTensorMapEncodeIm2col_v12000 g_encode_i2c = nullptr;
static std::once_flag g_encode_i2c_once;

// im2col view of a channel-blocked NHWC activation: dims {cs, W, H, B, nblk};
// each load = `pixels` walked output positions x 64 channels (128 B rows, 128B swizzle).
static int make_im2col_map(CUtensorMap* map, const void* ptr, int cs, int W, int H, int B, int nblk,
                           long long cstride, int pixels, int lw, int lh, int uw, int uh, int stride,
                           int chans = 64) {
  std::call_once(g_encode_i2c_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_i2c = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
  });
  PC_REQUIRE(g_encode_i2c != nullptr, PC_ECUDA, "cuTensorMapEncodeIm2col unavailable");
  PC_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && cs % 8 == 0 && cs >= 64, PC_EVALUE,
             "im2col view misaligned");
  cuuint64_t dims[5] = {(cuuint64_t)cs, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)nblk};
  cuuint64_t strides[4] = {(cuuint64_t)cs * 2, (cuuint64_t)W * cs * 2, (cuuint64_t)H * W * cs * 2,
                           (cuuint64_t)(nblk > 1 ? cstride : (long long)B * H * W * cs) * 2};
  int lower[3] = {lw, lh, 0}, upper[3] = {uw, uh, 0};
  cuuint32_t estr[5] = {1u, (cuuint32_t)stride, (cuuint32_t)stride, 1u, 1u};
  CUresult r = g_encode_i2c(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr), dims, strides, lower,
                            upper, (cuuint32_t)chans, (cuuint32_t)pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            chans == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  PC_REQUIRE(r == CUDA_SUCCESS, PC_ECUDA, "cuTensorMapEncodeIm2col failed (%d)", (int)r);
  return PC_OK;
}

static std::atomic<unsigned long long> g_tc_launches{0}, g_simt_launches{0};
// Per-thread cap on the persistent grid of the next tensor-core launches
// (pc_set_grid_cap): lets a step program run two GEMM chains side by side on
// disjoint SM sets (the CUDA graph records the grid of each launch).
static thread_local int t_grid_cap = 0;

// Programmatic dependent launch for the GEMM kernels (PC_PDL=0 disables): a
// GEMM's prologue overlaps the tail of the kernel before it on the stream.
static bool pdl_enabled() {
  static const int on = [] {
    const char* e = getenv("PC_PDL");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
static unsigned long long* g_trace = nullptr;  // pc_debug_trace_gemm

// fp32 output view for the TMA-store epilogue: {N, M, splits} with row stride
// o_ld and slice stride split_stride (elements). 0 = not expressible (or
// PC_F32_TMA=0): the kernel falls back to per-lane row stores.
static int f32_out_map(CUtensorMap* map, const Params& p, int splits) {
  static const int on = [] {
    const char* e = getenv("PC_F32_TMA");
    return e ? atoi(e) : 1;
  }();
  if (!on || !get_encode() || (reinterpret_cast<uintptr_t>(p.out) & 15) || p.o_ld % 4 ||
      (splits > 1 && p.split_stride % 4) || p.N < 1 || p.M < 1)
    return 0;
  cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)p.M, (cuuint64_t)std::max(splits, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)p.o_ld * 4,
                           (cuuint64_t)(splits > 1 ? p.split_stride : p.o_ld * (long long)p.M) * 4};
  cuuint32_t box[3] = {32u, 32u, 1u};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p.out, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 1 : 0;
}

template <int AM, int BMODE, int EPI, int BN, int STAGES, int CG>
static int launch(const Params& p, int splits, cudaStream_t st) {
  auto kern = umma_gemm_k<AM, BMODE, EPI, BN, STAGES, CG>;
  constexpr int smem = kernel_smem<EPI, BN, STAGES, CG, AM, BMODE == B_TMA_MN>();
  static_assert(smem <= 227 * 1024, "stage ring exceeds shared memory");
  constexpr int threads = kernel_threads<AM>();
  static int resident = 0;  // persistent CTAs the device holds at once
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (!resident) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (CG == 1) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
      const int tmem_cap = macc_of<AM>() > 1 ? 1 : 512 / (tmem_cols<BN>() * acc_count<BN>());
      per_sm = std::max(1, std::min(per_sm, tmem_cap));
      resident = sms * per_sm;
    } else {
      int clusters = 0;
      cfg.gridDim = dim3(sms & ~1);
      if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1) {
        cudaGetLastError();
        clusters = sms / 2;
      }
      resident = 2 * clusters;
    }
  }
  Params q = p;
  q.trace = g_trace;
  q.mt_rows = BM * CG * macc_of<AM>();
  static const int nostore = [] {
    const char* e = getenv("PC_DEBUG_NOSTORE");
    return e ? atoi(e) : 0;
  }();
  q.dbg_nostore = nostore;
  static const int noload = [] {
    const char* e = getenv("PC_DEBUG_NOLOAD");
    return e ? atoi(e) : 0;
  }();
  q.dbg_noload = noload;
  static const int kr_direct = [] {
    const char* e = getenv("PC_KR_DIRECT");
    return e ? atoi(e) : 0;
  }();
  q.epi_direct = kr_direct;
  if constexpr (f32_tma_epi<EPI, BN, STAGES, CG, AM, BMODE == B_TMA_MN>()) q.out_tma = f32_out_map(&q.tma_out, q, splits);
  q.tiles = ceil_div(p.N, BN) * ceil_div(p.M, q.mt_rows) * splits;
  static const int max_ctas = [] {  // debug: cap the persistent grid (PC_MAX_CTAS)
    const char* e = getenv("PC_MAX_CTAS");
    return e ? atoi(e) : 0;
  }();
  int cap = resident;
  if (max_ctas > 0) cap = std::min(cap, max_ctas);
  if (t_grid_cap > 0) cap = std::min(cap, std::max(t_grid_cap, CG));
  const int units = std::min(q.tiles, cap / CG);
  cfg.gridDim = dim3(units * CG);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, q);
  PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "umma_gemm launch: %s", cudaGetErrorString(e));
  g_tc_launches.fetch_add(1, std::memory_order_relaxed);
  PC_CUDA_CHECK_LAUNCH("umma_gemm");
  return PC_OK;
}

// Tile shape: BN (the MMA's N) and CG (1 = one SM, M = 128; 2 = CTA pair,
// M = 256, each SM holding half of B). Wide tiles cut the operand bytes each
// SM pulls from L2 per FLOP — the limit of these kernels — so the pair is used
// whenever the A operand comes by TMA and there are enough M tiles to occupy
// the 74 pairs; small-M FC layers (M = batch) stay single-SM and narrow N until
// the grid fills the machine. For a K-major B the TMA box height is BN / CG;
// an MN-major B is loaded in 64-column chunks, so BN / CG must be 64 or 128.
struct Tile {
  int bn, cg;
};

static bool mn192_enabled() {
  static const int on = [] {
    const char* e = getenv("PC_MN192");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
static bool cg2_enabled() {
  static const int on = [] {
    const char* e = getenv("PC_CG2");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}

static int bn_for(int N, int M = 1 << 30) {
  int bn = N <= 64 ? 64 : N <= 96 ? 96 : N <= 128 ? 128 : N % 192 == 0 ? 192 : 256;
  const long long tm = (M + BM - 1) / BM;
  while (bn > 64 && tm * ((N + bn - 1) / bn) < 148) bn = bn > 128 ? 128 : 64;
  return bn;
}
static int bn_for_mn(int N, int M = 1 << 30) {
  int bn = N <= 64 ? 64 : N <= 128 ? 128 : N % 192 == 0 ? 192 : 256;
  const long long tm = (M + BM - 1) / BM;
  while (bn > 64 && tm * ((N + bn - 1) / bn) < 148) bn = bn > 128 ? 128 : 64;
  return bn;
}

static Tile pick_k(int M, int N, bool pair_ok, int splits = 1) {
  if (pair_ok && cg2_enabled()) {
    const int bn = N <= 64 ? 64 : N <= 96 ? 96 : N <= 128 ? 128 : N % 192 == 0 ? 192 : 256;
    const long long units = (long long)((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn) * splits;
    if (units >= 74) return {bn, 2};
  }
  return {bn_for(N, splits > 1 ? 1 << 30 : M), 1};
}
static Tile pick_mn(int M, int N, bool pair_ok, int splits = 1) {
  if (pair_ok && cg2_enabled()) {
    // N = 384 (AlexNet conv3 / conv4 filters): two 192-wide tiles instead of 256 + 128
    const int bn = N <= 128 ? 128 : (N % 192 == 0 && N % 256 != 0 && mn192_enabled()) ? 192 : 256;
    const long long units = (long long)((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn) * splits;
    if (units >= 74) return {bn, 2};
  }
  return {bn_for_mn(N, splits > 1 ? 1 << 30 : M), 1};
}

template <int AM, int EPI>
static int launch_kb(const Params& p, Tile t, int splits, cudaStream_t st) {
  if constexpr (AM == A_HALO_KR2) {  // 42 KB window stages + resident B (CTA pair, N == 96)
    if (t.cg == 2 && t.bn == 96) return launch<AM, B_TMA_K, EPI, 96, 3, 2>(p, splits, st);
    PC_REQUIRE(false, PC_ESHAPE, "resident-B halo x2: CTA pair with N == 96 only");
  } else if constexpr (AM == A_IM2COL_KR) {  // 16 KB im2col stages + resident B (CTA pair, N == 96)
    if (t.cg == 2 && t.bn == 96) return launch<AM, B_TMA_K, EPI, 96, 8, 2>(p, splits, st);
    PC_REQUIRE(false, PC_ESHAPE, "resident-B im2col: CTA pair with N == 96 only");
  } else if constexpr (AM == A_HALO_KR) {  // window stages + resident B (CTA pair, N <= 96)
    static const int kr_stages = [] {  // tuning knob PC_KR_STAGES (4 or 5)
      const char* e = getenv("PC_KR_STAGES");
      return e ? atoi(e) : 5;
    }();
    if (t.cg == 2 && t.bn <= 96 && kr_stages == 4) return launch<AM, B_TMA_K, EPI, 96, 4, 2>(p, splits, st);
    if (t.cg == 2 && t.bn <= 96) return launch<AM, B_TMA_K, EPI, 96, 5, 2>(p, splits, st);
    PC_REQUIRE(false, PC_ESHAPE, "resident-B halo: CTA pair with N <= 96 only");
  } else if constexpr (AM == A_IM2COL_K2) {  // two 16 KB A boxes + the B half per stage; CTA pair only
    if (t.cg == 2 && t.bn == 256) return launch<AM, B_TMA_K, EPI, 256, 3, 2>(p, splits, st);
    if (t.cg == 2 && t.bn == 192) return launch<AM, B_TMA_K, EPI, 192, 3, 2>(p, splits, st);
    if (t.cg == 2 && t.bn == 128) return launch<AM, B_TMA_K, EPI, 128, 4, 2>(p, splits, st);
    PC_REQUIRE(false, PC_ESHAPE, "two-accumulator im2col: CTA pair with N in {128, 192, 256}");
  } else if constexpr (AM == A_HALO_K) {  // stages of (window + k B tiles)
    if (t.cg == 2 && t.bn == 256) return launch<AM, B_TMA_K, EPI, 256, 2, 2>(p, splits, st);  // 2 x 112 KB
    if (t.cg == 2 && t.bn == 192) return launch<AM, B_TMA_K, EPI, 192, 2, 2>(p, splits, st);
    PC_REQUIRE(t.bn <= 128, PC_ESHAPE, "halo A: tile width %d unsupported", t.bn);
    if (t.cg == 2) {
      if (t.bn <= 64) return launch<AM, B_TMA_K, EPI, 64, 4, 2>(p, splits, st);
      if (t.bn <= 96) return launch<AM, B_TMA_K, EPI, 96, 3, 2>(p, splits, st);
      return launch<AM, B_TMA_K, EPI, 128, 3, 2>(p, splits, st);
    }
    if (t.bn <= 64) return launch<AM, B_TMA_K, EPI, 64, 3, 1>(p, splits, st);
    if (t.bn <= 96) return launch<AM, B_TMA_K, EPI, 96, 2, 1>(p, splits, st);
    return launch<AM, B_TMA_K, EPI, 128, 2, 1>(p, splits, st);
  } else {
  if constexpr (!a_is_gather<AM>()) {
    if (t.cg == 2) {
      switch (t.bn) {
        case 64: return launch<AM, B_TMA_K, EPI, 64, fst<EPI, 64, 8, 2>(), 2>(p, splits, st);
        case 96: return launch<AM, B_TMA_K, EPI, 96, fst<EPI, 96, 8, 2>(), 2>(p, splits, st);
        case 128: return launch<AM, B_TMA_K, EPI, 128, fst<EPI, 128, 8, 2>(), 2>(p, splits, st);
        case 192: return launch<AM, B_TMA_K, EPI, 192, fst<EPI, 192, 7, 2>(), 2>(p, splits, st);
        default: return launch<AM, B_TMA_K, EPI, 256, fst<EPI, 256, 6, 2>(), 2>(p, splits, st);
      }
    }
  }
  switch (t.bn) {
    case 64: return launch<AM, B_TMA_K, EPI, 64, fst<EPI, 64, 8, 1>(), 1>(p, splits, st);
    case 96: return launch<AM, B_TMA_K, EPI, 96, fst<EPI, 96, 7, 1>(), 1>(p, splits, st);
    case 128: return launch<AM, B_TMA_K, EPI, 128, fst<EPI, 128, 6, 1>(), 1>(p, splits, st);
    case 192: return launch<AM, B_TMA_K, EPI, 192, fst<EPI, 192, 5, 1>(), 1>(p, splits, st);
    default: return launch<AM, B_TMA_K, EPI, 256, fst<EPI, 256, 4, 1>(), 1>(p, splits, st);
  }  }
}
template <int AM, int EPI>
static int launch_mn(const Params& p, Tile t, int splits, cudaStream_t st) {
  if constexpr (AM == A_GATHER_WGRAD) {
    if (t.cg == 2) {
      if (t.bn == 128) return launch<AM, B_TMA_MN, EPI, 128, 8, 2>(p, splits, st);
      return launch<AM, B_TMA_MN, EPI, 256, 6, 2>(p, splits, st);
    }
  }
  if constexpr (!a_is_gather<AM>()) {
    if (t.cg == 2) {
      if (t.bn == 128) return launch<AM, B_TMA_MN, EPI, 128, fst<EPI, 128, 8, 2, true>(), 2>(p, splits, st);
      if (t.bn == 192) return launch<AM, B_TMA_MN, EPI, 192, fst<EPI, 192, 6, 2, true>(), 2>(p, splits, st);
      return launch<AM, B_TMA_MN, EPI, 256, fst<EPI, 256, 6, 2, true>(), 2>(p, splits, st);
    }
  }
  switch (t.bn) {
    case 64: return launch<AM, B_TMA_MN, EPI, 64, fst<EPI, 64, 8, 1, true>(), 1>(p, splits, st);
    case 128: return launch<AM, B_TMA_MN, EPI, 128, fst<EPI, 128, 6, 1, true>(), 1>(p, splits, st);
    case 192: return launch<AM, B_TMA_MN, EPI, 192, fst<EPI, 192, 5, 1, true>(), 1>(p, splits, st);
    default: return launch<AM, B_TMA_MN, EPI, 256, fst<EPI, 256, 4, 1, true>(), 1>(p, splits, st);
  }
}

// MN-major B for tile t: prefer the chunked single-op view ({64 cols, BK rows,
// BN/CG/64 chunks} per CTA); fall back to one 3-D load per 64-column chunk.
static int setup_mn_b(Params& p, const void* ptr, long long cb, long long rows, long long blocks, long long ld,
                      long long bstride, Tile t) {
  const int bnc = t.bn / t.cg;
  p.b_chunked = bnc % 64 == 0 && (blocks == 1 || cb % bnc == 0) &&
                make_mn_chunked_map(&p.tma_b, ptr, cb, rows, blocks, ld, bstride, bnc / 64);
  if (p.b_chunked) return PC_OK;
  return make_map(&p.tma_b, ptr, cb, rows, blocks, ld, bstride, 64);
}

static Params base_params(int M, int N, int K) {
  Params p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.K = K;
  p.num_kb = ceil_div(K, BK);
  p.kb_per_split = p.num_kb;
  p.a_cb = p.b_cb = 0;
  p.o_cb = 1LL << 40;
  return p;
}

}  // namespace umma

using namespace umma;

void set_grid_cap(int ctas) { umma::t_grid_cap = ctas; }

bool umma_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0 && get_encode();
}

// TMA im2col needs 64-channel (128 B) pixel rows within one channel block.
static bool half_chunk_enabled() {  // PC_HALF_CHUNK=0: zero-filled 64-channel boxes instead
  static const int on = [] {
    const char* e = getenv("PC_HALF_CHUNK");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
static bool im2col_enabled() {
  static const int enabled = [] {
    const char* e = getenv("PC_IM2COL");
    return e ? atoi(e) : 1;
  }();
  return enabled != 0;
}
static bool im2col_ok(int cs, int C, long long cstride) {
  return im2col_enabled() && cs % 64 == 0 && C % cs == 0 && (C == cs || cstride % 8 == 0);
}

// K-major im2col (forward): also a single (unblocked) channel block of any
// multiple of 8 channels — the last 64-channel chunk is zero-filled by TMA.
static bool im2col_k_ok(int cs, int C, long long cstride) {
  return im2col_ok(cs, C, cstride) || (im2col_enabled() && C == cs && C % 8 == 0 && C >= 64);
}

static void set_i2c(Params& p, int C, int cs, int k, int s, int lo, int Wo, int Ho) {
  p.i2c_C = C;
  p.i2c_cs = cs;
  p.i2c_k = k;
  p.i2c_s = s;
  p.i2c_lw = p.i2c_lh = lo;
  p.i2c_Wo = Wo;
  p.i2c_Ho = Ho;
  p.i2c_cpt = (C + BK - 1) / BK;
}

// K-major im2col GEMM over k*k taps x ceil(C/64) channel chunks.
static void set_i2c_kloop(Params& p, int C, int k) {
  p.num_kb = k * k * ((C + BK - 1) / BK);
  p.kb_per_split = p.num_kb;
}

static bool conv_tc_shape(const pc_conv_geom& g) {
  return g.C % 8 == 0 && g.cs % 8 == 0 && g.N % 8 == 0 && (g.C == g.cs || g.cstride % 8 == 0);
}

// Halo (shifted-window) A operand for a stride-1 conv whose GEMM N is narrow
// (N <= 128: the im2col operand dominates the TMA traffic there). IN is the
// unblocked NHWC input [B][Hi][Wi][Ci]; output pixel (y, x) reads IN(y + i + lo,
// x + j + lo) for tap (i, j). Returns false when the geometry does not fit.
// Default: narrow N (<= 128) with >= 16 taps per channel (AlexNet conv2 data
// gradient: N = 96, 5x5). Few taps (3x3) leave the 128-row epilogue per tile
// exposed, where the im2col path is faster. PC_HALO=0 off, 2 = whenever it fits.
static bool halo_wanted(int N, int k) {
  static const int mode = [] {
    const char* e = getenv("PC_HALO");
    return e ? atoi(e) : 1;
  }();
  return mode == 2 || (mode == 1 && N <= 128 && k * k >= 16);
}
// hsub > 1 (A_HALO_KR2): a CTA tile is hsub vertically adjacent sub-tiles of R rows;
// the window box spans hsub * R + k - 1 rows and halo_tpi counts CTA tiles.
static bool setup_halo(Params& p, const void* in, int B, int Hi, int Wi, int Ci, int k, int lo, int Ho, int Wo,
                       int hsub = 1, int chans = 64) {
  const int Wv = (Wo + 7) / 8 * 8;
  if (Wv > 128 || Ci % 8 || Ci < 64 || (reinterpret_cast<uintptr_t>(in) & 15) || !get_encode()) return false;
  const int R = BM / Wv;
  if (BM + (k - 1) * Wv > HALO_SLOT_BYTES / 128 || R + k - 1 > 256 || k > HALO_KMAX) return false;
  if (hsub > 1 && (hsub * R + k - 1) * Wv * 128 > HALO_R2_SLOT_BYTES) return false;
  cuuint64_t dims[4] = {(cuuint64_t)Ci, (cuuint64_t)Wi, (cuuint64_t)Hi, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)Ci * 2, (cuuint64_t)Wi * Ci * 2, (cuuint64_t)Hi * Wi * Ci * 2};
  // chans = 48: the input layer's structural-zero channels 48..63 are not loaded (the
  // forward skips their k16 step; the rows keep the 128-byte swizzled pitch)
  cuuint32_t box[4] = {(cuuint32_t)chans, (cuuint32_t)Wv, (cuuint32_t)(hsub * R + k - 1), 1u};
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  if (g_encode(&p.tma_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(in), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  p.halo_R = R;
  p.halo_tpi = (Ho + hsub * R - 1) / (hsub * R);
  p.halo_Wv = Wv;
  p.halo_lo = lo;
  p.halo_bytes = chans * Wv * (hsub * R + k - 1) * 2;
  p.M = B * p.halo_tpi * BM * hsub;  // virtual rows: hsub 128-row sub-tiles per halo tile
  p.i2c_k = k;
  p.i2c_C = Ci;
  p.i2c_Ho = Ho;
  p.i2c_Wo = Wo;
  p.num_kb = k * ((Ci + BK - 1) / BK);  // k-blocks = (channel chunk, filter column)
  p.kb_per_split = p.num_kb;
  return true;
}

// Resident-B halo (A_HALO_KR): a CTA pair with N <= 96 whose filters fit in
// RES_B_BYTES per SM and whose windows fit a HALO_R_SLOT_BYTES slot — the
// space-to-depth input layer (9 taps x 64 channels x 96 filters). PC_HALO_RES=0 off.
static bool halo_res_fits(const Params& p, int N) {
  static const int on = [] {
    const char* e = getenv("PC_HALO_RES");
    return e ? atoi(e) : 1;
  }();
  if (!on || !cg2_enabled() || N != 96) return false;
  const long long res = (long long)p.num_kb * p.i2c_k * 48 * BK * 2;
  const long long pair_tiles = (p.M + 2 * BM - 1) / (2 * BM);
  return res <= RES_B_BYTES && (long long)(p.halo_R + p.i2c_k - 1) * p.halo_Wv * 128 <= HALO_R_SLOT_BYTES &&
         pair_tiles >= 74;
}

// Plain NHWC bf16 output [M][N] as a TMA store view {N, M}, box {64 channels, 32 rows},
// 128B swizzle (epilogue_bf16_tma); sets p.out_tma.
static int bf16_out_map(Params* p, void* y, int N, long long M) {
  PC_REQUIRE(get_encode(), PC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if (N % 8 || (reinterpret_cast<uintptr_t>(y) & 15)) return PC_OK;   // generic epilogue
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {64u, 32u}, estr[2] = {1u, 1u};
  PC_REQUIRE(g_encode(&p->tma_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS,
             PC_ECUDA, "bf16 output tensor map");
  p->out_tma = 1;
  return PC_OK;
}

// A_IM2COL_K2 (two accumulators per CTA) instead of A_IM2COL_K: the 512-row pair
// tiles cut the TMA rows per MMA cycle by a quarter — the per-tile trace shows the
// main loop MMA-bound at 1009 cycles per k-block (1024 ideal) where A_IM2COL_K needs
// 719 for half the work — and with the TMA-store epilogue (6k cycles per tile, not
// overlapped) conv2's forward runs 181 -> 159 us; but the tiles are twice as large,
// so they pay only where they still fill the pairs' waves: the share of busy pair
// slots, weighted by that gain, must beat the 256-row tiling's. Only with the TMA
// epilogue (plain NHWC output, no ReLU mask). PC_K2=0: never, 2: always.
static bool k2_wanted(long long M, int N, const Tile& t) {
  static const int mode = [] {
    const char* e = getenv("PC_K2");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || t.cg != 2 || (t.bn != 128 && t.bn != 192 && t.bn != 256)) return false;
  if (mode == 2) return true;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long pairs = sms / 2, nt = (N + t.bn - 1) / t.bn;
  const long long u1 = (M + 2 * BM - 1) / (2 * BM) * nt, u2 = (M + 4 * BM - 1) / (4 * BM) * nt;
  const double e1 = (double)u1 / (double)(((u1 + pairs - 1) / pairs) * pairs);
  const double e2 = (double)u2 / (double)(((u2 + pairs - 1) / pairs) * pairs);
  return e2 * 1.25 > e1;
}

int umma_conv_forward(const pc_conv_geom& g, const void* x, const void* w, const float* bias, void* y,
                      int flags, cudaStream_t st) {
  if (!conv_tc_shape(g)) {
    g_simt_launches++;
    return simt_conv_forward(g, x, w, bias, y, PC_BF16, flags, st);
  }
  int M = g.B * g.Ho * g.Wo, K = g.k * g.k * g.C;
  Params p = base_params(M, g.N, K);
  // N = 96 with 64-channel rows whose filters fit in shared memory (the space-to-depth
  // input layer): TMA im2col A + resident filters (A_IM2COL_KR), opt-in with
  // PC_I2C_KR=1; by default the resident-filter halo path below (fewer bytes per tile).
  static const int i2c_kr = [] {  // measured slower than the halo path (141 vs 122 us): opt-in
    const char* e = getenv("PC_I2C_KR");
    return e ? atoi(e) : 0;
  }();
  if (i2c_kr && g.N == 96 && g.C % BK == 0 && im2col_ok(g.cs, g.C, g.cstride) && cg2_enabled() &&
      (long long)g.k * g.k * (g.C / BK) * 48 * BK * 2 <= RES_B_BYTES && (M + 2 * BM - 1) / (2 * BM) >= 74) {
    const Tile t{96, 2};
    int rc = make_map(&p.tma_b, w, K, g.N, 1, K, 0, t.bn / t.cg);
    if (!rc) rc = make_im2col_map(&p.tma_a, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, BM, -g.pad, -g.pad,
                                  g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride);
    if (rc) return rc;
    p.b_cb = 0;
    p.gsrc = static_cast<const __nv_bfloat16*>(x);
    p.g = g;
    p.out = y;
    p.o_ld = g.N;
    p.bias = bias;
    p.relu = (flags & PC_RELU) != 0;
    set_i2c(p, g.C, g.cs, g.k, g.stride, -g.pad, g.Wo, g.Ho);
    set_i2c_kloop(p, g.C, g.k);
    return launch_kb<A_IM2COL_KR, EPI_BF16>(p, t, 1, st);
  }
  bool halo = g.stride == 1 && g.C == g.cs && halo_wanted(g.N, g.k) &&
             setup_halo(p, x, g.B, g.H, g.W, g.C, g.k, -g.pad, g.Ho, g.Wo);
  bool res = false, res2 = false;
  if (!halo && g.stride == 1 && g.C == g.cs && g.N <= 96) {
    static const int kr2 = [] {  // two sub-tiles per CTA (A_HALO_KR2); PC_KR2=0: one
      const char* e = getenv("PC_KR2");
      return e ? atoi(e) : 1;
    }();
    Params q = p;
    static const int h48 = [] {  // PC_HALO48=0: load all 64 channels of the input-layer windows
      const char* e = getenv("PC_HALO48");
      return e ? atoi(e) : 1;
    }();
    const int wch = h48 && (flags & PC_ZERO_TAIL16) && g.C == BK ? 48 : 64;
    if (kr2 && setup_halo(q, x, g.B, g.H, g.W, g.C, g.k, -g.pad, g.Ho, g.Wo, 2, wch) && halo_res_fits(q, g.N)) {
      p = q;
      halo = res = res2 = true;
    } else if (setup_halo(q, x, g.B, g.H, g.W, g.C, g.k, -g.pad, g.Ho, g.Wo) && halo_res_fits(q, g.N)) {
      p = q;
      halo = res = true;
    }
  }
  const bool i2c = !halo && im2col_k_ok(g.cs, g.C, g.cstride);
  const Tile t = res ? Tile{96, 2} : pick_k(p.M, g.N, i2c || halo);
  int rc = make_map(&p.tma_b, w, K, g.N, 1, K, 0, t.bn / t.cg);
  if (rc) return rc;
  p.b_cb = 0;
  p.gsrc = static_cast<const __nv_bfloat16*>(x);
  p.g = g;
  p.out = y;
  p.o_ld = g.N;
  p.bias = bias;
  p.relu = (flags & PC_RELU) != 0;
  p.zero_tail16 = (flags & PC_ZERO_TAIL16) && halo && g.C % BK == 0 && g.C == BK;
  if (res) {
    // output view {N, Wo, B*Ho}, box {N/2, 8 rows, 1} (epilogue_bf16_halo_tma)
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.Wo, (cuuint64_t)g.B * g.Ho};
    cuuint64_t strides[2] = {(cuuint64_t)g.N * 2, (cuuint64_t)g.Wo * g.N * 2};
    cuuint32_t box[3] = {(cuuint32_t)(t.bn / 2), 8u, 1u}, estr[3] = {1u, 1u, 1u};
    PC_REQUIRE(g.N == t.bn && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                   g_encode(&p.tma_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS,
               PC_ECUDA, "resident-B halo: output tensor map");
    p.out_tma = 1;
    return res2 ? launch_kb<A_HALO_KR2, EPI_BF16>(p, t, 1, st) : launch_kb<A_HALO_KR, EPI_BF16>(p, t, 1, st);
  }
  if (halo) return launch_kb<A_HALO_K, EPI_BF16>(p, t, 1, st);
  if (i2c) {
    rc = make_im2col_map(&p.tma_a, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, BM, -g.pad, -g.pad,
                         g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride);
    if (rc) return rc;
    set_i2c(p, g.C, g.cs, g.k, g.stride, -g.pad, g.Wo, g.Ho);
    set_i2c_kloop(p, g.C, g.k);
    if (g.C == g.cs && g.C % BK != 0 && g.C % BK <= 32 && half_chunk_enabled()) {
      rc = make_im2col_map(&p.tma_a32, x, g.cs, g.W, g.H, g.B, 1, g.cstride, BM, -g.pad, -g.pad,
                           g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride, 32);
      if (!rc) rc = make_map(&p.tma_b32, w, K, g.N, 1, K, 0, t.bn / t.cg, 32);
      if (rc) return rc;
      p.half_chunk = 1;
    }
    if (g.N % 64 == 0 && k2_wanted(g.B * g.Ho * g.Wo, g.N, t)) {
      rc = bf16_out_map(&p, y, g.N, (long long)g.B * g.Ho * g.Wo);
      if (rc) return rc;
      if (p.out_tma) return launch_kb<A_IM2COL_K2, EPI_BF16>(p, t, 1, st);
    }
    return launch_kb<A_IM2COL_K, EPI_BF16>(p, t, 1, st);
  }
  return launch_kb<A_GATHER_FWD, EPI_BF16>(p, t, 1, st);
}

// wt[c][ij][n] = w[n][ij'][c], ij' = flip ? KK-1-ij : ij (180-degree filter
// rotation). Per tap a 2-D transpose of [N][C] (row stride KK*C) into [C][N]
// (row stride KK*N) through a 32x32 SMEM tile: coalesced on both sides.
__global__ void __launch_bounds__(256) transpose_w_k(const __nv_bfloat16* __restrict__ w,
                                                     __nv_bfloat16* __restrict__ wt, int N, int KK, int C,
                                                     int flip) {
  PC_PDL_TRIGGER();
  __shared__ __nv_bfloat16 tile[32][33];
  const int ij = blockIdx.z, src_ij = flip ? KK - 1 - ij : ij;
  const int c0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows per pass
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int n = n0 + r, c = c0 + tx;
    if (n < N && c < C) tile[r][tx] = w[((long long)n * KK + src_ij) * C + c];
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int c = c0 + r, n = n0 + tx;
    if (n < N && c < C) wt[((long long)c * KK + ij) * N + n] = tile[tx][r];
  }
}

static void transpose_w(const void* w, __nv_bfloat16* wt, int N, int KK, int C, int flip, cudaStream_t st) {
  const dim3 grid((C + 31) / 32, (N + 31) / 32, KK);
  transpose_w_k<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w), wt, N, KK, C, flip);
}

size_t umma_conv_extra_ws(const pc_conv_geom& g, int prec) {
  return prec == PC_BF16 ? (size_t)g.N * g.k * g.k * g.C * 2 + 256 : 0;
}

// The data gradient reads its filters as wt[c][ij][n] (N contiguous), rotated by
// 180 degrees (flip) when it runs as a forward conv of gy (TMA im2col or halo
// paths). dgrad_flip() is that choice, made from the geometry alone, so the
// caller can prepare wt ahead of time (pc_conv2d_dgrad_weights).
static bool halo_geom_ok(int Ci, int k, int Wo) {
  const int Wv = (Wo + 7) / 8 * 8;
  if (Wv > 128 || Ci % 8 || Ci < 64 || k > HALO_KMAX) return false;
  const int R = BM / Wv;
  return BM + (k - 1) * Wv <= HALO_SLOT_BYTES / 128 && R + k - 1 <= 256;
}
static int dgrad_flip(const pc_conv_geom& g) {
  const bool rot = g.stride == 1 && g.H + 2 * g.pad - g.k + 1 == g.Ho;  // dgrad = conv of gy with the rotated filter
  const bool i2c = rot && im2col_ok(g.N, g.N, 0);
  const bool halo = rot && halo_wanted(g.C, g.k) && halo_geom_ok(g.N, g.k, g.W);
  return (i2c || halo) ? 1 : 0;
}

int umma_conv_dgrad_weights(const pc_conv_geom& g, const void* w, void* wt, cudaStream_t st) {
  transpose_w(w, static_cast<__nv_bfloat16*>(wt), g.N, g.k * g.k, g.C, dgrad_flip(g), st);
  PC_CUDA_CHECK_LAUNCH("transpose_w");
  return PC_OK;
}

int umma_conv_dgrad(const pc_conv_geom& g, const void* w, const void* gy, void* gx, const void* mask,
                    cudaStream_t st, void* ws, size_t ws_bytes, bool w_preset) {
  if (!conv_tc_shape(g)) {
    PC_REQUIRE(!w_preset, PC_EVALUE, "conv dgrad: prepared weights need the tensor-core path");
    g_simt_launches++;
    return simt_conv_dgrad(g, w, gy, gx, mask, st, PC_BF16);
  }
  const int KK = g.k * g.k;
  size_t need = (size_t)g.N * KK * g.C * 2;
  const int flip = dgrad_flip(g);
  const bool rot = g.stride == 1 && g.H + 2 * g.pad - g.k + 1 == g.Ho;
  const bool i2c = rot && im2col_ok(g.N, g.N, 0);
  const bool halo_ok = rot && halo_wanted(g.C, g.k);
  int M = g.B * g.H * g.W, K = KK * g.N;
  Params p = base_params(M, g.C, K);
  const bool halo = halo_ok && setup_halo(p, gy, g.B, g.Ho, g.Wo, g.N, g.k, g.pad - (g.k - 1), g.H, g.W);
  PC_REQUIRE(!w_preset || (i2c || halo) == (flip != 0), PC_EVALUE,
             "conv dgrad: prepared weights do not match the data-gradient path");
  const void* wt = w;
  if (!w_preset) {
    PC_REQUIRE(ws != nullptr && ws_bytes >= need, PC_EVALUE, "conv dgrad: workspace too small");
    // the transposed weights live at the END of the workspace (wgrad partials use the front)
    __nv_bfloat16* wt_ws = reinterpret_cast<__nv_bfloat16*>(
        (reinterpret_cast<uintptr_t>(ws) + ws_bytes - need) & ~uintptr_t(127));
    transpose_w(w, wt_ws, g.N, KK, g.C, (i2c || halo) ? 1 : 0, st);
    PC_CUDA_CHECK_LAUNCH("transpose_w");
    wt = wt_ws;
  }
  const Tile t = pick_k(p.M, g.C, i2c || halo);
  int rc = make_map(&p.tma_b, wt, K, g.C, 1, K, 0, t.bn / t.cg);
  if (rc) return rc;
  p.b_cb = 0;
  p.gsrc = static_cast<const __nv_bfloat16*>(gy);
  p.g = g;
  p.out = gx;
  p.o_ld = g.cs;
  p.o_cb = g.cs;
  p.o_bstride = g.cstride;
  p.mask = static_cast<const __nv_bfloat16*>(mask);
  if (halo) return launch_kb<A_HALO_K, EPI_BF16>(p, t, 1, st);
  if (i2c) {
    // dgrad = forward conv of gy with the rotated filter, corner p-(k-1), walking dx's H x W
    const int lo = g.pad - (g.k - 1);
    rc = make_im2col_map(&p.tma_a, gy, g.N, g.Wo, g.Ho, g.B, 1, 0, BM, lo, lo, lo + g.W - g.Wo,
                         lo + g.H - g.Ho, 1);
    if (rc) return rc;
    set_i2c(p, g.N, g.N, g.k, 1, lo, g.W, g.H);
    set_i2c_kloop(p, g.N, g.k);
    if (!mask && g.cs == g.C && g.C % 64 == 0 && k2_wanted(M, g.C, t)) {
      rc = bf16_out_map(&p, gx, g.C, M);
      if (rc) return rc;
      if (p.out_tma) return launch_kb<A_IM2COL_K2, EPI_BF16>(p, t, 1, st);
    }
    return launch_kb<A_IM2COL_K, EPI_BF16>(p, t, 1, st);
  }
  return launch_kb<A_GATHER_DGRAD, EPI_BF16>(p, t, 1, st);
}

// Split-K count for a long reduction: the persistent grid runs ceil(units/148)
// waves of ceil(kbs/s) k-blocks each (plus ~4 k-blocks of per-unit fill/drain),
// and every extra slice costs a partial tile write + read in the reduction.
// Pick the s with the smallest modelled time (wave quantisation matters:
// 297 units on 148 SMs is three waves, 296 is two).
static long long choose_splits(long long tiles, long long kbs, int bn, int cg = 1) {
  long long best = 1;
  double best_cost = 1e30;
  const int cap = 148 / cg;                                  // concurrent units (SMs or SM pairs)
  const double tile_bytes = (double)BM * cg * bn * 4 * 2;    // partial write + reduce read
  const double kb_bytes = (double)(BM * cg + bn) * BK * 2;   // operand bytes per k-block
  for (long long sp = 1; sp <= 64; ++sp) {
    if (sp > 1 && kbs / sp < 8) break;
    const long long units = tiles * sp, kb_per = (kbs + sp - 1) / sp;
    const long long waves = (units + cap - 1) / cap;
    double cost = (double)waves * (kb_per + 4);
    if (sp > 1) cost += (double)units * tile_bytes / (cap * kb_bytes);
    if (cost < best_cost * 0.999) best_cost = cost, best = sp;
  }
  return best;
}

// Weight gradient tiling: M = kh*kw*C, N = Cout, K = pixels (long) -> split-K.
// The CTA pair applies when the A operand comes by TMA im2col.
struct WgradPlan {
  Tile t;
  int splits;
  bool mn2;  // A_IM2COL_MN2: two M accumulators per CTA of the pair
  bool g32;  // ... over 32-channel groups (A_IM2COL_MN2_32)
};
// 32-channel MN-major groups: unblocked input whose channel count is a multiple of
// 32 but not of 64 (the 64-channel chunks would carry zero padding). PC_GRP32=0 off.
static bool grp32_ok(const pc_conv_geom& g) {
  static const int on = [] {
    const char* e = getenv("PC_GRP32");
    return e ? atoi(e) : 1;
  }();
  return on && g.C == g.cs && g.C % 64 != 0 && g.C % 32 == 0 && g.C >= 32;
}
static bool mn2_enabled() {
  static const int on = [] {
    const char* e = getenv("PC_MN2");
    return e ? atoi(e) : 1;
  }();
  return on != 0;
}
// Weight gradient of an unblocked input whose channel count is not a multiple
// of 64 (conv2: 96) by TMA im2col with zero-filled padding channels: a third more
// MMA rows than the cp.async gather, but the operand arrives at TMA rate.
static bool wgrad_pad_ok(const pc_conv_geom& g) {
  static const int on = [] {
    const char* e = getenv("PC_WGRAD_PAD");
    return e ? atoi(e) : 1;
  }();
  return on && im2col_enabled() && g.C == g.cs && g.C % 64 != 0 && g.C % 8 == 0 && g.C >= 64;
}

static WgradPlan wgrad_plan(const pc_conv_geom& g) {
  const bool padded = wgrad_pad_ok(g);
  const long long Kc0 = (long long)g.k * g.k * (padded ? (g.C + 63) / 64 * 64 : g.C), P = (long long)g.B * g.Ho * g.Wo;
  const bool i2c = im2col_ok(g.cs, g.C, g.cstride) || padded;
  static const int gather_cg2 = [] {
    const char* e = getenv("PC_GATHER_CG2");
    return e ? atoi(e) : 1;
  }();
  const bool pair = cg2_enabled() && (i2c || (gather_cg2 && g.N % 128 == 0));
  // N = 384 (conv3 / conv4 filters): two 192-wide pair tiles instead of 256 + 128
  const int pbn = g.N <= 128 ? 128 : (i2c && g.N % 192 == 0 && g.N % 256 != 0 && mn192_enabled()) ? 192 : 256;
  const Tile t = pair ? Tile{pbn, 2} : Tile{bn_for_mn(g.N), 1};
  // N = 256 on TMA im2col (conv2, conv5): 512-row pair tiles, two accumulators per CTA
  const bool mn2 = pair && i2c && (g.N == 256 || (g.N % 192 == 0 && g.N % 256 != 0)) && mn2_enabled();
  const long long rows = BM * t.cg * (mn2 ? 2 : 1);
  const bool g32 = mn2 && grp32_ok(g);
  const long long Kc = g32 ? (long long)g.k * g.k * g.C : Kc0;
  const long long tiles = ((Kc + rows - 1) / rows) * ((g.N + t.bn - 1) / t.bn);
  const long long kbs = (P + BK - 1) / BK;
  long long sp = choose_splits(tiles, kbs, t.bn * (mn2 ? 2 : 1), t.cg);
  const long long per = (kbs + sp - 1) / sp;
  return {t, (int)((kbs + per - 1) / per), mn2, g32};
}

static bool macc_wgrad_ok(const pc_conv_geom& g);
static int macc_splits(const pc_conv_geom& g);
long long umma_wgrad_splits(const pc_conv_geom& g) {
  return macc_wgrad_ok(g) ? macc_splits(g) : wgrad_plan(g).splits;
}

// Multi-accumulator weight gradient (A_IM2COL_MN5): M = k*k*C in (256, 640], N <= 128.
static bool macc_wgrad_ok(const pc_conv_geom& g) {
  static const int on = [] {
    const char* e = getenv("PC_MACC");
    return e ? atoi(e) : 1;
  }();
  const int Kc = g.k * g.k * g.C;
  // one TMEM accumulator of N fp32 columns per 128 rows of M: all of them within 512 columns
  return on && Kc > 2 * BM && Kc <= 5 * BM && g.N <= 128 && g.N % 16 == 0 &&
         (long long)((Kc + BM - 1) / BM) * g.N <= 512 && im2col_ok(g.cs, g.C, g.cstride);
}
// The pair variant (A_IM2COL_MN3P): M <= 768 rows in three accumulators per CTA,
// N <= 96 (3 x N <= 512 TMEM columns; the pair splits B in 64-column halves).
static bool macc_pair_ok(const pc_conv_geom& g) {
  static const int on = [] {
    const char* e = getenv("PC_MACC_PAIR");
    return e ? atoi(e) : 1;
  }();
  return on && cg2_enabled() && g.k * g.k * g.C <= 6 * BM && g.N <= 96 && g.N % 16 == 0;
}
static int macc_splits(const pc_conv_geom& g) {
  const long long kbs = ((long long)g.B * g.Ho * g.Wo + BK - 1) / BK;
  const int units = macc_pair_ok(g) ? 74 : 148;  // CTA pairs or CTAs
  long long sp = std::min<long long>(units, std::max<long long>(1, kbs / 16));
  const long long per = (kbs + sp - 1) / sp;
  return (int)((kbs + per - 1) / per);
}

int umma_conv_wgrad(const pc_conv_geom& g, const void* x, const void* gy, float* gw, float* part,
                    cudaStream_t st, const pc_sgd_fuse* upd) {
  if (!conv_tc_shape(g)) {
    g_simt_launches++;
    long long P = (long long)g.B * g.Ho * g.Wo;
    int rc = simt_conv_wgrad(g, x, gy, gw, part, simt_splits(g.N, g.k * g.k * g.C, P), st, PC_BF16);
    return rc || !upd ? rc : apply_sgd(gw, (long long)g.N * g.k * g.k * g.C, upd, st);
  }
  int Kc = g.k * g.k * g.C;
  long long P = (long long)g.B * g.Ho * g.Wo;
  Params p = base_params(Kc, g.N, (int)P);
  if (macc_wgrad_ok(g)) {
    int splits = macc_splits(g);
    p.kb_per_split = ceil_div(p.num_kb, splits);
    splits = ceil_div(p.num_kb, p.kb_per_split);
    const bool macc_pair = macc_pair_ok(g);
    // pair: each CTA holds N/2 = 48 of the B columns (one 64-column MN chunk loaded)
    const Tile t = macc_pair ? Tile{96, 2} : Tile{128, 1};
    int rc = setup_mn_b(p, gy, g.N, P, 1, g.N, 0, t);
    if (rc) return rc;
    p.b_cb = 0;
    p.gsrc = static_cast<const __nv_bfloat16*>(x);
    p.g = g;
    p.o_ld = Kc;
    rc = make_im2col_map(&p.tma_a, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, 64, -g.pad, -g.pad,
                         g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride);
    if (rc) return rc;
    set_i2c(p, g.C, g.cs, g.k, g.stride, -g.pad, g.Wo, g.Ho);
    p.macc_chunks = (Kc + 63) / 64;
    p.out = splits > 1 ? static_cast<void*>(part) : static_cast<void*>(gw);
    p.split_stride = splits > 1 ? (long long)g.N * Kc : 0;
    if (macc_pair) {
      p.macc_chunks = (Kc + 63) / 64;  // real 64-row chunks over the whole pair tile
      rc = launch<A_IM2COL_MN3P, B_TMA_MN, EPI_F32_T, 96, 4, 2>(p, splits, st);
    } else {
      rc = launch<A_IM2COL_MN5, B_TMA_MN, EPI_F32_T, 128, 2, 1>(p, splits, st);
    }
    if (rc) return rc;
    if (splits == 1) return upd ? apply_sgd(gw, (long long)g.N * Kc, upd, st) : PC_OK;
    return reduce_partials(part, splits, (long long)g.N * Kc, gw, st, upd);
  }
  const WgradPlan wp = wgrad_plan(g);
  int splits = wp.splits;
  p.kb_per_split = ceil_div(p.num_kb, splits);
  splits = ceil_div(p.num_kb, p.kb_per_split);
  int rc = setup_mn_b(p, gy, g.N, P, 1, g.N, 0, wp.t);
  if (rc) return rc;
  p.b_cb = 0;
  p.gsrc = static_cast<const __nv_bfloat16*>(x);
  p.g = g;
  p.o_ld = Kc;
  const bool padded = wgrad_pad_ok(g);
  const bool i2c = im2col_ok(g.cs, g.C, g.cstride) || padded;
  if (padded) {
    p.m_cp = (g.C + 63) / 64 * 64;
    p.M = g.k * g.k * p.m_cp;
  }
  if (i2c) {
    rc = make_im2col_map(&p.tma_a, x, g.cs, g.W, g.H, g.B, g.C / g.cs, g.cstride, 64, -g.pad, -g.pad,
                         g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride);
    if (rc) return rc;
    set_i2c(p, g.C, g.cs, g.k, g.stride, -g.pad, g.Wo, g.Ho);
  }
  p.out = splits > 1 ? static_cast<void*>(part) : static_cast<void*>(gw);
  p.split_stride = splits > 1 ? (long long)g.N * Kc : 0;

  if (wp.g32) {
    p.m_cp = 0;
    p.M = Kc;
    p.m_grp = g.C / 32;
    rc = make_im2col_map(&p.tma_a32, x, g.cs, g.W, g.H, g.B, 1, g.cstride, 64, -g.pad, -g.pad,
                         g.pad - (g.k - 1), g.pad - (g.k - 1), g.stride, 32);
    if (rc) return rc;
    set_i2c(p, g.C, g.cs, g.k, g.stride, -g.pad, g.Wo, g.Ho);
    p.macc_chunks = 4;
    rc = launch<A_IM2COL_MN2_32, B_TMA_MN, EPI_F32_T, 256, 4, 2>(p, splits, st);
  } else if (wp.mn2) {
    p.macc_chunks = 4;  // every chunk row exists or is clamped (rows past M are discarded)
    rc = wp.t.bn == 192 ? launch<A_IM2COL_MN2, B_TMA_MN, EPI_F32_T, 192, 4, 2>(p, splits, st)
                        : launch<A_IM2COL_MN2, B_TMA_MN, EPI_F32_T, 256, 4, 2>(p, splits, st);
  } else {
    rc = i2c ? launch_mn<A_IM2COL_MN, EPI_F32_T>(p, wp.t, splits, st)
             : launch_mn<A_GATHER_WGRAD, EPI_F32_T>(p, wp.t, splits, st);
  }
  if (rc) return rc;
  if (splits == 1) return upd ? apply_sgd(gw, (long long)g.N * Kc, upd, st) : PC_OK;
  return reduce_partials(part, splits, (long long)g.N * Kc, gw, st, upd);
}

static bool tma_view_ok(const pc_mat& v, long long inner_total) {
  bool blocked = v.cb < inner_total;
  return v.ld % 8 == 0 && (reinterpret_cast<uintptr_t>(v.ptr) & 15) == 0 &&
         (!blocked || (v.cb % 64 == 0 && v.bstride % 8 == 0));
}

// Small-M FC GEMMs (M = batch): the weights must stream through the SMs once,
// so the K loop is split over enough CTA pairs to fill the machine and the fp32
// partials are summed (in slice order: deterministic) by a fused epilogue kernel
// (bias, ReLU, producer mask, bf16 store). Large-M calls keep the direct epilogue.
struct FcPlan {
  Tile t;
  int splits;
};
static FcPlan fc_split_plan(int M, int N, int K) {
  const int cg = (M > BM && cg2_enabled()) ? 2 : 1;
  const Tile t{256, cg};
  const long long tiles = (long long)((M + BM * cg - 1) / (BM * cg)) * ((N + t.bn - 1) / t.bn);
  const int cap = 148 / cg, kbs = (K + BK - 1) / BK;
  if (tiles * 2 > cap || kbs < 8) return {t, 1};
  int sp = (int)std::min<long long>(cap / tiles, kbs / 4);
  static const int sp_cap = [] {  // tuning knob: PC_FC_SPLIT_CAP
    const char* e = getenv("PC_FC_SPLIT_CAP");
    return e ? atoi(e) : 0;
  }();
  if (sp_cap > 0) sp = std::min(sp, sp_cap);
  if (sp < 2) return {t, 1};
  const int per = (kbs + sp - 1) / sp;
  return {t, (kbs + per - 1) / per};
}

__global__ void fc_reduce_epilogue_k(const float* __restrict__ part, int splits, int M, int N,
                                     const float* __restrict__ bias, int relu, const __nv_bfloat16* __restrict__ mask,
                                     __nv_bfloat16* __restrict__ out, long long o_ld, long long o_cb,
                                     long long o_bstride) {
  // launched programmatically dependent on the split-K GEMM (which leaves SMs idle:
  // 64 of 74 pairs for fc6): CTAs placed early wait here for the GEMM's partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  PC_PDL_TRIGGER();
  const int groups = N / 8;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)M * groups) return;
  const int m = (int)(t / groups), n0 = (int)(t - (long long)m * groups) * 8;
  const size_t stride = (size_t)M * N;
  const float* src = part + (size_t)m * N + n0;
  float4 a = __ldg(reinterpret_cast<const float4*>(src)), b = __ldg(reinterpret_cast<const float4*>(src) + 1);
#pragma unroll 4
  for (int z = 1; z < splits; ++z) {  // unrolled: the slices' loads are in flight together
    const float4 c = __ldg(reinterpret_cast<const float4*>(src + z * stride));
    const float4 d = __ldg(reinterpret_cast<const float4*>(src + z * stride) + 1);
    a.x += c.x; a.y += c.y; a.z += c.z; a.w += c.w;
    b.x += d.x; b.y += d.y; b.z += d.z; b.w += d.w;
  }
  float o[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (bias) o[q] += __ldg(bias + n0 + q);
    if (relu) o[q] = o[q] > 0.f ? o[q] : 0.f;
  }
  const long long blk = n0 / o_cb;
  const long long idx = blk * o_bstride + (long long)m * o_ld + (n0 - blk * o_cb);
  if (mask) {
    const uint4 mk = *reinterpret_cast<const uint4*>(mask + idx);
    const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mk);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = __bfloat162float(mb[q]) > 0.f ? o[q] : 0.f;
  }
  uint4 u;
  __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) hh[q] = __floats2bfloat162_rn(o[2 * q], o[2 * q + 1]);
  *reinterpret_cast<uint4*>(out + idx) = u;
}

// PC_FC_REDUCE_PDL=1: launch the split-K reduction programmatically dependent on its
// GEMM (measured +12-16 us per step on AlexNet b256: its waiting CTAs take SMs the
// side stream's weight gradients would use), so off by default
static bool fc_reduce_pdl() {
  static const int on = [] {
    const char* e = getenv("PC_FC_REDUCE_PDL");
    return e ? atoi(e) : 0;
  }();
  return on != 0 && pdl_enabled();
}

static int fc_reduce_epilogue(const float* part, int splits, int M, int N, const float* bias, int relu,
                              const void* mask, void* out, long long o_ld, long long o_cb, long long o_bstride,
                              cudaStream_t st) {
  const long long work = (long long)M * (N / 8);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)((work + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = fc_reduce_pdl() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fc_reduce_epilogue_k, part, splits, M, N, bias, relu,
                                     static_cast<const __nv_bfloat16*>(mask), static_cast<__nv_bfloat16*>(out), o_ld,
                                     o_cb, o_bstride);
  PC_REQUIRE(e == cudaSuccess, PC_ECUDA, "fc_reduce_epilogue launch: %s", cudaGetErrorString(e));
  PC_CUDA_CHECK_LAUNCH("fc_reduce_epilogue");
  return PC_OK;
}

static size_t fc_split_bytes(int M, int N, int K) {
  const FcPlan fp = fc_split_plan(M, N, K);
  return fp.splits > 1 && N % 8 == 0 ? (size_t)fp.splits * M * N * sizeof(float) : 0;
}
size_t umma_fc_forward_ws(int B, int D, int U) { return fc_split_bytes(B, U, D); }

int umma_fc_forward(int B, int D, int U, const pc_mat& x, const void* w, const float* bias, void* y, int flags,
                    cudaStream_t st, void* ws, size_t ws_bytes) {
  if (!(tma_view_ok(x, D) && D % 8 == 0 && U % 8 == 0)) {
    g_simt_launches++;
    return simt_fc_forward(B, D, U, x, w, bias, y, PC_BF16, flags, st);
  }
  Params p = base_params(B, U, D);
  long long cb = x.cb < D ? x.cb : D;
  int rc = make_map(&p.tma_a, x.ptr, cb, B, D / cb, x.ld, x.bstride, BM);
  if (rc) return rc;
  p.a_cb = cb < D ? (int)cb : 0;
  const size_t need = fc_split_bytes(B, U, D);
  if (need && ws && ws_bytes >= need) {
    const FcPlan fp = fc_split_plan(B, U, D);
    if ((rc = make_map(&p.tma_b, w, D, U, 1, D, 0, fp.t.bn / fp.t.cg))) return rc;
    p.b_cb = 0;
    p.kb_per_split = ceil_div(p.num_kb, fp.splits);
    p.out = ws;
    p.o_ld = U;
    p.split_stride = (long long)B * U;
    if ((rc = launch_kb<A_TMA_K, EPI_F32>(p, fp.t, fp.splits, st))) return rc;
    return fc_reduce_epilogue(static_cast<const float*>(ws), fp.splits, B, U, bias, (flags & PC_RELU) != 0, nullptr,
                              y, U, 1LL << 40, 0, st);
  }
  const Tile t = pick_k(B, U, true);
  if ((rc = make_map(&p.tma_b, w, D, U, 1, D, 0, t.bn / t.cg))) return rc;
  p.b_cb = 0;
  p.out = y;
  p.o_ld = U;
  p.bias = bias;
  p.relu = (flags & PC_RELU) != 0;
  return launch_kb<A_TMA_K, EPI_BF16>(p, t, 1, st);
}

size_t umma_fc_dgrad_ws(int B, int D, int U) { return fc_split_bytes(B, D, U); }

int umma_fc_dgrad(int B, int D, int U, const void* w, const void* gy, const pc_mat& gx, const void* mask,
                  cudaStream_t st, void* ws, size_t ws_bytes) {
  if (!(D % 8 == 0 && U % 8 == 0 && gx.ld % 8 == 0 && (gx.cb >= D || gx.cb % 8 == 0))) {
    g_simt_launches++;
    return simt_fc_dgrad(B, D, U, w, gy, gx, mask, st, PC_BF16);
  }
  Params p = base_params(B, D, U);
  int rc = make_map(&p.tma_a, gy, U, B, 1, U, 0, BM);
  if (rc) return rc;
  p.a_cb = 0;
  const size_t need = fc_split_bytes(B, D, U);
  if (need && ws && ws_bytes >= need) {
    const FcPlan fp = fc_split_plan(B, D, U);
    if ((rc = setup_mn_b(p, w, D, U, 1, D, 0, fp.t))) return rc;
    p.b_cb = 0;
    p.kb_per_split = ceil_div(p.num_kb, fp.splits);
    p.out = ws;
    p.o_ld = D;
    p.split_stride = (long long)B * D;
    if ((rc = launch_mn<A_TMA_K, EPI_F32>(p, fp.t, fp.splits, st))) return rc;
    return fc_reduce_epilogue(static_cast<const float*>(ws), fp.splits, B, D, nullptr, 0, mask, gx.ptr, gx.ld,
                              gx.cb, gx.bstride, st);
  }
  const Tile t = pick_mn(B, D, true);
  if ((rc = setup_mn_b(p, w, D, U, 1, D, 0, t))) return rc;
  p.b_cb = 0;
  p.out = gx.ptr;
  p.o_ld = gx.ld;
  p.o_cb = gx.cb;
  p.o_bstride = gx.bstride;
  p.mask = static_cast<const __nv_bfloat16*>(mask);
  return launch_mn<A_TMA_K, EPI_BF16>(p, t, 1, st);
}

// EPI_SGD views of the parameters {D, U}: fp32 p and v (128B-swizzled 32x32
// boxes) and the bf16 shadow (64B-swizzled). false: not expressible (or
// PC_SGD_EPI=0) -> gradient store + separate update pass.
static bool sgd_epilogue_maps(Params& p, const pc_sgd_fuse* u, int U, int D) {
  static const int on = [] {
    const char* e = getenv("PC_SGD_EPI");
    return e ? atoi(e) : 1;
  }();
  if (!on || !get_encode() || !u->p || !u->v || !u->p_lowp || D % 8 ||
      ((reinterpret_cast<uintptr_t>(u->p) | reinterpret_cast<uintptr_t>(u->v) |
        reinterpret_cast<uintptr_t>(u->p_lowp)) & 15))
    return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)U, 1};
  cuuint64_t s32[2] = {(cuuint64_t)D * 4, (cuuint64_t)D * U * 4}, s16[2] = {(cuuint64_t)D * 2, (cuuint64_t)D * U * 2};
  cuuint32_t box[3] = {32u, 32u, 1u}, estr[3] = {1u, 1u, 1u};
  auto enc = [&](CUtensorMap* m, void* ptr, CUtensorMapDataType dt, cuuint64_t* str, CUtensorMapSwizzle sw) {
    return g_encode(m, dt, 3, ptr, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!enc(&p.tma_p, u->p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, s32, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !enc(&p.tma_v, u->v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, s32, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !enc(&p.tma_pl, u->p_lowp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, s16, CU_TENSOR_MAP_SWIZZLE_64B))
    return false;
  p.lr = u->lr;
  p.mom = u->momentum;
  p.wd = u->weight_decay;
  return true;
}

// Split-K for the weight gradient when the reduction (the batch, or the pixel
// count of an explicit-im2col convolution) is long and the output tiles few.
static int fc_wgrad_splits(int B, int D, int U) {
  const int bn = bn_for_mn(D);
  long long tiles = (long long)ceil_div(U, BM) * ceil_div(D, bn);
  return (int)choose_splits(tiles, (B + BK - 1) / BK, bn);
}

int umma_fc_wgrad(int B, int D, int U, const pc_mat& x, const void* gy, float* gw, float* part, cudaStream_t st,
                  const pc_sgd_fuse* upd) {
  if (!(tma_view_ok(x, D) && D % 8 == 0 && U % 8 == 0)) {
    g_simt_launches++;
    int rc = simt_fc_wgrad(B, D, U, x, gy, gw, st, PC_BF16);
    return rc || !upd ? rc : apply_sgd(gw, (long long)U * D, upd, st);
  }
  Params p = base_params(U, D, B);
  int rc = make_map(&p.tma_a, gy, U, B, 1, U, 0, 64);
  if (rc) return rc;
  p.a_cb = 0;
  long long cb = x.cb < D ? x.cb : D;
  int splits = fc_wgrad_splits(B, D, U);
  const Tile t{bn_for_mn(D, splits > 1 ? 1 << 30 : U), 1};
  if ((rc = setup_mn_b(p, x.ptr, cb, B, D / cb, x.ld, x.bstride, t))) return rc;
  p.b_cb = cb < D ? (int)cb : 0;
  p.o_ld = D;
  p.kb_per_split = ceil_div(p.num_kb, splits);
  splits = ceil_div(p.num_kb, p.kb_per_split);
  if (splits == 1 || part == nullptr) {
    p.kb_per_split = p.num_kb;
    if (upd && sgd_epilogue_maps(p, upd, U, D)) return launch_mn<A_TMA_MN, EPI_SGD>(p, t, 1, st);
    p.out = gw;
    rc = launch_mn<A_TMA_MN, EPI_F32>(p, t, 1, st);
    return rc || !upd ? rc : apply_sgd(gw, (long long)U * D, upd, st);
  }
  p.out = part;
  p.split_stride = (long long)U * D;
  rc = launch_mn<A_TMA_MN, EPI_F32>(p, t, splits, st);
  if (rc) return rc;
  return reduce_partials(part, splits, (long long)U * D, gw, st, upd);
}

size_t umma_fc_extra_ws(int B, int D, int U, int prec) {
  if (prec != PC_BF16) return 0;
  int s = fc_wgrad_splits(B, D, U);
  return s > 1 ? (size_t)s * U * D * sizeof(float) : 0;
}

}  // namespace pc

// Debug only (tools/trace_gemm.py): device buffer of >= grid * 64 * 8 u64 that
// every following tensor-core GEMM launch stamps with clock64 per tile; NULL stops.
extern "C" PC_API void pc_debug_trace_gemm(void* buf) {
  pc::umma::g_trace = static_cast<unsigned long long*>(buf);
}

extern "C" PC_API void pc_contraction_counts(unsigned long long* tensor_core, unsigned long long* simt) {
  if (tensor_core) *tensor_core = pc::umma::g_tc_launches.load();
  if (simt) *simt = pc::umma::g_simt_launches.load();
}
