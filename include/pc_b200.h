/*
 * pc_b200.h — C ABI of the B200 training-step library (libpcb200.so).
 *
 * Drop-in boundary for the hot path of the reference package `parconv`
 * (pure Python/numpy, /root/reference/pkg/src/parconv). Each entry point
 * replaces one reference kernel call made by the step engine
 * `schemes.column_fwd_bwd` (schemes.py:342-419) or the data-parallel leg of
 * `schemes.hybrid_step` (schemes.py:540-558); the Python drop-in binds them
 * with ctypes (paper_1312_5853_b200/_lib.py; INTEGRATION.md shows the stub).
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless noted; sizes are element counts.
 *  - Activations are NHWC ("channels last"), row = pixel (b, y, x), in the
 *    storage precision `prec` (PC_FP32 -> float, PC_BF16 -> __nv_bfloat16).
 *    The contraction entry points (conv / FC forward and backward and their
 *    workspace queries) also take PC_TF32: float storage, tcgen05 kind::tf32
 *    tensor-core math (geometries it cannot tile fall back to the fp32 SIMT path).
 *    Master weights, velocities and weight gradients are always float.
 *  - A channel-blocked activation (the cross-layer concatenation of m column
 *    slices) stores channel c at  base + (c / cs) * cstride + pixel * cs + c % cs.
 *    cs == C (cstride ignored) is plain NHWC.
 *  - Conv weights are stored [N][kh][kw][C] (reference: [N][C][kh][kw]).
 *  - FC weights are stored [U][D] (reference: [D][U], kernels.py:160-168).
 *  - Every function is asynchronous on `stream` and returns a status:
 *      0 ok, 1 shape error, 2 validation error, 3 CUDA error, 4 NCCL error.
 *    pc_last_error() returns the message of the calling thread's last error.
 *  - Functions never allocate device memory; callers pass workspaces.
 *  - Reentrant; the caller selects the device (cudaSetDevice) beforehand.
 */
#ifndef PC_B200_H
#define PC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PC_API __attribute__((visibility("default")))
#else
#define PC_API
#endif

typedef void* pc_stream_t; /* cudaStream_t */

enum pc_prec { PC_FP32 = 0, PC_BF16 = 1, PC_TF32 = 2,
               PC_FP64 = 3 /* source images only: pc_space_to_depth_ex / _f32 */ };
enum pc_status { PC_OK = 0, PC_ESHAPE = 1, PC_EVALUE = 2, PC_ECUDA = 3, PC_ENCCL = 4 };
enum pc_conv_flags { PC_RELU = 1, PC_WANT_DX = 2, PC_WANT_DW = 4, PC_MASK_DX = 8, PC_WT_PRESET = 16,
                     /* forward: the last 16 input channels have structural-zero filter
                      * weights (the space-to-depth input layer: 48 real of 64) — the
                      * tensor-core path may skip their MMA steps */
                     PC_ZERO_TAIL16 = 32 };

/* Conv geometry (reference ConvParams + input shape, kernels.py:37-83). */
typedef struct {
  int B, H, W, C;      /* input extents (C = full, possibly concatenated, channels) */
  int N, k, stride, pad;
  int Ho, Wo;          /* output extents; must equal (H+2p-k)/s+1 exactly */
  int cs;              /* channels per input block (== C when not blocked) */
  long long cstride;   /* elements between input channel blocks */
} pc_conv_geom;

/* Matrix view: element (r, c) at ptr + (c / cb) * bstride + r * ld + c % cb. */
typedef struct {
  void* ptr;
  long long ld, cb, bstride;
} pc_mat;

PC_API const char* pc_last_error(void);
PC_API int pc_version(void);
/* Number of kernels this library has launched in the process (all devices). */
PC_API unsigned long long pc_launch_count(void);
/* bf16 contraction launches by engine: tcgen05 tensor-core kernels vs the
 * CUDA-core kernel used only for extents the tensor-core path cannot tile
 * (e.g. a 10-class head: rows not 16-byte aligned). */
PC_API void pc_contraction_counts(unsigned long long* tensor_core, unsigned long long* simt);
/* Launches of the tf32 tensor-core kernels (tcgen05.mma kind::tf32) so far. */
PC_API unsigned long long pc_tf32_contractions(void);
/* Debug (tools/trace_gemm.py): per-tile clock64 timeline of the following tensor-core
 * GEMM launches into a device buffer of >= grid x 64 tiles x 8 u64; NULL turns it off. */
PC_API void pc_debug_trace_gemm(void* buf);
/* 1 when the tcgen05/TMA tensor-core path is compiled in and the device is sm_100. */
PC_API int pc_has_tcgen05(void);

/* --- conv: replaces kernels.conv2d_forward (kernels.py:104-116) ------------- */
/* y[pixel][n] = bias[n] + sum_{i,j,c} x[b, oy*s+i-p, ox*s+j-p, c] * w[n][i][j][c]
 * (PC_RELU: y = max(y, 0)). x may be channel-blocked; y is plain NHWC. */
PC_API int pc_conv2d_forward(const pc_conv_geom* g, const void* x, const void* w, const float* bias,
                      void* y, int prec, int flags, pc_stream_t stream);

/* --- conv: replaces kernels.conv2d_backward (kernels.py:119-152) ------------ */
/* PC_WANT_DX: gx (same blocked layout as x) = conv-transpose of gy;
 *   PC_MASK_DX: gx = 0 where mask <= 0 (fused ReLU backward of the producer;
 *   mask has gx's layout, normally the ReLU output that fed this conv).
 * PC_WANT_DW: gw[n][i][j][c] (float) and gb[n] (float) = weight/bias grads.
 * workspace: pc_conv2d_backward_workspace() bytes (split-K partials). */
PC_API size_t pc_conv2d_backward_workspace(const pc_conv_geom* g, int prec);
PC_API int pc_conv2d_backward(const pc_conv_geom* g, const void* x, const void* w, const void* gy,
                       void* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                       void* workspace, size_t workspace_bytes, pc_stream_t stream);

/* --- fc: replaces kernels.fc_forward / fc_backward (kernels.py:160-182) ----- */
/* y[b][u] = bias[u] + sum_d x(b, d) * w[u][d]; x is a pc_mat view (blocked
 * when the FC consumes a cross concatenation). y is plain [B][U]. */
PC_API int pc_fc_forward(int B, int D, int U, const pc_mat* x, const void* w, const float* bias,
                  void* y, int prec, int flags, pc_stream_t stream);
/* Same with a caller workspace of pc_fc_forward_workspace() bytes: small-batch
 * calls then split the K loop over the machine and sum the fp32 partials in a
 * fixed order (bias/ReLU applied after the sum). pc_fc_forward == _ex without one. */
PC_API size_t pc_fc_forward_workspace(int B, int D, int U, int prec);
PC_API int pc_fc_forward_ex(int B, int D, int U, const pc_mat* x, const void* w, const float* bias, void* y,
                            int prec, int flags, void* workspace, size_t workspace_bytes, pc_stream_t stream);
/* gx(b, d) = sum_u gy[b][u] w[u][d] (written through the pc_mat view, masked
 * by `mask` viewed identically when PC_MASK_DX); gw[u][d] = sum_b gy[b][u] x(b, d);
 * gb[u] = sum_b gy[b][u]. */
PC_API size_t pc_fc_backward_workspace(int B, int D, int U, int prec);
PC_API int pc_fc_backward(int B, int D, int U, const pc_mat* x, const void* w, const void* gy,
                   const pc_mat* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                   void* workspace, size_t workspace_bytes, pc_stream_t stream);

/* --- relu: kernels.relu_forward / relu_backward (kernels.py:190-197) -------- */
PC_API int pc_relu_forward(long long n, const void* x, void* y, int prec, pc_stream_t stream);
/* gx = g where x > 0 else 0 (x may be the ReLU input or output: same mask). */
PC_API int pc_relu_backward(long long n, const void* x, const void* g, void* gx, int prec,
                     pc_stream_t stream);

/* --- maxpool: kernels.maxpool_forward / backward (kernels.py:200-244) ------- */
/* NHWC; argmax = local window index i*k+j (row-major, first max wins, NaN wins)
 * stored as uint8. */
PC_API int pc_maxpool_forward(int B, int H, int W, int C, int k, int s, const void* x, void* y,
                       uint8_t* argmax, int prec, pc_stream_t stream);
/* Deterministic gather form of the np.add.at scatter: each input element sums
 * the windows whose argmax hits it in ascending (oy, ox) order. If mask != NULL
 * the result is zeroed where mask <= 0 (fused ReLU backward). */
PC_API int pc_maxpool_backward(int B, int H, int W, int C, int k, int s, const void* gy,
                        const uint8_t* argmax, const void* mask, void* gx, int prec,
                        pc_stream_t stream);
/* pc_maxpool_backward (bf16, 3x3 / stride 2, 256 % (C/8) == 0) that also writes
 * gb[c] = sum over (b, y, x) of the stored gx: the bias gradient of the conv whose
 * ReLU output this pool reads (gx is that conv's upstream gradient), reduced in a
 * fixed order while gx is written instead of by a second pass over it.
 * gb == NULL: plain pc_maxpool_backward. Workspace:
 * pc_maxpool_backward_bias_workspace(C) bytes. */
PC_API size_t pc_maxpool_backward_bias_workspace(int C);
PC_API int pc_maxpool_backward_bias(int B, int H, int W, int C, int k, int s, const void* gy, const uint8_t* argmax,
                                    const void* mask, void* gx, int prec, float* gb, void* ws, size_t ws_bytes,
                                    pc_stream_t stream);

/* --- softmax cross-entropy: kernels.softmax_xent_scaled (kernels.py:252-276) */
/* grad[b][k] = (softmax - onehot) * scale (stored in prec); row_loss[b] =
 * -scale * log softmax[b][label_b] (double). Out-of-range labels set *bad_label
 * to 1 (device int; checked at the loss read-back). */
PC_API int pc_softmax_xent(int B, int K, const void* logits, const int32_t* labels, double scale,
                    void* grad, double* row_loss, int* bad_label, int prec, pc_stream_t stream);
/* out[0] = sum_i v[i] in ascending order (one block; deterministic). */
PC_API int pc_sum_f64(int n, const double* v, double* out, pc_stream_t stream);
/* pc_softmax_xent + pc_sum_f64 in one launch: the last block to finish (device
 * ticket, zero-initialised, reset by the kernel) sums row_loss into *loss in
 * pc_sum_f64's order (bit-identical). Falls back to the two launches for K > 1024. */
PC_API int pc_softmax_xent_loss(int B, int K, const void* logits, const int32_t* labels, double scale, void* grad,
                                double* row_loss, int* bad_label, double* loss, unsigned* ticket, int prec,
                                pc_stream_t stream);

/* Fused momentum-SGD epilogue for a weight gradient (single-replica plans, where
 * no cross-replica reduction sits between the gradient and the update): instead
 * of storing gw, the producing kernel applies v = momentum*v - lr*(g + wd*p),
 * p += v (and rewrites the bf16 shadow) to the parameters at gw's flat layout —
 * kernels.sgd_step's arithmetic (kernels.py:319-341) without the gradient round
 * trip through HBM. */
typedef struct {
  float* p;          /* fp32 master weights, same layout as the gradient */
  float* v;          /* fp32 velocity */
  void* p_lowp;      /* bf16 shadow of p (NULL: none) */
  float lr, momentum, weight_decay;
} pc_sgd_fuse;

/* pc_conv2d_backward / pc_fc_backward with an optional fused update of the
 * weights (upd != NULL: gw is not written; gb is). */
PC_API int pc_conv2d_backward_ex(const pc_conv_geom* g, const void* x, const void* w, const void* gy,
                                 void* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                                 void* workspace, size_t workspace_bytes, const pc_sgd_fuse* upd,
                                 pc_stream_t stream);
PC_API int pc_fc_backward_ex(int B, int D, int U, const pc_mat* x, const void* w, const void* gy,
                             const pc_mat* gx, const void* mask, float* gw, float* gb, int prec, int flags,
                             void* workspace, size_t workspace_bytes, const pc_sgd_fuse* upd, pc_stream_t stream);

/* --- SGD: kernels.sgd_step (kernels.py:319-341), multi-tensor, one launch -- */
typedef struct {
  float* p;          /* fp32 master parameters (updated in place) */
  float* v;          /* fp32 velocity (updated in place) */
  const float* g;    /* fp32 gradient */
  void* p_lowp;      /* optional bf16 shadow copy rewritten from p (NULL: none) */
  long long n;
} pc_sgd_tensor;
/* `table` is a DEVICE array of n_tensors descriptors. */
PC_API int pc_sgd_step(int n_tensors, const pc_sgd_tensor* table, long long max_numel, float lr,
                float momentum, float weight_decay, pc_stream_t stream);
/* Same update as a background launch: at most ctas_per_sm 256-thread CTAs per SM
 * in total, so it can run on a side stream beside a persistent GEMM that holds
 * one CTA per SM (ctas_per_sm <= 0: identical to pc_sgd_step). */
PC_API int pc_sgd_step_ex(int n_tensors, const pc_sgd_tensor* table, long long max_numel, float lr,
                   float momentum, float weight_decay, int ctas_per_sm, pc_stream_t stream);

/* --- extensions beyond the reference (the reference has no such
 * layers, netdef.py:219-220): definitions in oracle/ref_kernels.py ----------- */
/* Local response normalisation across the C channels of each of P NHWC pixels:
 * y = x * (k + alpha * sum_{|c'-c| <= size/2} x_c'^2)^-beta (lrn_forward). */
PC_API int pc_lrn_forward(long long P, int C, int size, float k, float alpha, float beta, const void* x, void* y,
                          int prec, pc_stream_t stream);
/* gx from x and gy (lrn_backward; the scale is recomputed from x). */
PC_API int pc_lrn_backward(long long P, int C, int size, float k, float alpha, float beta, const void* x,
                           const void* gy, void* gx, int prec, pc_stream_t stream);
/* Dropout on an NHWC slice [B][H][W][C] of a dense NCHW activation with C_dense
 * channels (slice channels c_off.., global rows row0..): y = x / (1 - p) where
 * kept, else 0. Element i of the dense activation is kept iff
 * (mix64(state + (i+1)*GOLDEN) >> 11) >= thresh, state = rng.dropout_state(seed,
 * *step, layer), thresh = rng.dropout_threshold(p); *step is a DEVICE counter.
 * The same call computes the backward (x = gy, y = gx). */
PC_API int pc_dropout(int B, int H, int W, int C, int C_dense, int c_off, long long row0, unsigned long long seed,
                      const unsigned long long* step, int layer, unsigned long long thresh, float p, const void* x,
                      void* y, int prec, pc_stream_t stream);
/* *counter += delta (device; advances the dropout step inside a CUDA graph). */
PC_API int pc_counter_add(unsigned long long* counter, long long delta, pc_stream_t stream);

/* --- single-process multi-GPU fabric (spawn(n) over the visible GPUs) --------
 * Replaces the reference's in-process message fabric (`fabric.py:102-339`):
 * the column exchange and the replica reduction read peer memory directly. */
/* Let the calling thread's current device read `peer`'s memory (idempotent). */
PC_API int pc_enable_peer_access(int peer);
/* Asynchronous copy between any two device (or pinned host) buffers on `stream`. */
PC_API int pc_copy_async(void* dst, const void* src, size_t bytes, pc_stream_t stream);

/* --- trainer feed on the device ------------------------------ */
/* Rows idx[0..n) (DEVICE int64 sample indices) of the synthetic split
 * gen_synthetic(classes, per_class, shape, seed) with prod(shape) = dim, written
 * as NCHW rows in out_prec (PC_FP32 = the reference's float32-quantised values;
 * PC_BF16 = those rounded to bf16). domain = rng.DOMAIN_TRAIN (4) / DOMAIN_TEST (5),
 * std_ = the blob standard deviation (0.5). Replaces the host loop of
 * `pkg/src/parconv/data.py:52-96` (templates `rng.py:94-100`, noise `rng.py:75-88`). */
PC_API int pc_synthetic_rows(int classes, int per_class, long long dim, unsigned long long seed, int domain,
                             const long long* idx, int n, float std_, void* out, int out_prec, pc_stream_t stream);
/* dst[r] = src[idx[r]] for n rows of row_bytes (multiple of 4, 4-byte aligned
 * buffers): the batch of an HBM-resident split by the epoch permutation
 * (`pkg/src/parconv/trainer.py:120-133` indexes the host array instead). */
PC_API int pc_gather_rows(int n, long long row_bytes, const void* src, const long long* idx, void* dst,
                          pc_stream_t stream);

/* --- layout / reduction helpers used by the engine -------------------------- */
/* Explicit im2col of the NCHW network input (float32 or bf16 in, bf16 out):
 * col[(b*Ho + oy)*Wo + ox][(c*k + i)*k + j] = x[b][c][oy*s+i-p][ox*s+j-p] (0 outside),
 * columns zero-padded to Kp (multiple of 8). Used for the input layer, whose
 * 3 channels are too narrow for 16-byte im2col rows; the conv then runs as
 * pc_fc_forward / pc_fc_backward over pixels with weights [N][Kp]. */
PC_API int pc_im2col(int B, int C, int H, int W, int k, int s, int p, int Kp, const void* src, int src_prec,
                     void* dst, pc_stream_t stream);
/* Same with the output precision selectable (PC_BF16 or PC_FP32: the tf32 mode's
 * input layer, columns padded to a multiple of 32). */
PC_API int pc_im2col_ex(int B, int C, int H, int W, int k, int s, int p, int Kp, const void* src, int src_prec,
                        void* dst, int dst_prec, pc_stream_t stream);
/* Space-to-depth of the NCHW network input (float32 or bf16 in, bf16 out) for a
 * strided input conv: dst[b][Y][X][(dy*s + dx)*C + c] = x[b][c][Y*s+dy-p][X*s+dx-p]
 * (0 outside the image and for channels >= s*s*C), Y < ceil((H+2p)/s), channels
 * padded to Cs (multiple of 8; 64 for the TMA im2col path). A k x k / stride-s
 * conv of x equals a ceil(k/s)^2 / stride-1 / pad-0 conv of dst with the weights
 * regrouped the same way (taps beyond k zero), so the input layer runs on the
 * tensor-core implicit GEMM with 128-byte channel rows. */
PC_API int pc_space_to_depth(int B, int C, int H, int W, int s, int p, int Cs, const void* src, int src_prec,
                             void* dst, pc_stream_t stream);
/* Bias gradient gb[n] = sum_p gy[p][n] (gy [P][N] in prec, N % 8 == 0) by a
 * fixed grid of `ctas` CTAs using no shared memory, so it can run on a side
 * stream beside the persistent tensor-core kernels; deterministic order.
 * Workspace: pc_bias_grad_workspace(P, N, ctas) bytes. (The data/weight gradient
 * entry points skip their own bias reduction when gb is NULL.) */
PC_API size_t pc_bias_grad_workspace(long long P, int N, int ctas);
PC_API int pc_bias_grad(long long P, int N, const void* gy, int prec, float* gb, float* ws, size_t ws_bytes,
                        int ctas, pc_stream_t stream);
/* bf16 conv data gradient, prepared filters: wt = the filters in the layout
 * (transposed, rotated as the data-gradient path needs) that pc_conv2d_backward
 * otherwise rebuilds in its workspace on every call. With PC_WT_PRESET in the
 * backward flags, `w` is taken to be this wt for the data gradient — so a step
 * can prepare every layer's wt off the critical path (a side stream at the
 * start of the step). wt holds N*k*k*C bf16. */
PC_API int pc_conv2d_dgrad_weights(const pc_conv_geom* g, const void* w, void* wt, int prec, pc_stream_t stream);
/* Cap (0 = none) on the number of CTAs of the persistent tensor-core kernels
 * launched next by the calling thread; a step program uses it to run the FC
 * weight-gradient + update chain on a side stream beside the convolution
 * backward on disjoint SM sets. */
PC_API int pc_set_grid_cap(int ctas);
/* As pc_space_to_depth, with padding channel `ones` (s*s*C <= ones < Cs; -1 =
 * none) set to 1.0 in every block: the input layer's weight gradient at that
 * channel and tap (0, 0) is then its bias gradient (pc_s2d_wgrad_finish), so the
 * bias needs no separate reduction over the upstream gradient. */
PC_API int pc_space_to_depth_ex(int B, int C, int H, int W, int s, int p, int Cs, const void* src, int src_prec,
                                int ones, void* dst, pc_stream_t stream);
/* pc_space_to_depth_ex with float32 output (the tf32 mode's input layer). */
PC_API int pc_space_to_depth_f32(int B, int C, int H, int W, int s, int p, int Cs, const void* src, int src_prec,
                                 int ones, float* dst, pc_stream_t stream);
/* gb[n] = gw[n * K + ones] for n < N, then gw[i] = 0 where keep[i] == 0 (the
 * structural zeros of the regrouped input-layer weights, including `ones`). */
PC_API int pc_s2d_wgrad_finish(int N, int K, int ones, const uint8_t* keep, float* gw, float* gb,
                               pc_stream_t stream);
/* buf[i] = 0 where keep[i] == 0 (fp32): pins the regrouped conv's structural-zero
 * weights by zeroing their gradients before the SGD update. */
PC_API int pc_mask_f32(long long n, const uint8_t* keep, float* buf, pc_stream_t stream);
/* NCHW float (reference layout) -> NHWC prec with C padded to Cp (zeros). */
PC_API int pc_nchw_to_nhwc(int B, int C, int H, int W, int Cp, const float* src, void* dst, int prec,
                    pc_stream_t stream);
/* dst[i] = sum_{j<k} src[j][i] in ascending j, accumulated in fp32 and rounded
 * once to prec (k buffers; `src` is a DEVICE array of k device pointers). */
PC_API int pc_sum_buffers(int k, long long n, const void* const* src, void* dst, int prec,
                          pc_stream_t stream);
/* float <-> prec conversions of a flat buffer. */
PC_API int pc_cast(long long n, const void* src, int src_prec, void* dst, int dst_prec,
            pc_stream_t stream);
/* dst = src * alpha (prec storage), used for the shared-head 1/m contribution. */
PC_API int pc_scale(long long n, const void* src, void* dst, float alpha, int prec, pc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PC_B200_H */
