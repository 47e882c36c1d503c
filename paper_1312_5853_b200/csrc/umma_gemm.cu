// bf16 contraction entry points. BRING-UP STAGE: routed through the SIMT
// implicit GEMM with bf16 storage until the tcgen05 kernel lands.
#include "gemm_ops.cuh"
#include "umma.cuh"

namespace pc {

bool umma_available() { return false; }

int umma_conv_forward(const pc_conv_geom& g, const void* x, const void* w, const float* bias, void* y,
                      int flags, cudaStream_t st) {
  return simt_conv_forward(g, x, w, bias, y, PC_BF16, flags, st);
}
int umma_conv_dgrad(const pc_conv_geom& g, const void* w, const void* gy, void* gx, const void* mask,
                    cudaStream_t st, void*, size_t) {
  return simt_conv_dgrad(g, w, gy, gx, mask, st, PC_BF16);
}
long long umma_wgrad_splits(const pc_conv_geom& g) {
  return simt_splits(g.N, g.k * g.k * g.C, (long long)g.B * g.Ho * g.Wo);
}
int umma_conv_wgrad(const pc_conv_geom& g, const void* x, const void* gy, float* gw, float* part,
                    cudaStream_t st) {
  return simt_conv_wgrad(g, x, gy, gw, part, (int)umma_wgrad_splits(g), st, PC_BF16);
}
size_t umma_conv_extra_ws(const pc_conv_geom&, int) { return 0; }
int umma_fc_forward(int B, int D, int U, const pc_mat& x, const void* w, const float* bias, void* y,
                    int flags, cudaStream_t st) {
  return simt_fc_forward(B, D, U, x, w, bias, y, PC_BF16, flags, st);
}
int umma_fc_dgrad(int B, int D, int U, const void* w, const void* gy, const pc_mat& gx, const void* mask,
                  cudaStream_t st) {
  return simt_fc_dgrad(B, D, U, w, gy, gx, mask, st, PC_BF16);
}
int umma_fc_wgrad(int B, int D, int U, const pc_mat& x, const void* gy, float* gw, float*, cudaStream_t st) {
  return simt_fc_wgrad(B, D, U, x, gy, gw, st, PC_BF16);
}
size_t umma_fc_extra_ws(int, int, int, int) { return 0; }

}  // namespace pc
