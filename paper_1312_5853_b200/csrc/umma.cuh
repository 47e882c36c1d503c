// bf16 tensor-core path (tcgen05 / TMEM / TMA): entry points used by api.cu.
#pragma once
#include "common.cuh"

namespace pc {

bool umma_available();
void set_grid_cap(int ctas);
int umma_conv_forward(const pc_conv_geom& g, const void* x, const void* w, const float* bias, void* y,
                      int flags, cudaStream_t st);
int umma_conv_dgrad(const pc_conv_geom& g, const void* w, const void* gy, void* gx, const void* mask,
                    cudaStream_t st, void* ws, size_t ws_bytes, bool w_preset = false);
int umma_conv_dgrad_weights(const pc_conv_geom& g, const void* w, void* wt, cudaStream_t st);
int umma_conv_wgrad(const pc_conv_geom& g, const void* x, const void* gy, float* gw, float* part,
                    cudaStream_t st, const pc_sgd_fuse* upd = nullptr);
long long umma_wgrad_splits(const pc_conv_geom& g);
size_t umma_conv_extra_ws(const pc_conv_geom& g, int prec);

int umma_fc_forward(int B, int D, int U, const pc_mat& x, const void* w, const float* bias, void* y,
                    int flags, cudaStream_t st, void* ws, size_t ws_bytes);
size_t umma_fc_forward_ws(int B, int D, int U);
int umma_fc_dgrad(int B, int D, int U, const void* w, const void* gy, const pc_mat& gx, const void* mask,
                  cudaStream_t st, void* ws, size_t ws_bytes);
size_t umma_fc_dgrad_ws(int B, int D, int U);
int umma_fc_wgrad(int B, int D, int U, const pc_mat& x, const void* gy, float* gw, float* part,
                  cudaStream_t st, const pc_sgd_fuse* upd = nullptr);
size_t umma_fc_extra_ws(int B, int D, int U, int prec);

}  // namespace pc
