// tf32 tensor-core path (tcgen05.mma kind::tf32, float storage): entry points used by api.cu.
#pragma once
#include "common.cuh"

namespace pc {

bool tf32_conv_ok(const pc_conv_geom& g);
int tf32_conv_forward(const pc_conv_geom& g, const float* x, const float* w, const float* bias, float* y, int flags,
                      cudaStream_t st);
size_t tf32_dgrad_ws(const pc_conv_geom& g);
int tf32_conv_dgrad(const pc_conv_geom& g, const float* w, const float* gy, float* gx, const float* mask,
                    float* wt, cudaStream_t st);
long long tf32_wgrad_splits(const pc_conv_geom& g);
int tf32_conv_wgrad(const pc_conv_geom& g, const float* x, const float* gy, float* gw, float* part, cudaStream_t st);

bool tf32_fc_ok(int D, int U, const pc_mat& x);
int tf32_fc_forward(int B, int D, int U, const pc_mat& x, const float* w, const float* bias, float* y, int flags,
                    cudaStream_t st);
int tf32_fc_dgrad(int B, int D, int U, const float* w, const float* gy, const pc_mat& gx, const float* mask,
                  cudaStream_t st);
long long tf32_fc_wgrad_splits(int B, int D, int U);
int tf32_fc_wgrad(int B, int D, int U, const pc_mat& x, const float* gy, float* gw, float* part, cudaStream_t st);

}  // namespace pc
