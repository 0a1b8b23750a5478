// ops.hpp — host launchers of the op-level kernels (ops.cu). All pointers are
// device pointers; validation mirrors the reference's ConfigError checks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.hpp"

namespace sige_b200 {

void op_difference_mask(const float* o, const float* e, int n, int c, int h, int w, float thr,
                        uint8_t* mask, cudaStream_t st);
void op_downsample_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out,
                        cudaStream_t st);
void op_dilate_mask(const uint8_t* m, int h, int w, int r, uint8_t* out, uint8_t* tmp,
                    cudaStream_t st);
void op_mask_to_block_indices(const uint8_t* m, int h, int w, int b, int batch, int32_t* idx,
                              int capacity, int32_t* count, cudaStream_t st);
void op_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count, int b,
               int ih, int iw, int k, int s, const DevEpilogue& epi, float* out, cudaStream_t st);
void op_scatter(const float* blocks, int count, int channels, int b, const int32_t* idx, float* base,
                int n, int c, int h, int w, bool add, cudaStream_t st);
int op_build_scatter_map(const int32_t* idx, int count, int b, int h, int w,
                         sige_scatter_entry* map, int* scratch2, cudaStream_t st);
void op_scatter_gather(const float* blocks, int count, int pb, const float* orig, int n, int c,
                       int h, int w, const sige_scatter_entry* map, int bps, const int32_t* cidx,
                       int ccount, int cb, int ch, int cw, int k, int s, const DevEpilogue& epi,
                       float* out, cudaStream_t st);
void op_residual_pass(const float* blocks, int count, int c, int b, const int32_t* idx,
                      const float* orig_sc, float* out, int n, int h, int w, bool shortcut_pass,
                      cudaStream_t st);
void op_combine(const float* a, const float* b, float sign, size_t n, float* out, cudaStream_t st);
void op_epilogue_blocks(float* blocks, int count, int c, int bh, const int32_t* idx,
                        const DevEpilogue& epi, cudaStream_t st);
void op_conv_cc(const float* in, long long in_stride, int ci, int ih, int iw, const float* wt,
                const float* bias, int co, int k, int s, int pad, float* out, long long out_stride,
                int oh, int ow, int items, int math, cudaStream_t st);

void op_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                     const int32_t* idx, int count, int b, int ih, int iw, int k, int s, const DevEpilogue& epi,
                     int act, float* out, cudaStream_t st);
void op_resize_nearest(const float* in, int n, int c, int h, int w, int oh, int ow, float* out, cudaStream_t st);
void op_cov_footprint(const int32_t* idx, const int32_t* count, int capacity, int b, int h, int w, uint8_t* m,
                      cudaStream_t st);
void op_cov_up2(const uint8_t* m, int h, int w, uint8_t* out, cudaStream_t st);
void op_cov_final(uint8_t* m, long long n, const int32_t* any, int mode, cudaStream_t st);
void op_expf_sweep(uint32_t first, long long count, int mode, float* out, cudaStream_t st);

}  // namespace sige_b200
