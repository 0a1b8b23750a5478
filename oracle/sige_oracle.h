/* sige_oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement of the SIGE
 * reference path (/root/reference/proj) used as the parity checker for the
 * CUDA library. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never does.
 *
 * Every function mirrors one reference function (cited at its definition in
 * sige_oracle.c) with the same arithmetic order, no FMA contraction
 * (-ffp-contract=off, as proj/CMakeLists.txt:11-13) and libm expf for SiLU.
 * Layouts are the reference's: NCHW tensors, (G,C,bh,bw) block stacks, index
 * triplets {n,r,c}. Return codes follow sige_b200.h (0 ok, 2 config error).
 */
#ifndef SIGE_ORACLE_H_
#define SIGE_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "sige_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

uint64_t orc_fnv1a64(const void* p, size_t n, uint64_t seed);
int orc_rng_stream(uint32_t seed, int count, uint32_t* out_u32, float* out_uniform, float lo,
                   float hi);
float orc_expf(float x);

int orc_make_edit_fixture(const char* kind, int n, int c, int h, int w, uint32_t seed,
                          float* orig, float* edited);

int orc_compute_difference_mask(const float* o, const float* e, int n, int c, int h, int w,
                                float thr, uint8_t* out);
int orc_downsample_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out);
int orc_dilate_mask(const uint8_t* m, int h, int w, int r, uint8_t* out);
int orc_mask_to_block_indices(const uint8_t* m, int h, int w, int b, int batch, int32_t* idx,
                              int cap, int* count, uint64_t* hash);
uint64_t orc_index_set_hash(const int32_t* idx, int count, int b, int h, int w);

int orc_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count, int b,
               int ih, int iw, int k, int s, const sige_epilogue* epi, float* out);
int orc_scatter(const float* blocks, int count, int channels, int block, const int32_t* idx,
                const float* base, float* out, int n, int c, int h, int w);
int orc_scatter_add_inplace(const float* blocks, int count, int channels, int block,
                            const int32_t* idx, float* base, int n, int c, int h, int w);
int orc_build_scatter_map(const int32_t* idx, int count, int block, int h, int w,
                          sige_scatter_entry* out, int* bps);
int orc_scatter_gather(const float* blocks, int count, int block, const int32_t* prod_idx,
                       const float* orig_out, int n, int c, int h, int w,
                       const int32_t* cons_idx, int cons_count, int cons_block, int ch, int cw,
                       int k, int s, const sige_epilogue* epi, float* out);
int orc_scatter_with_block_residual(const float* mb, int mcount, int mblock, const int32_t* midx,
                                    const float* sb, int scount, int sblock, const int32_t* sidx,
                                    const float* sum, const float* orig_sc, float* out, int n,
                                    int c, int h, int w, int fused);
int orc_combine_blocks(const float* a, const float* b, float sign, size_t numel, float* out);
int orc_apply_epilogue_on_blocks(float* blocks, int count, int channels, int bh,
                                 const int32_t* idx, int idx_h, int idx_w,
                                 const sige_epilogue* epi);
int orc_conv_on_blocks(const float* blocks, int count, int window, const sige_conv_desc* conv,
                       int with_bias, float* out, int block);
int orc_conv2d(const float* x, int n, int c, int h, int w, const sige_conv_desc* conv,
               int with_bias, float* out);
int orc_group_norm_fold(const float* x, int n, int c, int h, int w, int groups, float eps,
                        const float* gamma, const float* beta, float* scale, float* shift);

/* models: name in {conv3x3_128, mini_unet_gn, mini_unet_bn, gaugan_stack_in,
 * single_conv64, ddim_stack, ddim_stack_64x32}; returns an owned descriptor. */
sige_model_desc* orc_model_build(const char* name);
sige_model_desc* orc_model_clone(const sige_model_desc* d);
void orc_model_free(sige_model_desc* d);
uint64_t orc_model_weight_hash(const sige_model_desc* d);
int orc_model_required_dilation(const sige_model_desc* d);
int orc_model_output_shape(const sige_model_desc* d, int* c, int* h, int* w);

typedef struct orc_cache orc_cache;
orc_cache* orc_cache_precompute(const sige_model_desc* m, const float* orig, int n, int c, int h,
                                int w);
void orc_cache_free(orc_cache* c);
int orc_cache_tensor(orc_cache* c, int step, const char* key, float* out, size_t cap, int* dims);
int orc_cache_norm(orc_cache* c, int step, const char* key, float* scale, float* shift,
                   size_t cap, int* count);
int orc_cache_count(orc_cache* c);
/* i-th entry: kind 0 tensor / 1 norm; key copied into buf. */
int orc_cache_entry(orc_cache* c, int i, int* kind, char* key, size_t keycap, size_t* numel);
uint64_t orc_cache_total_elements(orc_cache* c);

int orc_sparse_forward(const sige_model_desc* m, orc_cache* cache, const float* edited, int n,
                       int c, int h, int w, const uint8_t* mask, const sige_run_config* cfg,
                       float* out, uint64_t* trace_rows, int trace_cap, int* trace_n);
int orc_dense_forward(const sige_model_desc* m, const float* in, int n, int c, int h, int w,
                      float* out);
int orc_dense_forward_reused_stats(const sige_model_desc* m, const float* in, int n, int c,
                                   int h, int w, orc_cache* cache, int step, float* out);

/* SPADE ops (config 3): restatements, not reference functions. */
int orc_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                     const int32_t* idx, int count, int b, int ih, int iw, int k, int s,
                     const sige_epilogue* norm, int act, float* out);
int orc_resize_nearest(const float* in, int n, int c, int h, int w, int oh, int ow, float* out);

#ifdef __cplusplus
}
#endif

#endif
