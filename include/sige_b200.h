/*
 * sige_b200.h — C-ABI drop-in boundary for SIGE's spatially sparse update path
 * on NVIDIA B200 (sm_100a).
 *
 * The reference (/root/reference/proj, namespace `sige`) exposes this path as a
 * C++ free-function API over host std::vector tensors. It has no FFI; each
 * entry point below replaces one of its functions and names the reference
 * declaration it stands in for. All tensor/block pointers are DEVICE pointers
 * (except where a function says "host"), every call takes a cudaStream_t (as
 * `sige_stream_t`, NULL = legacy default stream), and every call returns an
 * int status. On failure `sige_last_error()` returns the message, with the
 * reference's op prefix (e.g. "gather: kernel size must be 1 or 3", from
 * proj/src/kernels.cpp:41) so the C++ wrapper can rethrow `ConfigError`.
 *
 * Data layouts at the boundary are the reference's own:
 *   tensor       : NCHW fp32, tightly packed          (proj/include/sige/tensor.hpp:12-39)
 *   difference mask: u8 H*W, row-major, 0/1         (proj/include/sige/mask.hpp:11-27)
 *   index set    : `count` triplets int32 {n, r, c}, sorted (n, r, c)
 *                                                    (proj/include/sige/mask.hpp:44-57)
 *   block stack  : (G, C, bh, bw) fp32               (proj/include/sige/kernels.hpp:17-39)
 *   conv weight  : (c_out, c_in, k, k) fp32          (proj/include/sige/conv.hpp:11-23)
 * The engine (sige_engine_*) keeps activations internally in NHWC and is the
 * production path; the op-level entry points are the per-function drop-ins.
 */
#ifndef SIGE_B200_H_
#define SIGE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ------------------------------------------------------------ */
#define SIGE_OK 0
#define SIGE_ERR_CONFIG 2   /* reference ConfigError (CLI exit code 2, sige_cli.cpp:337-344) */
#define SIGE_ERR_CUDA 3     /* CUDA runtime / launch failure */
#define SIGE_ERR_INTERNAL 4 /* anything else */

typedef void* sige_stream_t; /* cudaStream_t */

/* Thread-local message of the last failing call on this thread. */
const char* sige_last_error(void);
const char* sige_version(void);
/* Number of CUDA kernels this library has launched (process lifetime). */
uint64_t sige_kernel_launch_count(void);

/* ---- shared descriptors -------------------------------------------------- */
enum { SIGE_ACT_NONE = 0, SIGE_ACT_RELU = 1, SIGE_ACT_SILU = 2 }; /* eltwise.hpp:12 */
/* LeakyReLU(0.2) of GauGAN's SPADE blocks: only sige_gather_spade takes it
 * (the reference's Epilogue has no such step). */
enum { SIGE_ACT_LEAKY_RELU = 3 };
enum { SIGE_EPI_SCALE_SHIFT = 0, SIGE_EPI_ACTIVATION = 1 };      /* eltwise.hpp:31-34 */
#define SIGE_MAX_EPI_STEPS 4

/* One step of the deferred element-wise chain `sige::Epilogue`
 * (eltwise.hpp:30-59). ScaleShift params hold either C values (broadcast over
 * the batch) or N*C values (sample-major), as eltwise.cpp:48-58 resolves them. */
typedef struct sige_epilogue_step {
  int kind;            /* SIGE_EPI_* */
  int act;             /* SIGE_ACT_* for activation steps */
  int nparams;         /* scale/shift length: C or N*C */
  const float* scale;  /* device pointer (host pointer for oracle/ref shims) */
  const float* shift;
} sige_epilogue_step;

typedef struct sige_epilogue {
  int num_steps;
  sige_epilogue_step steps[SIGE_MAX_EPI_STEPS];
} sige_epilogue;

/* `sige::ConvLayer` (conv.hpp:11-23). bias == NULL means empty bias. */
typedef struct sige_conv_desc {
  int c_in, c_out, k, stride;
  const float* weight; /* (c_out, c_in, k, k) */
  const float* bias;   /* c_out or NULL */
} sige_conv_desc;

enum { SIGE_NORM_GROUP = 0, SIGE_NORM_INSTANCE = 1, SIGE_NORM_BATCH = 2 }; /* norm.hpp:10 */

/* `sige::NormLayer` (graph.hpp:18-28). */
typedef struct sige_norm_desc {
  int kind, groups, channels;
  float eps;
  const float* gamma;
  const float* beta;
  const float* running_mean; /* batch kind only, else NULL */
  const float* running_var;
} sige_norm_desc;

/* `sige::LayerKind` (graph.hpp:37). */
enum {
  SIGE_LAYER_CONV = 0,
  SIGE_LAYER_NORM = 1,
  SIGE_LAYER_ACTIVATION = 2,
  SIGE_LAYER_RESBLOCK = 3,
  SIGE_LAYER_DOWNSAMPLE = 4,
  SIGE_LAYER_UPSAMPLE = 5,
  /* Config 3 (GauGAN; no reference counterpart): */
  SIGE_LAYER_SPADE_RESBLOCK = 6, /* SPADE residual block, see sige_spade_desc */
  SIGE_LAYER_RESIZE = 7          /* the model INPUT resized (nearest) to resize_h x resize_w (integer factors) */
};

/* One SPADE normalisation (Park et al. 2019): the param-free instance norm of
 * its input x (per sample and channel, eps), modulated per pixel by the
 * segmentation map s (the model input, nearest-resized to x's resolution):
 *   a = ReLU(shared(s)),  SPADE(x) = norm(x) * (1 + gamma(a)) + beta(a)
 * shared: 3x3 label_nc -> nhidden; gamma, beta: 3x3 nhidden -> C. */
typedef struct sige_spade_desc {
  float eps;
  sige_conv_desc shared;
  sige_conv_desc gamma;
  sige_conv_desc beta;
} sige_spade_desc;

/* `sige::Layer` (graph.hpp:53-61) flattened. For RESBLOCK: conv = conv1,
 * conv2, norm, act and (has_shortcut) shortcut, as ResBlockSpec
 * (graph.hpp:45-51). Weight pointers are HOST pointers: the engine uploads. */
typedef struct sige_layer_desc {
  int kind;
  int policy_sparse;  /* SparsePolicy::sparse (graph.hpp:30-35) */
  int min_resolution; /* SparsePolicy::min_resolution */
  sige_conv_desc conv;
  sige_norm_desc norm;
  int act;
  sige_conv_desc conv2;
  int has_shortcut;
  sige_conv_desc shortcut;
  /* SPADE_RESBLOCK (config 3): conv = conv_0 (3x3 fin -> fmiddle), conv2 =
   * conv_1 (3x3 fmiddle -> fout), shortcut = conv_s (1x1, no bias) when
   * has_shortcut, act = the block activation (SIGE_ACT_LEAKY_RELU);
   * spade[0] normalises conv_0's input, spade[1] conv_1's, spade[2] the
   * shortcut's. out = (has_shortcut ? conv_s(SPADE_s(x)) : x)
   *                 + conv_1(act(SPADE_1(conv_0(act(SPADE_0(x)))))). */
  const sige_spade_desc* spade;
  int resize_h, resize_w; /* RESIZE */
} sige_layer_desc;

/* `sige::ModelSpec` (graph.hpp:63-71). */
typedef struct sige_model_desc {
  const char* name;
  int in_channels, in_h, in_w;
  int num_layers;
  const sige_layer_desc* layers;
} sige_model_desc;

/* `sige::RunConfig` (graph.hpp:86-104). */
typedef struct sige_run_config {
  int step;
  float mask_threshold;
  int dilate_full;
  int dilate_scale;
  int block3;
  int block1;
  int min_sparse_res;
  int sparse;
  int norm_precompute;
  /* Ablation toggles of the reference's schedule (graph.cpp:571-582). Their
   * output is identical by the reference's own tests (test_graph.cpp:215-250);
   * the device executor always runs the fused schedule, so any value gives the
   * same result (tests/test_gpu_engine.py). */
  int elem_fusion;
  int scatter_fusion;
  uint32_t seed;
} sige_run_config;

/* Fills the reference defaults (graph.hpp:87-101). */
void sige_run_config_default(sige_run_config* cfg);

/* `sige::ScatterMap::Entry` (kernels.hpp:65-68): 8 bytes per pixel. */
typedef struct sige_scatter_entry {
  int32_t block;
  int16_t dy, dx;
} sige_scatter_entry;

/* Conv arithmetic for conv kernels and the engine. */
enum {
  SIGE_MATH_EXACT = 0, /* fp32 CUDA cores, reference accumulation order, no FMA: bit-exact */
  SIGE_MATH_TF32 = 1,  /* tcgen05.mma kind::tf32, fp32 accumulators in TMEM */
  SIGE_MATH_FP32_FMA = 2, /* fp32 CUDA cores with FMA (1e-4 check mode) */
  SIGE_MATH_F16 = 3 /* tcgen05.mma kind::f16 with fp16 operands, fp32 accumulators in TMEM */
};

/* ---- mask reduction (proj/include/sige/mask.hpp) -------------------------- */

/* compute_difference_mask (mask.hpp:31-32, mask.cpp:14-32). */
int sige_compute_difference_mask(const float* original, const float* edited, int n, int c,
                                 int h, int w, float threshold, uint8_t* mask_out,
                                 sige_stream_t stream);
/* downsample_mask (mask.hpp:36, mask.cpp:34-53). */
int sige_downsample_mask(const uint8_t* mask, int h, int w, int out_h, int out_w,
                         uint8_t* out, sige_stream_t stream);
/* dilate_mask (mask.hpp:40, mask.cpp:55-80). */
int sige_dilate_mask(const uint8_t* mask, int h, int w, int radius, uint8_t* out,
                     sige_stream_t stream);
/* mask_to_block_indices (mask.hpp:62-63, mask.cpp:103-136). Writes the
 * deterministic (n, r, c)-ordered set into `indices` (capacity triplets) and
 * the count into *count_device (device int). No host synchronisation. */
int sige_mask_to_block_indices_async(const uint8_t* mask, int h, int w, int block_size,
                                     int batch, int32_t* indices, int capacity,
                                     int32_t* count_device, sige_stream_t stream);
/* Same, then synchronises the stream and returns the count in *count_host. */
int sige_mask_to_block_indices(const uint8_t* mask, int h, int w, int block_size, int batch,
                               int32_t* indices, int capacity, int* count_host,
                               sige_stream_t stream);

/* ---- block kernels (proj/include/sige/kernels.hpp) ----------------------- */

/* gather (kernels.hpp:48-49, kernels.cpp:39-86). idx lives at the conv output
 * resolution idx_h x idx_w; out is (count, c, win, win), win = s*b + k - s. */
int sige_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count,
                int block_size, int idx_h, int idx_w, int k, int stride,
                const sige_epilogue* epilogue, float* out, sige_stream_t stream);
/* scatter_inplace (kernels.hpp:54, kernels.cpp:88-106): overlap-free blocks
 * (count, c, b, b) into base (n, c, h, w), clipped at the fringe. */
int sige_scatter_inplace(const float* blocks, int count, int channels, int block,
                         const int32_t* idx, float* base, int n, int c, int h, int w,
                         sige_stream_t stream);
/* scatter (kernels.hpp:53): out = copy of base, then scatter_inplace. */
int sige_scatter(const float* blocks, int count, int channels, int block, const int32_t* idx,
                 const float* base, float* out, int n, int c, int h, int w,
                 sige_stream_t stream);
/* scatter_add_inplace (kernels.hpp:57, kernels.cpp:114-132). */
int sige_scatter_add_inplace(const float* blocks, int count, int channels, int block,
                             const int32_t* idx, float* base, int n, int c, int h, int w,
                             sige_stream_t stream);
/* build_scatter_map (kernels.hpp:77, kernels.cpp:134-169): per-pixel
 * provenance over the first `per_sample` indices. Fails (ConfigError message)
 * if the tile pattern differs across the batch. */
int sige_build_scatter_map(const int32_t* idx, int count, int block, int h, int w,
                           sige_scatter_entry* map_out, int* blocks_per_sample_host,
                           sige_stream_t stream);
/* BlockIndexSet::content_hash (mask.cpp:91-101) of a device index set
 * (fnv1a64 over block, h, w, then every {n, r, c}); synchronises the stream. */
int sige_block_index_hash(const int32_t* idx, int count, int block, int h, int w, uint64_t* hash_out,
                          sige_stream_t stream);
/* ScatterMapCache::instance().get/size/clear (kernels.hpp:80-91,
 * kernels.cpp:171-202): a process-wide, mutex-protected memo of DEVICE scatter
 * maps keyed by the index set's content hash. get() builds the map on a miss
 * and returns the cache-owned map (h x w entries), blocks-per-sample and the
 * key; the map stays valid until sige_scatter_map_cache_clear(), which waits
 * for the device before freeing. */
int sige_scatter_map_cache_get(const int32_t* idx, int count, int block, int h, int w,
                               const sige_scatter_entry** map_out, int* blocks_per_sample,
                               uint64_t* key_out, sige_stream_t stream);
size_t sige_scatter_map_cache_size(void);
void sige_scatter_map_cache_clear(void);
/* scatter_gather (kernels.hpp:98-100, kernels.cpp:204-275). */
int sige_scatter_gather(const float* blocks, int count, int block, const float* original_out,
                        int n, int c, int h, int w, const sige_scatter_entry* map,
                        int blocks_per_sample, const int32_t* consumer_idx, int consumer_count,
                        int consumer_block, int consumer_h, int consumer_w, int k, int stride,
                        const sige_epilogue* epilogue, float* out, sige_stream_t stream);
/* scatter_with_block_residual (kernels.hpp:107-110, kernels.cpp:291-337). */
int sige_scatter_with_block_residual(const float* main_blocks, int main_count, int main_block,
                                     const int32_t* main_idx, const float* shortcut_blocks,
                                     int shortcut_count, int shortcut_block,
                                     const int32_t* shortcut_idx, const float* precomputed_sum,
                                     const float* original_shortcut, float* out, int n, int c,
                                     int h, int w, sige_stream_t stream);
/* scatter_with_block_residual_unfused (kernels.hpp:115-118, kernels.cpp:339-355). */
int sige_scatter_with_block_residual_unfused(
    const float* main_blocks, int main_count, int main_block, const int32_t* main_idx,
    const float* shortcut_blocks, int shortcut_count, int shortcut_block,
    const int32_t* shortcut_idx, const float* precomputed_sum, const float* original_shortcut,
    float* out, int n, int c, int h, int w, sige_stream_t stream);
/* add_blocks / subtract_blocks (kernels.hpp:121-122): out = a + sign*b over numel. */
int sige_combine_blocks(const float* a, const float* b, float sign, size_t numel, float* out,
                        sige_stream_t stream);
/* apply_epilogue_on_blocks (kernels.hpp:125, kernels.cpp:382-389). */
int sige_apply_epilogue_on_blocks(float* blocks, int count, int channels, int bh,
                                  const int32_t* idx, const sige_epilogue* epilogue,
                                  sige_stream_t stream);
/* conv_on_blocks (kernels.hpp:130-131, kernels.cpp:391-421): windows
 * (count, c_in, win, win) -> (count, c_out, b, b). conv weights are DEVICE. */
int sige_conv_on_blocks(const float* blocks, int count, int window, const sige_conv_desc* conv,
                        int with_bias, int math_mode, float* out, int block,
                        sige_stream_t stream);
/* conv2d dense (conv.hpp:35, conv.cpp:83-102). */
int sige_conv2d(const float* x, int n, int c, int h, int w, const sige_conv_desc* conv,
                int with_bias, int math_mode, float* out, sige_stream_t stream);

/* ---- engine: cached-activation state + sparse executor (graph.hpp) -------- */

typedef struct sige_engine sige_engine;

/* Uploads the model (host weight pointers) and allocates the device
 * ActivationCache (graph.hpp:116-156) and working buffers for `batch`. */
int sige_engine_create(const sige_model_desc* model, int batch, int math_mode,
                       sige_engine** out);
void sige_engine_destroy(sige_engine* eng);
/* precompute (graph.hpp:168-171, graph.cpp:426-435) on the device: one dense
 * pass over `original` (device NCHW) that fills the cache for `step`. */
int sige_engine_precompute(sige_engine* eng, const float* original, int step,
                           sige_stream_t stream);
/* ActivationCache lifecycle (graph.hpp:116-176). drop_step erases one step's
 * entries and frees their device memory (ActivationCache::drop_step,
 * graph.cpp:271-274); refresh_step replaces a step from a new original
 * (graph.cpp:437-444). The cache carries the structure hash of the model it
 * was built for (precompute sets the engine's own; a cache imported with
 * put_tensor/put_norm declares its producer's with set_cache_model_hash), and
 * sparse_forward fails with the reference's check_cache_model ConfigError
 * when it differs from the engine model's (graph.cpp:596-603). */
int sige_engine_drop_step(sige_engine* eng, int step);
/* Multi-step caches in host memory: offload_step copies one
 * step's entries to pinned host memory (kept as the step's home; the cache is
 * immutable after precompute) and frees their device memory; prefetch_step
 * uploads them again asynchronously on `stream` — order the step's next
 * sparse_forward after it. A sparse_forward on an offloaded step fails with the
 * reference's "precompute required" ConfigError. */
int sige_engine_offload_step(sige_engine* eng, int step, sige_stream_t stream);
int sige_engine_prefetch_step(sige_engine* eng, int step, sige_stream_t stream);
/* output_coverage (graph.hpp:190-192, graph.cpp:1078-1129) on the device: the
 * out_h x out_w u8 map (device buffer) of output pixels a sparse_forward of
 * this edit may change — computed from the same on-device IndexPlan the
 * executor runs (mask = NULL: difference against the cached original). */
int sige_engine_output_coverage(sige_engine* eng, const float* edited, const uint8_t* mask,
                                const sige_run_config* cfg, uint8_t* out, int* out_h, int* out_w,
                                sige_stream_t stream);
int sige_engine_refresh_step(sige_engine* eng, const float* original, int step, sige_stream_t stream);
int sige_engine_cache_model_hash(const sige_engine* eng, uint64_t* cache_hash, uint64_t* model_hash);
int sige_engine_set_cache_model_hash(sige_engine* eng, uint64_t cache_hash);
/* ModelSpec::structure_hash (graph.cpp:89-127). */
uint64_t sige_model_structure_hash(const sige_model_desc* model);
/* Upload one cache entry (host NCHW tensor or n*C folded norm) from a CPU
 * precompute, for parity runs. key follows graph.cpp:356-410 ("L3.conv1.out",
 * "L0.norm", "final", ...). For norms pass scale and shift (n*C each). */
int sige_engine_put_tensor(sige_engine* eng, int step, const char* key, const float* host_nchw,
                           size_t numel);
int sige_engine_put_norm(sige_engine* eng, int step, const char* key, const float* host_scale,
                         const float* host_shift, size_t numel);
/* Download a cache entry (host NCHW) — for tests. */
int sige_engine_get_tensor(sige_engine* eng, int step, const char* key, float* host_nchw,
                           size_t numel);
/* Download a folded norm entry (scale, shift: `numel` values each). */
int sige_engine_get_norm(sige_engine* eng, int step, const char* key, float* host_scale,
                         float* host_shift, size_t numel);
/* sparse_forward (graph.hpp:224-226, graph.cpp:619-901). edited is device NCHW;
 * mask (device u8 H*W) may be NULL, in which case the engine computes it
 * against the cached original input with cfg->mask_threshold (mask.cpp:14-32).
 * out is device NCHW of the model output shape. No host synchronisation. */
int sige_engine_sparse_forward(sige_engine* eng, const float* edited, const uint8_t* mask,
                               const sige_run_config* cfg, float* out, sige_stream_t stream);
/* Grouped independent requests (config 5; no reference counterpart — the
 * reference runs one request per call, graph.hpp:224-226): every batch sample
 * of the engine is its own request, with its own original (precompute), edited
 * input and difference mask (`masks`: batch x H x W u8, or NULL to compute
 * each sample's mask against its cached original with cfg->mask_threshold).
 * Per-sample IndexPlans are concatenated n-major into each layer's tile list,
 * so one launch per layer serves all requests; sample n's output equals a
 * batch-1 sparse_forward of request n (empty mask -> its cached final). */
int sige_engine_sparse_forward_grouped(sige_engine* eng, const float* edited, const uint8_t* masks,
                                       const sige_run_config* cfg, float* out, sige_stream_t stream);
/* Same through HOST buffers: H2D of edited (and mask when non-NULL), run,
 * D2H of the output, stream synchronised on return. */
int sige_engine_sparse_forward_host(sige_engine* eng, const float* edited_host,
                                    const uint8_t* mask_host, const sige_run_config* cfg,
                                    float* out_host, sige_stream_t stream);
/* dense_forward (graph.hpp:179) on the device; reused_stats != 0 gives
 * dense_forward_reused_stats (graph.hpp:184-186) with cached folded norms. */
int sige_engine_dense_forward(sige_engine* eng, const float* input, int reused_stats, int step,
                              float* out, sige_stream_t stream);
/* Output shape of the model. */
int sige_engine_output_shape(const sige_engine* eng, int* n, int* c, int* h, int* w);
/* Host-side plan summary of the last sparse_forward launch list (for traces):
 * number of kernels launched per sparse_forward call. */
int sige_engine_last_launch_count(const sige_engine* eng);
/* Per-layer trace (RunTrace, graph.hpp:194-216) of the last run: copies up
 * to `cap` rows of {active_blocks, gathered_elems, scattered_elems, macs,
 * dense_macs, ran_sparse} as uint64 sextuples; returns rows in *rows.
 * Synchronises the stream. */
int sige_engine_trace(sige_engine* eng, uint64_t* rows, int cap, int* nrows,
                      sige_stream_t stream);
/* Per-conv-launch profiling (CUDA events around each fused conv launch of
 * subsequent engine calls; off by default). sige_engine_profile_read
 * synchronises the stream and returns up to `cap` rows of {ms, algorithmic
 * flops (2*MACs over the tiles actually processed), tensor-core flag}, then
 * clears the record. */
int sige_engine_set_profiling(sige_engine* eng, int enable);
/* CUDA-graph replay of sparse_forward (on by default): after one direct run,
 * each (edited, mask, out) pointer binding is captured once and replayed with a
 * single graph launch. Results are identical either way. */
int sige_engine_set_graphs(sige_engine* eng, int enable);
/* SM budget of this engine's launches (0 = every SM): with several engines
 * (independent requests) in flight on one GPU each launch sizes its grid and
 * N tile for its share, so the requests' latency-bound kernels run side by
 * side instead of each filling the GPU. No reference counterpart (the
 * reference runs one request per call, graph.hpp:224-226). */
int sige_engine_set_sm_budget(sige_engine* eng, int sms);
int sige_engine_profile_read(sige_engine* eng, double* rows, int cap, int* nrows,
                             sige_stream_t stream);
/* Graph timeline (measurement; no reference counterpart): with it on, every
 * tensor-core conv launch of a call stamps %globaltimer at its first CTA's
 * start, its dependency-wait exit and its last CTA's end — inside replayed
 * CUDA graphs, so PDL overlap is kept (captured graphs are re-captured when
 * the switch changes). sige_engine_timeline_read synchronises the device and
 * returns up to `cap` rows {start_ns, end_ns, wait_ns, algorithmic flops,
 * sparse flag} of the last call's launches (times relative to the first
 * start), then resets the stamps. */
int sige_engine_set_timeline(sige_engine* eng, int enable);
int sige_engine_timeline_read(sige_engine* eng, double* rows, int cap, int* nrows);
/* Newline-separated cache listing for `step`: "T <key> <n> <c> <h> <w>" for
 * tensors (reference NCHW shape) and "N <key> <count>" for folded norms.
 * Returns the needed buffer size in *needed. */
int sige_engine_cache_entries(const sige_engine* eng, int step, char* buf, size_t cap,
                              size_t* needed);
/* Bytes of device memory held by the cache (ActivationCache::element_breakdown
 * * 4, graph.cpp:287-302). */
size_t sige_engine_cache_bytes(const sige_engine* eng);

/* ---- synthetic inputs (fixtures.hpp, models.hpp) -------------------------- */

/* Config 3 input: a one-hot segmentation map (n, label_nc, h, w) of random
 * labelled rectangles and its edit — a rect1-style square (1.2 % of the
 * pixels) relabelled, the GauGAN edit of SIGE. Host buffers. */
int sige_make_seg_fixture(int n, int label_nc, int h, int w, uint32_t seed, float* orig, float* edited);
/* make_edit_fixture (fixtures.hpp:23-24, fixtures.cpp:105-128) into host
 * buffers of n*c*h*w floats. Returns SIGE_ERR_CONFIG for unknown kinds. */
int sige_make_edit_fixture(const char* kind, int n, int c, int h, int w, uint32_t seed,
                           float* original_host, float* edited_host);
/* Builds one of the named synthetic models ("conv3x3_128", "mini_unet_gn",
 * "mini_unet_bn", "gaugan_stack_in" (models.cpp:91-161), "single_conv64"
 * (config 1), "ddim_stack" (config 2)). The returned descriptor and its
 * weights stay valid until sige_model_free. */
int sige_model_build(const char* name, sige_model_desc** out);
void sige_model_free(sige_model_desc* model);
/* required_dilation (graph.hpp:81, graph.cpp:195-218). */
int sige_model_required_dilation(const sige_model_desc* model, int* out);
/* model_weight_hash (models.hpp:17, models.cpp:185-207). */
uint64_t sige_model_weight_hash(const sige_model_desc* model);

/* ---- SPADE ops (BASELINE config 3, GauGAN SPADE ResBlocks) -----------------
 * Not in the reference API (per-pixel gamma/beta exceed Epilogue's
 * per-channel params; no label-map resample); restated in
 * oracle/sige_oracle.c (orc_gather_spade, orc_resize_nearest), parity bit-exact.
 *
 * gather with SPADE modulation: for every in-canvas cell of each window
 * (geometry and validation exactly as sige_gather), v = x, then the `norm`
 * chain (the folded, param-free norm as scale-shift steps: p = a*v, v = p + b),
 * then v = v * (1 + gamma) + beta with gamma/beta the per-pixel modulation
 * maps (n, c, h, w) at the same cell (two roundings each), then `act`
 * (SIGE_ACT_*). Out-of-canvas cells stay +0. */
int sige_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                      const int32_t* idx, int count, int block, int idx_h, int idx_w, int k, int stride,
                      const sige_epilogue* norm, int act, float* out, sige_stream_t s);
/* Nearest resample of a (segmentation / label) map by integer factors per
 * axis (down: sample (y*f, x*f); up: replicate), = torch nearest for integer
 * ratios. Non-integer ratios fail with "resize_nearest: non-integer scale". */
int sige_resize_nearest(const float* in, int n, int c, int h, int w, int out_h, int out_w, float* out,
                        sige_stream_t s);

/* ---- on-disk exchange formats (io.hpp:12-36, io.cpp) ----------------------
 * Host buffers, host files. Same byte layouts and ConfigError messages as the
 * reference; files written here load in the reference and vice versa. */

/* save_tensor (io.hpp:14, io.cpp:34-51,87-91): SIGT v1, little-endian. */
int sige_save_tensor(const char* path, const float* host, int n, int c, int h, int w);
/* load_tensor (io.hpp:15, io.cpp:58-85,93-102): dims[4] = n,c,h,w; pass
 * host = NULL to read the header only. Zero dimensions are rejected. */
int sige_load_tensor(const char* path, float* host, size_t cap, int* dims);
/* save_mask_pbm (io.hpp:18, io.cpp:104-114): plain PBM (P1). */
int sige_save_mask_pbm(const char* path, const uint8_t* mask, int h, int w);
/* load_mask_pbm (io.hpp:19, io.cpp:118-160): *h, *w always; mask = NULL for
 * the header only. Comments and unseparated digits are accepted. */
int sige_load_mask_pbm(const char* path, uint8_t* mask, size_t cap, int* h, int* w);
/* save_block_stack (io.hpp:33, io.cpp:405-421): <prefix>.sigt payload
 * (count, channels, block+overlap, block+overlap) + <prefix>.json sidecar
 * ("sige_blocks_v1", byte-identical to the reference's dump). */
int sige_save_block_stack(const char* prefix, const float* host, int count, int channels, int block, int overlap,
                          int origin_block, int origin_h, int origin_w, const int32_t* idx);
/* load_block_stack (io.hpp:34, io.cpp:423-457): meta[7] = {count, channels,
 * block, overlap, origin_block, origin_h, origin_w}; host / idx may be NULL
 * (header only). */
int sige_load_block_stack(const char* prefix, float* host, size_t cap, int32_t* idx, size_t idx_cap, int* meta);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SIGE_B200_H_ */
