// engine.hpp — device-resident ActivationCache + sparse executor.
//
// Mirrors, on the device, the reference's graph layer
// (proj/include/sige/graph.hpp:116-226, proj/src/graph.cpp:343-901):
//   * ActivationCache: (step, key) -> NHWC device tensor / folded norm params;
//   * precompute / dense_forward(_reused_stats): the dense walk;
//   * sparse_forward: the Flow executor, compiled once per (step, RunConfig)
//     into a "program" — an ordered list of kernel launches over device-side
//     index sets produced by the on-device IndexPlan, so a call never
//     synchronises with the host.
// Scatters write tiles into per-key working copies of the cached outputs
// ("W" buffers) instead of copying whole tensors (kernels.cpp:108-112); the
// tiles a call dirtied are restored from the cache at the start of the next
// call, so the cache itself stays immutable.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "common.hpp"
#include "engine_kernels.hpp"
#include "models.hpp"

namespace sige_b200 {

struct DevTensor {
  float* p = nullptr;  // fp32 storage, or fp16 when `half` (activation buffers)
  int n = 0, c = 0, h = 0, w = 0;
  int layout = kNHWC;
  int half = 0;
  void* h16 = nullptr;  // fp16 twin (F16 mode, tensors that feed convolutions)
  size_t numel() const { return static_cast<size_t>(n) * c * h * w; }
  size_t bytes() const { return numel() * (half ? 2 : 4); }
};

struct DevNorm {
  float* scale = nullptr;
  float* shift = nullptr;
  int np = 0;
};

struct LayerDev {
  int kind = 0, act = 0, has_shortcut = 0, policy_sparse = 1, min_resolution = 16;
  ConvW conv, conv2, shortcut;
  int norm_kind = 0, groups = 1, channels = 0;
  float eps = 1e-5f;
  float *gamma = nullptr, *beta = nullptr, *rmean = nullptr, *rvar = nullptr;
  // SPADE_RESBLOCK (config 3): per SPADE norm k (0: conv_0's input, 1:
  // conv_1's, 2: the shortcut's) the shared conv (segmentation -> hidden,
  // then ReLU) and gamma/beta stacked into one conv (hidden -> 2C: gamma
  // channels first), the instance-norm eps and its param-free affine (ones,
  // zeros) for the fold.
  int n_spade = 0;
  ConvW spade_shared[3], spade_gb[3];
  float spade_eps[3] = {1e-5f, 1e-5f, 1e-5f};
  float *spade_ones[3] = {}, *spade_zeros[3] = {};
  int resize_h = 0, resize_w = 0;  // RESIZE
};

struct TraceInfo {
  int entry = -1;  // plan entry (sparse) or -1 (dense)
  int c_in = 0, c_out = 0, k = 1, stride = 1, oh = 0, ow = 0, batch = 1;
};

struct Program;


class Engine {
 public:
  Engine(const sige_model_desc* model, int batch, int math);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void precompute(const float* original_nchw, int step, cudaStream_t st);
  // ActivationCache lifecycle (graph.hpp:116-176): drop_step erases one
  // step's entries (graph.cpp:271-274); refresh_step replaces them from a new
  // original (graph.cpp:437-444); the cache's model hash guards sparse_forward
  // against a cache built for another model (check_cache_model, graph.cpp:596-603).
  void drop_step(int step);
  void refresh_step(const float* original_nchw, int step, cudaStream_t st);
  // Multi-step caches in host memory ("store the activations in
  // CPU memory and load the on-demand ones on GPU"): offload_step moves one
  // step's entries to pinned host memory and frees their device memory;
  // prefetch_step brings them back asynchronously on `st` (the caller orders
  // the step's next sparse_forward after it, e.g. with an event).
  void offload_step(int step, cudaStream_t st);
  void prefetch_step(int step, cudaStream_t st);
  bool step_offloaded(int step) const;
  uint64_t structure_hash() const { return structure_hash_; }
  uint64_t cache_model_hash() const { return cache_model_hash_; }
  void set_cache_model_hash(uint64_t h) { cache_model_hash_ = h; }
  void put_tensor(int step, const std::string& key, const float* host_nchw, size_t numel);
  void put_norm(int step, const std::string& key, const float* sc, const float* sh, size_t np);
  void get_tensor(int step, const std::string& key, float* host_nchw, size_t numel);
  void get_norm(int step, const std::string& key, float* sc, float* sh, size_t np);
  // grouped: every batch sample is an independent request with its own
  // difference mask (mask: batch x H x W when given) — per-sample IndexPlans
  // concatenated n-major into each layer's tile list, one launch per layer for
  // all requests; each sample's output equals a batch-1 sparse_forward of that
  // request (graph.cpp:619-901). Otherwise one mask is shared by the batch.
  void sparse_forward(const float* edited, const uint8_t* mask, const sige_run_config& cfg,
                      float* out, cudaStream_t st, bool grouped = false);
  void dense_forward(const float* in, bool reused_stats, int step, float* out, cudaStream_t st);

  void output_shape(int* n, int* c, int* h, int* w) const;
  int last_launch_count() const { return last_launches_; }
  int trace(uint64_t* rows, int cap, cudaStream_t st);
  void output_coverage(const float* edited, const uint8_t* mask, const sige_run_config& cfg, uint8_t* out, int* oh,
                       int* ow, cudaStream_t st);
  size_t cache_bytes() const;
  void set_profiling(bool on);
  void set_graphs(bool on);
  // Graph timeline of the conv launches (device stamps inside replayed
  // graphs): on/off, and read rows [start_ns, end_ns, wait_ns, flops, sparse]
  // (times relative to the first launch's start) of the last call, then reset.
  void set_timeline(bool on);
  int timeline_read(double* rows, int cap);
  void set_sm_budget(int sms);
  int profile_read(double* rows, int cap, cudaStream_t st);
  std::string cache_entries(int step) const;
  int in_channels() const { return in_c_; }
  int in_h() const { return in_h_; }
  int in_w() const { return in_w_; }
  int batch() const { return batch_; }

 private:
  friend struct ProgramBuilder;
  // conv dispatch by math mode
  void conv(const Src& src, const Tiles& t, const ConvW& cw, const Dst& dst, cudaStream_t st) const;
  const DevTensor& cache_tensor(int step, const std::string& key) const;
  const DevNorm& cache_norm(int step, const std::string& key) const;
  DevTensor& cache_slot(int step, const std::string& key, int c, int h, int w, int layout, int half = 0);
  // F16 mode: layer outputs that later convolutions read (".out" of Conv /
  // Downsample layers, ".sum" of ResBlocks) carry an fp16 twin written by the
  // producing kernel's epilogue.
  bool wants_twin(const std::string& key, int layout, int half) const;
  void attach_twin(DevTensor& t, const std::string& key);
  void force_twin(DevTensor& t);
  // F16 + GroupNorm/InstanceNorm ResBlocks with fresh statistics (dense
  // fallback, dense_forward): conv1's epilogue accumulates the statistics,
  // conv2 folds them and applies norm + act to its staged window in shared
  // memory (no separate statistics / fold / activation kernels).
  // (The folded table of n x C scale/shift pairs lives in shared memory:
  // batches beyond 4096 / C channels take the separate fold + act path.)
  bool fused_gn(const LayerDev& L) const {
    return math_ == SIGE_MATH_F16 && L.norm_kind != SIGE_NORM_BATCH &&
           static_cast<long long>(batch_) * std::max(L.channels, L.conv2.c_in) <= 4096;
  }
  double* dense_stats_ = nullptr;  // statistics arena of dense walks (zeroed per walk)
  // F16: fp16 channels-last copy of the current input (channels padded to 8),
  // written by k_input_twin at the start of each call; the first conv streams it.
  void* in_twin_ = nullptr;
  int in_twin_c_ = 0;
  Src input_src(const float* ptr, cudaStream_t st, bool convert);
  size_t dense_stats_len_ = 0;
  size_t stats_len() const;        // doubles needed by all ResBlocks of the model
  DevNorm& norm_slot(int step, const std::string& key, int np);
  DevTensor& work_buffer(int step, const std::string& key);
  DevTensor& scratch(const std::string& key, int c, int h, int w, int layout, int half = 0);
  // Activation buffers (tensor-core modes): conv2 of a ResBlock stages
  // act1 = act(norm1(conv1.out)) instead of re-applying the chain.
  bool use_act() const { return tensor_cores(); }
  int act_half() const { return math_ == SIGE_MATH_F16 ? 1 : 0; }
  const DevTensor& ensure_act(int step, const std::string& key, int layer, cudaStream_t st);
  DevNorm& scratch_norm(const std::string& key, int np);
  Tiles dense_tiles(int oh, int ow, int k, int s);
  std::pair<int, int> dense_shape(int oh, int ow, int k, int s) const;
  bool tensor_cores() const { return math_ == SIGE_MATH_TF32 || math_ == SIGE_MATH_F16; }
  static constexpr int kGnScratch = 1 << 16;
  double* gn_scratch_ = nullptr;
  void invalidate_programs();
  void drop_act(int step);
  void dense_walk(const Src& input, int step, bool capture, bool reused, float* out_nchw,
                  cudaStream_t st);
  Program& program(const sige_run_config& cfg, bool grouped);
  void run_program(Program& P, const float* edited, const uint8_t* mask, const sige_run_config& cfg,
                   cudaStream_t st);
  bool use_graphs_ = true;
  int sm_budget_ = 0;  // 0 = every SM
  cudaStream_t cap_stream_ = nullptr;
  // fork/join for work off the launch chain (the input twin)
  cudaStream_t side_stream_ = nullptr;
  cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
  // Program branch (SPADE): the label-map convs of every SPADE norm depend on
  // the input only and run on this stream ahead of the main chain; events
  // order them (graph edges when captured). Created at program build time.
  cudaStream_t br_stream_ = nullptr;
  std::vector<cudaEvent_t> br_events_;
  static constexpr size_t kBrDense = 64;  // spade_dense's events: [64, 68) (programs use 0..63)
  cudaEvent_t br_event(size_t i) {
    while (br_events_.size() <= i) {
      cudaEvent_t e;
      SIGE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      br_events_.push_back(e);
    }
    if (!br_stream_) SIGE_CUDA(cudaStreamCreateWithFlags(&br_stream_, cudaStreamNonBlocking));
    return br_events_[i];
  }
  void fold_norm(const LayerDev& L, const Src& x, DevNorm& out, cudaStream_t st);
  // Config 3: a SPADE residual block over every pixel (dense walk / dense
  // fallback; buffers from `tensor` / `norm`, statistics folded unless
  // `reused`) — returns the block output; and the segmentation map (the model
  // input `in`, NCHW) nearest-resized to (h, w) as an NHWC source.
  Src spade_dense(const LayerDev& L, int li, const Src& x, const Src& seg, bool reused,
                  const std::function<DevTensor&(const std::string&, int, int)>& tensor,
                  const std::function<DevNorm&(const std::string&, int)>& norm, cudaStream_t st);
  Src seg_at(const float* in, int h, int w, DevTensor& buf, cudaStream_t st);

  std::string name_;
  struct HostEntry {  // an offloaded cache entry (pinned host copies)
    DevTensor meta;     // shape / layout (device pointers unset)
    void* host = nullptr;
    void* host16 = nullptr;  // fp16 twin, if the entry had one
  };
  struct HostNorm {
    int np = 0;
    float* scale = nullptr;  // pinned, np each
    float* shift = nullptr;
  };
  std::map<std::pair<int, std::string>, HostEntry> host_cache_;
  std::map<std::pair<int, std::string>, HostNorm> host_norms_;
  uint64_t structure_hash_ = 0;     // of the engine's model
  uint64_t cache_model_hash_ = 0;   // of the model the cache was built for
  int batch_, math_, in_c_, in_h_, in_w_;
  int out_c_ = 0, out_h_ = 0, out_w_ = 0;
  std::vector<LayerDev> layers_;
  std::vector<LayerShape> shapes_;
  std::vector<void*> allocations_;
  std::map<std::pair<int, std::string>, DevTensor> cache_;
  std::map<std::pair<int, std::string>, DevNorm> norms_;
  std::map<std::pair<int, std::string>, DevTensor> work_;
  std::map<std::string, DevTensor> scratch_;
  std::map<std::string, DevNorm> scratch_norms_;
  std::map<std::tuple<int, int, int, int>, std::pair<int32_t*, int>> dense_tiles_;
  std::map<std::string, std::unique_ptr<Program>> programs_;
  Program* last_program_ = nullptr;
  int last_launches_ = 0;
  struct ProfRec {
    cudaEvent_t a, b;
    const int32_t* count_dev;
    int count;
    double flops_per_tile;
    int tc;
  };
  bool profiling_ = false;
  mutable std::vector<ProfRec> prof_;
  // Graph timeline (set_timeline): every tensor-core conv launch of a call
  // stamps [start, end, dependency-wait exit] with %globaltimer into tl_buf_,
  // indexed by launch order within the call; valid inside replayed graphs.
  struct TlMeta {
    const int32_t* count_dev;
    int count;
    double flops_per_tile;
    int sparse;
  };
  bool timeline_ = false;
  unsigned long long* tl_buf_ = nullptr;
  mutable int tl_next_ = 0;
  mutable std::vector<TlMeta> tl_meta_;
  void timeline_reset();
  void drop_graphs();
  mutable std::vector<cudaEvent_t> ev_pool_;
  // per-call bindings read by program steps
  const float* cur_in_ = nullptr;
  float* cur_out_ = nullptr;
  void* alloc(size_t bytes);
  void release(void* p);  // frees an alloc() block early (dropped cache entries)
  void free_device_step(int step);
  void free_host_step(int step);
};

}  // namespace sige_b200
