// engine.cpp — device ActivationCache, dense walk (precompute / dense_forward)
// and the compiled sparse_forward executor. See engine.hpp.
#include "engine.hpp"
#include "ops.hpp"

#include <algorithm>
#include <cstdio>
#include <tuple>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>

namespace sige_b200 {

namespace {

std::string lk(int i) { return "L" + std::to_string(i); }

// layer_runs_sparse (graph.cpp:478-483).
bool runs_sparse(const LayerDev& L, int h, int w, const sige_run_config& cfg) {
  if (!cfg.sparse || !L.policy_sparse) return false;
  int thr = cfg.min_sparse_res >= 0 ? cfg.min_sparse_res : L.min_resolution;
  return std::min(h, w) >= thr;
}

void epi_push_ss(DevEpilogue& e, const float* sc, const float* sh, int np, int channels) {
  if (e.num_steps >= SIGE_MAX_EPI_STEPS)
    throw ConfigError("epilogue: more than " + std::to_string(SIGE_MAX_EPI_STEPS) +
                      " pending element-wise steps");
  const int s = e.num_steps++;
  e.kind[s] = SIGE_EPI_SCALE_SHIFT;
  e.per_sample[s] = np != channels ? 1 : 0;
  e.scale[s] = sc;
  e.shift[s] = sh;
}

void epi_push_act(DevEpilogue& e, int act) {
  if (act == SIGE_ACT_NONE) return;  // Epilogue::add_activation (eltwise.cpp:99-105)
  if (e.num_steps >= SIGE_MAX_EPI_STEPS)
    throw ConfigError("epilogue: more than " + std::to_string(SIGE_MAX_EPI_STEPS) +
                      " pending element-wise steps");
  const int s = e.num_steps++;
  e.kind[s] = SIGE_EPI_ACTIVATION;
  e.act[s] = act;
}

Src plain(const DevTensor& t) {
  Src s;
  s.ptr = t.p;
  s.layout = t.layout;
  s.n = t.n;
  s.c = t.c;
  s.h = t.h;
  s.w = t.w;
  s.half = t.half;
  s.epi.fma_expf = host_expf_is_fma() ? 1 : 0;
  s.twin = t.h16;
  return s;
}

Dst to_dst(const DevTensor& t, int mode = kStore) {
  Dst d;
  d.ptr = t.p;
  d.n = t.n;
  d.c = t.c;
  d.h = t.h;
  d.w = t.w;
  d.mode = mode;
  if (t.h16) {  // the epilogue also writes the fp16 twin (identity chain)
    d.act = t.h16;
    d.act_half = 1;
  }
  return d;
}

bool ends_with(const std::string& s, const char* suf) {
  const size_t n = std::strlen(suf);
  return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}

}  // namespace

// A compiled sparse_forward for one (step, RunConfig): plan entries, ordered
// launches, restore jobs, trace metadata.
struct Program {
  std::vector<PlanEntryDev> entries;
  PlanEntryDev* entries_dev = nullptr;
  std::vector<std::function<void(cudaStream_t)>> steps;
  std::vector<RestoreJob> restores;
  RestoreJob* restores_dev = nullptr;
  long long restore_max = 0;
  std::vector<TraceInfo> trace;
  uint32_t* bits = nullptr;
  int32_t* any = nullptr;
  int full_h = 0, full_w = 0, dilate_full = 0, dilate_scale = 0;
  int launches = 0;
  bool ran = false;
  bool grouped = false;  // per-sample masks (independent requests)
  // Tile-based result: the call's output starts as a copy of the cached final
  // (off the critical path, beside the mask / IndexPlan) and the last layer's
  // tiles are written straight into it — no full-tensor finalize at the tail.
  const float* out_from_cache = nullptr;
  size_t out_bytes = 0;
  double* stats = nullptr;  // GroupNorm statistics arena (fused dense-fallback ResBlocks), zeroed per call
  size_t stats_len = 0, stats_used = 0;
  // captured calls keyed by (edited, mask, out, threshold bits): without a
  // mask the threshold is baked into the captured k_mask_bits launch
  std::map<std::tuple<const void*, const void*, const void*, uint32_t>, std::pair<cudaGraphExec_t, int>> graphs;
  ~Program() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.first);
  }
};

// ----------------------------------------------------------- basics -----

Engine::Engine(const sige_model_desc* m, int batch, int math) : batch_(batch), math_(math) {
  if (batch < 1) throw ConfigError("engine: batch must be >= 1");
  if (math != SIGE_MATH_EXACT && math != SIGE_MATH_TF32 && math != SIGE_MATH_FP32_FMA &&
      math != SIGE_MATH_F16)
    throw ConfigError("engine: unknown math mode " + std::to_string(math));
  shapes_ = walk_shapes(m);
  name_ = m->name ? m->name : "";
  structure_hash_ = cache_model_hash_ = model_structure_hash(m);
  in_c_ = m->in_channels;
  in_h_ = m->in_h;
  in_w_ = m->in_w;
  out_c_ = shapes_.back().c_out;
  out_h_ = shapes_.back().h_out;
  out_w_ = shapes_.back().w_out;
  auto upload = [&](const float* host, size_t n) -> float* {
    if (!host) return nullptr;
    float* d = static_cast<float*>(alloc(n * sizeof(float)));
    SIGE_CUDA(cudaMemcpy(d, host, n * sizeof(float), cudaMemcpyHostToDevice));
    return d;
  };
  auto up_conv = [&](const sige_conv_desc& c) {
    ConvW w;
    w.c_in = c.c_in;
    w.c_out = c.c_out;
    w.k = c.k;
    w.stride = c.stride;
    w.w = upload(c.weight, static_cast<size_t>(c.c_out) * c.c_in * c.k * c.k);
    w.bias = upload(c.bias, c.c_out);
    if (tensor_cores()) {
      pack_weights_tc(w.w, c.c_out, c.c_in, c.k, math_ == SIGE_MATH_F16 ? 1 : 0, &w, nullptr);
      allocations_.push_back(const_cast<void*>(w.w_tc));
    }
    return w;
  };
  for (int i = 0; i < m->num_layers; ++i) {
    const sige_layer_desc& d = m->layers[i];
    LayerDev L;
    L.kind = d.kind;
    L.act = d.act;
    L.policy_sparse = d.policy_sparse;
    L.min_resolution = d.min_resolution;
    if (d.kind == SIGE_LAYER_CONV || d.kind == SIGE_LAYER_DOWNSAMPLE || d.kind == SIGE_LAYER_RESBLOCK)
      L.conv = up_conv(d.conv);
    if (d.kind == SIGE_LAYER_RESBLOCK) {
      L.conv2 = up_conv(d.conv2);
      L.has_shortcut = d.has_shortcut;
      if (d.has_shortcut) L.shortcut = up_conv(d.shortcut);
    }
    if (d.kind == SIGE_LAYER_SPADE_RESBLOCK) {
      L.conv = up_conv(d.conv);
      L.conv2 = up_conv(d.conv2);
      L.has_shortcut = d.has_shortcut;
      if (d.has_shortcut) L.shortcut = up_conv(d.shortcut);
      L.n_spade = d.has_shortcut ? 3 : 2;
      for (int k = 0; k < L.n_spade; ++k) {
        const sige_spade_desc& sp = d.spade[k];
        L.spade_shared[k] = up_conv(sp.shared);
        L.spade_eps[k] = sp.eps;
        // gamma and beta as one conv: output channels [gamma | beta]
        const int C = sp.gamma.c_out, nh = sp.gamma.c_in;
        const size_t wn = static_cast<size_t>(C) * nh * 9;
        std::vector<float> w2(2 * wn), b2(2 * static_cast<size_t>(C), 0.0f);
        std::memcpy(w2.data(), sp.gamma.weight, wn * sizeof(float));
        std::memcpy(w2.data() + wn, sp.beta.weight, wn * sizeof(float));
        if (sp.gamma.bias) std::memcpy(b2.data(), sp.gamma.bias, C * sizeof(float));
        if (sp.beta.bias) std::memcpy(b2.data() + C, sp.beta.bias, C * sizeof(float));
        const sige_conv_desc gb{nh, 2 * C, 3, 1, w2.data(), b2.data()};
        L.spade_gb[k] = up_conv(gb);
        const std::vector<float> ones(C, 1.0f), zeros(C, 0.0f);
        L.spade_ones[k] = upload(ones.data(), C);
        L.spade_zeros[k] = upload(zeros.data(), C);
      }
    }
    if (d.kind == SIGE_LAYER_RESIZE) {
      if (i != 0) throw ConfigError("model layer L" + std::to_string(i) + ": resize is supported on the input only");
      L.resize_h = d.resize_h;
      L.resize_w = d.resize_w;
    }
    if (d.kind == SIGE_LAYER_NORM || d.kind == SIGE_LAYER_RESBLOCK) {
      const sige_norm_desc& n = d.norm;
      L.norm_kind = n.kind;
      L.groups = n.groups;
      L.channels = n.channels;
      L.eps = n.eps;
      L.gamma = upload(n.gamma, n.channels);
      L.beta = upload(n.beta, n.channels);
      L.rmean = upload(n.running_mean, n.channels);
      L.rvar = upload(n.running_var, n.channels);
      if (n.kind == SIGE_NORM_BATCH && (!L.rmean || !L.rvar))
        throw ConfigError("norm: batch kind requires per-channel running stats");
    }
    layers_.push_back(L);
  }
  for (const LayerDev& L : layers_)  // SPADE models: branch stream + events up front (never created under capture)
    if (L.kind == SIGE_LAYER_SPADE_RESBLOCK) {
      br_event(kBrDense + 3);
      break;
    }
}

Engine::~Engine() {
  cudaDeviceSynchronize();
  programs_.clear();  // destroys captured graphs
  for (auto& r : prof_) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  if (cap_stream_) cudaStreamDestroy(cap_stream_);
  if (side_stream_) cudaStreamDestroy(side_stream_);
  if (br_stream_) cudaStreamDestroy(br_stream_);
  for (cudaEvent_t e : br_events_) cudaEventDestroy(e);
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  if (join_ev_) cudaEventDestroy(join_ev_);
  for (void* p : allocations_) cudaFree(p);
  for (auto& kv : host_cache_) {
    cudaFreeHost(kv.second.host);
    if (kv.second.host16) cudaFreeHost(kv.second.host16);
  }
  for (auto& kv : host_norms_) {
    cudaFreeHost(kv.second.scale);
    cudaFreeHost(kv.second.shift);
  }
}

void* Engine::alloc(size_t bytes) {
  void* p = nullptr;
  SIGE_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
  allocations_.push_back(p);
  return p;
}

void Engine::output_shape(int* n, int* c, int* h, int* w) const {
  *n = batch_;
  *c = out_c_;
  *h = out_h_;
  *w = out_w_;
}

size_t Engine::cache_bytes() const {
  size_t b = 0;
  for (auto& kv : cache_)
    if (kv.first.second != "input") b += kv.second.numel() * sizeof(float);
  for (auto& kv : norms_) b += 2 * sizeof(float) * kv.second.np;
  return b;
}

const DevTensor& Engine::cache_tensor(int step, const std::string& key) const {
  auto it = cache_.find({step, key});
  if (it == cache_.end())
    throw ConfigError("precompute required: no cache entry for step " + std::to_string(step) +
                      ", layer " + key);  // graph.cpp:242-248
  return it->second;
}

const DevNorm& Engine::cache_norm(int step, const std::string& key) const {
  auto it = norms_.find({step, key});
  if (it == norms_.end())
    throw ConfigError("precompute required: no cached norm params for step " +
                      std::to_string(step) + ", layer " + key);  // graph.cpp:250-258
  return it->second;
}

bool Engine::wants_twin(const std::string& key, int layout, int half) const {
  if (math_ != SIGE_MATH_F16 || layout != kNHWC || half) return false;
  if (ends_with(key, ".sum") || ends_with(key, ".mod")) return true;
  if (ends_with(key, ".conv0.out") || ends_with(key, ".sc.out")) return false;  // read by the modulation / join only
  return ends_with(key, ".out") && !ends_with(key, "conv1.out") && !ends_with(key, "conv2.out") &&
         !ends_with(key, "shortcut.out");
}

void Engine::attach_twin(DevTensor& t, const std::string& key) {
  if (wants_twin(key, t.layout, t.half) && !t.h16) t.h16 = alloc(t.numel() * 2);
}

// The NCHW input as a Src; in F16 mode with its fp16 channels-last twin
// (converted here when `convert`, i.e. outside the captured step).
Src Engine::input_src(const float* ptr, cudaStream_t st, bool convert) {
  DevTensor in;
  in.p = const_cast<float*>(ptr);
  in.n = batch_;
  in.c = in_c_;
  in.h = in_h_;
  in.w = in_w_;
  in.layout = kNCHW;
  Src s = plain(in);
  if (math_ == SIGE_MATH_F16) {
    if (!in_twin_) {
      in_twin_c_ = (in_c_ + 7) / 8 * 8;
      in_twin_ = alloc(static_cast<size_t>(batch_) * in_h_ * in_w_ * in_twin_c_ * 2);
    }
    if (convert) launch_input_twin(ptr, batch_, in_c_, in_h_, in_w_, in_twin_c_, in_twin_, st);
    s.twin = in_twin_;
    s.twin_c = in_twin_c_;
  }
  return s;
}

void Engine::force_twin(DevTensor& t) {
  if (math_ == SIGE_MATH_F16 && t.layout == kNHWC && !t.half && !t.h16) t.h16 = alloc(t.numel() * 2);
}

size_t Engine::stats_len() const {
  size_t n = 0;
  for (const LayerDev& L : layers_)
    if (L.kind == SIGE_LAYER_RESBLOCK && L.norm_kind != SIGE_NORM_BATCH) n += 2 * static_cast<size_t>(batch_) * L.groups;
  return n;
}

// Src / Dst wiring of a fused-statistics ResBlock: conv1 writes m1 (+ fp16
// twin) and accumulates GroupNorm statistics of m1; conv2 stages the twin and
// applies norm (folded from the statistics) + act in shared memory.
static void wire_fused_gn(const LayerDev& L, const DevTensor& m1, double* stats, Dst& d1, Src& mid) {
  d1.gn_stats = stats;
  d1.gn_groups = L.groups;
  mid.gn_stats = stats;
  mid.gn_groups = L.groups;
  mid.gn_eps = L.eps;
  mid.gn_count = static_cast<double>(m1.c / L.groups) * m1.h * m1.w;
  mid.gn_gamma = L.gamma;
  mid.gn_beta = L.beta;
}

DevTensor& Engine::cache_slot(int step, const std::string& key, int c, int h, int w, int layout, int half) {
  DevTensor& t = cache_[{step, key}];
  if (!t.p || t.c != c || t.h != h || t.w != w || t.n != batch_ || t.layout != layout || t.half != half) {
    t.p = static_cast<float*>(alloc(static_cast<size_t>(batch_) * c * h * w * (half ? 2 : 4)));
    t.n = batch_;
    t.c = c;
    t.h = h;
    t.w = w;
    t.layout = layout;
    t.half = half;
    t.h16 = nullptr;
  }
  attach_twin(t, key);
  return t;
}

// act1 of ResBlock `layer` for `step`: computed by precompute, or derived here
// from conv1.out + norm1 when the cache was uploaded from a CPU precompute.
const DevTensor& Engine::ensure_act(int step, const std::string& key, int layer, cudaStream_t st) {
  auto it = cache_.find({step, key + ".act1"});
  if (it != cache_.end()) return it->second;
  const LayerDev& L = layers_[layer];
  const DevTensor& m1 = cache_tensor(step, key + ".conv1.out");
  const DevNorm& f = cache_norm(step, key + ".norm1");
  Src s = plain(m1);
  epi_push_ss(s.epi, f.scale, f.shift, f.np, m1.c);
  epi_push_act(s.epi, L.act);
  DevTensor& a = cache_slot(step, key + ".act1", m1.c, m1.h, m1.w, kNHWC, act_half());
  launch_materialize_act(s, a.p, a.half, st);
  SIGE_CUDA(cudaStreamSynchronize(st));
  return a;
}

DevNorm& Engine::norm_slot(int step, const std::string& key, int np) {
  DevNorm& n = norms_[{step, key}];
  if (!n.scale || n.np != np) {
    n.scale = static_cast<float*>(alloc(np * sizeof(float)));
    n.shift = static_cast<float*>(alloc(np * sizeof(float)));
    n.np = np;
  }
  return n;
}

DevTensor& Engine::scratch(const std::string& key, int c, int h, int w, int layout, int half) {
  DevTensor& t = scratch_[key];
  if (!t.p || t.c != c || t.h != h || t.w != w || t.layout != layout || t.half != half) {
    t.p = static_cast<float*>(alloc(static_cast<size_t>(batch_) * c * h * w * (half ? 2 : 4)));
    t.n = batch_;
    t.c = c;
    t.h = h;
    t.w = w;
    t.layout = layout;
    t.half = half;
    t.h16 = nullptr;
  }
  attach_twin(t, key);
  return t;
}

DevNorm& Engine::scratch_norm(const std::string& key, int np) {
  DevNorm& n = scratch_norms_[key];
  if (!n.scale || n.np < np) {
    n.scale = static_cast<float*>(alloc(np * sizeof(float)));
    n.shift = static_cast<float*>(alloc(np * sizeof(float)));
  }
  n.np = np;
  return n;
}

// Working copy of a cached output: equals the cache entry except for the
// tiles the current call scattered (restored at the start of the next call).
DevTensor& Engine::work_buffer(int step, const std::string& key) {
  auto it = work_.find({step, key});
  if (it != work_.end()) return it->second;
  const DevTensor& src = cache_tensor(step, key);
  DevTensor w = src;
  w.p = static_cast<float*>(alloc(src.bytes()));
  SIGE_CUDA(cudaMemcpy(w.p, src.p, src.bytes(), cudaMemcpyDeviceToDevice));
  if (src.h16) {
    w.h16 = alloc(src.numel() * 2);
    SIGE_CUDA(cudaMemcpy(w.h16, src.h16, src.numel() * 2, cudaMemcpyDeviceToDevice));
  }
  return work_[{step, key}] = w;
}

// All tiles of an (oh, ow) grid, 8x8, n-major: the dense path runs the same
// fused kernels over every tile (equal to conv2d, test_kernels.cpp:288-351).
// Tile shape for the dense path. CUDA-core kernel: 8x8. Tensor cores: the
// widest tile (<= 16 columns) whose GEMM rows (bh-1)*P + bw fit one M=128 MMA.
std::pair<int, int> Engine::dense_shape(int oh, int ow, int k, int s) const {
  if (!tensor_cores()) return {8, 8};
  const int bw = std::min(ow, 16);
  const int P = s == 1 ? bw + k - 1 : bw + 1;
  const int bh = std::max(1, std::min(oh, (128 - bw) / P + 1));
  return {bh, bw};
}

Tiles Engine::dense_tiles(int oh, int ow, int k, int s) {
  const auto shape = dense_shape(oh, ow, k, s);
  const int bh = shape.first, bw = shape.second;
  auto key = std::make_tuple(oh, ow, bh, bw);
  auto it = dense_tiles_.find(key);
  if (it == dense_tiles_.end()) {
    std::vector<int32_t> idx;
    for (int n = 0; n < batch_; ++n)
      for (int r = 0; r < oh; r += bh)
        for (int c = 0; c < ow; c += bw) {
          idx.push_back(n);
          idx.push_back(r);
          idx.push_back(c);
        }
    int32_t* d = static_cast<int32_t*>(alloc(idx.size() * sizeof(int32_t)));
    SIGE_CUDA(cudaMemcpy(d, idx.data(), idx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    it = dense_tiles_.emplace(key, std::make_pair(d, static_cast<int>(idx.size() / 3))).first;
  }
  Tiles t;
  t.idx = it->second.first;
  t.count = it->second.second;
  t.capacity = t.count;
  t.bh = bh;
  t.bw = bw;
  return t;
}

void Engine::conv(const Src& src, const Tiles& t, const ConvW& cw, const Dst& dst,
                  cudaStream_t st) const {
  ProfRec rec{};
  if (profiling_) {
    for (cudaEvent_t* e : {&rec.a, &rec.b}) {
      if (ev_pool_.empty()) {
        SIGE_CUDA(cudaEventCreate(e));
      } else {
        *e = ev_pool_.back();
        ev_pool_.pop_back();
      }
    }
    SIGE_CUDA(cudaEventRecord(rec.a, st));
  }
  if (tensor_cores() && timeline_) {
    const int idx = tl_next_++;
    if (idx < kTimelineSlots) {
      TlMeta m{};
      m.count_dev = t.count_dev;
      m.count = t.count;
      // algorithmic FLOPs (graph.cpp:712-714): 2 C_out C_in k^2 b^2 per tile,
      // exact output pixels for the static (dense) launches
      m.flops_per_tile = t.count_dev ? 2.0 * cw.c_out * cw.c_in * cw.k * cw.k * t.bh * t.bw
                                     : 2.0 * cw.c_out * cw.c_in * cw.k * cw.k * dst.h * dst.w * dst.n /
                                           std::max(1, t.count);
      m.sparse = t.count_dev ? 1 : 0;
      tl_meta_.push_back(m);
    }
    launch_conv_tc(src, t, cw, dst, math_ == SIGE_MATH_F16 ? 1 : 0, st, sm_budget_, tl_buf_, idx);
  } else if (tensor_cores())
    launch_conv_tc(src, t, cw, dst, math_ == SIGE_MATH_F16 ? 1 : 0, st, sm_budget_);
  else
    launch_conv_exact(src, t, cw, dst, math_, st);
  if (profiling_) {
    SIGE_CUDA(cudaEventRecord(rec.b, st));
    rec.count_dev = t.count_dev;
    rec.count = t.count;
    // algorithmic FLOPs per tile: 2 * C_out * C_in * k^2 * (pixels of the
    // tile inside the canvas ~ bh*bw; fringe clipping ignored)
    rec.flops_per_tile = 2.0 * cw.c_out * cw.c_in * cw.k * cw.k * t.bh * t.bw;
    if (!t.count_dev) {  // dense pass: the tiles clip at the canvas edge, count exact output pixels
      rec.flops_per_tile = 2.0 * cw.c_out * cw.c_in * cw.k * cw.k * dst.h * dst.w * dst.n / std::max(1, t.count);
    }
    rec.tc = tensor_cores() ? 1 : 0;
    prof_.push_back(rec);
  }
}

void Engine::set_profiling(bool on) { profiling_ = on; }

void Engine::timeline_reset() {
  std::vector<unsigned long long> init(3 * kTimelineSlots, ~0ull);  // [start, end] pairs, then wait exits
  for (int i = 0; i < kTimelineSlots; ++i) init[2 * i + 1] = 0;
  SIGE_CUDA(cudaMemcpy(tl_buf_, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
}

void Engine::drop_graphs() {
  SIGE_CUDA(cudaDeviceSynchronize());
  for (auto& kv : programs_) {
    for (auto& g : kv.second->graphs) cudaGraphExecDestroy(g.second.first);
    kv.second->graphs.clear();
  }
}

void Engine::set_timeline(bool on) {
  if (on == timeline_) return;
  if (on && !tl_buf_) {
    tl_buf_ = static_cast<unsigned long long*>(alloc(3 * kTimelineSlots * sizeof(unsigned long long)));
    timeline_reset();
  }
  drop_graphs();  // captured launches carry (or lack) the stamp buffer
  timeline_ = on;
}

int Engine::timeline_read(double* rows, int cap) {
  if (!tl_buf_) return 0;
  SIGE_CUDA(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(3 * kTimelineSlots);
  SIGE_CUDA(cudaMemcpy(h.data(), tl_buf_, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  int n = 0;
  unsigned long long t0 = ~0ull;
  for (size_t i = 0; i < tl_meta_.size(); ++i)
    if (h[2 * i + 1]) t0 = std::min(t0, h[2 * i]);
  for (size_t i = 0; i < tl_meta_.size(); ++i) {
    const TlMeta& m = tl_meta_[i];
    if (!h[2 * i + 1]) continue;  // not launched (or no CTA ran)
    int32_t cnt = m.count;
    if (m.count_dev) SIGE_CUDA(cudaMemcpy(&cnt, m.count_dev, sizeof cnt, cudaMemcpyDeviceToHost));
    if (n < cap && rows) {
      double* r = rows + 5 * n;
      r[0] = static_cast<double>(h[2 * i] - t0);
      r[1] = static_cast<double>(h[2 * i + 1] - t0);
      const unsigned long long w = h[2 * kTimelineSlots + i];
      r[2] = w == ~0ull ? r[0] : static_cast<double>(w - t0);
      r[3] = m.flops_per_tile * cnt;
      r[4] = m.sparse;
    }
    ++n;
  }
  timeline_reset();
  return n;
}

int Engine::profile_read(double* rows, int cap, cudaStream_t st) {
  SIGE_CUDA(cudaStreamSynchronize(st));
  int n = 0;
  for (const ProfRec& r : prof_) {
    if (n < cap && rows) {
      float ms = 0.0f;
      SIGE_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      int32_t cnt = r.count;
      if (r.count_dev) SIGE_CUDA(cudaMemcpy(&cnt, r.count_dev, sizeof cnt, cudaMemcpyDeviceToHost));
      rows[3 * n] = ms;
      rows[3 * n + 1] = r.flops_per_tile * cnt;
      rows[3 * n + 2] = r.tc;
    }
    ev_pool_.push_back(r.a);
    ev_pool_.push_back(r.b);
    ++n;
  }
  prof_.clear();
  return n;
}

std::string Engine::cache_entries(int step) const {
  std::ostringstream o;
  for (auto& kv : cache_) {
    if (kv.first.first != step || kv.first.second == "input" || kv.second.half) continue;
    const DevTensor& t = kv.second;
    if (kv.first.second.size() > 5 && kv.first.second.compare(kv.first.second.size() - 5, 5, ".act1") == 0)
      continue;  // engine-internal activation buffer, not a reference cache entry
    o << "T " << kv.first.second << ' ' << t.n << ' ' << t.c << ' ' << t.h << ' ' << t.w << '\n';
  }
  for (auto& kv : norms_) {
    if (kv.first.first != step) continue;
    o << "N " << kv.first.second << ' ' << kv.second.np << '\n';
  }
  return o.str();
}

// fold_norm_layer (graph.cpp:310-322).
void Engine::fold_norm(const LayerDev& L, const Src& x, DevNorm& out, cudaStream_t st) {
  if (L.norm_kind == SIGE_NORM_BATCH) {
    launch_bn_fold(L.channels, L.eps, L.gamma, L.beta, L.rmean, L.rvar, out.scale, out.shift, st);
  } else {
    if (!gn_scratch_) gn_scratch_ = static_cast<double*>(alloc(kGnScratch * sizeof(double)));
    launch_gn_fold(x, L.groups, L.eps, L.gamma, L.beta, out.scale, out.shift, gn_scratch_, kGnScratch,
                   tensor_cores() ? 0 : 1, st);
  }
}

// Derived activation buffers go stale when their inputs are replaced.
void Engine::drop_act(int step) {
  for (auto it = cache_.begin(); it != cache_.end();) {
    const std::string& k = it->first.second;
    if (it->first.first == step && k.size() > 5 && k.compare(k.size() - 5, 5, ".act1") == 0)
      it = cache_.erase(it);
    else
      ++it;
  }
}

void Engine::invalidate_programs() {
  // Working buffers mirror cache contents; any cache write drops them. The
  // memory stays in allocations_ until the engine dies (cache writes are rare).
  SIGE_CUDA(cudaDeviceSynchronize());  // captured graphs may still be running
  work_.clear();
  programs_.clear();
  last_program_ = nullptr;
}

// ---------------------------------------------------------- dense walk --
// dense_walk (graph.cpp:343-412) on the device. capture=true stores every
// cache entry (precompute); reused=true takes folded norms from the cache.
// ---------------------------------------------------- SPADE (config 3) --
Src Engine::seg_at(const float* in, int h, int w, DevTensor& buf, cudaStream_t st) {
  if (math_ == SIGE_MATH_F16 && !buf.h16) buf.h16 = alloc(static_cast<size_t>(batch_) * h * w * ((in_c_ + 7) / 8 * 8) * 2);
  const int c16 = (in_c_ + 7) / 8 * 8;
  launch_resize_nhwc(in, batch_, in_c_, in_h_, in_w_, h, w, buf.p, buf.h16, c16, st);
  Src s = plain(buf);
  s.twin = buf.h16;
  s.twin_c = c16;
  return s;
}

// One SPADE residual block over every pixel, in the restatement's order
// (oracle/spade.py): per SPADE norm k, a = ReLU(shared(seg)), [gamma|beta] =
// gb(a), mod = act(instnorm(input) (1 + gamma) + beta); conv_0(mod_0) ->
// conv_1(mod_1) + (conv_s(mod_s) | x).
Src Engine::spade_dense(const LayerDev& L, int li, const Src& x, const Src& seg, bool reused,
                        const std::function<DevTensor&(const std::string&, int, int)>& tensor,
                        const std::function<DevNorm&(const std::string&, int)>& norm, cudaStream_t st) {
  (void)li;
  const int h = x.h, w = x.w;
  const Tiles t3 = dense_tiles(h, w, 3, 1), t1 = dense_tiles(h, w, 1, 1);
  // The label-map convs of the block's norms depend on seg only: they run on
  // the branch stream (fork here, one event per norm, join at the end), so
  // the gamma/beta of norm_s and norm_1 overlap conv_0 (as in the sparse program).
  static const bool no_branch = std::getenv("SIGE_NO_SPADE_BRANCH") != nullptr;
  const bool branch = !no_branch && br_stream_ != nullptr;
  cudaStream_t bs = branch ? br_stream_ : st;
  if (branch) {
    SIGE_CUDA(cudaEventRecord(br_events_[kBrDense], st));
    SIGE_CUDA(cudaStreamWaitEvent(bs, br_events_[kBrDense], 0));
  }
  DevTensor* gbt[3] = {nullptr, nullptr, nullptr};
  auto label_convs = [&](int k, int C) {
    const std::string sk = ".spade" + std::to_string(k);
    const int nh = L.spade_shared[k].c_out;
    DevTensor& a = tensor(sk + ".a", nh, 0);
    Dst da = to_dst(a);
    Src as = plain(a);
    if (use_act()) {  // the gamma/beta conv stages ReLU(a) once per pixel (fp16 in F16)
      DevTensor& aa = tensor(sk + ".aact", nh, act_half());
      da.act = aa.p;
      da.act_half = aa.half;
      da.act_epi.fma_expf = host_expf_is_fma() ? 1 : 0;
      epi_push_act(da.act_epi, SIGE_ACT_RELU);
      as = plain(aa);
    } else {
      epi_push_act(as.epi, SIGE_ACT_RELU);
    }
    conv(seg, t3, L.spade_shared[k], da, bs);
    gbt[k] = &tensor(sk + ".gb", 2 * C, 0);
    conv(as, t3, L.spade_gb[k], to_dst(*gbt[k]), bs);
    if (branch) SIGE_CUDA(cudaEventRecord(br_events_[kBrDense + 1 + k], bs));
  };
  label_convs(0, x.c);
  if (L.has_shortcut) label_convs(2, x.c);
  label_convs(1, L.conv.c_out);
  auto modulate = [&](int k, const Src& in, int act) -> Src {
    const std::string sk = ".spade" + std::to_string(k);
    const int C = in.c;
    DevNorm& nf = norm(sk + ".norm", batch_ * C);
    if (!reused) {
      if (!gn_scratch_) gn_scratch_ = static_cast<double*>(alloc(kGnScratch * sizeof(double)));
      launch_gn_fold(in, C, L.spade_eps[k], L.spade_ones[k], L.spade_zeros[k], nf.scale, nf.shift, gn_scratch_,
                     kGnScratch, tensor_cores() ? 0 : 1, st);
    }
    if (branch) SIGE_CUDA(cudaStreamWaitEvent(st, br_events_[kBrDense + 1 + k], 0));
    DevTensor& mod = tensor(sk + ".mod", C, 0);
    launch_spade_mod(in, nf.scale, nf.shift, gbt[k]->p, act, nullptr, mod.p, mod.h16, st);
    return plain(mod);
  };
  const Src m0 = modulate(0, x, L.act);
  DevTensor& c0 = tensor(".conv0.out", L.conv.c_out, 0);
  conv(m0, t3, L.conv, to_dst(c0), st);
  Src addend = x;
  if (L.has_shortcut) {
    const Src ms = modulate(2, x, SIGE_ACT_NONE);
    DevTensor& sc = tensor(".sc.out", L.shortcut.c_out, 0);
    conv(ms, t1, L.shortcut, to_dst(sc), st);
    addend = plain(sc);
  }
  const Src m1 = modulate(1, plain(c0), L.act);
  DevTensor& sum = tensor(".sum", L.conv2.c_out, 0);
  Dst d = to_dst(sum, kAddSrc);
  d.addend = addend;
  conv(m1, t3, L.conv2, d, st);
  return plain(sum);  // (every branch event was waited on by a modulation: joined)
}

void Engine::dense_walk(const Src& input, int step, bool capture, bool reused, float* out_nchw,
                        cudaStream_t st) {
  Src x = input;
  std::map<std::string, Src> seg_done;  // SPADE label maps resized in this walk
  size_t dense_stats_used = 0;
  if (!capture && !reused && math_ == SIGE_MATH_F16) {
    if (!dense_stats_) {
      dense_stats_len_ = std::max<size_t>(stats_len(), 1);
      dense_stats_ = static_cast<double*>(alloc(dense_stats_len_ * sizeof(double)));
    }
    SIGE_CUDA(cudaMemsetAsync(dense_stats_, 0, dense_stats_len_ * sizeof(double), st));
  }
  for (size_t i = 0; i < layers_.size(); ++i) {
    const LayerDev& L = layers_[i];
    const LayerShape& sh = shapes_[i];
    const std::string key = lk(static_cast<int>(i));
    switch (L.kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE: {
        DevTensor& o = capture ? cache_slot(step, key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC)
                               : scratch("dense." + key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC);
        conv(x, dense_tiles(sh.h_out, sh.w_out, L.conv.k, L.conv.stride), L.conv, to_dst(o), st);
        x = plain(o);
        break;
      }
      case SIGE_LAYER_NORM: {
        DevNorm* f;
        const int np = L.norm_kind == SIGE_NORM_BATCH ? L.channels : batch_ * L.channels;
        if (reused) {
          f = const_cast<DevNorm*>(&cache_norm(step, key + ".norm"));
        } else {
          f = capture ? &norm_slot(step, key + ".norm", np) : &scratch_norm("dense." + key + ".norm", np);
          fold_norm(L, x, *f, st);
        }
        epi_push_ss(x.epi, f->scale, f->shift, f->np, x.c);
        break;
      }
      case SIGE_LAYER_ACTIVATION:
        epi_push_act(x.epi, L.act);
        break;
      case SIGE_LAYER_UPSAMPLE:
        x.up += 1;
        x.h *= 2;
        x.w *= 2;
        break;
      case SIGE_LAYER_RESIZE: {
        DevTensor& o = capture ? cache_slot(step, key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC)
                               : scratch("dense." + key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC);
        launch_resize_nhwc(input.ptr, batch_, in_c_, in_h_, in_w_, sh.h_out, sh.w_out, o.p, o.h16,
                           in_c_, st);
        x = plain(o);
        break;
      }
      case SIGE_LAYER_SPADE_RESBLOCK: {
        // the label map at this resolution: the input itself at full
        // resolution (its fp16 twin already exists), else one resize per
        // resolution and walk (blocks sharing a resolution reuse it)
        Src seg;
        if (sh.h_in == in_h_ && sh.w_in == in_w_) {
          seg = input;
        } else {
          const std::string sk = "dense.seg@" + std::to_string(sh.h_in) + "x" + std::to_string(sh.w_in);
          DevTensor& segb = scratch(sk, in_c_, sh.h_in, sh.w_in, kNHWC);
          auto hit = seg_done.find(sk);
          if (hit == seg_done.end()) hit = seg_done.emplace(sk, seg_at(input.ptr, sh.h_in, sh.w_in, segb, st)).first;
          seg = hit->second;
        }
        auto tensor = [&](const std::string& sfx, int c, int half) -> DevTensor& {
          return capture ? cache_slot(step, key + sfx, c, sh.h_in, sh.w_in, kNHWC, half)
                         : scratch("dense." + key + sfx, c, sh.h_in, sh.w_in, kNHWC, half);
        };
        auto norm = [&](const std::string& sfx, int np) -> DevNorm& {
          if (reused) return const_cast<DevNorm&>(cache_norm(step, key + sfx));
          return capture ? norm_slot(step, key + sfx, np) : scratch_norm("dense." + key + sfx, np);
        };
        x = spade_dense(L, static_cast<int>(i), x, seg, reused, tensor, norm, st);
        break;
      }
      case SIGE_LAYER_RESBLOCK: {
        const int c1 = L.conv.c_out, co = L.conv2.c_out, h = sh.h_in, w = sh.w_in;
        if (!capture && !reused && fused_gn(L)) {
          // conv1 (+ statistics) -> [shortcut] -> conv2 (norm + act in smem) with the join add(m, sc).
          DevTensor& m1 = scratch("dense." + key + ".conv1.out", c1, h, w, kNHWC);
          force_twin(m1);
          double* stats = dense_stats_ + dense_stats_used;
          dense_stats_used += 2 * static_cast<size_t>(batch_) * L.groups;
          Dst d1 = to_dst(m1);
          Src mid = plain(m1);
          wire_fused_gn(L, m1, stats, d1, mid);
          epi_push_act(mid.epi, L.act);
          conv(x, dense_tiles(h, w, 3, 1), L.conv, d1, st);
          DevTensor& sc = scratch("dense." + key + ".shortcut.out", co, h, w, kNHWC);
          if (L.has_shortcut)
            conv(x, dense_tiles(h, w, 1, 1), L.shortcut, to_dst(sc), st);
          DevTensor& sum = scratch("dense." + key + ".sum", co, h, w, kNHWC);
          Dst d = to_dst(sum, kAddSrc);
          d.addend = L.has_shortcut ? plain(sc) : x;
          conv(mid, dense_tiles(h, w, 3, 1), L.conv2, d, st);
          x = plain(sum);
          break;
        }
        DevTensor& m1 = capture ? cache_slot(step, key + ".conv1.out", c1, h, w, kNHWC)
                                : scratch("dense." + key + ".conv1.out", c1, h, w, kNHWC);
        conv(x, dense_tiles(h, w, 3, 1), L.conv, to_dst(m1), st);
        const int np = L.norm_kind == SIGE_NORM_BATCH ? L.channels : batch_ * L.channels;
        DevNorm* f;
        if (reused) {
          f = const_cast<DevNorm*>(&cache_norm(step, key + ".norm1"));
        } else {
          f = capture ? &norm_slot(step, key + ".norm1", np) : &scratch_norm("dense." + key + ".norm1", np);
          fold_norm(L, plain(m1), *f, st);
        }
        Src mid = plain(m1);
        epi_push_ss(mid.epi, f->scale, f->shift, f->np, c1);
        epi_push_act(mid.epi, L.act);
        if (use_act()) {  // conv2 stages act1 = act(norm1(m1)) evaluated once per pixel
          DevTensor& a1 = capture ? cache_slot(step, key + ".act1", c1, h, w, kNHWC, act_half())
                                  : scratch("dense." + key + ".act1", c1, h, w, kNHWC, act_half());
          launch_materialize_act(mid, a1.p, a1.half, st);
          mid = plain(a1);
        }
        DevTensor& sc = capture ? cache_slot(step, key + ".shortcut.out", co, h, w, kNHWC)
                                : scratch("dense." + key + ".shortcut.out", co, h, w, kNHWC);
        if (L.has_shortcut)
          conv(x, dense_tiles(h, w, 1, 1), L.shortcut, to_dst(sc), st);
        else
          launch_materialize(x, sc.p, kNHWC, st);
        DevTensor& sum = capture ? cache_slot(step, key + ".sum", co, h, w, kNHWC)
                                 : scratch("dense." + key + ".sum", co, h, w, kNHWC);
        if (capture) {
          DevTensor& m2 = cache_slot(step, key + ".conv2.out", co, h, w, kNHWC);
          conv(mid, dense_tiles(h, w, 3, 1), L.conv2, to_dst(m2), st);
          launch_add_h(m2.p, sc.p, sum.p, sum.h16, sum.numel(), st);  // add(m, sc), graph.cpp:404
        } else {
          Dst d = to_dst(sum, kAddSrc);
          d.addend = plain(sc);
          conv(mid, dense_tiles(h, w, 3, 1), L.conv2, d, st);
        }
        x = plain(sum);
        break;
      }
    }
  }
  if (capture) {
    DevTensor& fin = cache_slot(step, "final", out_c_, out_h_, out_w_, kNCHW);
    launch_materialize(x, fin.p, kNCHW, st);
    if (out_nchw) SIGE_CUDA(cudaMemcpyAsync(out_nchw, fin.p, fin.numel() * sizeof(float),
                                            cudaMemcpyDeviceToDevice, st));
  } else {
    launch_materialize(x, out_nchw, kNCHW, st);
  }
}

void Engine::precompute(const float* original, int step, cudaStream_t st) {
  cache_model_hash_ = structure_hash_;  // precompute (graph.cpp:426-435)
  invalidate_programs();
  free_host_step(step);  // an offloaded copy of this step is stale now
  DevTensor& in = cache_slot(step, "input", in_c_, in_h_, in_w_, kNCHW);
  SIGE_CUDA(cudaMemcpyAsync(in.p, original, in.numel() * sizeof(float), cudaMemcpyDeviceToDevice, st));
  dense_walk(plain(in), step, /*capture=*/true, /*reused=*/false, nullptr, st);
}

void Engine::dense_forward(const float* input, bool reused, int step, float* out, cudaStream_t st) {
  tl_next_ = 0;
  tl_meta_.clear();
  dense_walk(input_src(input, st, true), step, false, reused, out, st);
}

// ------------------------------------------------------ cache exchange --
namespace {
bool is_nchw_key(const std::string& key) { return key == "final" || key == "input"; }
}  // namespace

void Engine::put_tensor(int step, const std::string& key, const float* host, size_t numel) {
  // Shape from the model walk (graph.cpp:356-410 keys).
  int c = 0, h = 0, w = 0;
  if (key == "final") {
    c = out_c_, h = out_h_, w = out_w_;
  } else if (key == "input") {
    c = in_c_, h = in_h_, w = in_w_;
  } else {
    int li = -1;
    char rest[64] = {0};
    if (std::sscanf(key.c_str(), "L%d.%63s", &li, rest) != 2 || li < 0 ||
        li >= static_cast<int>(layers_.size()))
      throw ConfigError("cache: unknown key " + key);
    const LayerShape& s = shapes_[li];
    const std::string r = rest;
    if (r == "out") {
      c = s.c_out, h = s.h_out, w = s.w_out;
    } else if (r == "conv1.out") {
      c = layers_[li].conv.c_out, h = s.h_in, w = s.w_in;
    } else if (r == "conv2.out" || r == "shortcut.out" || r == "sum") {
      c = s.c_out, h = s.h_out, w = s.w_out;
    } else {
      throw ConfigError("cache: unknown key " + key);
    }
  }
  if (numel != static_cast<size_t>(batch_) * c * h * w)
    throw ConfigError("cache entry " + key + ": expected " +
                      std::to_string(static_cast<size_t>(batch_) * c * h * w) + " values");
  invalidate_programs();
  drop_act(step);
  free_host_step(step);
  const int layout = is_nchw_key(key) ? kNCHW : kNHWC;
  DevTensor& t = cache_slot(step, key, c, h, w, layout);
  std::vector<float> buf(numel);
  if (layout == kNHWC) {
    for (int n = 0; n < batch_; ++n)
      for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < h; ++y)
          for (int x = 0; x < w; ++x)
            buf[((static_cast<size_t>(n) * h + y) * w + x) * c + ch] =
                host[((static_cast<size_t>(n) * c + ch) * h + y) * w + x];
  } else {
    std::memcpy(buf.data(), host, numel * sizeof(float));
  }
  SIGE_CUDA(cudaMemcpy(t.p, buf.data(), numel * sizeof(float), cudaMemcpyHostToDevice));
  if (t.h16) {
    launch_to_half(t.p, t.h16, numel, nullptr);
    SIGE_CUDA(cudaStreamSynchronize(nullptr));
  }
}

void Engine::put_norm(int step, const std::string& key, const float* sc, const float* sh, size_t np) {
  invalidate_programs();
  drop_act(step);
  free_host_step(step);
  DevNorm& n = norm_slot(step, key, static_cast<int>(np));
  SIGE_CUDA(cudaMemcpy(n.scale, sc, np * sizeof(float), cudaMemcpyHostToDevice));
  SIGE_CUDA(cudaMemcpy(n.shift, sh, np * sizeof(float), cudaMemcpyHostToDevice));
}

void Engine::get_norm(int step, const std::string& key, float* sc, float* sh, size_t np) {
  const DevNorm& n = cache_norm(step, key);
  if (np != static_cast<size_t>(n.np)) throw ConfigError("cache norm " + key + ": size mismatch");
  SIGE_CUDA(cudaDeviceSynchronize());
  SIGE_CUDA(cudaMemcpy(sc, n.scale, np * sizeof(float), cudaMemcpyDeviceToHost));
  SIGE_CUDA(cudaMemcpy(sh, n.shift, np * sizeof(float), cudaMemcpyDeviceToHost));
}

void Engine::get_tensor(int step, const std::string& key, float* host, size_t numel) {
  const DevTensor& t = cache_tensor(step, key);
  if (numel != t.numel()) throw ConfigError("cache entry " + key + ": size mismatch");
  if (t.half) throw ConfigError("cache entry " + key + ": fp16 activation buffer (engine-internal)");
  std::vector<float> buf(numel);
  SIGE_CUDA(cudaDeviceSynchronize());
  SIGE_CUDA(cudaMemcpy(buf.data(), t.p, numel * sizeof(float), cudaMemcpyDeviceToHost));
  if (t.layout == kNHWC) {
    for (int n = 0; n < t.n; ++n)
      for (int ch = 0; ch < t.c; ++ch)
        for (int y = 0; y < t.h; ++y)
          for (int x = 0; x < t.w; ++x)
            host[((static_cast<size_t>(n) * t.c + ch) * t.h + y) * t.w + x] =
                buf[((static_cast<size_t>(n) * t.h + y) * t.w + x) * t.c + ch];
  } else {
    std::memcpy(host, buf.data(), numel * sizeof(float));
  }
}

// ------------------------------------------------------- sparse program --
namespace {
std::string config_key(const sige_run_config& c) {
  std::ostringstream o;
  o << c.step << '|' << c.dilate_full << '|' << c.dilate_scale << '|' << c.block3 << '|' << c.block1
    << '|' << c.min_sparse_res << '|' << c.norm_precompute;
  return o.str();
}
}  // namespace

struct ProgramBuilder {
  Engine& E;
  Program& P;
  const sige_run_config& cfg;
  std::map<std::tuple<int, int, int>, int> memo;
  size_t br_next = 0;    // next branch event
  bool br_forked = false;  // the SPADE branch stream has forked from the main chain
  static bool branch_on() {
    static const bool off = std::getenv("SIGE_NO_SPADE_BRANCH") != nullptr;  // A/B: one serial chain
    return !off;
  }
  // Branch helpers: fork once (after the IndexPlan), record / wait events.
  void br_fork() {
    if (br_forked) return;
    br_forked = true;
    Engine* eng = &E;
    const cudaEvent_t ev = E.br_event(br_next++);
    add([eng, ev](cudaStream_t st) {
      SIGE_CUDA(cudaEventRecord(ev, st));
      SIGE_CUDA(cudaStreamWaitEvent(eng->br_stream_, ev, 0));
    }, 0);
  }
  cudaEvent_t br_record() {
    Engine* eng = &E;
    const cudaEvent_t ev = E.br_event(br_next++);
    add([eng, ev](cudaStream_t) { SIGE_CUDA(cudaEventRecord(ev, eng->br_stream_)); }, 0);
    return ev;
  }

  int entry(int h, int w, int b) {  // IndexPlan::at (graph.cpp:517-528)
    auto key = std::make_tuple(h, w, b);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    const int H = E.in_h_, W = E.in_w_;
    if (h <= H && w <= W) {
      if (H % h != 0 || W % w != 0)
        throw ConfigError("downsample_mask: non-integer scale factor (" + std::to_string(H) + "x" +
                          std::to_string(W) + " -> " + std::to_string(h) + "x" + std::to_string(w) + ")");
    } else if (h % H != 0 || w % W != 0) {
      throw ConfigError("mask: cannot scale " + std::to_string(H) + "x" + std::to_string(W) +
                        " up to " + std::to_string(h) + "x" + std::to_string(w) +
                        " (non-integer factor)");
    }
    PlanEntryDev e;
    e.h = h;
    e.w = w;
    e.b = b;
    e.capacity = ((h + b - 1) / b) * ((w + b - 1) / b) * E.batch_;
    e.idx = static_cast<int32_t*>(E.alloc(static_cast<size_t>(e.capacity) * 3 * sizeof(int32_t)));
    e.count = static_cast<int32_t*>(E.alloc(sizeof(int32_t)));
    SIGE_CUDA(cudaMemset(e.count, 0, sizeof(int32_t)));
    const int grid_tiles = ((h + b - 1) / b) * ((w + b - 1) / b);
    e.bm = static_cast<uint32_t*>(
        E.alloc(static_cast<size_t>((grid_tiles + 31) / 32) * (P.grouped ? E.batch_ : 1) * sizeof(uint32_t)));
    P.entries.push_back(e);
    return memo[key] = static_cast<int>(P.entries.size()) - 1;
  }

  Tiles tiles(int ei) const {
    const PlanEntryDev& e = P.entries[ei];
    Tiles t;
    t.idx = e.idx;
    t.count_dev = e.count;
    t.capacity = e.capacity;
    t.bh = t.bw = e.b;
    return t;
  }

  void restore(const DevTensor& wbuf, const DevTensor& cache, int ei) {
    const PlanEntryDev& e = P.entries[ei];
    RestoreJob j;
    j.dst = wbuf.p;
    j.src = cache.p;
    j.idx = e.idx;
    j.count = e.count;
    j.n = wbuf.n;
    j.c = wbuf.c;
    j.h = wbuf.h;
    j.w = wbuf.w;
    j.b = e.b;
    j.layout = wbuf.layout;
    j.half = wbuf.half;
    P.restores.push_back(j);
    if (wbuf.h16 && cache.h16) {  // the fp16 twin's dirtied tiles too
      j.dst = static_cast<float*>(wbuf.h16);
      j.src = static_cast<const float*>(cache.h16);
      j.half = 1;
      P.restores.push_back(j);
    }
    P.restore_max = std::max<long long>(P.restore_max, static_cast<long long>(e.capacity) * e.b * e.b * wbuf.c);
  }

  void add(std::function<void(cudaStream_t)> f, int launches = 1) {
    P.steps.push_back(std::move(f));
    P.launches += launches;
  }

  void conv_step(const Src& s, const Tiles& t, const ConvW& cw, const Dst& d) {
    Engine* eng = &E;
    add([eng, s, t, cw, d](cudaStream_t st) { eng->conv(s, t, cw, d, st); });
  }

  void build() {
    const int step = cfg.step;
    const int N = E.batch_;
    // Flow (graph.cpp:538-569). The input source pointer is bound per call.
    Src flow;
    flow.ptr = nullptr;  // bound to cur_in_ below
    flow.layout = kNCHW;
    flow.n = N;
    flow.c = E.in_c_;
    flow.h = E.in_h_;
    flow.w = E.in_w_;
    flow.epi.fma_expf = host_expf_is_fma() ? 1 : 0;
    bool flow_is_input = true;
    bool has_blocks = false;
    int blocks_entry = -1;
    Engine* eng = &E;
    std::set<std::string> seg_keys;  // SPADE label-map resolutions already resized in this program
    // Source pointer resolution at launch time for steps that read the input.
    // The first layers read the per-call input (and, in F16, its fp16 twin
    // written by k_input_twin at the start of the call).
    const Src in_src = E.input_src(nullptr, nullptr, false);
    auto bind = [eng, in_src](Src s, bool is_input) {
      if (is_input) {
        s.ptr = eng->cur_in_;
        s.twin = in_src.twin;
        s.twin_c = in_src.twin_c;
      }
      return s;
    };
    for (size_t i = 0; i < E.layers_.size(); ++i) {
      const LayerDev& L = E.layers_[i];
      const LayerShape& sh = E.shapes_[i];
      const std::string key = lk(static_cast<int>(i));
      const bool fin = flow_is_input;
      switch (L.kind) {
        case SIGE_LAYER_CONV:
        case SIGE_LAYER_DOWNSAMPLE: {
          const ConvW cw = L.conv;
          TraceInfo tr{-1, cw.c_in, cw.c_out, cw.k, cw.stride, sh.h_out, sh.w_out, N};
          Src s = flow;
          if (!runs_sparse(L, flow.h, flow.w, cfg)) {
            DevTensor& o = E.scratch("sparse." + key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC);
            Tiles t = E.dense_tiles(sh.h_out, sh.w_out, cw.k, cw.stride);
            Dst d = to_dst(o);
            add([eng, s, t, cw, d, fin, bind](cudaStream_t st) { eng->conv(bind(s, fin), t, cw, d, st); });
            flow = plain(o);
            has_blocks = false;
          } else {
            const int ei = entry(sh.h_out, sh.w_out, cw.k == 3 ? cfg.block3 : cfg.block1);
            tr.entry = ei;
            DevTensor& wb = E.work_buffer(step, key + ".out");
            const DevTensor& cb = E.cache_tensor(step, key + ".out");
            Tiles t = tiles(ei);
            Dst d = to_dst(wb);
            add([eng, s, t, cw, d, fin, bind](cudaStream_t st) { eng->conv(bind(s, fin), t, cw, d, st); });
            restore(wb, cb, ei);
            flow = plain(wb);
            has_blocks = true;
            blocks_entry = ei;
          }
          P.trace.push_back(tr);
          flow_is_input = false;
          break;
        }
        case SIGE_LAYER_NORM: {
          if (L.norm_kind == SIGE_NORM_BATCH || cfg.norm_precompute) {
            const DevNorm& f = E.cache_norm(step, key + ".norm");
            epi_push_ss(flow.epi, f.scale, f.shift, f.np, flow.c);
          } else {
            // flush + fresh statistics (graph.cpp:745-750).
            DevTensor& full = E.scratch("sparse." + key + ".flush", flow.c, flow.h, flow.w, kNHWC);
            const int np = N * L.channels;
            DevNorm& f = E.scratch_norm("sparse." + key + ".norm", np);
            Src s = flow;
            DevTensor fullc = full;
            DevNorm fc = f;
            LayerDev Lc = L;
            add([eng, s, fullc, fc, Lc, fin, bind](cudaStream_t st) mutable {
              launch_materialize(bind(s, fin), fullc.p, kNHWC, st);
              eng->fold_norm(Lc, plain(fullc), fc, st);
            }, 2);
            flow = plain(full);
            epi_push_ss(flow.epi, f.scale, f.shift, np, flow.c);
            flow_is_input = false;
            has_blocks = false;
          }
          break;
        }
        case SIGE_LAYER_ACTIVATION:
          epi_push_act(flow.epi, L.act);
          break;
        case SIGE_LAYER_UPSAMPLE:
          flow.up += 1;
          flow.h *= 2;
          flow.w *= 2;
          has_blocks = false;  // materialize (graph.cpp:762-770)
          break;
        case SIGE_LAYER_RESIZE: {
          // the input resized per call, dense (a few KB to a few MB)
          DevTensor& o = E.scratch("sparse." + key + ".out", sh.c_out, sh.h_out, sh.w_out, kNHWC);
          const DevTensor oc = o;
          const int ic = E.in_c_, ih = E.in_h_, iw = E.in_w_, n = N;
          add([eng, oc, ic, ih, iw, n](cudaStream_t st) {
            launch_resize_nhwc(eng->cur_in_, n, ic, ih, iw, oc.h, oc.w, oc.p, oc.h16, ic, st);
          });
          flow = plain(o);
          flow_is_input = false;
          has_blocks = false;
          break;
        }
        case SIGE_LAYER_SPADE_RESBLOCK: {
          const int h = flow.h, w = flow.w;
          const Src x0 = flow;
          const int li = static_cast<int>(i);
          const int c16 = (E.in_c_ + 7) / 8 * 8;
          // full resolution: the label map is the input itself (bound per call,
          // fp16 twin from the call's input conversion); lower resolutions are
          // resized once per call and resolution (blocks sharing one reuse it)
          const bool seg_full = h == E.in_h_ && w == E.in_w_;
          const std::string seg_key = "sparse.seg@" + std::to_string(h) + "x" + std::to_string(w);
          DevTensor& segb = E.scratch(seg_key, E.in_c_, seg_full ? 1 : h, seg_full ? 1 : w, kNHWC);
          if (!seg_full && E.math_ == SIGE_MATH_F16 && !segb.h16)
            segb.h16 = E.alloc(static_cast<size_t>(N) * h * w * c16 * 2);
          const DevTensor segc = segb;
          const bool branch = ProgramBuilder::branch_on();
          auto add_trace = [&](int entry_idx) {
            for (int k = 0; k < L.n_spade; ++k) {
              P.trace.push_back({entry_idx, L.spade_shared[k].c_in, L.spade_shared[k].c_out, 3, 1, h, w, N});
              P.trace.push_back({entry_idx, L.spade_gb[k].c_in, L.spade_gb[k].c_out, 3, 1, h, w, N});
            }
            P.trace.push_back({entry_idx, L.conv.c_in, L.conv.c_out, 3, 1, h, w, N});
            if (L.has_shortcut) P.trace.push_back({entry_idx, L.shortcut.c_in, L.shortcut.c_out, 1, 1, h, w, N});
            P.trace.push_back({entry_idx, L.conv2.c_in, L.conv2.c_out, 3, 1, h, w, N});
          };
          if (!runs_sparse(L, h, w, cfg) || !cfg.norm_precompute) {
            // dense fallback with fresh statistics (as ResBlocks, graph.cpp:799-815)
            DevTensor& sum = E.scratch("sparse." + key + ".sum", L.conv2.c_out, h, w, kNHWC);
            const LayerDev Lc = L;
            Src in_seg = in_src;
            in_seg.ptr = nullptr;
            DevTensor segfb = seg_full ? segc
                                       : E.scratch("sparse.segfb@" + std::to_string(h) + "x" + std::to_string(w),
                                                   E.in_c_, h, w, kNHWC);
            if (!seg_full && E.math_ == SIGE_MATH_F16 && !segfb.h16) {
              DevTensor& sf = E.scratch("sparse.segfb@" + std::to_string(h) + "x" + std::to_string(w), E.in_c_, h,
                                        w, kNHWC);
              sf.h16 = E.alloc(static_cast<size_t>(N) * h * w * c16 * 2);
              segfb = sf;
            }
            add([eng, Lc, li, x0, fin, bind, segfb, key, seg_full, in_seg](cudaStream_t st) {
              DevTensor seg_buf = segfb;
              const Src seg = seg_full ? bind(in_seg, true) : eng->seg_at(eng->cur_in_, x0.h, x0.w, seg_buf, st);
              auto tensor = [&](const std::string& sfx, int c, int half) -> DevTensor& {
                return eng->scratch("sparse." + key + sfx, c, x0.h, x0.w, kNHWC, half);
              };
              auto norm = [&](const std::string& sfx, int np) -> DevNorm& {
                return eng->scratch_norm("sparse." + key + sfx, np);
              };
              eng->spade_dense(Lc, li, bind(x0, fin), seg, false, tensor, norm, st);
            }, 0);
            add_trace(-1);
            flow = plain(sum);
            has_blocks = false;
          } else {
            // sparse: every SPADE conv, the modulation and conv_0/conv_s/conv_1
            // run on the main tiles; working buffers restored afterwards.
            const int em = entry(h, w, cfg.block3);
            const Tiles tm = tiles(em);
            auto W = [&](const std::string& sfx) -> DevTensor& {
              DevTensor& wb = E.work_buffer(step, key + sfx);
              restore(wb, E.cache_tensor(step, key + sfx), em);
              return wb;
            };
            const bool seg_new = !seg_full && seg_keys.insert(seg_key).second;
            if (branch) br_fork();
            if (seg_new) {
              add([eng, segc, branch](cudaStream_t st) {  // this resolution's segmentation map
                DevTensor seg_buf = segc;
                eng->seg_at(eng->cur_in_, segc.h, segc.w, seg_buf, branch ? eng->br_stream_ : st);
              });
            }
            Src seg = plain(segb);
            seg.twin = segb.h16;
            seg.twin_c = c16;
            if (seg_full) {
              seg = in_src;  // NCHW input + twin, pointers bound at launch
              seg.ptr = nullptr;
            }
            auto modulate = [&](int k, const Src& in, int act, bool in_is_input) -> Src {
              const std::string sk = ".spade" + std::to_string(k);
              DevTensor& a = W(sk + ".a");
              Dst da = to_dst(a);
              Src as = plain(a);
              if (E.use_act()) {
                DevTensor& aa = W(sk + ".aact");
                da.act = aa.p;
                da.act_half = aa.half;
                da.act_epi.fma_expf = host_expf_is_fma() ? 1 : 0;
                epi_push_act(da.act_epi, SIGE_ACT_RELU);
                as = plain(aa);
              } else {
                epi_push_act(as.epi, SIGE_ACT_RELU);
              }
              // the label-map convs (input only): on the branch stream
              DevTensor& gb = W(sk + ".gb");
              {
                const ConvW sw = L.spade_shared[k], gw = L.spade_gb[k];
                const Dst dgb = to_dst(gb);
                add([eng, seg, tm, sw, da, bind, seg_full, as, gw, dgb, branch](cudaStream_t st) {
                  cudaStream_t bs = branch ? eng->br_stream_ : st;
                  eng->conv(bind(seg, seg_full), tm, sw, da, bs);
                  eng->conv(as, tm, gw, dgb, bs);
                }, 2);
              }
              const cudaEvent_t gb_ready = branch ? br_record() : nullptr;
              const DevNorm& nf = E.cache_norm(step, key + sk + ".norm");
              DevTensor& mod = W(sk + ".mod");
              const float* scp = nf.scale;
              const float* shp = nf.shift;
              const float* gbp = gb.p;
              float* mp = mod.p;
              void* m16 = mod.h16;
              add([in, in_is_input, bind, scp, shp, gbp, act, tm, mp, m16, gb_ready](cudaStream_t st) {
                if (gb_ready) SIGE_CUDA(cudaStreamWaitEvent(st, gb_ready, 0));
                launch_spade_mod(bind(in, in_is_input), scp, shp, gbp, act, &tm, mp, m16, st);
              });
              return plain(mod);
            };
            const Src m0 = modulate(0, x0, L.act, fin);
            DevTensor& c0 = W(".conv0.out");
            conv_step(m0, tm, L.conv, to_dst(c0));
            Src addend = x0;
            if (L.has_shortcut) {
              const Src ms = modulate(2, x0, SIGE_ACT_NONE, fin);
              DevTensor& sc = W(".sc.out");
              conv_step(ms, tm, L.shortcut, to_dst(sc));
              addend = plain(sc);
            }
            const Src m1 = modulate(1, plain(c0), L.act, false);
            DevTensor& sum = W(".sum");
            Dst d = to_dst(sum, kAddSrc);
            d.addend = addend;
            const bool add_in = !L.has_shortcut && fin;
            const ConvW c2w = L.conv2;
            add([eng, m1, tm, c2w, d, add_in, bind](cudaStream_t st) {
              Dst dd = d;
              if (add_in) dd.addend = bind(d.addend, true);
              eng->conv(m1, tm, c2w, dd, st);
            });
            add_trace(em);
            flow = plain(sum);
            has_blocks = true;
            blocks_entry = em;
          }
          flow_is_input = false;
          break;
        }
        case SIGE_LAYER_RESBLOCK: {
          const int h = flow.h, w = flow.w, c1 = L.conv.c_out, co = L.conv2.c_out;
          Src x0 = flow;
          if (!runs_sparse(L, h, w, cfg) && E.fused_gn(L)) {
            // Dense fallback (graph.cpp:799-815), fresh statistics: conv1's
            // epilogue accumulates them, conv2 folds + applies norm/act in smem.
            DevTensor& m1 = E.scratch("sparse." + key + ".conv1", c1, h, w, kNHWC);
            E.force_twin(m1);
            DevTensor& o = E.scratch("sparse." + key + ".sum", co, h, w, kNHWC);
            double* stats = P.stats + P.stats_used;
            P.stats_used += 2 * static_cast<size_t>(N) * L.groups;
            Dst d1 = to_dst(m1);
            Src mid = plain(m1);
            wire_fused_gn(L, m1, stats, d1, mid);
            epi_push_act(mid.epi, L.act);
            Tiles t = E.dense_tiles(h, w, 3, 1), t1 = E.dense_tiles(h, w, 1, 1);
            ConvW c1w = L.conv, c2w = L.conv2, scw = L.shortcut;
            DevTensor scc{};
            if (L.has_shortcut) scc = E.scratch("sparse." + key + ".shortcut", co, h, w, kNHWC);
            Dst d = to_dst(o, kAddSrc);
            const bool has_sc = L.has_shortcut != 0;
            add([eng, x0, t, t1, c1w, c2w, scw, d1, mid, d, scc, has_sc, fin, bind](cudaStream_t st) {
              Src xin = bind(x0, fin);
              eng->conv(xin, t, c1w, d1, st);
              Dst dd = d;
              if (has_sc) {
                eng->conv(xin, t1, scw, to_dst(scc), st);
                dd.addend = plain(scc);
              } else {
                dd.addend = xin;
              }
              eng->conv(mid, t, c2w, dd, st);
            }, L.has_shortcut ? 3 : 2);
            P.trace.push_back({-1, L.conv.c_in, c1, 3, 1, h, w, N});
            P.trace.push_back({-1, c1, co, 3, 1, h, w, N});
            if (L.has_shortcut) P.trace.push_back({-1, L.shortcut.c_in, co, 1, 1, h, w, N});
            flow = plain(o);
          } else if (!runs_sparse(L, h, w, cfg)) {
            // Dense fallback (graph.cpp:799-815): fresh statistics always.
            DevTensor& m1 = E.scratch("sparse." + key + ".conv1", c1, h, w, kNHWC);
            DevTensor& o = E.scratch("sparse." + key + ".sum", co, h, w, kNHWC);
            const int np = L.norm_kind == SIGE_NORM_BATCH ? L.channels : N * L.channels;
            DevNorm& f = E.scratch_norm("sparse." + key + ".norm1", np);
            Tiles t = E.dense_tiles(h, w, 3, 1), t1 = E.dense_tiles(h, w, 1, 1);
            ConvW c1w = L.conv, c2w = L.conv2, scw = L.shortcut;
            LayerDev Lc = L;
            DevTensor m1c = m1;
            DevNorm fc = f;
            Src mid = plain(m1);
            epi_push_ss(mid.epi, f.scale, f.shift, np, c1);
            epi_push_act(mid.epi, L.act);
            DevTensor a1c{};
            if (E.use_act()) a1c = E.scratch("sparse." + key + ".act1", c1, h, w, kNHWC, E.act_half());
            Dst d = to_dst(o, kAddSrc);
            DevTensor* scd = nullptr;
            if (L.has_shortcut) scd = &E.scratch("sparse." + key + ".shortcut", co, h, w, kNHWC);
            DevTensor scc = scd ? *scd : DevTensor{};
            const bool has_sc = L.has_shortcut != 0;
            add([eng, x0, t, t1, c1w, c2w, scw, Lc, m1c, fc, mid, a1c, d, scc, has_sc, fin, bind](cudaStream_t st) mutable {
              Src xin = bind(x0, fin);
              eng->conv(xin, t, c1w, to_dst(m1c), st);
              eng->fold_norm(Lc, plain(m1c), fc, st);
              if (a1c.p) {  // act1 once per pixel, conv2 stages plain copies
                launch_materialize_act(mid, a1c.p, a1c.half, st);
                mid = plain(a1c);
              }
              Dst dd = d;
              if (has_sc) {
                eng->conv(xin, t1, scw, to_dst(scc), st);
                dd.addend = plain(scc);
              } else {
                dd.addend = xin;
              }
              eng->conv(mid, t, c2w, dd, st);
            }, L.has_shortcut ? 4 : 3);
            P.trace.push_back({-1, L.conv.c_in, c1, 3, 1, h, w, N});
            P.trace.push_back({-1, c1, co, 3, 1, h, w, N});
            if (L.has_shortcut) P.trace.push_back({-1, L.shortcut.c_in, co, 1, 1, h, w, N});
            flow = plain(o);
          } else {
            const int em = entry(h, w, cfg.block3), es = entry(h, w, cfg.block1);
            DevTensor& w1 = E.work_buffer(step, key + ".conv1.out");
            const DevTensor& c1c = E.cache_tensor(step, key + ".conv1.out");
            DevTensor& ws = E.work_buffer(step, key + ".sum");
            const DevTensor& csum = E.cache_tensor(step, key + ".sum");
            const DevTensor& osc = E.cache_tensor(step, key + ".shortcut.out");
            Tiles tm = tiles(em), ts = tiles(es);
            ConvW c1w = L.conv, c2w = L.conv2, scw = L.shortcut;
            // 1. conv1 over main tiles -> W(conv1.out)
            Dst d1 = to_dst(w1);
            // 2. conv2 on scatter_gather(m1) with norm1 + act (graph.cpp:821-846)
            Src mid = plain(w1);
            const bool reuse = L.norm_kind == SIGE_NORM_BATCH || cfg.norm_precompute;
            if (reuse && E.use_act()) {
              // conv1's epilogue also writes act1 = act(norm1(value)) for its
              // tiles into W(act1); conv2 stages plain copies of W(act1).
              const DevNorm& f = E.cache_norm(step, key + ".norm1");
              const DevTensor& ca = E.ensure_act(step, key, static_cast<int>(i), nullptr);
              DevTensor& wa = E.work_buffer(step, key + ".act1");
              d1.act = wa.p;
              d1.act_half = wa.half;
              d1.act_epi.fma_expf = host_expf_is_fma() ? 1 : 0;
              epi_push_ss(d1.act_epi, f.scale, f.shift, f.np, c1);
              epi_push_act(d1.act_epi, L.act);
              restore(wa, ca, em);
              mid = plain(wa);
              // conv2 reads act1 only: W(conv1.out) is never read in this mode,
              // so conv1 skips its fp32 store (2/3 of its epilogue bytes) and
              // the buffer needs no restore.
              d1.no_main = c1 % 16 == 0 && w1.c % 4 == 0 && !std::getenv("SIGE_KEEP_CONV1_OUT") ? 1 : 0;
            }
            add([eng, x0, tm, c1w, d1, fin, bind](cudaStream_t st) { eng->conv(bind(x0, fin), tm, c1w, d1, st); });
            if (!d1.no_main) restore(w1, c1c, em);
            if (reuse && E.use_act()) {
              // mid already reads W(act1)
            } else if (reuse) {
              const DevNorm& f = E.cache_norm(step, key + ".norm1");
              epi_push_ss(mid.epi, f.scale, f.shift, f.np, c1);
            } else {
              const int np = N * L.channels;
              DevNorm& f = E.scratch_norm("sparse." + key + ".norm1", np);
              LayerDev Lc = L;
              DevNorm fc = f;
              Src w1s = plain(w1);
              add([eng, Lc, fc, w1s](cudaStream_t st) mutable { eng->fold_norm(Lc, w1s, fc, st); });
              epi_push_ss(mid.epi, f.scale, f.shift, np, c1);
            }
            if (!(reuse && E.use_act())) epi_push_act(mid.epi, L.act);
            Dst d2 = to_dst(ws, kResMain);
            d2.aux = osc.p;
            // Identity shortcut on the tensor cores: the join (graph.cpp:854-879,
            // kernels.cpp:320-334) is fused into conv2 — no separate launch.
            const bool fuse_join = !L.has_shortcut && E.tensor_cores();
            if (fuse_join) {
              d2.join_bm = P.entries[es].bm;
              d2.main_bm = P.entries[em].bm;
              if (P.grouped) {  // one activity bitmap per request
                const auto words = [](const PlanEntryDev& e) {
                  return (((e.h + e.b - 1) / e.b) * ((e.w + e.b - 1) / e.b) + 31) / 32;
                };
                d2.join_bm_words = words(P.entries[es]);
                d2.main_bm_words = words(P.entries[em]);
              }
              d2.join_b = P.entries[es].b;
              d2.main_b = P.entries[em].b;
              d2.join_tiles = ts;
              add([eng, mid, tm, c2w, d2, x0, fin, bind](cudaStream_t st) {
                Dst dd = d2;
                dd.join_x = bind(x0, fin);
                eng->conv(mid, tm, c2w, dd, st);
              });
            } else {
              conv_step(mid, tm, c2w, d2);
            }
            restore(ws, csum, em);
            // 3. shortcut tiles (graph.cpp:854-879)
            Dst d3 = to_dst(ws, kResShortcut);
            d3.aux = osc.p;
            if (L.has_shortcut) {
              add([eng, x0, ts, scw, d3, fin, bind](cudaStream_t st) { eng->conv(bind(x0, fin), ts, scw, d3, st); });
            } else if (!fuse_join) {
              add([x0, ts, d3, fin, bind](cudaStream_t st) { launch_identity_join(bind(x0, fin), ts, d3, st); });
            }
            restore(ws, csum, es);
            P.trace.push_back({em, L.conv.c_in, c1, 3, 1, h, w, N});
            P.trace.push_back({em, c1, co, 3, 1, h, w, N});
            if (L.has_shortcut) P.trace.push_back({es, L.shortcut.c_in, co, 1, 1, h, w, N});
            flow = plain(ws);
          }
          flow_is_input = false;
          has_blocks = false;
          break;
        }
      }
    }
    if (br_forked) {  // the branch rejoins the main chain (before the final copy and the restores)
      const cudaEvent_t ev = br_record();
      add([ev](cudaStream_t st) { SIGE_CUDA(cudaStreamWaitEvent(st, ev, 0)); }, 0);
    }
    // Final output (graph.cpp:891-900).
    const DevTensor& cfin = E.cache_tensor(step, "final");
    static const bool old_tail = std::getenv("SIGE_FINALIZE_TAIL") != nullptr;  // A/B: the full-copy tail
    if (has_blocks && !old_tail) {
      // out = cached final (copied at the start of the call, run_program),
      // then the last layer's tiles; empty masks / samples without an edit keep
      // the copy (graph.cpp:665-668), exactly what the full finalize produced
      P.out_from_cache = cfin.p;
      P.out_bytes = cfin.numel() * sizeof(float);
      const Tiles t = tiles(blocks_entry);
      const Src sres = flow;
      add([eng, sres, t](cudaStream_t st) { launch_tiles_apply(sres, t, eng->cur_out_, kNCHW, st); });
      return;
    }
    Src result = flow;
    bool result_is_input = flow_is_input;
    if (has_blocks) {
      DevTensor& wf = E.work_buffer(step, "final");
      Tiles t = tiles(blocks_entry);
      Src s = flow;
      DevTensor wfc = wf;
      add([s, t, wfc](cudaStream_t st) { launch_tiles_apply(s, t, wfc.p, kNCHW, st); });
      restore(wf, cfin, blocks_entry);
      result = plain(wf);
      result_is_input = false;
    }
    // finalize: out = any(mask) ? result : cached final (empty-mask
    // short-circuit, graph.cpp:665-668), full NCHW copy.
    const float* cfp = cfin.p;
    int32_t* anyp = P.any;
    const int per_sample = P.grouped ? 1 : 0;
    add([eng, result, result_is_input, cfp, anyp, bind, per_sample](cudaStream_t st) {
      launch_finalize(bind(result, result_is_input), cfp, anyp, eng->cur_out_, st, per_sample);
    });
  }
};

Program& Engine::program(const sige_run_config& cfg, bool grouped) {
  const std::string key = config_key(cfg) + (grouped ? "|grouped" : "");
  auto it = programs_.find(key);
  if (it != programs_.end()) return *it->second;
  auto P = std::make_unique<Program>();
  P->grouped = grouped;
  const int masks = grouped ? batch_ : 1;
  P->full_h = in_h_;
  P->full_w = in_w_;
  P->dilate_full = cfg.dilate_full;
  P->dilate_scale = cfg.dilate_scale;
  P->bits = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * in_h_ * ((in_w_ + 31) / 32) * masks));
  P->any = static_cast<int32_t*>(alloc(sizeof(int32_t) * masks));
  P->stats_len = std::max<size_t>(stats_len(), 1);
  P->stats = static_cast<double*>(alloc(P->stats_len * sizeof(double)));
  ProgramBuilder b{*this, *P, cfg, {}};
  b.build();
  if (!P->entries.empty()) {
    P->entries_dev = static_cast<PlanEntryDev*>(alloc(P->entries.size() * sizeof(PlanEntryDev)));
    SIGE_CUDA(cudaMemcpy(P->entries_dev, P->entries.data(), P->entries.size() * sizeof(PlanEntryDev),
                         cudaMemcpyHostToDevice));
  }
  if (!P->restores.empty()) {
    P->restores_dev = static_cast<RestoreJob*>(alloc(P->restores.size() * sizeof(RestoreJob)));
    SIGE_CUDA(cudaMemcpy(P->restores_dev, P->restores.data(), P->restores.size() * sizeof(RestoreJob),
                         cudaMemcpyHostToDevice));
  }
  Program& ref = *P;
  programs_[key] = std::move(P);
  return ref;
}

void Engine::sparse_forward(const float* edited, const uint8_t* mask, const sige_run_config& cfg,
                            float* out, cudaStream_t st, bool grouped) {
  // RunConfig::validate (graph.cpp:220-227)
  if (cfg.mask_threshold < 0.0f) throw ConfigError("config: threshold must be >= 0");
  if (cfg.dilate_full < 0 || cfg.dilate_scale < 0) throw ConfigError("config: dilation radii must be >= 0");
  if (cfg.block3 < 1 || cfg.block1 < 1) throw ConfigError("config: block sizes must be >= 1");
  if (cfg.step < 0) throw ConfigError("config: step must be >= 0");
  if (cfg.sparse && cache_model_hash_ != structure_hash_)  // check_cache_model (graph.cpp:596-603)
    throw ConfigError("cache was precomputed for a different model than '" + name_ + "' (cache hash " +
                      std::to_string(cache_model_hash_) + ", model hash " + std::to_string(structure_hash_) + ")");
  const uint64_t before = g_launches.load();
  if (!cfg.sparse) {  // graph.cpp:626-663: plain dense forward
    dense_forward(edited, false, cfg.step, out, st);
    last_launches_ = static_cast<int>(g_launches.load() - before);
    return;
  }
  Program& P = program(cfg, grouped && batch_ > 1);
  cur_in_ = edited;
  cur_out_ = out;
  last_program_ = &P;
  // Replay: after one direct run the whole call (mask, plan, every fused conv,
  // final copy, restore) is captured once per (input, mask, output) binding
  // into a CUDA graph on an internal stream and replayed with one launch.
  if (use_graphs_ && !profiling_ && P.ran) {
    uint32_t thr_bits = 0;
    if (!mask) std::memcpy(&thr_bits, &cfg.mask_threshold, sizeof(thr_bits));
    auto key = std::make_tuple(static_cast<const void*>(edited), static_cast<const void*>(mask),
                               static_cast<const void*>(out), thr_bits);
    auto it = P.graphs.find(key);
    if (it == P.graphs.end()) {
      if (!cap_stream_) SIGE_CUDA(cudaStreamCreateWithFlags(&cap_stream_, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      const uint64_t b0 = g_launches.load();
      SIGE_CUDA(cudaStreamBeginCapture(cap_stream_, cudaStreamCaptureModeThreadLocal));
      try {
        run_program(P, edited, mask, cfg, cap_stream_);
      } catch (...) {
        cudaStreamEndCapture(cap_stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      SIGE_CUDA(cudaStreamEndCapture(cap_stream_, &g));
      const int kernels = static_cast<int>(g_launches.load() - b0);
      g_launches.fetch_sub(static_cast<uint64_t>(kernels));  // counted when the graph runs
      cudaGraphExec_t ex = nullptr;
      SIGE_CUDA(cudaGraphInstantiate(&ex, g, 0));
      cudaGraphDestroy(g);
      it = P.graphs.emplace(key, std::make_pair(ex, kernels)).first;
    }
    SIGE_CUDA(cudaGraphLaunch(it->second.first, st));
    g_launches.fetch_add(static_cast<uint64_t>(it->second.second));
    last_launches_ = it->second.second;
    return;
  }
  run_program(P, edited, mask, cfg, st);
  P.ran = true;
  last_launches_ = static_cast<int>(g_launches.load() - before);
}

// One sparse_forward call on `st`: mask -> bits (compute_difference_mask
// against the cached original input when no mask is given), the IndexPlan,
// every compiled step, then the restore of the tiles this call dirtied.
void Engine::run_program(Program& P, const float* edited, const uint8_t* mask,
                         const sige_run_config& cfg, cudaStream_t st) {
  tl_next_ = 0;
  tl_meta_.clear();
  static const bool no_fork = std::getenv("SIGE_NO_FORK") != nullptr;  // A/B switch
  const bool fork = in_twin_ && !no_fork;
  if (fork) {
    // The fp16 input twin depends on the edited input only: it runs on a side
    // branch (a parallel graph node when captured) beside the mask and the
    // IndexPlan instead of between the plan and the first conv.
    if (!side_stream_) {
      SIGE_CUDA(cudaStreamCreateWithFlags(&side_stream_, cudaStreamNonBlocking));
      SIGE_CUDA(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming));
      SIGE_CUDA(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming));
    }
    SIGE_CUDA(cudaEventRecord(fork_ev_, st));
    SIGE_CUDA(cudaStreamWaitEvent(side_stream_, fork_ev_, 0));
    launch_input_twin(edited, batch_, in_c_, in_h_, in_w_, in_twin_c_, in_twin_, side_stream_);
    if (P.out_from_cache)
      SIGE_CUDA(cudaMemcpyAsync(cur_out_, P.out_from_cache, P.out_bytes, cudaMemcpyDeviceToDevice, side_stream_));
    SIGE_CUDA(cudaEventRecord(join_ev_, side_stream_));
  } else if (P.out_from_cache) {
    SIGE_CUDA(cudaMemcpyAsync(cur_out_, P.out_from_cache, P.out_bytes, cudaMemcpyDeviceToDevice, st));
  }
  const int masks = P.grouped ? batch_ : 1;
  SIGE_CUDA(cudaMemsetAsync(P.any, 0, sizeof(int32_t) * masks, st));
  if (P.stats_used) SIGE_CUDA(cudaMemsetAsync(P.stats, 0, P.stats_used * sizeof(double), st));
  if (mask) {
    launch_mask_u8_to_bits(mask, in_h_, in_w_, P.bits, P.any, st, masks);
  } else {
    const DevTensor& orig = cache_tensor(cfg.step, "input");
    launch_mask_bits(orig.p, edited, batch_, in_c_, in_h_, in_w_, cfg.mask_threshold, P.bits,
                     nullptr, P.any, st, P.grouped ? 1 : 0);
  }
  launch_plan(P.bits, in_h_, in_w_, cfg.dilate_full, cfg.dilate_scale, batch_, P.entries_dev,
              static_cast<int>(P.entries.size()), st, P.grouped ? 1 : 0);
  if (fork)
    SIGE_CUDA(cudaStreamWaitEvent(st, join_ev_, 0));
  else if (in_twin_)
    launch_input_twin(edited, batch_, in_c_, in_h_, in_w_, in_twin_c_, in_twin_, st);
  for (auto& f : P.steps) f(st);
  if (!P.restores.empty())
    launch_restore(P.restores_dev, static_cast<int>(P.restores.size()),
                   static_cast<int>(std::min<long long>(P.restore_max, 1LL << 30)), st);
}

void Engine::set_graphs(bool on) { use_graphs_ = on; }

void Engine::release(void* p) {
  if (!p) return;
  auto it = std::find(allocations_.begin(), allocations_.end(), p);
  if (it == allocations_.end()) return;
  cudaFree(p);
  allocations_.erase(it);
}

void Engine::drop_step(int step) {  // ActivationCache::drop_step (graph.cpp:271-274)
  free_device_step(step);
  free_host_step(step);  // an offloaded copy goes too
}

void Engine::free_device_step(int step) {
  invalidate_programs();  // programs and captured graphs point into the dropped entries
  for (auto it = cache_.begin(); it != cache_.end();) {
    if (it->first.first != step) {
      ++it;
      continue;
    }
    release(it->second.p);  // the step's device memory goes back (multi-step caches)
    release(it->second.h16);
    it = cache_.erase(it);
  }
  for (auto it = norms_.begin(); it != norms_.end();) {
    if (it->first.first != step) {
      ++it;
      continue;
    }
    release(it->second.scale);
    release(it->second.shift);
    it = norms_.erase(it);
  }
}

void Engine::free_host_step(int step) {
  for (auto it = host_cache_.begin(); it != host_cache_.end();) {
    if (it->first.first != step) {
      ++it;
      continue;
    }
    cudaFreeHost(it->second.host);
    if (it->second.host16) cudaFreeHost(it->second.host16);
    it = host_cache_.erase(it);
  }
  for (auto it = host_norms_.begin(); it != host_norms_.end();) {
    if (it->first.first != step) {
      ++it;
      continue;
    }
    cudaFreeHost(it->second.scale);
    cudaFreeHost(it->second.shift);
    it = host_norms_.erase(it);
  }
}

// The host copy is the step's home once offloaded (the cache is immutable
// after precompute); a later offload of the same, unchanged step only frees
// the device memory again.
void Engine::offload_step(int step, cudaStream_t st) {
  bool any = false;
  for (auto& kv : cache_) {
    if (kv.first.first != step) continue;
    any = true;
    if (host_cache_.count(kv.first)) continue;  // host copy already current
    const DevTensor& t = kv.second;
    HostEntry& h = host_cache_[kv.first];
    h.meta = t;
    h.meta.p = nullptr;
    h.meta.h16 = nullptr;
    SIGE_CUDA(cudaMallocHost(&h.host, std::max<size_t>(t.bytes(), 16)));
    SIGE_CUDA(cudaMemcpyAsync(h.host, t.p, t.bytes(), cudaMemcpyDeviceToHost, st));
    if (t.h16) {
      SIGE_CUDA(cudaMallocHost(&h.host16, std::max<size_t>(t.numel() * 2, 16)));
      SIGE_CUDA(cudaMemcpyAsync(h.host16, t.h16, t.numel() * 2, cudaMemcpyDeviceToHost, st));
    }
  }
  for (auto& kv : norms_) {
    if (kv.first.first != step || host_norms_.count(kv.first)) continue;
    HostNorm& h = host_norms_[kv.first];
    h.np = kv.second.np;
    SIGE_CUDA(cudaMallocHost(&h.scale, std::max<size_t>(h.np * sizeof(float), 16)));
    SIGE_CUDA(cudaMallocHost(&h.shift, std::max<size_t>(h.np * sizeof(float), 16)));
    SIGE_CUDA(cudaMemcpyAsync(h.scale, kv.second.scale, h.np * sizeof(float), cudaMemcpyDeviceToHost, st));
    SIGE_CUDA(cudaMemcpyAsync(h.shift, kv.second.shift, h.np * sizeof(float), cudaMemcpyDeviceToHost, st));
  }
  if (!any) throw ConfigError("offload_step: no cache entry for step " + std::to_string(step));
  SIGE_CUDA(cudaStreamSynchronize(st));  // the copies landed: the device memory can go
  free_device_step(step);
}

// Asynchronous on `st`: the H2D copies overlap whatever runs on other streams
// (PAPER.md:389); the step's sparse_forward must be ordered after them.
void Engine::prefetch_step(int step, cudaStream_t st) {
  bool any = false;
  for (auto& kv : host_cache_) {
    if (kv.first.first != step) continue;
    any = true;
    const HostEntry& h = kv.second;
    if (cache_.count(kv.first)) continue;  // already resident
    DevTensor& t = cache_slot(step, kv.first.second, h.meta.c, h.meta.h, h.meta.w, h.meta.layout, h.meta.half);
    SIGE_CUDA(cudaMemcpyAsync(t.p, h.host, t.bytes(), cudaMemcpyHostToDevice, st));
    if (h.host16) {
      if (!t.h16) t.h16 = alloc(t.numel() * 2);
      SIGE_CUDA(cudaMemcpyAsync(t.h16, h.host16, t.numel() * 2, cudaMemcpyHostToDevice, st));
    }
  }
  for (auto& kv : host_norms_) {
    if (kv.first.first != step || norms_.count(kv.first)) continue;
    DevNorm& n = norm_slot(step, kv.first.second, kv.second.np);
    SIGE_CUDA(cudaMemcpyAsync(n.scale, kv.second.scale, kv.second.np * sizeof(float), cudaMemcpyHostToDevice, st));
    SIGE_CUDA(cudaMemcpyAsync(n.shift, kv.second.shift, kv.second.np * sizeof(float), cudaMemcpyHostToDevice, st));
  }
  if (!any) throw ConfigError("prefetch_step: step " + std::to_string(step) + " was not offloaded");
}

bool Engine::step_offloaded(int step) const {
  for (auto& kv : host_cache_)
    if (kv.first.first == step && !cache_.count(kv.first)) return true;
  return false;
}

void Engine::refresh_step(const float* original, int step, cudaStream_t st) {  // graph.cpp:437-444
  drop_step(step);
  precompute(original, step, st);
}

void Engine::set_sm_budget(int sms) {
  if (sms < 0) throw ConfigError("engine: SM budget must be >= 0");
  if (sms != sm_budget_) invalidate_programs();  // captured launches carry the old grids
  sm_budget_ = sms;
}

// output_coverage (graph.cpp:1078-1129) on the device: the output pixels a
// sparse_forward with this mask / config may change — the same layer walk over
// the same on-device IndexPlan the executor uses (tile footprints of sparse
// layers, dilation / downsample / 2x upsample of the running coverage for
// dense ones, everything for fresh-statistics norms). A cross-check of the
// executor's coverage against the reference's (tests/test_gpu_engine.py).
void Engine::output_coverage(const float* edited, const uint8_t* mask, const sige_run_config& cfg, uint8_t* out,
                             int* oh, int* ow, cudaStream_t st) {
  if (cfg.mask_threshold < 0.0f) throw ConfigError("config: threshold must be >= 0");
  if (cfg.dilate_full < 0 || cfg.dilate_scale < 0) throw ConfigError("config: dilation radii must be >= 0");
  if (cfg.block3 < 1 || cfg.block1 < 1) throw ConfigError("config: block sizes must be >= 1");
  *oh = out_h_;
  *ow = out_w_;
  Program& P = program(cfg, false);
  size_t cap = static_cast<size_t>(in_h_) * in_w_;
  for (const LayerShape& sh : shapes_) cap = std::max(cap, static_cast<size_t>(sh.h_out) * sh.w_out);
  uint8_t* a = static_cast<uint8_t*>(alloc(cap));
  uint8_t* b = static_cast<uint8_t*>(alloc(cap));
  uint8_t* t = static_cast<uint8_t*>(alloc(cap));
  struct Free {
    Engine* e;
    std::vector<void*> p;
    ~Free() {
      cudaDeviceSynchronize();
      for (void* q : p) e->release(q);
    }
  } fr{this, {a, b, t}};
  SIGE_CUDA(cudaMemsetAsync(P.any, 0, sizeof(int32_t), st));
  if (mask) {
    launch_mask_u8_to_bits(mask, in_h_, in_w_, P.bits, P.any, st);
    SIGE_CUDA(cudaMemcpyAsync(a, mask, static_cast<size_t>(in_h_) * in_w_, cudaMemcpyDeviceToDevice, st));
  } else {
    const DevTensor& orig = cache_tensor(cfg.step, "input");
    launch_mask_bits(orig.p, edited, batch_, in_c_, in_h_, in_w_, cfg.mask_threshold, P.bits, a, P.any, st);
  }
  int h = in_h_, w = in_w_;
  auto entry = [&](int eh, int ew, int eb) -> const PlanEntryDev& {
    for (const PlanEntryDev& e : P.entries)
      if (e.h == eh && e.w == ew && e.b == eb) return e;
    throw ConfigError("output_coverage: no plan entry for " + std::to_string(eh) + "x" + std::to_string(ew));
  };
  auto footprint = [&](const PlanEntryDev& e, bool clear) {
    if (clear) SIGE_CUDA(cudaMemsetAsync(a, 0, static_cast<size_t>(e.h) * e.w, st));
    op_cov_footprint(e.idx, e.count, e.capacity, e.b, e.h, e.w, a, st);
  };
  auto dilate = [&](int r) {
    if (r <= 0) return;
    op_dilate_mask(a, h, w, r, b, t, st);
    std::swap(a, b);
  };
  if (cfg.sparse) {
    launch_plan(P.bits, in_h_, in_w_, cfg.dilate_full, cfg.dilate_scale, batch_, P.entries_dev,
                static_cast<int>(P.entries.size()), st);
    dilate(cfg.dilate_full);
    for (size_t i = 0; i < layers_.size(); ++i) {
      const LayerDev& L = layers_[i];
      const LayerShape& s = shapes_[i];
      const bool sp = runs_sparse(L, s.h_in, s.w_in, cfg);
      switch (L.kind) {
        case SIGE_LAYER_CONV:
        case SIGE_LAYER_DOWNSAMPLE:
          if (sp) {
            footprint(entry(s.h_out, s.w_out, L.conv.k == 3 ? cfg.block3 : cfg.block1), true);
          } else {
            dilate((L.conv.k - 1) / 2);
            if (L.conv.stride == 2) {
              op_downsample_mask(a, h, w, s.h_out, s.w_out, b, st);
              std::swap(a, b);
            }
          }
          break;
        case SIGE_LAYER_NORM:
          if (L.norm_kind != SIGE_NORM_BATCH && !cfg.norm_precompute)
            SIGE_CUDA(cudaMemsetAsync(a, 1, static_cast<size_t>(s.h_out) * s.w_out, st));
          break;
        case SIGE_LAYER_UPSAMPLE:
          op_cov_up2(a, h, w, b, st);
          std::swap(a, b);
          break;
        case SIGE_LAYER_SPADE_RESBLOCK:
        case SIGE_LAYER_RESIZE:
          throw ConfigError("output_coverage: SPADE models (config 3) are not supported");
        case SIGE_LAYER_RESBLOCK:
          if (sp) {
            footprint(entry(s.h_out, s.w_out, cfg.block3), true);
            footprint(entry(s.h_out, s.w_out, cfg.block1), false);
          } else {
            dilate(2);
            if (L.norm_kind != SIGE_NORM_BATCH && !cfg.norm_precompute)
              SIGE_CUDA(cudaMemsetAsync(a, 1, static_cast<size_t>(s.h_out) * s.w_out, st));
          }
          break;
        default:
          break;
      }
      h = s.h_out;
      w = s.w_out;
    }
  }
  const long long n = static_cast<long long>(out_h_) * out_w_;
  op_cov_final(a, n, P.any, cfg.sparse ? 0 : 1, st);  // empty mask -> nothing; dense -> everything
  if (!cfg.sparse) op_cov_final(a, n, P.any, 0, st);
  SIGE_CUDA(cudaMemcpyAsync(out, a, n, cudaMemcpyDeviceToDevice, st));
}

int Engine::trace(uint64_t* rows, int cap, cudaStream_t st) {
  if (!last_program_) return 0;
  Program& P = *last_program_;
  std::vector<int32_t> counts(P.entries.size());
  for (size_t i = 0; i < P.entries.size(); ++i)
    SIGE_CUDA(cudaMemcpyAsync(&counts[i], P.entries[i].count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> anys(P.grouped ? batch_ : 1, 0);
  SIGE_CUDA(cudaMemcpyAsync(anys.data(), P.any, sizeof(int32_t) * anys.size(), cudaMemcpyDeviceToHost, st));
  SIGE_CUDA(cudaStreamSynchronize(st));
  bool any = false;
  for (int32_t a : anys) any = any || a != 0;
  if (!any) return 0;  // short-circuit: no trace rows (graph.cpp:665-668)
  int n = 0;
  for (const TraceInfo& t : P.trace) {
    if (n < cap && rows) {
      uint64_t* r = rows + 6 * n;
      const uint64_t dense = static_cast<uint64_t>(t.c_out) * t.c_in * t.k * t.k * t.oh * t.ow * t.batch;
      if (t.entry < 0) {
        r[0] = r[1] = r[2] = 0;
        r[3] = r[4] = dense;
        r[5] = 0;
      } else {
        const int b = P.entries[t.entry].b;
        const uint64_t g = static_cast<uint64_t>(counts[t.entry]);
        const int win = t.stride * b + t.k - t.stride;
        r[0] = g;
        r[1] = g * t.c_in * win * win;
        r[2] = g * t.c_out * b * b;
        r[3] = g * t.c_out * t.c_in * t.k * t.k * b * b;
        r[4] = dense;
        r[5] = 1;
      }
    }
    ++n;
  }
  return n;
}

}  // namespace sige_b200
