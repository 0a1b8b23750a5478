// models.cpp — synthetic inputs and model weights for the BASELINE workloads.
//
// The reference generates every input from its seeded Rng (std::mt19937 with
// the toolchain-portable float mapping of proj/include/sige/common.hpp:25-43):
// edit fixtures (proj/src/fixtures.cpp:26-128) and toy models
// (proj/src/models.cpp:8-161). The bench and the parity tests need the very
// same bytes on the device side, so this file restates those generators plus
// the two BASELINE models (single_conv64 = config 1, ddim_stack = config 2;
// DESIGN.md "Synthetic workloads"). model_weight_hash / content hashes pin
// them to the reference (tests/test_oracle_golden.py, tests/test_models.py).
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "common.hpp"
#include "models.hpp"

namespace sige_b200 {

uint64_t fnv1a64(const void* data, size_t bytes, uint64_t h) {
  const auto* p = static_cast<const uint8_t*>(data);
  for (size_t i = 0; i < bytes; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

namespace {

struct Rng {
  std::mt19937 st;
  explicit Rng(uint32_t seed) : st(seed) {}
  uint32_t u32() { return st(); }
  float uniform(float lo, float hi) {  // common.hpp:33-36
    double u = u32() * (1.0 / 4294967296.0);
    return static_cast<float>(lo + (static_cast<double>(hi) - lo) * u);
  }
  int uniform_int(int lo, int hi) {  // common.hpp:39-41
    return lo + static_cast<int>(u32() % static_cast<uint32_t>(hi - lo + 1));
  }
};

struct Region {
  int h, w;
  std::vector<uint8_t> on;
  void rect(int y0, int x0, int he, int we) {
    for (int y = y0; y < y0 + he; ++y)
      for (int x = x0; x < x0 + we; ++x) on[static_cast<size_t>(y) * w + x] = 1;
  }
};

void square(Region& g, Rng& r, double px, int x_lo, int x_hi) {  // fixtures.cpp:26-34
  int side = std::max(1, static_cast<int>(std::lround(std::sqrt(px))));
  int we = std::min(side, x_hi - x_lo);
  int he = std::min(std::max(1, static_cast<int>(std::lround(px / we))), g.h);
  int y0 = r.uniform_int(0, g.h - he);
  int x0 = x_lo + r.uniform_int(0, (x_hi - x_lo) - we);
  g.rect(y0, x0, he, we);
}

void blob(Region& g, Rng& r, int target) {  // fixtures.cpp:37-60
  std::vector<std::pair<int, int>> fr{{r.uniform_int(g.h / 4, 3 * g.h / 4), 0}};
  fr[0].second = r.uniform_int(g.w / 4, 3 * g.w / 4);
  int painted = 0;
  const int dy[4] = {-1, 1, 0, 0}, dx[4] = {0, 0, -1, 1};
  while (painted < target && !fr.empty()) {
    int pick = r.uniform_int(0, static_cast<int>(fr.size()) - 1);
    auto [y, x] = fr[pick];
    fr[pick] = fr.back();
    fr.pop_back();
    uint8_t& cell = g.on[static_cast<size_t>(y) * g.w + x];
    if (cell) continue;
    cell = 1;
    ++painted;
    for (int d = 0; d < 4; ++d) {
      int ny = y + dy[d], nx = x + dx[d];
      if (ny >= 0 && ny < g.h && nx >= 0 && nx < g.w && !g.on[static_cast<size_t>(ny) * g.w + nx])
        fr.push_back({ny, nx});
    }
  }
}

// ------------------------------------------------------------- model IR --
struct OwnedModel {
  sige_model_desc desc{};  // must stay first: sige_model_free casts back
  std::string name;
  std::vector<sige_layer_desc> layers;
  std::vector<std::unique_ptr<std::vector<float>>> buffers;
  std::vector<std::unique_ptr<sige_spade_desc[]>> spades;

  const float* keep(std::vector<float> v) {
    buffers.push_back(std::make_unique<std::vector<float>>(std::move(v)));
    return buffers.back()->data();
  }
  std::vector<float> uni(Rng& r, size_t n, float lo, float hi) {
    std::vector<float> v(n);
    for (float& x : v) x = r.uniform(lo, hi);
    return v;
  }
  sige_conv_desc conv(Rng& r, int ci, int co, int k, int s) {  // models.cpp:8-27
    sige_conv_desc c{ci, co, k, s, nullptr, nullptr};
    float bound = 1.0f / std::sqrt(static_cast<float>(ci * k * k));
    c.weight = keep(uni(r, static_cast<size_t>(co) * ci * k * k, -bound, bound));
    c.bias = keep(uni(r, co, -0.05f, 0.05f));
    return c;
  }
  sige_norm_desc norm(Rng& r, int kind, int ch, int groups) {  // models.cpp:29-45
    sige_norm_desc n{kind, kind == SIGE_NORM_INSTANCE ? ch : groups, ch, 1e-5f,
                     nullptr, nullptr, nullptr, nullptr};
    n.gamma = keep(uni(r, ch, 0.8f, 1.2f));
    n.beta = keep(uni(r, ch, -0.1f, 0.1f));
    if (kind == SIGE_NORM_BATCH) {
      n.running_mean = keep(uni(r, ch, -0.3f, 0.3f));
      n.running_var = keep(uni(r, ch, 0.5f, 1.5f));
    }
    return n;
  }
  static sige_layer_desc blank(int kind) {
    sige_layer_desc L;
    std::memset(&L, 0, sizeof L);
    L.kind = kind;
    L.policy_sparse = 1;
    L.min_resolution = 16;  // SparsePolicy defaults (graph.hpp:30-35)
    return L;
  }
  void add_conv(Rng& r, int ci, int co, int k, int s) {
    sige_layer_desc L = blank(s == 2 ? SIGE_LAYER_DOWNSAMPLE : SIGE_LAYER_CONV);
    L.conv = conv(r, ci, co, k, s);
    layers.push_back(L);
  }
  void add_norm(Rng& r, int kind, int ch, int groups) {
    sige_layer_desc L = blank(SIGE_LAYER_NORM);
    L.norm = norm(r, kind, ch, groups);
    layers.push_back(L);
  }
  void add_act(int act) {
    sige_layer_desc L = blank(SIGE_LAYER_ACTIVATION);
    L.act = act;
    layers.push_back(L);
  }
  void add_up() { layers.push_back(blank(SIGE_LAYER_UPSAMPLE)); }
  void add_res(Rng& r, int ci, int co, int nk, int groups, int act) {  // models.cpp:76-89
    sige_layer_desc L = blank(SIGE_LAYER_RESBLOCK);
    L.conv = conv(r, ci, co, 3, 1);
    L.norm = norm(r, nk, co, groups);
    L.act = act;
    L.conv2 = conv(r, co, co, 3, 1);
    if (ci != co) {
      L.has_shortcut = 1;
      L.shortcut = conv(r, ci, co, 1, 1);
    }
    layers.push_back(L);
  }
  void add_resize(int h, int w) {
    sige_layer_desc L = blank(SIGE_LAYER_RESIZE);
    L.resize_h = h;
    L.resize_w = w;
    layers.push_back(L);
  }
  // SPADE residual block (SPADEResnetBlock of Park et al. 2019): fmiddle =
  // min(fin, fout), learned 1x1 shortcut (no bias) when fin != fout, LeakyReLU(0.2),
  // three SPADE norms (instance norm, nhidden-wide shared 3x3 + ReLU, 3x3 gamma/beta).
  void add_spade_res(Rng& r, int fin, int fout, int label_nc, int nhidden) {
    sige_layer_desc L = blank(SIGE_LAYER_SPADE_RESBLOCK);
    const int fmid = std::min(fin, fout);
    L.conv = conv(r, fin, fmid, 3, 1);
    L.conv2 = conv(r, fmid, fout, 3, 1);
    L.act = SIGE_ACT_LEAKY_RELU;
    if (fin != fout) {
      L.has_shortcut = 1;
      L.shortcut = conv(r, fin, fout, 1, 1);
      L.shortcut.bias = nullptr;
    }
    auto sp = std::make_unique<sige_spade_desc[]>(3);
    const int chans[3] = {fin, fmid, fin};
    for (int k = 0; k < (fin != fout ? 3 : 2); ++k) {
      sp[k].eps = 1e-5f;
      sp[k].shared = conv(r, label_nc, nhidden, 3, 1);
      sp[k].gamma = conv(r, nhidden, chans[k], 3, 1);
      sp[k].beta = conv(r, nhidden, chans[k], 3, 1);
    }
    L.spade = sp.get();
    spades.push_back(std::move(sp));
    layers.push_back(L);
  }
  sige_model_desc* finish(const std::string& nm, int ci, int h, int w) {
    name = nm;
    desc.name = name.c_str();
    desc.in_channels = ci;
    desc.in_h = h;
    desc.in_w = w;
    desc.num_layers = static_cast<int>(layers.size());
    desc.layers = layers.data();
    return &desc;
  }
};

sige_model_desc* build_mini_unet(OwnedModel* m, int nk, const std::string& name, uint32_t seed) {
  Rng r(seed);  // models.cpp:102-121
  m->add_conv(r, 3, 16, 3, 1);
  m->add_norm(r, nk, 16, 4);
  m->add_act(SIGE_ACT_SILU);
  m->add_res(r, 16, 16, nk, 4, SIGE_ACT_SILU);
  m->add_conv(r, 16, 32, 3, 2);
  m->add_res(r, 32, 32, nk, 8, SIGE_ACT_SILU);
  m->add_conv(r, 32, 64, 3, 2);
  m->add_res(r, 64, 64, nk, 8, SIGE_ACT_SILU);
  m->add_up();
  m->add_res(r, 64, 32, nk, 8, SIGE_ACT_SILU);
  m->add_up();
  m->add_res(r, 32, 16, nk, 4, SIGE_ACT_SILU);
  m->add_conv(r, 16, 3, 3, 1);
  return m->finish(name, 3, 64, 64);
}

// DDIM-UNet-shaped post-norm residual stack (BASELINE config 2; SURVEY
// §8(d)): conv_in 3->base, six levels of two ResBlocks (mult 1,1,2,2,4,4)
// with a 3x3 s2 Downsample between levels, two middle ResBlocks, six decoder
// levels of three ResBlocks with Upsample + 3x3 conv between, GN32 + SiLU +
// conv_out. At (256, 128): 51 layers, 80 conv sites, required_dilation 822.
sige_model_desc* build_ddim(OwnedModel* m, int res, int base) {
  Rng r(2211);
  const int mult[6] = {1, 1, 2, 2, 4, 4};
  m->add_conv(r, 3, base, 3, 1);
  int c = base;
  for (int lvl = 0; lvl < 6; ++lvl) {
    for (int j = 0; j < 2; ++j) {
      m->add_res(r, c, base * mult[lvl], SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
      c = base * mult[lvl];
    }
    if (lvl < 5) m->add_conv(r, c, c, 3, 2);
  }
  for (int j = 0; j < 2; ++j) m->add_res(r, c, c, SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
  for (int lvl = 0; lvl < 6; ++lvl) {
    int dc = base * mult[5 - lvl];
    for (int j = 0; j < 3; ++j) {
      m->add_res(r, c, dc, SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
      c = dc;
    }
    if (lvl < 5) {
      m->add_up();
      m->add_conv(r, c, c, 3, 1);
    }
  }
  m->add_norm(r, SIGE_NORM_GROUP, c, 32);
  m->add_act(SIGE_ACT_SILU);
  m->add_conv(r, c, 3, 3, 1);
  return m->finish("ddim_stack", 3, res, res);
}

// GauGAN SPADE generator (BASELINE config 3; SPADEGenerator, Park et al. 2019,
// "normal" upsampling): the segmentation map (label_nc channels) is resized to
// (h/32, w/32) and mapped by a 3x3 conv to 16 nf channels, then 7 SPADE
// residual blocks with nearest 2x upsampling between levels (16nf, 16nf, 16nf,
// 8nf, 4nf, 2nf, nf), LeakyReLU(0.2) and a 3x3 conv to RGB (the final tanh is
// a pointwise map on the result and not part of the sparse path). Random init,
// Rng seed 3003.
sige_model_desc* build_gaugan(OwnedModel* m, const std::string& name, int label_nc, int h, int w, int nf,
                              int nhidden) {
  Rng r(3003);
  m->add_resize(h / 32, w / 32);
  m->add_conv(r, label_nc, 16 * nf, 3, 1);
  m->add_spade_res(r, 16 * nf, 16 * nf, label_nc, nhidden);  // head_0
  m->add_up();
  m->add_spade_res(r, 16 * nf, 16 * nf, label_nc, nhidden);  // G_middle_0
  m->add_spade_res(r, 16 * nf, 16 * nf, label_nc, nhidden);  // G_middle_1
  const int ch[5] = {16 * nf, 8 * nf, 4 * nf, 2 * nf, nf};
  for (int i = 0; i < 4; ++i) {
    m->add_up();
    m->add_spade_res(r, ch[i], ch[i + 1], label_nc, nhidden);  // up_0 .. up_3
  }
  m->add_act(SIGE_ACT_LEAKY_RELU);
  m->add_conv(r, nf, 3, 3, 1);  // conv_img
  return m->finish(name, label_nc, h, w);
}

}  // namespace

// A synthetic segmentation map (config 3): one-hot over label_nc classes of
// random axis-aligned regions on a background class, and an edited copy where
// a rect1-style square (fixtures.cpp:26-34, 1.2 % of the pixels) is relabelled
// — the SIGE GauGAN edit (change the label of a region).
void make_seg_fixture(int n, int label_nc, int h, int w, uint32_t seed, float* orig, float* edited) {
  Rng r(seed);
  std::vector<int> lab(static_cast<size_t>(h) * w, 0);
  for (int k = 0; k < 12; ++k) {
    const int cls = r.uniform_int(1, label_nc - 1);
    const int he = r.uniform_int(h / 8, h / 2), we = r.uniform_int(w / 8, w / 2);
    const int y0 = r.uniform_int(0, h - he), x0 = r.uniform_int(0, w - we);
    for (int y = y0; y < y0 + he; ++y)
      for (int x = x0; x < x0 + we; ++x) lab[static_cast<size_t>(y) * w + x] = cls;
  }
  Region g{h, w, std::vector<uint8_t>(static_cast<size_t>(h) * w, 0)};
  square(g, r, 0.012 * h * w, 0, w);
  const int new_cls = r.uniform_int(1, label_nc - 1);
  for (int in = 0; in < n; ++in)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const size_t px = static_cast<size_t>(y) * w + x;
        const int lo = lab[px], le = g.on[px] ? new_cls : lo;
        for (int c = 0; c < label_nc; ++c) {
          const size_t at = ((static_cast<size_t>(in) * label_nc + c) * h + y) * w + x;
          orig[at] = c == lo ? 1.0f : 0.0f;
          edited[at] = c == le ? 1.0f : 0.0f;
        }
      }
}

void make_edit_fixture(const std::string& kind, int n, int c, int h, int w, uint32_t seed,
                       float* orig, float* edited) {
  Rng r(seed);
  size_t total = static_cast<size_t>(n) * c * h * w;
  for (size_t i = 0; i < total; ++i) orig[i] = r.uniform(-1.0f, 1.0f);
  Region g{h, w, std::vector<uint8_t>(static_cast<size_t>(h) * w, 0)};
  double px = static_cast<double>(h) * w;
  if (kind == "rect1") {
    square(g, r, 0.012 * px, 0, w);
  } else if (kind == "rect5") {
    square(g, r, 0.05 * px, 0, w);
  } else if (kind == "rect15") {
    square(g, r, 0.15 * px, 0, w);
  } else if (kind == "rect35") {
    square(g, r, 0.35 * px, 0, w);
  } else if (kind == "blob5") {
    blob(g, r, static_cast<int>(std::lround(0.05 * px)));
  } else if (kind == "multi15") {
    for (int band = 0; band < 3; ++band) square(g, r, 0.15 * px / 3.0, band * w / 3, (band + 1) * w / 3);
  } else if (kind.rfind("rect_", 0) == 0) {
    // rect_<percent>: a square of arbitrary area (edit-area sweep)
    square(g, r, std::stod(kind.substr(5)) / 100.0 * px, 0, w);
  } else {
    throw ConfigError("unknown edit fixture: " + kind +
                      " (expected one of rect1, rect5, rect15, rect35, blob5, multi15, rect_<pct>)");
  }
  std::memcpy(edited, orig, total * sizeof(float));
  for (int in = 0; in < n; ++in)
    for (int ic = 0; ic < c; ++ic)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          if (!g.on[static_cast<size_t>(y) * w + x]) continue;
          float mag = r.uniform(0.05f, 0.5f);
          float sign = r.uniform(0.0f, 1.0f) < 0.5f ? -1.0f : 1.0f;
          size_t at = ((static_cast<size_t>(in) * c + ic) * h + y) * w + x;
          edited[at] += sign * mag;
        }
}

sige_model_desc* build_model(const std::string& name) {
  auto m = std::make_unique<OwnedModel>();
  sige_model_desc* d = nullptr;
  if (name == "conv3x3_128" || name == "single_conv64") {
    int c = name == "conv3x3_128" ? 128 : 64;
    Rng r(1001);  // models.cpp:91-100
    m->add_conv(r, c, c, 3, 1);
    d = m->finish(name, c, 256, 256);
  } else if (name == "mini_unet_gn") {
    d = build_mini_unet(m.get(), SIGE_NORM_GROUP, name, 1002);
  } else if (name == "mini_unet_bn") {
    d = build_mini_unet(m.get(), SIGE_NORM_BATCH, name, 1003);
  } else if (name == "gaugan_stack_in") {
    Rng r(1004);  // models.cpp:123-140
    m->add_conv(r, 3, 16, 3, 2);
    m->add_act(SIGE_ACT_RELU);
    m->add_conv(r, 16, 32, 3, 2);
    m->add_act(SIGE_ACT_RELU);
    m->add_res(r, 32, 32, SIGE_NORM_INSTANCE, 32, SIGE_ACT_RELU);
    m->add_up();
    m->add_res(r, 32, 16, SIGE_NORM_INSTANCE, 16, SIGE_ACT_RELU);
    m->add_up();
    m->add_conv(r, 16, 3, 3, 1);
    d = m->finish(name, 3, 64, 64);
  } else if (name == "ddim_stack") {
    d = build_ddim(m.get(), 256, 128);
  } else if (name == "ddim_stack_64x32") {
    d = build_ddim(m.get(), 64, 32);
  } else if (name == "gaugan_spade") {  // BASELINE config 3: Cityscapes 256x512, 36 labels, nf 64
    d = build_gaugan(m.get(), name, 36, 256, 512, 64, 128);
  } else if (name == "gaugan_spade_mini") {  // the same generator at 64x128, nf 8 (tests)
    d = build_gaugan(m.get(), name, 8, 64, 128, 8, 16);
  } else {
    throw ConfigError("unknown model: " + name +
                      " (expected one of conv3x3_128, mini_unet_gn, mini_unet_bn, gaugan_stack_in,"
                      " single_conv64, ddim_stack, ddim_stack_64x32, gaugan_spade, gaugan_spade_mini)");
  }
  m.release();
  return d;
}

void free_model(sige_model_desc* d) { delete reinterpret_cast<OwnedModel*>(d); }

namespace {
uint64_t hv(const float* p, size_t n, uint64_t h) { return p ? fnv1a64(p, n * sizeof(float), h) : h; }
uint64_t hconv(const sige_conv_desc& c, uint64_t h) {
  h = hv(c.weight, static_cast<size_t>(c.c_out) * c.c_in * c.k * c.k, h);
  return hv(c.bias, c.bias ? c.c_out : 0, h);
}
uint64_t hnorm(const sige_norm_desc& n, uint64_t h) {
  h = hv(n.gamma, n.channels, h);
  h = hv(n.beta, n.channels, h);
  h = hv(n.running_mean, n.channels, h);
  return hv(n.running_var, n.channels, h);
}
}  // namespace

// ModelSpec::structure_hash (graph.cpp:89-127): name, input dims, then per
// layer its kind, sparse policy and parameters (hash_conv / hash_norm,
// graph.cpp:68-85) — the guard that ties an ActivationCache to its model.
namespace {
uint64_t sconv(const sige_conv_desc& c, uint64_t h) {
  const int dims[4] = {c.c_in, c.c_out, c.k, c.stride};
  h = fnv1a64(dims, sizeof(dims), h);
  h = hv(c.weight, static_cast<size_t>(c.c_out) * c.c_in * c.k * c.k, h);
  return hv(c.bias, c.bias ? c.c_out : 0, h);
}
uint64_t snorm(const sige_norm_desc& n, uint64_t h) {
  const int meta[2] = {n.kind, n.groups};
  h = fnv1a64(meta, sizeof(meta), h);
  h = fnv1a64(&n.eps, sizeof(n.eps), h);
  return hnorm(n, h);
}
}  // namespace

uint64_t model_structure_hash(const sige_model_desc* d) {
  uint64_t h = fnv1a64(d->name, std::strlen(d->name), kFnvSeed);
  const int dims[3] = {d->in_channels, d->in_h, d->in_w};
  h = fnv1a64(dims, sizeof(dims), h);
  for (int i = 0; i < d->num_layers; ++i) {
    const sige_layer_desc& L = d->layers[i];
    h = fnv1a64(&L.kind, sizeof(L.kind), h);
    const int pol[2] = {L.policy_sparse ? 1 : 0, L.min_resolution};
    h = fnv1a64(pol, sizeof(pol), h);
    switch (L.kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE:
        h = sconv(L.conv, h);
        break;
      case SIGE_LAYER_NORM:
        h = snorm(L.norm, h);
        break;
      case SIGE_LAYER_ACTIVATION:
        h = fnv1a64(&L.act, sizeof(L.act), h);
        break;
      case SIGE_LAYER_RESBLOCK: {
        h = sconv(L.conv, h);
        h = sconv(L.conv2, h);
        h = snorm(L.norm, h);
        h = fnv1a64(&L.act, sizeof(L.act), h);
        const int has_sc = L.has_shortcut ? 1 : 0;
        h = fnv1a64(&has_sc, sizeof(has_sc), h);
        if (has_sc) h = sconv(L.shortcut, h);
        break;
      }
      case SIGE_LAYER_RESIZE: {
        const int rs[2] = {L.resize_h, L.resize_w};
        h = fnv1a64(rs, sizeof(rs), h);
        break;
      }
      case SIGE_LAYER_SPADE_RESBLOCK: {  // no reference counterpart: the same scheme over every weight
        h = sconv(L.conv, h);
        h = sconv(L.conv2, h);
        h = fnv1a64(&L.act, sizeof(L.act), h);
        const int has_sc = L.has_shortcut ? 1 : 0;
        h = fnv1a64(&has_sc, sizeof(has_sc), h);
        if (has_sc) h = sconv(L.shortcut, h);
        for (int k = 0; k < (has_sc ? 3 : 2); ++k) {
          h = fnv1a64(&L.spade[k].eps, sizeof(float), h);
          h = sconv(L.spade[k].shared, h);
          h = sconv(L.spade[k].gamma, h);
          h = sconv(L.spade[k].beta, h);
        }
        break;
      }
      default:
        break;
    }
  }
  return h;
}

uint64_t model_weight_hash(const sige_model_desc* d) {  // models.cpp:185-207
  uint64_t h = fnv1a64(d->name, std::strlen(d->name), kFnvSeed);
  for (int i = 0; i < d->num_layers; ++i) {
    const sige_layer_desc& L = d->layers[i];
    switch (L.kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE:
        h = hconv(L.conv, h);
        break;
      case SIGE_LAYER_NORM:
        h = hnorm(L.norm, h);
        break;
      case SIGE_LAYER_RESBLOCK:
        h = hconv(L.conv, h);
        h = hnorm(L.norm, h);
        h = hconv(L.conv2, h);
        if (L.has_shortcut) h = hconv(L.shortcut, h);
        break;
      case SIGE_LAYER_SPADE_RESBLOCK:
        h = hconv(L.conv, h);
        h = hconv(L.conv2, h);
        if (L.has_shortcut) h = hconv(L.shortcut, h);
        for (int k = 0; k < (L.has_shortcut ? 3 : 2); ++k) {
          h = hconv(L.spade[k].shared, h);
          h = hconv(L.spade[k].gamma, h);
          h = hconv(L.spade[k].beta, h);
        }
        break;
      default:
        break;
    }
  }
  return h;
}

std::vector<LayerShape> walk_shapes(const sige_model_desc* m) {  // graph.cpp:129-193
  std::vector<LayerShape> shapes;
  int c = m->in_channels, h = m->in_h, w = m->in_w;
  if (c < 1 || h < 1 || w < 1) throw ConfigError("model: input shape must be positive");
  if (m->num_layers < 1) throw ConfigError("model: no layers");
  auto check_conv = [&](const sige_conv_desc& cv, int i) {
    if (cv.k != 1 && cv.k != 3)
      throw ConfigError("conv: kernel size must be 1 or 3, got " + std::to_string(cv.k));
    if (cv.stride != 1 && cv.stride != 2)
      throw ConfigError("conv: stride must be 1 or 2, got " + std::to_string(cv.stride));
    if (cv.c_in < 1 || cv.c_out < 1) throw ConfigError("conv: channel counts must be >= 1");
    if (!cv.weight) throw ConfigError("conv: weight size does not match (c_out, c_in, k, k)");
    (void)i;
  };
  for (int i = 0; i < m->num_layers; ++i) {
    const sige_layer_desc& L = m->layers[i];
    LayerShape s{c, h, w, 0, 0, 0};
    auto fail = [&](const std::string& why) {
      throw ConfigError("model layer L" + std::to_string(i) + ": " + why);
    };
    switch (L.kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE:
        check_conv(L.conv, i);
        if (L.conv.c_in != c)
          fail("expects " + std::to_string(L.conv.c_in) + " channels, gets " + std::to_string(c));
        c = L.conv.c_out;
        h = conv_out_dim(h, L.conv.k, L.conv.stride);
        w = conv_out_dim(w, L.conv.k, L.conv.stride);
        break;
      case SIGE_LAYER_NORM:
        if (L.norm.channels != c) fail("norm channel mismatch");
        if (L.norm.groups < 1 || L.norm.channels % L.norm.groups) fail("norm groups must divide channels");
        break;
      case SIGE_LAYER_ACTIVATION:
        break;
      case SIGE_LAYER_RESBLOCK:
        check_conv(L.conv, i);
        check_conv(L.conv2, i);
        if (L.conv.k != 3 || L.conv.stride != 1 || L.conv2.k != 3 || L.conv2.stride != 1)
          fail("resblock main convs must be 3x3 stride 1");
        if (L.conv.c_in != c) fail("resblock channel mismatch");
        if (L.norm.channels != L.conv.c_out) fail("resblock norm channels");
        if (L.conv2.c_in != L.conv.c_out) fail("resblock conv chaining");
        if (L.has_shortcut) {
          check_conv(L.shortcut, i);
          if (L.shortcut.k != 1 || L.shortcut.stride != 1) fail("resblock shortcut must be 1x1 stride 1");
          if (L.shortcut.c_in != c || L.shortcut.c_out != L.conv2.c_out)
            fail("resblock shortcut channel mismatch");
        } else if (L.conv2.c_out != c) {
          fail("identity shortcut requires c_in == c_out");
        }
        c = L.conv2.c_out;
        break;
      case SIGE_LAYER_UPSAMPLE:
        h *= 2;
        w *= 2;
        break;
      case SIGE_LAYER_RESIZE:
        if (L.resize_h < 1 || L.resize_w < 1) fail("resize to a non-positive size");
        if ((L.resize_h <= h ? h % L.resize_h : L.resize_h % h) || (L.resize_w <= w ? w % L.resize_w : L.resize_w % w))
          fail("resize by a non-integer factor");
        h = L.resize_h;
        w = L.resize_w;
        break;
      case SIGE_LAYER_SPADE_RESBLOCK: {
        check_conv(L.conv, i);
        check_conv(L.conv2, i);
        if (L.conv.k != 3 || L.conv.stride != 1 || L.conv2.k != 3 || L.conv2.stride != 1)
          fail("spade block convs must be 3x3 stride 1");
        if (L.conv.c_in != c || L.conv2.c_in != L.conv.c_out) fail("spade block channel mismatch");
        if (!L.spade) fail("spade block without SPADE norms");
        if (L.has_shortcut) {
          check_conv(L.shortcut, i);
          if (L.shortcut.k != 1 || L.shortcut.c_in != c || L.shortcut.c_out != L.conv2.c_out)
            fail("spade block shortcut mismatch");
        } else if (L.conv2.c_out != c) {
          fail("identity shortcut requires c_in == c_out");
        }
        const int chans[3] = {c, L.conv.c_out, c};
        for (int k = 0; k < (L.has_shortcut ? 3 : 2); ++k) {
          const sige_spade_desc& sp = L.spade[k];
          check_conv(sp.shared, i);
          check_conv(sp.gamma, i);
          check_conv(sp.beta, i);
          if (sp.shared.k != 3 || sp.gamma.k != 3 || sp.beta.k != 3 || sp.shared.stride != 1 || sp.gamma.stride != 1 ||
              sp.beta.stride != 1)
            fail("SPADE convs must be 3x3 stride 1");
          if (sp.shared.c_in != m->in_channels) fail("SPADE shared conv must read the segmentation map");
          if (sp.gamma.c_in != sp.shared.c_out || sp.beta.c_in != sp.shared.c_out) fail("SPADE hidden width");
          if (sp.gamma.c_out != chans[k] || sp.beta.c_out != chans[k]) fail("SPADE modulation channels");
          if (!(sp.eps > 0.0f)) fail("SPADE eps must be > 0");
        }
        c = L.conv2.c_out;
        break;
      }
      default:
        fail("unknown layer kind");
    }
    s.c_out = c;
    s.h_out = h;
    s.w_out = w;
    shapes.push_back(s);
  }
  return shapes;
}

int required_dilation(const sige_model_desc* m) {  // graph.cpp:195-218
  auto shapes = walk_shapes(m);
  int g = 0;
  for (int i = 0; i < m->num_layers; ++i) {
    const sige_layer_desc& L = m->layers[i];
    int f = std::max(1, m->in_h / shapes[i].h_in);
    if (L.kind == SIGE_LAYER_CONV || L.kind == SIGE_LAYER_DOWNSAMPLE)
      g += ((L.conv.k - 1) / 2) * f;
    else if (L.kind == SIGE_LAYER_RESBLOCK)
      g += ((L.conv.k - 1) / 2 + (L.conv2.k - 1) / 2) * f;
    else if (L.kind == SIGE_LAYER_SPADE_RESBLOCK)  // segmentation -> shared -> gamma/beta -> conv_0 -> conv_1
      g += 4 * f;
  }
  return g;
}

}  // namespace sige_b200
