/* sige_oracle.c — TEST INFRASTRUCTURE ONLY (header: sige_oracle.h).
 *
 * A plain-C restatement of the reference's sparse-update path, written from
 * the reference's behaviour (file:line citations on each function) and used
 * only as the checker for the CUDA library. Built by oracle/Makefile with
 * -ffp-contract=off so every float multiply and add rounds separately, as
 * the reference build does (proj/CMakeLists.txt:11-13).
 */
#include "sige_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static _Thread_local char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return SIGE_ERR_CONFIG;
}

#define TRY(x)              \
  do {                      \
    int rc_ = (x);          \
    if (rc_ != 0) return rc_; \
  } while (0)

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) abort();
  return p;
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* --------------------------------------------------------------- hashing --
 * fnv1a64: proj/src/common.cpp:11-19. */
uint64_t orc_fnv1a64(const void* p, size_t n, uint64_t h) {
  const uint8_t* b = (const uint8_t*)p;
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}
#define FNV_SEED 1469598103934665603ull

/* ------------------------------------------------------------------- Rng --
 * std::mt19937 (the standard-mandated generator) plus the toolchain-portable
 * float mapping of proj/include/sige/common.hpp:25-43. */
typedef struct {
  uint32_t mt[624];
  int i;
} Rng;

static void rng_seed(Rng* r, uint32_t seed) {
  r->mt[0] = seed;
  for (int k = 1; k < 624; ++k)
    r->mt[k] = 1812433253u * (r->mt[k - 1] ^ (r->mt[k - 1] >> 30)) + (uint32_t)k;
  r->i = 624;
}

static uint32_t rng_u32(Rng* r) {
  if (r->i >= 624) {
    for (int k = 0; k < 624; ++k) {
      uint32_t y = (r->mt[k] & 0x80000000u) | (r->mt[(k + 1) % 624] & 0x7fffffffu);
      r->mt[k] = r->mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    r->i = 0;
  }
  uint32_t y = r->mt[r->i++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* common.hpp:33-36 */
static float rng_uniform(Rng* r, float lo, float hi) {
  double u = rng_u32(r) * (1.0 / 4294967296.0);
  return (float)((double)lo + ((double)hi - (double)lo) * u);
}

/* common.hpp:39-41 */
static int rng_int(Rng* r, int lo, int hi) {
  return lo + (int)(rng_u32(r) % (uint32_t)(hi - lo + 1));
}

int orc_rng_stream(uint32_t seed, int count, uint32_t* out_u32, float* out_uniform, float lo,
                   float hi) {
  Rng a, b;
  rng_seed(&a, seed);
  rng_seed(&b, seed);
  for (int k = 0; k < count; ++k) {
    if (out_u32) out_u32[k] = rng_u32(&a);
    if (out_uniform) out_uniform[k] = rng_uniform(&b, lo, hi);
  }
  return 0;
}

float orc_expf(float x) { return expf(x); }

/* -------------------------------------------------------------- fixtures --
 * make_edit_fixture and its region builders: proj/src/fixtures.cpp:26-128. */
typedef struct {
  int h, w;
  uint8_t* on;
} Region;

static void region_rect(Region* g, int y0, int x0, int he, int we) {
  for (int y = y0; y < y0 + he; ++y)
    for (int x = x0; x < x0 + we; ++x) g->on[(size_t)y * g->w + x] = 1;
}

/* fixtures.cpp:26-34 */
static void region_square(Region* g, Rng* r, double target_px, int x_lo, int x_hi) {
  int side = imax(1, (int)lround(sqrt(target_px)));
  int we = imin(side, x_hi - x_lo);
  int he = imax(1, (int)lround(target_px / we));
  he = imin(he, g->h);
  int y0 = rng_int(r, 0, g->h - he);
  int x0 = x_lo + rng_int(r, 0, (x_hi - x_lo) - we);
  region_rect(g, y0, x0, he, we);
}

/* fixtures.cpp:37-60: 4-connected growth from a seeded start. The frontier
 * is a swap-remove array. */
static void region_blob(Region* g, Rng* r, int target_px) {
  int y0 = rng_int(r, g->h / 4, 3 * g->h / 4);
  int x0 = rng_int(r, g->w / 4, 3 * g->w / 4);
  size_t cap = 1024, len = 0;
  int* fy = (int*)xcalloc(cap, sizeof(int));
  int* fx = (int*)xcalloc(cap, sizeof(int));
  fy[0] = y0;
  fx[0] = x0;
  len = 1;
  int painted = 0;
  static const int DY[4] = {-1, 1, 0, 0}, DX[4] = {0, 0, -1, 1};
  while (painted < target_px && len > 0) {
    int pick = rng_int(r, 0, (int)len - 1);
    int y = fy[pick], x = fx[pick];
    fy[pick] = fy[len - 1];
    fx[pick] = fx[len - 1];
    --len;
    if (g->on[(size_t)y * g->w + x]) continue;
    g->on[(size_t)y * g->w + x] = 1;
    ++painted;
    for (int d = 0; d < 4; ++d) {
      int ny = y + DY[d], nx = x + DX[d];
      if (ny < 0 || ny >= g->h || nx < 0 || nx >= g->w || g->on[(size_t)ny * g->w + nx]) continue;
      if (len == cap) {
        cap *= 2;
        fy = (int*)realloc(fy, cap * sizeof(int));
        fx = (int*)realloc(fx, cap * sizeof(int));
      }
      fy[len] = ny;
      fx[len] = nx;
      ++len;
    }
  }
  free(fy);
  free(fx);
}

int orc_make_edit_fixture(const char* kind, int n, int c, int h, int w, uint32_t seed,
                          float* orig, float* edited) {
  Rng r;
  rng_seed(&r, seed);
  size_t total = (size_t)n * c * h * w;
  for (size_t i = 0; i < total; ++i) orig[i] = rng_uniform(&r, -1.0f, 1.0f);
  Region g = {h, w, (uint8_t*)xcalloc((size_t)h * w, 1)};
  double px = (double)h * w;
  if (!strcmp(kind, "rect1")) {
    region_square(&g, &r, 0.012 * px, 0, w);
  } else if (!strcmp(kind, "rect5")) {
    region_square(&g, &r, 0.05 * px, 0, w);
  } else if (!strcmp(kind, "rect15")) {
    region_square(&g, &r, 0.15 * px, 0, w);
  } else if (!strcmp(kind, "rect35")) {
    region_square(&g, &r, 0.35 * px, 0, w);
  } else if (!strcmp(kind, "blob5")) {
    region_blob(&g, &r, (int)lround(0.05 * px));
  } else if (!strcmp(kind, "multi15")) {
    for (int band = 0; band < 3; ++band)
      region_square(&g, &r, 0.15 * px / 3.0, band * w / 3, (band + 1) * w / 3);
  } else {
    free(g.on);
    return fail("unknown edit fixture: %s", kind);
  }
  memcpy(edited, orig, total * sizeof(float));
  for (int in = 0; in < n; ++in)
    for (int ic = 0; ic < c; ++ic)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
          if (!g.on[(size_t)y * w + x]) continue;
          float mag = rng_uniform(&r, 0.05f, 0.5f);
          float sign = rng_uniform(&r, 0.0f, 1.0f) < 0.5f ? -1.0f : 1.0f;
          size_t at = (((size_t)in * c + ic) * h + y) * w + x;
          edited[at] = edited[at] + sign * mag;
        }
  free(g.on);
  return 0;
}

/* ----------------------------------------------------------------- masks */

/* compute_difference_mask: proj/src/mask.cpp:14-32 (strict '>' on |e-o|). */
int orc_compute_difference_mask(const float* o, const float* e, int n, int c, int h, int w,
                                float thr, uint8_t* out) {
  if (thr < 0.0f) return fail("compute_difference_mask: threshold must be >= 0");
  size_t hw = (size_t)h * w;
  memset(out, 0, hw);
  for (size_t plane = 0; plane < (size_t)n * c; ++plane) {
    const float* a = o + plane * hw;
    const float* b = e + plane * hw;
    for (size_t i = 0; i < hw; ++i)
      if (fabsf(b[i] - a[i]) > thr) out[i] = 1;
  }
  return 0;
}

/* downsample_mask (max-pool by an integer factor): mask.cpp:34-53. */
int orc_downsample_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out) {
  if (oh < 1 || ow < 1 || oh > h || ow > w)
    return fail("downsample_mask: target must be >= 1 and <= source");
  if (h % oh || w % ow)
    return fail("downsample_mask: non-integer scale factor (%dx%d -> %dx%d)", h, w, oh, ow);
  int fy = h / oh, fx = w / ow;
  memset(out, 0, (size_t)oh * ow);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x)
      if (m[(size_t)y * w + x]) out[(size_t)(y / fy) * ow + x / fx] = 1;
  return 0;
}

/* nearest replication up by an integer factor: graph.cpp:485-500. */
static int replicate_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out) {
  if (oh % h || ow % w)
    return fail("mask: cannot scale %dx%d up to %dx%d (non-integer factor)", h, w, oh, ow);
  int fy = oh / h, fx = ow / w;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) out[(size_t)y * ow + x] = m[(size_t)(y / fy) * w + x / fx];
  return 0;
}

/* dilate_mask: Chebyshev radius r, clipped; r = 0 copies. mask.cpp:55-80.
 * Restated as a row pass then a column pass over running window counts. */
int orc_dilate_mask(const uint8_t* m, int h, int w, int r, uint8_t* out) {
  if (r < 0) return fail("dilate_mask: radius must be >= 0");
  size_t hw = (size_t)h * w;
  if (r == 0) {
    memcpy(out, m, hw);
    return 0;
  }
  uint8_t* tmp = (uint8_t*)xcalloc(hw, 1);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      uint8_t v = 0;
      for (int t = imax(0, x - r); t <= imin(w - 1, x + r) && !v; ++t) v = m[(size_t)y * w + t];
      tmp[(size_t)y * w + x] = v ? 1 : 0;
    }
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      uint8_t v = 0;
      for (int t = imax(0, y - r); t <= imin(h - 1, y + r) && !v; ++t) v = tmp[(size_t)t * w + x];
      out[(size_t)y * w + x] = v ? 1 : 0;
    }
  free(tmp);
  return 0;
}

/* BlockIndexSet::content_hash: mask.cpp:91-101 (fields hashed as int32). */
uint64_t orc_index_set_hash(const int32_t* idx, int count, int b, int h, int w) {
  uint64_t hs = orc_fnv1a64(&b, 4, FNV_SEED);
  hs = orc_fnv1a64(&h, 4, hs);
  hs = orc_fnv1a64(&w, 4, hs);
  for (int i = 0; i < count; ++i) hs = orc_fnv1a64(idx + 3 * i, 12, hs);
  return hs;
}

/* mask_to_block_indices: stride-b grid anchored at (0,0); a tile is active if
 * any set pixel lies inside it (fringe tiles clipped to the canvas); tiles in
 * row-major order, replicated n-major. mask.cpp:103-136. */
int orc_mask_to_block_indices(const uint8_t* m, int h, int w, int b, int batch, int32_t* idx,
                              int cap, int* count, uint64_t* hash) {
  if (b < 1) return fail("mask_to_block_indices: block size must be >= 1");
  if (batch < 1) return fail("mask_to_block_indices: batch must be >= 1");
  int ty = (h + b - 1) / b, tx = (w + b - 1) / b;
  int* act = (int*)xcalloc((size_t)ty * tx, sizeof(int));
  int tiles = 0;
  for (int R = 0; R < ty; ++R)
    for (int C = 0; C < tx; ++C) {
      int on = 0;
      for (int y = R * b; y < imin(h, R * b + b) && !on; ++y)
        for (int x = C * b; x < imin(w, C * b + b) && !on; ++x) on = m[(size_t)y * w + x] != 0;
      if (on) act[tiles++] = R * tx + C;
    }
  int total = tiles * batch;
  if (count) *count = total;
  for (int in = 0, k = 0; in < batch; ++in)
    for (int t = 0; t < tiles; ++t, ++k) {
      if (k >= cap) continue;
      idx[3 * k] = in;
      idx[3 * k + 1] = (act[t] / tx) * b;
      idx[3 * k + 2] = (act[t] % tx) * b;
    }
  if (hash && total <= cap) *hash = orc_index_set_hash(idx, total, b, h, w);
  free(act);
  return 0;
}

/* -------------------------------------------------------------- epilogue --
 * Epilogue chain (eltwise.hpp:30-59): ScaleShift a*x+b with two roundings,
 * Relu x>0?x:0, Silu x/(1+expf(-x)). eltwise.cpp:23-36, 110-150. */
static float act1(float v, int kind) {
  if (kind == SIGE_ACT_RELU) return v > 0.0f ? v : 0.0f;
  if (kind == SIGE_ACT_LEAKY_RELU) return v > 0.0f ? v : 0.2f * v;
  if (kind == SIGE_ACT_SILU) return v / (1.0f + expf(-v));
  return v;
}

/* param_slice: eltwise.cpp:48-58 */
static int param_slice(const sige_epilogue_step* s, int channels, int sample, int* offset) {
  if (s->nparams == channels) {
    *offset = 0;
    return 0;
  }
  if (channels > 0 && s->nparams % channels == 0 && (sample + 1) * channels <= s->nparams) {
    *offset = sample * channels;
    return 0;
  }
  return fail("epilogue: affine param size %d does not match channels %d", s->nparams, channels);
}

/* One value of channel ch of sample n through the whole chain. */
static int epi_value(const sige_epilogue* e, float* v, int ch, int channels, int n) {
  if (!e) return 0;
  for (int k = 0; k < e->num_steps; ++k) {
    const sige_epilogue_step* s = &e->steps[k];
    if (s->kind == SIGE_EPI_ACTIVATION) {
      *v = act1(*v, s->act);
    } else {
      int off;
      TRY(param_slice(s, channels, n, &off));
      float a = s->scale[off + ch], b = s->shift[off + ch];
      float p = a * *v;
      *v = p + b;
    }
  }
  return 0;
}

static int epi_empty(const sige_epilogue* e) { return !e || e->num_steps == 0; }

/* ----------------------------------------------------------------- blocks */

static int conv_out_dim(int in, int k, int s) { return (in + 2 * ((k - 1) / 2) - k) / s + 1; }

/* gather: kernels.cpp:39-86. Windows of side s*b+k-s at (r*s-pad, c*s-pad);
 * out-of-canvas cells stay +0 and never see the epilogue. */
int orc_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count, int b,
               int ih, int iw, int k, int s, const sige_epilogue* epi, float* out) {
  if (k != 1 && k != 3) return fail("gather: kernel size must be 1 or 3");
  if (s != 1 && s != 2) return fail("gather: stride must be 1 or 2");
  int oh = conv_out_dim(h, k, s), ow = conv_out_dim(w, k, s);
  if (ih != oh || iw != ow)
    return fail("gather: index set lives at %dx%d but conv output of (%d, %d, %d, %d) is %dx%d", ih,
                iw, n, c, h, w, oh, ow);
  int win = s * b + k - s, pad = (k - 1) / 2;
  size_t wsz = (size_t)win * win;
  memset(out, 0, (size_t)count * c * wsz * sizeof(float));
  for (int i = 0; i < count; ++i) {
    int bn = idx[3 * i], y0 = idx[3 * i + 1] * s - pad, x0 = idx[3 * i + 2] * s - pad;
    for (int ch = 0; ch < c; ++ch) {
      const float* src = x + ((size_t)bn * c + ch) * h * w;
      float* dst = out + ((size_t)i * c + ch) * wsz;
      for (int wy = 0; wy < win; ++wy) {
        int sy = y0 + wy;
        if (sy < 0 || sy >= h) continue;
        for (int wx = 0; wx < win; ++wx) {
          int sx = x0 + wx;
          if (sx < 0 || sx >= w) continue;
          float v = src[(size_t)sy * w + sx];
          TRY(epi_value(epi, &v, ch, c, bn));
          dst[(size_t)wy * win + wx] = v;
        }
      }
    }
  }
  return 0;
}

/* SPADE modulation gather (config 3; NOT a reference function — restated
 * from GauGAN's SPADE block, x_norm * (1 + gamma) + beta, over gather()'s
 * window geometry, kernels.cpp:39-86). Order: norm chain, m = 1 + gamma,
 * v = v * m, v = v + beta, act. Out-of-canvas cells stay +0. */
int orc_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                     const int32_t* idx, int count, int b, int ih, int iw, int k, int s,
                     const sige_epilogue* norm, int act, float* out) {
  if (k != 1 && k != 3) return fail("gather: kernel size must be 1 or 3");
  if (s != 1 && s != 2) return fail("gather: stride must be 1 or 2");
  int oh = conv_out_dim(h, k, s), ow = conv_out_dim(w, k, s);
  if (ih != oh || iw != ow)
    return fail("gather: index set lives at %dx%d but conv output of (%d, %d, %d, %d) is %dx%d", ih,
                iw, n, c, h, w, oh, ow);
  int win = s * b + k - s, pad = (k - 1) / 2;
  size_t wsz = (size_t)win * win;
  memset(out, 0, (size_t)count * c * wsz * sizeof(float));
  for (int i = 0; i < count; ++i) {
    int bn = idx[3 * i], y0 = idx[3 * i + 1] * s - pad, x0 = idx[3 * i + 2] * s - pad;
    for (int ch = 0; ch < c; ++ch) {
      size_t plane = ((size_t)bn * c + ch) * h * w;
      float* dst = out + ((size_t)i * c + ch) * wsz;
      for (int wy = 0; wy < win; ++wy) {
        int sy = y0 + wy;
        if (sy < 0 || sy >= h) continue;
        for (int wx = 0; wx < win; ++wx) {
          int sx = x0 + wx;
          if (sx < 0 || sx >= w) continue;
          size_t at = plane + (size_t)sy * w + sx;
          float v = x[at];
          TRY(epi_value(norm, &v, ch, c, bn));
          float m = 1.0f + gamma[at];
          v = v * m;
          v = v + beta[at];
          dst[(size_t)wy * win + wx] = act1(v, act);
        }
      }
    }
  }
  return 0;
}

/* Nearest resample by integer factors (config 3 label maps; not a reference
 * function): down samples (y*f, x*f), up replicates (y/u, x/u). */
int orc_resize_nearest(const float* in, int n, int c, int h, int w, int oh, int ow, float* out) {
  if (oh < 1 || ow < 1 || !((h % oh == 0) || (oh % h == 0)) || !((w % ow == 0) || (ow % w == 0)))
    return fail("resize_nearest: non-integer scale");
  for (int p = 0; p < n * c; ++p)
    for (int y = 0; y < oh; ++y) {
      int sy = oh <= h ? y * (h / oh) : y / (oh / h);
      for (int x = 0; x < ow; ++x) {
        int sx = ow <= w ? x * (w / ow) : x / (ow / w);
        out[((size_t)p * oh + y) * ow + x] = in[((size_t)p * h + sy) * w + sx];
      }
    }
  return 0;
}

static int check_scatter(int count, int channels, const int32_t* idx, int n, int c,
                         const char* op) {
  if (channels != c) return fail("%s: channel mismatch", op);
  for (int i = 0; i < count; ++i)
    if (idx[3 * i] < 0 || idx[3 * i] >= n) return fail("%s: block sample out of range", op);
  return 0;
}

/* scatter / scatter_inplace: kernels.cpp:88-112 (tiles clipped at the fringe). */
static int scatter_into(const float* blocks, int count, int channels, int block,
                        const int32_t* idx, float* t, int n, int c, int h, int w, int add) {
  TRY(check_scatter(count, channels, idx, n, c, add ? "scatter_add" : "scatter"));
  for (int i = 0; i < count; ++i) {
    int bn = idx[3 * i], r = idx[3 * i + 1], q = idx[3 * i + 2];
    int yl = imin(block, h - r), xl = imin(block, w - q);
    for (int ch = 0; ch < c; ++ch) {
      const float* src = blocks + ((size_t)i * c + ch) * block * block;
      float* dst = t + ((size_t)bn * c + ch) * h * w;
      for (int y = 0; y < yl; ++y)
        for (int x = 0; x < xl; ++x) {
          float* d = &dst[(size_t)(r + y) * w + q + x];
          *d = add ? *d + src[y * block + x] : src[y * block + x];
        }
    }
  }
  return 0;
}

int orc_scatter(const float* blocks, int count, int channels, int block, const int32_t* idx,
                const float* base, float* out, int n, int c, int h, int w) {
  memmove(out, base, (size_t)n * c * h * w * sizeof(float));
  return scatter_into(blocks, count, channels, block, idx, out, n, c, h, w, 0);
}

int orc_scatter_add_inplace(const float* blocks, int count, int channels, int block,
                            const int32_t* idx, float* base, int n, int c, int h, int w) {
  return scatter_into(blocks, count, channels, block, idx, base, n, c, h, w, 1);
}

/* per_sample: mask.cpp:81-89 (count of leading sample's entries). */
static int per_sample(const int32_t* idx, int count) {
  int p = 0;
  for (int i = 0; i < count; ++i) p += idx[3 * i] == idx[0];
  return count ? p : 0;
}

/* build_scatter_map: kernels.cpp:134-169. */
int orc_build_scatter_map(const int32_t* idx, int count, int block, int h, int w,
                          sige_scatter_entry* out, int* bps) {
  for (size_t p = 0; p < (size_t)h * w; ++p) {
    out[p].block = -1;
    out[p].dy = 0;
    out[p].dx = 0;
  }
  int per = per_sample(idx, count);
  *bps = per;
  if (!per) return 0;
  for (int i = per; i < count; ++i) {
    const int32_t* rep = idx + 3 * (i % per);
    if (idx[3 * i + 1] != rep[1] || idx[3 * i + 2] != rep[2])
      return fail("build_scatter_map: tile pattern differs across batch");
  }
  for (int o = 0; o < per; ++o) {
    int r = idx[3 * o + 1], q = idx[3 * o + 2];
    for (int y = r; y < imin(h, r + block); ++y)
      for (int x = q; x < imin(w, q + block); ++x) {
        sige_scatter_entry* e = &out[(size_t)y * w + x];
        e->block = o;
        e->dy = (int16_t)(y - r);
        e->dx = (int16_t)(x - q);
      }
  }
  return 0;
}

/* scatter_gather: kernels.cpp:204-275. Every in-canvas consumer cell comes
 * from the producer block when the map hits, else from original_out; the
 * epilogue runs on in-canvas cells only. */
static int scatter_gather_map(const float* blocks, int count, int block,
                              const sige_scatter_entry* map, int bps, const float* orig_out,
                              int n, int c, int h, int w, const int32_t* cidx, int ccount,
                              int cb, int ch_, int cw, int k, int s, const sige_epilogue* epi,
                              float* out) {
  if (bps * n != count) return fail("scatter_gather: map does not describe this block stack");
  if (ch_ != conv_out_dim(h, k, s) || cw != conv_out_dim(w, k, s))
    return fail("scatter_gather: consumer index resolution mismatch");
  int win = s * cb + k - s, pad = (k - 1) / 2;
  size_t wsz = (size_t)win * win;
  memset(out, 0, (size_t)ccount * c * wsz * sizeof(float));
  for (int i = 0; i < ccount; ++i) {
    int bn = cidx[3 * i], y0 = cidx[3 * i + 1] * s - pad, x0 = cidx[3 * i + 2] * s - pad;
    for (int wy = 0; wy < win; ++wy) {
      int sy = y0 + wy;
      if (sy < 0 || sy >= h) continue;
      for (int wx = 0; wx < win; ++wx) {
        int sx = x0 + wx;
        if (sx < 0 || sx >= w) continue;
        const sige_scatter_entry* e = &map[(size_t)sy * w + sx];
        for (int ch = 0; ch < c; ++ch) {
          float v = e->block < 0
                        ? orig_out[(((size_t)bn * c + ch) * h + sy) * w + sx]
                        : blocks[(((size_t)(bn * bps + e->block) * c + ch) * block + e->dy) * block +
                                 e->dx];
          TRY(epi_value(epi, &v, ch, c, bn));
          out[((size_t)i * c + ch) * wsz + (size_t)wy * win + wx] = v;
        }
      }
    }
  }
  return 0;
}

int orc_scatter_gather(const float* blocks, int count, int block, const int32_t* prod_idx,
                       const float* orig_out, int n, int c, int h, int w,
                       const int32_t* cons_idx, int cons_count, int cons_block, int ch, int cw,
                       int k, int s, const sige_epilogue* epi, float* out) {
  sige_scatter_entry* map = (sige_scatter_entry*)xcalloc((size_t)h * w, sizeof *map);
  int bps = 0;
  int rc = orc_build_scatter_map(prod_idx, count, block, h, w, map, &bps);
  if (!rc)
    rc = scatter_gather_map(blocks, count, block, map, bps, orig_out, n, c, h, w, cons_idx,
                            cons_count, cons_block, ch, cw, k, s, epi, out);
  free(map);
  return rc;
}

/* scatter_with_block_residual (fused): kernels.cpp:291-337; the unfused twin
 * kernels.cpp:339-355 goes through gather/add/scatter/subtract/scatter_add and
 * must agree bit for bit. */
int orc_scatter_with_block_residual(const float* mb, int mcount, int mblock, const int32_t* midx,
                                    const float* sb, int scount, int sblock, const int32_t* sidx,
                                    const float* sum, const float* orig_sc, float* out, int n,
                                    int c, int h, int w, int fused) {
  TRY(check_scatter(mcount, c, midx, n, c, "block_residual(main)"));
  TRY(check_scatter(scount, c, sidx, n, c, "block_residual(shortcut)"));
  size_t total = (size_t)n * c * h * w;
  memmove(out, sum, total * sizeof(float));
  if (fused) {
    for (int i = 0; i < mcount; ++i) {
      int bn = midx[3 * i], r = midx[3 * i + 1], q = midx[3 * i + 2];
      for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < imin(mblock, h - r); ++y)
          for (int x = 0; x < imin(mblock, w - q); ++x) {
            size_t p = (((size_t)bn * c + ch) * h + r + y) * w + q + x;
            out[p] = mb[(((size_t)i * c + ch) * mblock + y) * mblock + x] + orig_sc[p];
          }
    }
    for (int i = 0; i < scount; ++i) {
      int bn = sidx[3 * i], r = sidx[3 * i + 1], q = sidx[3 * i + 2];
      for (int ch = 0; ch < c; ++ch)
        for (int y = 0; y < imin(sblock, h - r); ++y)
          for (int x = 0; x < imin(sblock, w - q); ++x) {
            size_t p = (((size_t)bn * c + ch) * h + r + y) * w + q + x;
            float d = sb[(((size_t)i * c + ch) * sblock + y) * sblock + x] - orig_sc[p];
            out[p] = out[p] + d;
          }
    }
    return 0;
  }
  size_t msz = (size_t)mcount * c * mblock * mblock, ssz = (size_t)scount * c * sblock * sblock;
  float* g = (float*)xcalloc(msz > ssz ? msz : ssz, sizeof(float));
  float* t = (float*)xcalloc(msz > ssz ? msz : ssz, sizeof(float));
  int rc = orc_gather(orig_sc, n, c, h, w, midx, mcount, mblock, h, w, 1, 1, NULL, g);
  if (!rc) {
    orc_combine_blocks(mb, g, 1.0f, msz, t);
    rc = scatter_into(t, mcount, c, mblock, midx, out, n, c, h, w, 0);
  }
  if (!rc) rc = orc_gather(orig_sc, n, c, h, w, sidx, scount, sblock, h, w, 1, 1, NULL, g);
  if (!rc) {
    orc_combine_blocks(sb, g, -1.0f, ssz, t);
    rc = scatter_into(t, scount, c, sblock, sidx, out, n, c, h, w, 1);
  }
  free(g);
  free(t);
  return rc;
}

/* add_blocks / subtract_blocks: kernels.cpp:359-380 (a + sign*b). */
int orc_combine_blocks(const float* a, const float* b, float sign, size_t numel, float* out) {
  for (size_t i = 0; i < numel; ++i) {
    float p = sign * b[i];
    out[i] = a[i] + p;
  }
  return 0;
}

/* apply_epilogue_on_blocks: kernels.cpp:382-389 (apply_slab per block). */
int orc_apply_epilogue_on_blocks(float* blocks, int count, int channels, int bh,
                                 const int32_t* idx, int idx_h, int idx_w,
                                 const sige_epilogue* epi) {
  size_t hw = (size_t)bh * bh;
  for (int i = 0; i < count; ++i)
    for (int ch = 0; ch < channels; ++ch)
      for (size_t p = 0; p < hw; ++p)
        TRY(epi_value(epi, &blocks[((size_t)i * channels + ch) * hw + p], ch, channels,
                      idx[3 * i]));
  return 0;
}

/* ------------------------------------------------------------------ conv */

static int conv_validate(const sige_conv_desc* cv) {
  if (cv->k != 1 && cv->k != 3) return fail("conv: kernel size must be 1 or 3, got %d", cv->k);
  if (cv->stride != 1 && cv->stride != 2)
    return fail("conv: stride must be 1 or 2, got %d", cv->stride);
  if (cv->c_in < 1 || cv->c_out < 1) return fail("conv: channel counts must be >= 1");
  return 0;
}

/* detail::conv2d_raw: conv.cpp:33-79. Per output value: acc = +0, then for
 * ic, ky, kx (in-bounds taps only) acc = acc + w*x with separate roundings,
 * then acc + bias. */
static void conv_raw(const float* in, int ci, int ih, int iw, const float* wt, const float* bias,
                     int co, int k, int s, int pad, float* out, int oh, int ow) {
  for (int oc = 0; oc < co; ++oc)
    for (int oy = 0; oy < oh; ++oy)
      for (int ox = 0; ox < ow; ++ox) {
        float acc = 0.0f;
        for (int ic = 0; ic < ci; ++ic) {
          const float* plane = in + (size_t)ic * ih * iw;
          const float* wk = wt + ((size_t)oc * ci + ic) * k * k;
          for (int ky = 0; ky < k; ++ky) {
            int iy = oy * s + ky - pad;
            if (iy < 0 || iy >= ih) continue;
            for (int kx = 0; kx < k; ++kx) {
              int ix = ox * s + kx - pad;
              if (ix < 0 || ix >= iw) continue;
              float p = wk[ky * k + kx] * plane[(size_t)iy * iw + ix];
              acc = acc + p;
            }
          }
        }
        if (bias) acc = acc + bias[oc];
        out[((size_t)oc * oh + oy) * ow + ox] = acc;
      }
}

/* conv_on_blocks: kernels.cpp:391-421 (pad-0 conv per window). */
int orc_conv_on_blocks(const float* blocks, int count, int window, const sige_conv_desc* cv,
                       int with_bias, float* out, int block) {
  TRY(conv_validate(cv));
  int bo = (window - cv->k) / cv->stride + 1;
  if (bo != block)
    return fail("conv_on_blocks: window %d with k=%d s=%d yields %d, expected block %d", window,
                cv->k, cv->stride, bo, block);
  for (int i = 0; i < count; ++i)
    conv_raw(blocks + (size_t)i * cv->c_in * window * window, cv->c_in, window, window,
             cv->weight, with_bias ? cv->bias : NULL, cv->c_out, cv->k, cv->stride, 0,
             out + (size_t)i * cv->c_out * block * block, block, block);
  return 0;
}

/* conv2d: conv.cpp:83-102. */
int orc_conv2d(const float* x, int n, int c, int h, int w, const sige_conv_desc* cv,
               int with_bias, float* out) {
  TRY(conv_validate(cv));
  if (c != cv->c_in)
    return fail("conv2d: input has %d channels, layer expects %d", c, cv->c_in);
  int oh = conv_out_dim(h, cv->k, cv->stride), ow = conv_out_dim(w, cv->k, cv->stride);
  for (int in = 0; in < n; ++in)
    conv_raw(x + (size_t)in * c * h * w, c, h, w, cv->weight, with_bias ? cv->bias : NULL,
             cv->c_out, cv->k, cv->stride, (cv->k - 1) / 2,
             out + (size_t)in * cv->c_out * oh * ow, oh, ow);
  return 0;
}

/* ------------------------------------------------------------------ norm */

/* compute_norm_stats + fold_stats: norm.cpp:25-90 (double sums, two passes,
 * traversal channel-in-group, rows, columns). */
int orc_group_norm_fold(const float* x, int n, int c, int h, int w, int groups, float eps,
                        const float* gamma, const float* beta, float* scale, float* shift) {
  if (groups < 1 || c % groups)
    return fail("compute_norm_stats: groups %d must divide channels %d", groups, c);
  int cpg = c / groups;
  size_t hw = (size_t)h * w;
  double count = (double)cpg * (double)hw;
  for (int in = 0; in < n; ++in)
    for (int g = 0; g < groups; ++g) {
      double sum = 0.0;
      for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic) {
        const float* p = x + ((size_t)in * c + ic) * hw;
        for (size_t i = 0; i < hw; ++i) sum += p[i];
      }
      double mean = sum / count;
      double sq = 0.0;
      for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic) {
        const float* p = x + ((size_t)in * c + ic) * hw;
        for (size_t i = 0; i < hw; ++i) {
          double d = p[i] - mean;
          sq += d * d;
        }
      }
      float fmean = (float)mean, fvar = (float)(sq / count);
      for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic) {
        float sc = gamma[ic] / sqrtf(fvar + eps);
        float p = fmean * sc;
        scale[(size_t)in * c + ic] = sc;
        shift[(size_t)in * c + ic] = beta[ic] - p;
      }
    }
  return 0;
}

/* ---------------------------------------------------------------- models --
 * Toy models: proj/src/models.cpp:8-161. single_conv64 and ddim_stack are the
 * BASELINE configs 1 and 2. */
typedef struct {
  sige_layer_desc* v;
  int n, cap;
} LayerVec;

static void lv_push(LayerVec* lv, sige_layer_desc L) {
  if (lv->n == lv->cap) {
    lv->cap = lv->cap ? 2 * lv->cap : 16;
    lv->v = (sige_layer_desc*)realloc(lv->v, (size_t)lv->cap * sizeof *lv->v);
  }
  lv->v[lv->n++] = L;
}

static float* uniform_vec(Rng* r, size_t n, float lo, float hi) {
  float* v = (float*)xcalloc(n, sizeof(float));
  for (size_t i = 0; i < n; ++i) v[i] = rng_uniform(r, lo, hi);
  return v;
}

/* models.cpp:8-27 */
static sige_conv_desc mk_conv(Rng* r, int ci, int co, int k, int s) {
  sige_conv_desc c = {ci, co, k, s, NULL, NULL};
  float bound = 1.0f / sqrtf((float)(ci * k * k));
  c.weight = uniform_vec(r, (size_t)co * ci * k * k, -bound, bound);
  c.bias = uniform_vec(r, (size_t)co, -0.05f, 0.05f);
  return c;
}

/* models.cpp:29-45 */
static sige_norm_desc mk_norm(Rng* r, int kind, int ch, int groups) {
  sige_norm_desc n = {kind, kind == SIGE_NORM_INSTANCE ? ch : groups, ch, 1e-5f,
                      NULL, NULL, NULL, NULL};
  n.gamma = uniform_vec(r, ch, 0.8f, 1.2f);
  n.beta = uniform_vec(r, ch, -0.1f, 0.1f);
  if (kind == SIGE_NORM_BATCH) {
    n.running_mean = uniform_vec(r, ch, -0.3f, 0.3f);
    n.running_var = uniform_vec(r, ch, 0.5f, 1.5f);
  }
  return n;
}

static sige_layer_desc blank_layer(int kind) {
  sige_layer_desc L;
  memset(&L, 0, sizeof L);
  L.kind = kind;
  L.policy_sparse = 1;
  L.min_resolution = 16; /* SparsePolicy defaults, graph.hpp:30-35 */
  return L;
}

static void push_conv(LayerVec* lv, Rng* r, int ci, int co, int k, int s) {
  sige_layer_desc L = blank_layer(s == 2 ? SIGE_LAYER_DOWNSAMPLE : SIGE_LAYER_CONV);
  L.conv = mk_conv(r, ci, co, k, s);
  lv_push(lv, L);
}

static void push_norm(LayerVec* lv, Rng* r, int kind, int ch, int groups) {
  sige_layer_desc L = blank_layer(SIGE_LAYER_NORM);
  L.norm = mk_norm(r, kind, ch, groups);
  lv_push(lv, L);
}

static void push_act(LayerVec* lv, int act) {
  sige_layer_desc L = blank_layer(SIGE_LAYER_ACTIVATION);
  L.act = act;
  lv_push(lv, L);
}

static void push_up(LayerVec* lv) { lv_push(lv, blank_layer(SIGE_LAYER_UPSAMPLE)); }

/* models.cpp:76-89: conv1, norm, conv2, shortcut (when c_in != c_out). */
static void push_res(LayerVec* lv, Rng* r, int ci, int co, int nk, int groups, int act) {
  sige_layer_desc L = blank_layer(SIGE_LAYER_RESBLOCK);
  L.conv = mk_conv(r, ci, co, 3, 1);
  L.norm = mk_norm(r, nk, co, groups);
  L.act = act;
  L.conv2 = mk_conv(r, co, co, 3, 1);
  if (ci != co) {
    L.has_shortcut = 1;
    L.shortcut = mk_conv(r, ci, co, 1, 1);
  }
  lv_push(lv, L);
}

static char* dupstr(const char* s) {
  char* d = (char*)xcalloc(strlen(s) + 1, 1);
  strcpy(d, s);
  return d;
}

static sige_model_desc* finish(const char* name, int ci, int h, int w, LayerVec* lv) {
  sige_model_desc* m = (sige_model_desc*)xcalloc(1, sizeof *m);
  m->name = dupstr(name);
  m->in_channels = ci;
  m->in_h = h;
  m->in_w = w;
  m->num_layers = lv->n;
  m->layers = lv->v;
  return m;
}

static sige_model_desc* build_ddim(int res, int base) {
  Rng r;
  rng_seed(&r, 2211);
  LayerVec lv = {0};
  static const int mult[6] = {1, 1, 2, 2, 4, 4};
  push_conv(&lv, &r, 3, base, 3, 1);
  int c = base;
  for (int lvl = 0; lvl < 6; ++lvl) {
    for (int j = 0; j < 2; ++j) {
      push_res(&lv, &r, c, base * mult[lvl], SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
      c = base * mult[lvl];
    }
    if (lvl < 5) push_conv(&lv, &r, c, c, 3, 2);
  }
  for (int j = 0; j < 2; ++j) push_res(&lv, &r, c, c, SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
  for (int lvl = 0; lvl < 6; ++lvl) {
    int dc = base * mult[5 - lvl];
    for (int j = 0; j < 3; ++j) {
      push_res(&lv, &r, c, dc, SIGE_NORM_GROUP, 32, SIGE_ACT_SILU);
      c = dc;
    }
    if (lvl < 5) {
      push_up(&lv);
      push_conv(&lv, &r, c, c, 3, 1);
    }
  }
  push_norm(&lv, &r, SIGE_NORM_GROUP, c, 32);
  push_act(&lv, SIGE_ACT_SILU);
  push_conv(&lv, &r, c, 3, 3, 1);
  return finish("ddim_stack", 3, res, res, &lv);
}

static sige_model_desc* build_mini_unet(int nk, const char* name, uint32_t seed) {
  Rng r;
  rng_seed(&r, seed);
  LayerVec lv = {0};
  push_conv(&lv, &r, 3, 16, 3, 1);
  push_norm(&lv, &r, nk, 16, 4);
  push_act(&lv, SIGE_ACT_SILU);
  push_res(&lv, &r, 16, 16, nk, 4, SIGE_ACT_SILU);
  push_conv(&lv, &r, 16, 32, 3, 2);
  push_res(&lv, &r, 32, 32, nk, 8, SIGE_ACT_SILU);
  push_conv(&lv, &r, 32, 64, 3, 2);
  push_res(&lv, &r, 64, 64, nk, 8, SIGE_ACT_SILU);
  push_up(&lv);
  push_res(&lv, &r, 64, 32, nk, 8, SIGE_ACT_SILU);
  push_up(&lv);
  push_res(&lv, &r, 32, 16, nk, 4, SIGE_ACT_SILU);
  push_conv(&lv, &r, 16, 3, 3, 1);
  return finish(name, 3, 64, 64, &lv);
}

sige_model_desc* orc_model_build(const char* name) {
  Rng r;
  LayerVec lv = {0};
  if (!strcmp(name, "conv3x3_128") || !strcmp(name, "single_conv64")) {
    int c = name[0] == 'c' ? 128 : 64;
    rng_seed(&r, 1001);
    push_conv(&lv, &r, c, c, 3, 1);
    return finish(name, c, 256, 256, &lv);
  }
  if (!strcmp(name, "mini_unet_gn")) return build_mini_unet(SIGE_NORM_GROUP, name, 1002);
  if (!strcmp(name, "mini_unet_bn")) return build_mini_unet(SIGE_NORM_BATCH, name, 1003);
  if (!strcmp(name, "gaugan_stack_in")) {
    rng_seed(&r, 1004);
    push_conv(&lv, &r, 3, 16, 3, 2);
    push_act(&lv, SIGE_ACT_RELU);
    push_conv(&lv, &r, 16, 32, 3, 2);
    push_act(&lv, SIGE_ACT_RELU);
    push_res(&lv, &r, 32, 32, SIGE_NORM_INSTANCE, 32, SIGE_ACT_RELU);
    push_up(&lv);
    push_res(&lv, &r, 32, 16, SIGE_NORM_INSTANCE, 16, SIGE_ACT_RELU);
    push_up(&lv);
    push_conv(&lv, &r, 16, 3, 3, 1);
    return finish(name, 3, 64, 64, &lv);
  }
  if (!strcmp(name, "ddim_stack")) return build_ddim(256, 128);
  if (!strcmp(name, "ddim_stack_64x32")) return build_ddim(64, 32);
  fail("unknown model: %s", name);
  return NULL;
}

static float* dupf(const float* p, size_t n) {
  if (!p) return NULL;
  float* d = (float*)xcalloc(n, sizeof(float));
  memcpy(d, p, n * sizeof(float));
  return d;
}

static sige_conv_desc clone_conv(sige_conv_desc c) {
  c.weight = dupf(c.weight, (size_t)c.c_out * c.c_in * c.k * c.k);
  c.bias = dupf(c.bias, (size_t)c.c_out);
  return c;
}

static sige_norm_desc clone_norm(sige_norm_desc n) {
  n.gamma = dupf(n.gamma, n.channels);
  n.beta = dupf(n.beta, n.channels);
  n.running_mean = dupf(n.running_mean, n.channels);
  n.running_var = dupf(n.running_var, n.channels);
  return n;
}

sige_model_desc* orc_model_clone(const sige_model_desc* d) {
  LayerVec lv = {0};
  for (int i = 0; i < d->num_layers; ++i) {
    sige_layer_desc L = d->layers[i];
    if (L.kind == SIGE_LAYER_CONV || L.kind == SIGE_LAYER_DOWNSAMPLE || L.kind == SIGE_LAYER_RESBLOCK)
      L.conv = clone_conv(L.conv);
    if (L.kind == SIGE_LAYER_NORM || L.kind == SIGE_LAYER_RESBLOCK) L.norm = clone_norm(L.norm);
    if (L.kind == SIGE_LAYER_RESBLOCK) {
      L.conv2 = clone_conv(L.conv2);
      if (L.has_shortcut) L.shortcut = clone_conv(L.shortcut);
    }
    lv_push(&lv, L);
  }
  return finish(d->name ? d->name : "", d->in_channels, d->in_h, d->in_w, &lv);
}

static void free_conv(sige_conv_desc* c) {
  free((void*)c->weight);
  free((void*)c->bias);
}

static void free_norm(sige_norm_desc* n) {
  free((void*)n->gamma);
  free((void*)n->beta);
  free((void*)n->running_mean);
  free((void*)n->running_var);
}

void orc_model_free(sige_model_desc* d) {
  if (!d) return;
  for (int i = 0; i < d->num_layers; ++i) {
    sige_layer_desc* L = (sige_layer_desc*)&d->layers[i];
    if (L->kind == SIGE_LAYER_CONV || L->kind == SIGE_LAYER_DOWNSAMPLE || L->kind == SIGE_LAYER_RESBLOCK)
      free_conv(&L->conv);
    if (L->kind == SIGE_LAYER_NORM || L->kind == SIGE_LAYER_RESBLOCK) free_norm(&L->norm);
    if (L->kind == SIGE_LAYER_RESBLOCK) {
      free_conv(&L->conv2);
      if (L->has_shortcut) free_conv(&L->shortcut);
    }
  }
  free((void*)d->layers);
  free((void*)d->name);
  free(d);
}

/* model_weight_hash: models.cpp:185-207. */
static uint64_t hash_f(const float* p, size_t n, uint64_t h) {
  return p ? orc_fnv1a64(p, n * sizeof(float), h) : h;
}
static uint64_t hash_convw(const sige_conv_desc* c, uint64_t h) {
  h = hash_f(c->weight, (size_t)c->c_out * c->c_in * c->k * c->k, h);
  return hash_f(c->bias, c->bias ? (size_t)c->c_out : 0, h);
}
static uint64_t hash_normw(const sige_norm_desc* n, uint64_t h) {
  h = hash_f(n->gamma, n->channels, h);
  h = hash_f(n->beta, n->channels, h);
  h = hash_f(n->running_mean, n->channels, h);
  return hash_f(n->running_var, n->channels, h);
}

uint64_t orc_model_weight_hash(const sige_model_desc* d) {
  uint64_t h = orc_fnv1a64(d->name, strlen(d->name), FNV_SEED);
  for (int i = 0; i < d->num_layers; ++i) {
    const sige_layer_desc* L = &d->layers[i];
    switch (L->kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE:
        h = hash_convw(&L->conv, h);
        break;
      case SIGE_LAYER_NORM:
        h = hash_normw(&L->norm, h);
        break;
      case SIGE_LAYER_RESBLOCK:
        h = hash_convw(&L->conv, h);
        h = hash_normw(&L->norm, h);
        h = hash_convw(&L->conv2, h);
        if (L->has_shortcut) h = hash_convw(&L->shortcut, h);
        break;
      default:
        break;
    }
  }
  return h;
}

/* walk_shapes (graph.cpp:129-193): per-layer (c,h,w) in / out. */
typedef struct {
  int c_in, h_in, w_in, c_out, h_out, w_out;
} Shape;

static int walk(const sige_model_desc* m, int h, int w, Shape* out) {
  int c = m->in_channels;
  for (int i = 0; i < m->num_layers; ++i) {
    const sige_layer_desc* L = &m->layers[i];
    Shape s = {c, h, w, 0, 0, 0};
    switch (L->kind) {
      case SIGE_LAYER_CONV:
      case SIGE_LAYER_DOWNSAMPLE:
        TRY(conv_validate(&L->conv));
        if (L->conv.c_in != c) return fail("model layer L%d: expects %d channels, gets %d", i, L->conv.c_in, c);
        c = L->conv.c_out;
        h = conv_out_dim(h, L->conv.k, L->conv.stride);
        w = conv_out_dim(w, L->conv.k, L->conv.stride);
        break;
      case SIGE_LAYER_NORM:
        if (L->norm.channels != c) return fail("model layer L%d: norm channel mismatch", i);
        break;
      case SIGE_LAYER_RESBLOCK:
        if (L->conv.c_in != c) return fail("model layer L%d: resblock channel mismatch", i);
        c = L->conv2.c_out;
        break;
      case SIGE_LAYER_UPSAMPLE:
        h *= 2;
        w *= 2;
        break;
      default:
        break;
    }
    s.c_out = c;
    s.h_out = h;
    s.w_out = w;
    if (out) out[i] = s;
  }
  return 0;
}

int orc_model_output_shape(const sige_model_desc* d, int* c, int* h, int* w) {
  Shape* s = (Shape*)xcalloc(d->num_layers, sizeof(Shape));
  int rc = walk(d, d->in_h, d->in_w, s);
  if (!rc) {
    *c = s[d->num_layers - 1].c_out;
    *h = s[d->num_layers - 1].h_out;
    *w = s[d->num_layers - 1].w_out;
  }
  free(s);
  return rc;
}

/* required_dilation: graph.cpp:195-218. */
int orc_model_required_dilation(const sige_model_desc* d) {
  Shape* s = (Shape*)xcalloc(d->num_layers, sizeof(Shape));
  int g = 0;
  if (walk(d, d->in_h, d->in_w, s) == 0)
    for (int i = 0; i < d->num_layers; ++i) {
      const sige_layer_desc* L = &d->layers[i];
      int f = imax(1, d->in_h / s[i].h_in);
      if (L->kind == SIGE_LAYER_CONV || L->kind == SIGE_LAYER_DOWNSAMPLE)
        g += ((L->conv.k - 1) / 2) * f;
      else if (L->kind == SIGE_LAYER_RESBLOCK)
        g += ((L->conv.k - 1) / 2 + (L->conv2.k - 1) / 2) * f;
    }
  free(s);
  return g;
}

/* ----------------------------------------------------------------- tensors */
typedef struct {
  int n, c, h, w;
  float* d;
} T4;

static size_t t_numel(const T4* t) { return (size_t)t->n * t->c * t->h * t->w; }
static T4 t_new(int n, int c, int h, int w) {
  T4 t = {n, c, h, w, (float*)xcalloc((size_t)n * c * h * w, sizeof(float))};
  return t;
}
static T4 t_copy(const T4* s) {
  T4 t = t_new(s->n, s->c, s->h, s->w);
  memcpy(t.d, s->d, t_numel(s) * sizeof(float));
  return t;
}
static void t_free(T4* t) {
  free(t->d);
  t->d = NULL;
}

/* upsample_nearest2x: tensor.cpp:69-83. */
static T4 t_upsample(const T4* s) {
  T4 t = t_new(s->n, s->c, s->h * 2, s->w * 2);
  for (size_t pl = 0; pl < (size_t)s->n * s->c; ++pl)
    for (int y = 0; y < t.h; ++y)
      for (int x = 0; x < t.w; ++x)
        t.d[(pl * t.h + y) * t.w + x] = s->d[(pl * s->h + y / 2) * s->w + x / 2];
  return t;
}

static int t_apply_epi(T4* t, const sige_epilogue* e) {
  if (epi_empty(e)) return 0;
  size_t hw = (size_t)t->h * t->w;
  for (int in = 0; in < t->n; ++in)
    for (int ch = 0; ch < t->c; ++ch)
      for (size_t p = 0; p < hw; ++p)
        TRY(epi_value(e, &t->d[((size_t)in * t->c + ch) * hw + p], ch, t->c, in));
  return 0;
}

/* ------------------------------------------------------------------ cache
 * ActivationCache (graph.hpp:116-156): (step, key) -> tensor | folded norm. */
typedef struct {
  int step, kind; /* 0 tensor, 1 norm */
  char key[64];
  T4 t;
  float *scale, *shift;
  size_t np;
} Entry;

struct orc_cache {
  Entry* e;
  int n, cap;
};

static Entry* cache_find(orc_cache* c, int step, const char* key, int kind) {
  for (int i = 0; i < c->n; ++i)
    if (c->e[i].step == step && c->e[i].kind == kind && !strcmp(c->e[i].key, key)) return &c->e[i];
  return NULL;
}

static Entry* cache_slot(orc_cache* c, int step, const char* key, int kind) {
  Entry* e = cache_find(c, step, key, kind);
  if (e) {
    t_free(&e->t);
    free(e->scale);
    free(e->shift);
  } else {
    if (c->n == c->cap) {
      c->cap = c->cap ? 2 * c->cap : 32;
      c->e = (Entry*)realloc(c->e, (size_t)c->cap * sizeof(Entry));
    }
    e = &c->e[c->n++];
  }
  memset(e, 0, sizeof *e);
  e->step = step;
  e->kind = kind;
  snprintf(e->key, sizeof e->key, "%s", key);
  return e;
}

static void cache_put_tensor(orc_cache* c, int step, const char* key, const T4* t) {
  cache_slot(c, step, key, 0)->t = t_copy(t);
}

static void cache_put_norm(orc_cache* c, int step, const char* key, const float* sc,
                           const float* sh, size_t np) {
  Entry* e = cache_slot(c, step, key, 1);
  e->scale = dupf(sc, np);
  e->shift = dupf(sh, np);
  e->np = np;
}

/* tensor_entry / norm_entry: graph.cpp:242-262 ("precompute required"). */
static int cache_tensor(orc_cache* c, int step, const char* key, const T4** out) {
  Entry* e = cache_find(c, step, key, 0);
  if (!e) return fail("precompute required: no cache entry for step %d, layer %s", step, key);
  *out = &e->t;
  return 0;
}

static int cache_norm(orc_cache* c, int step, const char* key, Entry** out) {
  Entry* e = cache_find(c, step, key, 1);
  if (!e) return fail("precompute required: no cached norm params for step %d, layer %s", step, key);
  *out = e;
  return 0;
}

/* cache_base: graph.cpp:584-594 (shape check -> "cache is stale"). */
static int cache_base(orc_cache* c, int step, const char* key, int n, int ch, int h, int w,
                      const T4** out) {
  TRY(cache_tensor(c, step, key, out));
  const T4* t = *out;
  if (t->n != n || t->c != ch || t->h != h || t->w != w)
    return fail("cache entry %s has shape (%d, %d, %d, %d), run needs (%d, %d, %d, %d); cache is stale",
                key, t->n, t->c, t->h, t->w, n, ch, h, w);
  return 0;
}

void orc_cache_free(orc_cache* c) {
  if (!c) return;
  for (int i = 0; i < c->n; ++i) {
    t_free(&c->e[i].t);
    free(c->e[i].scale);
    free(c->e[i].shift);
  }
  free(c->e);
  free(c);
}

int orc_cache_tensor(orc_cache* c, int step, const char* key, float* out, size_t cap, int* dims) {
  const T4* t;
  TRY(cache_tensor(c, step, key, &t));
  dims[0] = t->n;
  dims[1] = t->c;
  dims[2] = t->h;
  dims[3] = t->w;
  if (out && cap >= t_numel(t)) memcpy(out, t->d, t_numel(t) * sizeof(float));
  return 0;
}

int orc_cache_norm(orc_cache* c, int step, const char* key, float* scale, float* shift,
                   size_t cap, int* count) {
  Entry* e;
  TRY(cache_norm(c, step, key, &e));
  *count = (int)e->np;
  if (scale && cap >= e->np) {
    memcpy(scale, e->scale, e->np * sizeof(float));
    memcpy(shift, e->shift, e->np * sizeof(float));
  }
  return 0;
}

int orc_cache_count(orc_cache* c) { return c->n; }

int orc_cache_entry(orc_cache* c, int i, int* kind, char* key, size_t keycap, size_t* numel) {
  if (i < 0 || i >= c->n) return fail("cache index out of range");
  *kind = c->e[i].kind;
  snprintf(key, keycap, "%s", c->e[i].key);
  *numel = c->e[i].kind ? c->e[i].np : t_numel(&c->e[i].t);
  return 0;
}

uint64_t orc_cache_total_elements(orc_cache* c) {
  uint64_t s = 0;
  for (int i = 0; i < c->n; ++i) s += c->e[i].kind ? 2 * c->e[i].np : t_numel(&c->e[i].t);
  return s;
}

/* ------------------------------------------------------------ dense walk */

static int conv_t(const T4* x, const sige_conv_desc* cv, T4* out) {
  *out = t_new(x->n, cv->c_out, conv_out_dim(x->h, cv->k, cv->stride),
               conv_out_dim(x->w, cv->k, cv->stride));
  return orc_conv2d(x->d, x->n, x->c, x->h, x->w, cv, 1, out->d);
}

/* fold_norm_layer: graph.cpp:310-322. Batch kind folds running stats into C
 * values; group/instance reduce over x into N*C values. */
static int fold_layer(const sige_norm_desc* nl, const T4* x, float** sc, float** sh, size_t* np) {
  int c = nl->channels;
  if (nl->kind == SIGE_NORM_BATCH) {
    *np = c;
    *sc = (float*)xcalloc(c, sizeof(float));
    *sh = (float*)xcalloc(c, sizeof(float));
    for (int ic = 0; ic < c; ++ic) {
      float s = nl->gamma[ic] / sqrtf(nl->running_var[ic] + nl->eps);
      float p = nl->running_mean[ic] * s;
      (*sc)[ic] = s;
      (*sh)[ic] = nl->beta[ic] - p;
    }
    return 0;
  }
  *np = (size_t)x->n * c;
  *sc = (float*)xcalloc(*np, sizeof(float));
  *sh = (float*)xcalloc(*np, sizeof(float));
  return orc_group_norm_fold(x->d, x->n, x->c, x->h, x->w, nl->groups, nl->eps, nl->gamma,
                             nl->beta, *sc, *sh);
}

static sige_epilogue epi_ss(const float* sc, const float* sh, size_t np) {
  sige_epilogue e;
  memset(&e, 0, sizeof e);
  e.num_steps = 1;
  e.steps[0].kind = SIGE_EPI_SCALE_SHIFT;
  e.steps[0].scale = sc;
  e.steps[0].shift = sh;
  e.steps[0].nparams = (int)np;
  return e;
}

static void epi_push_act(sige_epilogue* e, int act) {
  if (act == SIGE_ACT_NONE) return;
  e->steps[e->num_steps].kind = SIGE_EPI_ACTIVATION;
  e->steps[e->num_steps].act = act;
  e->num_steps++;
}

static sige_epilogue epi_act(int act) {
  sige_epilogue e;
  memset(&e, 0, sizeof e);
  epi_push_act(&e, act);
  return e;
}

/* dense_walk: graph.cpp:343-412; sink = precompute capture, stats = reuse. */
static int dense_walk(const sige_model_desc* m, const T4* input, orc_cache* sink,
                      orc_cache* stats, int step, T4* result) {
  char key[64], k2[80];
  T4 x = t_copy(input);
  int rc = 0;
  for (int i = 0; i < m->num_layers && !rc; ++i) {
    const sige_layer_desc* L = &m->layers[i];
    snprintf(key, sizeof key, "L%d", i);
    if (L->kind == SIGE_LAYER_CONV || L->kind == SIGE_LAYER_DOWNSAMPLE) {
      T4 y;
      rc = conv_t(&x, &L->conv, &y);
      t_free(&x);
      x = y;
      snprintf(k2, sizeof k2, "%s.out", key);
      if (!rc && sink) cache_put_tensor(sink, step, k2, &x);
    } else if (L->kind == SIGE_LAYER_NORM) {
      float *sc = NULL, *sh = NULL;
      size_t np = 0;
      snprintf(k2, sizeof k2, "%s.norm", key);
      if (stats) {
        Entry* e;
        rc = cache_norm(stats, step, k2, &e);
        if (!rc) {
          sc = dupf(e->scale, e->np);
          sh = dupf(e->shift, e->np);
          np = e->np;
        }
      } else {
        rc = fold_layer(&L->norm, &x, &sc, &sh, &np);
      }
      if (!rc && sink) cache_put_norm(sink, step, k2, sc, sh, np);
      if (!rc) {
        sige_epilogue e = epi_ss(sc, sh, np);
        rc = t_apply_epi(&x, &e);
      }
      free(sc);
      free(sh);
    } else if (L->kind == SIGE_LAYER_ACTIVATION) {
      sige_epilogue e = epi_act(L->act);
      rc = t_apply_epi(&x, &e);
    } else if (L->kind == SIGE_LAYER_UPSAMPLE) {
      T4 y = t_upsample(&x);
      t_free(&x);
      x = y;
    } else if (L->kind == SIGE_LAYER_RESBLOCK) {
      T4 mm, sc;
      rc = conv_t(&x, &L->conv, &mm);
      snprintf(k2, sizeof k2, "%s.conv1.out", key);
      if (!rc && sink) cache_put_tensor(sink, step, k2, &mm);
      float *fs = NULL, *fh = NULL;
      size_t np = 0;
      snprintf(k2, sizeof k2, "%s.norm1", key);
      if (!rc) {
        if (stats) {
          Entry* e;
          rc = cache_norm(stats, step, k2, &e);
          if (!rc) {
            fs = dupf(e->scale, e->np);
            fh = dupf(e->shift, e->np);
            np = e->np;
          }
        } else {
          rc = fold_layer(&L->norm, &mm, &fs, &fh, &np);
        }
      }
      if (!rc && sink) cache_put_norm(sink, step, k2, fs, fh, np);
      if (!rc) {
        sige_epilogue e = epi_ss(fs, fh, np);
        epi_push_act(&e, L->act);
        rc = t_apply_epi(&mm, &e);
      }
      free(fs);
      free(fh);
      if (!rc) {
        T4 m2;
        rc = conv_t(&mm, &L->conv2, &m2);
        t_free(&mm);
        mm = m2;
      }
      snprintf(k2, sizeof k2, "%s.conv2.out", key);
      if (!rc && sink) cache_put_tensor(sink, step, k2, &mm);
      if (!rc) {
        if (L->has_shortcut)
          rc = conv_t(&x, &L->shortcut, &sc);
        else
          sc = t_copy(&x);
      }
      snprintf(k2, sizeof k2, "%s.shortcut.out", key);
      if (!rc && sink) cache_put_tensor(sink, step, k2, &sc);
      if (!rc) {
        t_free(&x);
        x = t_new(mm.n, mm.c, mm.h, mm.w);
        for (size_t q = 0; q < t_numel(&x); ++q) x.d[q] = mm.d[q] + sc.d[q];
        snprintf(k2, sizeof k2, "%s.sum", key);
        if (sink) cache_put_tensor(sink, step, k2, &x);
      }
      t_free(&mm);
      t_free(&sc);
    }
  }
  if (!rc && sink) cache_put_tensor(sink, step, "final", &x);
  if (rc) {
    t_free(&x);
    return rc;
  }
  *result = x;
  return 0;
}

orc_cache* orc_cache_precompute(const sige_model_desc* m, const float* orig, int n, int c, int h,
                                int w) {
  orc_cache* cache = (orc_cache*)xcalloc(1, sizeof *cache);
  T4 in = {n, c, h, w, (float*)orig};
  T4 out;
  if (dense_walk(m, &in, cache, NULL, 0, &out)) {
    orc_cache_free(cache);
    return NULL;
  }
  t_free(&out);
  return cache;
}

int orc_dense_forward(const sige_model_desc* m, const float* in, int n, int c, int h, int w,
                      float* out) {
  T4 x = {n, c, h, w, (float*)in}, y;
  TRY(dense_walk(m, &x, NULL, NULL, 0, &y));
  memcpy(out, y.d, t_numel(&y) * sizeof(float));
  t_free(&y);
  return 0;
}

int orc_dense_forward_reused_stats(const sige_model_desc* m, const float* in, int n, int c,
                                   int h, int w, orc_cache* cache, int step, float* out) {
  T4 x = {n, c, h, w, (float*)in}, y;
  TRY(dense_walk(m, &x, NULL, cache, step, &y));
  memcpy(out, y.d, t_numel(&y) * sizeof(float));
  t_free(&y);
  return 0;
}

/* ---------------------------------------------------- sparse executor --- */

/* IndexPlan: graph.cpp:506-528. */
typedef struct {
  int h, w, b, count;
  int32_t* idx;
} PlanEntry;

typedef struct {
  uint8_t* full;
  int fh, fw, batch, dilate_scale;
  PlanEntry e[64];
  int n;
} Plan;

static int plan_at(Plan* p, int h, int w, int b, PlanEntry** out) {
  for (int i = 0; i < p->n; ++i)
    if (p->e[i].h == h && p->e[i].w == w && p->e[i].b == b) {
      *out = &p->e[i];
      return 0;
    }
  uint8_t* m = (uint8_t*)xcalloc((size_t)h * w, 1);
  int rc = (h <= p->fh && w <= p->fw) ? orc_downsample_mask(p->full, p->fh, p->fw, h, w, m)
                                      : replicate_mask(p->full, p->fh, p->fw, h, w, m);
  if (!rc && p->dilate_scale > 0) {
    uint8_t* d = (uint8_t*)xcalloc((size_t)h * w, 1);
    rc = orc_dilate_mask(m, h, w, p->dilate_scale, d);
    free(m);
    m = d;
  }
  if (rc) {
    free(m);
    return rc;
  }
  PlanEntry* e = &p->e[p->n++];
  e->h = h;
  e->w = w;
  e->b = b;
  int cap = ((h + b - 1) / b) * ((w + b - 1) / b) * p->batch;
  e->idx = (int32_t*)xcalloc((size_t)cap * 3 + 3, sizeof(int32_t));
  rc = orc_mask_to_block_indices(m, h, w, b, p->batch, e->idx, cap, &e->count, NULL);
  free(m);
  *out = e;
  return rc;
}

/* Flow: the activation in flight (graph.cpp:538-569). Either a full tensor
 * or raw conv blocks over a cached base, plus the pending element-wise chain. */
typedef struct {
  T4 full;
  sige_epilogue pending;
  int has_blocks;
  float* blocks;
  PlanEntry* bidx;
  int bc;
  const T4* base;
  int c, h, w;
} Flow;

static int materialize(Flow* f) {
  if (!f->has_blocks) return 0;
  f->full = t_new(f->base->n, f->base->c, f->base->h, f->base->w);
  int rc = orc_scatter(f->blocks, f->bidx->count, f->bc, f->bidx->b, f->bidx->idx, f->base->d,
                       f->full.d, f->base->n, f->base->c, f->base->h, f->base->w);
  free(f->blocks);
  f->blocks = NULL;
  f->has_blocks = 0;
  return rc;
}

static int flush(Flow* f) {
  TRY(materialize(f));
  TRY(t_apply_epi(&f->full, &f->pending));
  f->pending.num_steps = 0;
  return 0;
}

/* consume_windows: graph.cpp:571-582 (non-destructive). */
static int consume(Flow* f, PlanEntry* idx, int k, int s, float** out) {
  int c = f->c, win = s * idx->b + k - s;
  *out = (float*)xcalloc((size_t)idx->count * c * win * win, sizeof(float));
  if (f->has_blocks)
    return orc_scatter_gather(f->blocks, f->bidx->count, f->bidx->b, f->bidx->idx, f->base->d,
                              f->base->n, c, f->base->h, f->base->w, idx->idx, idx->count, idx->b,
                              idx->h, idx->w, k, s, &f->pending, *out);
  return orc_gather(f->full.d, f->full.n, c, f->full.h, f->full.w, idx->idx, idx->count, idx->b,
                    idx->h, idx->w, k, s, &f->pending, *out);
}

static int runs_sparse(const sige_layer_desc* L, int h, int w, const sige_run_config* cfg) {
  if (!cfg->sparse || !L->policy_sparse) return 0;
  int thr = cfg->min_sparse_res >= 0 ? cfg->min_sparse_res : L->min_resolution;
  return imin(h, w) >= thr;
}

static void trace_row(uint64_t* rows, int cap, int* n, uint64_t blocks, uint64_t gathered,
                      uint64_t scattered, uint64_t macs, uint64_t dense, int sparse) {
  if (rows && *n < cap) {
    uint64_t* r = rows + 6 * *n;
    r[0] = blocks;
    r[1] = gathered;
    r[2] = scattered;
    r[3] = macs;
    r[4] = dense;
    r[5] = (uint64_t)sparse;
  }
  ++*n;
}

static uint64_t dense_macs(const sige_conv_desc* c, int oh, int ow, int batch) {
  return (uint64_t)c->c_out * c->c_in * c->k * c->k * oh * ow * batch;
}

/* Runs conv on gathered windows and returns the raw blocks (count, co, b, b). */
static int conv_blocks(const float* in, PlanEntry* idx, const sige_conv_desc* cv, float** out) {
  int win = cv->stride * idx->b + cv->k - cv->stride;
  *out = (float*)xcalloc((size_t)idx->count * cv->c_out * idx->b * idx->b, sizeof(float));
  return orc_conv_on_blocks(in, idx->count, win, cv, 1, *out, idx->b);
}

/* sparse_forward: graph.cpp:619-901 with elem_fusion and scatter_fusion on
 * (the reference proves the toggles output-invariant, test_graph.cpp:222-254). */
int orc_sparse_forward(const sige_model_desc* m, orc_cache* cache, const float* edited, int n,
                       int c, int h, int w, const uint8_t* mask, const sige_run_config* cfg,
                       float* out, uint64_t* trace_rows, int trace_cap, int* trace_n) {
  int tn = 0, rc = 0, any = 0;
  char key[64], k2[80];
  if (trace_n) *trace_n = 0;
  if (c != m->in_channels) return fail("forward: input channel mismatch");
  if (!cfg->sparse) return orc_dense_forward(m, edited, n, c, h, w, out);
  for (size_t i = 0; i < (size_t)h * w; ++i) any |= mask[i];
  if (!any) {
    const T4* fin;
    TRY(cache_tensor(cache, cfg->step, "final", &fin));
    memcpy(out, fin->d, t_numel(fin) * sizeof(float));
    return 0;
  }
  int step = cfg->step;
  Plan plan;
  memset(&plan, 0, sizeof plan);
  plan.full = (uint8_t*)xcalloc((size_t)h * w, 1);
  plan.fh = h;
  plan.fw = w;
  plan.batch = n;
  plan.dilate_scale = cfg->dilate_scale;
  TRY(orc_dilate_mask(mask, h, w, cfg->dilate_full, plan.full));

  Flow f;
  memset(&f, 0, sizeof f);
  T4 ein = {n, c, h, w, (float*)edited};
  f.full = t_copy(&ein);
  f.c = c;
  f.h = h;
  f.w = w;

  for (int i = 0; i < m->num_layers && !rc; ++i) {
    const sige_layer_desc* L = &m->layers[i];
    snprintf(key, sizeof key, "L%d", i);
    if (L->kind == SIGE_LAYER_CONV || L->kind == SIGE_LAYER_DOWNSAMPLE) {
      const sige_conv_desc* cv = &L->conv;
      int oh = conv_out_dim(f.h, cv->k, cv->stride), ow = conv_out_dim(f.w, cv->k, cv->stride);
      if (!runs_sparse(L, f.h, f.w, cfg)) {
        T4 y = {0, 0, 0, 0, NULL};
        rc = flush(&f);
        if (!rc) rc = conv_t(&f.full, cv, &y);
        t_free(&f.full);
        f.full = y;
        trace_row(trace_rows, trace_cap, &tn, 0, 0, 0, dense_macs(cv, oh, ow, n),
                  dense_macs(cv, oh, ow, n), 0);
      } else {
        PlanEntry* idx;
        float *win = NULL, *blk = NULL;
        const T4* base;
        rc = plan_at(&plan, oh, ow, cv->k == 3 ? cfg->block3 : cfg->block1, &idx);
        if (!rc) rc = consume(&f, idx, cv->k, cv->stride, &win);
        if (!rc) rc = conv_blocks(win, idx, cv, &blk);
        free(win);
        snprintf(k2, sizeof k2, "%s.out", key);
        if (!rc) rc = cache_base(cache, step, k2, n, cv->c_out, oh, ow, &base);
        int wsz = cv->stride * idx->b + cv->k - cv->stride;
        trace_row(trace_rows, trace_cap, &tn, idx->count, (uint64_t)idx->count * f.c * wsz * wsz,
                  (uint64_t)idx->count * cv->c_out * idx->b * idx->b,
                  (uint64_t)idx->count * cv->c_out * cv->c_in * cv->k * cv->k * idx->b * idx->b,
                  dense_macs(cv, oh, ow, n), 1);
        if (f.has_blocks) free(f.blocks);
        t_free(&f.full);
        f.blocks = blk;
        f.bidx = idx;
        f.bc = cv->c_out;
        f.base = base;
        f.has_blocks = 1;
        f.pending.num_steps = 0;
      }
      f.c = cv->c_out;
      f.h = oh;
      f.w = ow;
    } else if (L->kind == SIGE_LAYER_NORM) {
      snprintf(k2, sizeof k2, "%s.norm", key);
      if (L->norm.kind == SIGE_NORM_BATCH || cfg->norm_precompute) {
        Entry* e;
        rc = cache_norm(cache, step, k2, &e);
        if (!rc) {
          sige_epilogue_step* s = &f.pending.steps[f.pending.num_steps++];
          s->kind = SIGE_EPI_SCALE_SHIFT;
          s->scale = e->scale;
          s->shift = e->shift;
          s->nparams = (int)e->np;
        }
      } else {
        float *sc = NULL, *sh = NULL;
        size_t np;
        rc = flush(&f);
        if (!rc) rc = fold_layer(&L->norm, &f.full, &sc, &sh, &np);
        if (!rc) {
          sige_epilogue e = epi_ss(sc, sh, np);
          rc = t_apply_epi(&f.full, &e);
        }
        free(sc);
        free(sh);
      }
    } else if (L->kind == SIGE_LAYER_ACTIVATION) {
      epi_push_act(&f.pending, L->act);
    } else if (L->kind == SIGE_LAYER_UPSAMPLE) {
      rc = materialize(&f);
      T4 y = t_upsample(&f.full);
      t_free(&f.full);
      f.full = y;
      f.h *= 2;
      f.w *= 2;
    } else if (L->kind == SIGE_LAYER_RESBLOCK) {
      int co = L->conv2.c_out;
      if (!runs_sparse(L, f.h, f.w, cfg)) {
        T4 mm = {0, 0, 0, 0, NULL}, sc = {0, 0, 0, 0, NULL};
        rc = flush(&f);
        if (!rc) rc = conv_t(&f.full, &L->conv, &mm);
        trace_row(trace_rows, trace_cap, &tn, 0, 0, 0, dense_macs(&L->conv, f.h, f.w, n),
                  dense_macs(&L->conv, f.h, f.w, n), 0);
        if (!rc) {
          float *fs, *fh;
          size_t np;
          rc = fold_layer(&L->norm, &mm, &fs, &fh, &np);
          if (!rc) {
            sige_epilogue e = epi_ss(fs, fh, np);
            epi_push_act(&e, L->act);
            rc = t_apply_epi(&mm, &e);
          }
          free(fs);
          free(fh);
        }
        if (!rc) {
          T4 m2;
          rc = conv_t(&mm, &L->conv2, &m2);
          t_free(&mm);
          mm = m2;
        }
        trace_row(trace_rows, trace_cap, &tn, 0, 0, 0, dense_macs(&L->conv2, f.h, f.w, n),
                  dense_macs(&L->conv2, f.h, f.w, n), 0);
        if (!rc) {
          if (L->has_shortcut) {
            rc = conv_t(&f.full, &L->shortcut, &sc);
            trace_row(trace_rows, trace_cap, &tn, 0, 0, 0, dense_macs(&L->shortcut, f.h, f.w, n),
                      dense_macs(&L->shortcut, f.h, f.w, n), 0);
          } else {
            sc = t_copy(&f.full);
          }
        }
        if (!rc) {
          for (size_t q = 0; q < t_numel(&mm); ++q) mm.d[q] = mm.d[q] + sc.d[q];
          t_free(&f.full);
          f.full = mm;
          t_free(&sc);
        }
      } else {
        PlanEntry *im, *is;
        float *min_ = NULL, *sin_ = NULL, *m1 = NULL, *m2in = NULL, *m2 = NULL, *scb = NULL;
        const T4 *b1 = NULL, *sum = NULL, *osc = NULL;
        int hh = f.h, ww = f.w, ci = f.c, c1 = L->conv.c_out;
        rc = plan_at(&plan, hh, ww, cfg->block3, &im);
        if (!rc) rc = plan_at(&plan, hh, ww, cfg->block1, &is);
        if (!rc) rc = consume(&f, im, 3, 1, &min_);
        if (!rc) rc = consume(&f, is, 1, 1, &sin_);
        if (!rc) rc = conv_blocks(min_, im, &L->conv, &m1);
        snprintf(k2, sizeof k2, "%s.conv1.out", key);
        if (!rc) rc = cache_base(cache, step, k2, n, c1, hh, ww, &b1);
        size_t g8 = (size_t)im->count * c1 * (im->b + 2) * (im->b + 2);
        if (!rc) {
          m2in = (float*)xcalloc(g8, sizeof(float));
          snprintf(k2, sizeof k2, "%s.norm1", key);
          if (L->norm.kind == SIGE_NORM_BATCH || cfg->norm_precompute) {
            Entry* e;
            rc = cache_norm(cache, step, k2, &e);
            if (!rc) {
              sige_epilogue ep = epi_ss(e->scale, e->shift, e->np);
              epi_push_act(&ep, L->act);
              rc = orc_scatter_gather(m1, im->count, im->b, im->idx, b1->d, n, c1, hh, ww,
                                      im->idx, im->count, im->b, hh, ww, 3, 1, &ep, m2in);
            }
          } else {
            T4 full1 = t_new(n, c1, hh, ww);
            float *fs = NULL, *fh = NULL;
            size_t np;
            rc = orc_scatter(m1, im->count, c1, im->b, im->idx, b1->d, full1.d, n, c1, hh, ww);
            if (!rc) rc = fold_layer(&L->norm, &full1, &fs, &fh, &np);
            if (!rc) {
              sige_epilogue ep = epi_ss(fs, fh, np);
              epi_push_act(&ep, L->act);
              rc = t_apply_epi(&full1, &ep);
            }
            if (!rc)
              rc = orc_gather(full1.d, n, c1, hh, ww, im->idx, im->count, im->b, hh, ww, 3, 1,
                              NULL, m2in);
            free(fs);
            free(fh);
            t_free(&full1);
          }
        }
        if (!rc) rc = conv_blocks(m2in, im, &L->conv2, &m2);
        size_t g_main = (size_t)im->count * ci * (im->b + 2) * (im->b + 2);
        size_t g_sc = (size_t)is->count * ci * is->b * is->b;
        trace_row(trace_rows, trace_cap, &tn, im->count, g_main,
                  (uint64_t)im->count * c1 * im->b * im->b,
                  (uint64_t)im->count * c1 * ci * 9 * im->b * im->b,
                  dense_macs(&L->conv, hh, ww, n), 1);
        trace_row(trace_rows, trace_cap, &tn, im->count, g8,
                  (uint64_t)im->count * co * im->b * im->b,
                  (uint64_t)im->count * co * c1 * 9 * im->b * im->b,
                  dense_macs(&L->conv2, hh, ww, n), 1);
        if (!rc) {
          if (L->has_shortcut) {
            rc = conv_blocks(sin_, is, &L->shortcut, &scb);
            trace_row(trace_rows, trace_cap, &tn, is->count, g_sc,
                      (uint64_t)is->count * co * is->b * is->b,
                      (uint64_t)is->count * co * ci * is->b * is->b,
                      dense_macs(&L->shortcut, hh, ww, n), 1);
          } else {
            scb = sin_;
            sin_ = NULL;
          }
        }
        snprintf(k2, sizeof k2, "%s.sum", key);
        if (!rc) rc = cache_base(cache, step, k2, n, co, hh, ww, &sum);
        snprintf(k2, sizeof k2, "%s.shortcut.out", key);
        if (!rc) rc = cache_base(cache, step, k2, n, co, hh, ww, &osc);
        if (!rc) {
          T4 o = t_new(n, co, hh, ww);
          rc = orc_scatter_with_block_residual(m2, im->count, im->b, im->idx, scb, is->count,
                                               is->b, is->idx, sum->d, osc->d, o.d, n, co, hh, ww,
                                               1);
          if (f.has_blocks) free(f.blocks);
          f.blocks = NULL;
          f.has_blocks = 0;
          t_free(&f.full);
          f.full = o;
          f.pending.num_steps = 0;
        }
        free(min_);
        free(sin_);
        free(m1);
        free(m2in);
        free(m2);
        free(scb);
      }
      f.c = co;
    }
  }
  if (!rc) {
    if (f.has_blocks) {
      const T4* fin;
      rc = orc_apply_epilogue_on_blocks(f.blocks, f.bidx->count, f.bc, f.bidx->b, f.bidx->idx,
                                        f.bidx->h, f.bidx->w, &f.pending);
      if (!rc) rc = cache_base(cache, step, "final", n, f.c, f.h, f.w, &fin);
      if (!rc)
        rc = orc_scatter(f.blocks, f.bidx->count, f.bc, f.bidx->b, f.bidx->idx, fin->d, out,
                         fin->n, fin->c, fin->h, fin->w);
    } else {
      rc = flush(&f);
      if (!rc) memcpy(out, f.full.d, t_numel(&f.full) * sizeof(float));
    }
  }
  if (f.has_blocks) free(f.blocks);
  t_free(&f.full);
  for (int i = 0; i < plan.n; ++i) free(plan.e[i].idx);
  free(plan.full);
  if (trace_n) *trace_n = tn;
  return rc;
}
