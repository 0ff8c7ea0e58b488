// oracle/hierarchy.cpp — TEST INFRASTRUCTURE ONLY (parity checker).
//
// Restatement of Algorithm 1 (run_scene_flow) and its three map operations,
// which the reference specifies but does not ship
// (proj/CMakeLists.txt:21 lists src/hierarchy.cpp; the file is absent).
// Parity for these functions is pinned only by SPEC.md's examples — see
// DESIGN.md §Oracle. Every ambiguity is resolved here
// ONCE and the device code follows it:
//   C.1 prolongation samples the coarse grid at fine-anchor/2 (no half-pixel
//       shift), clamped into coarse coverage; base = 2 * sample; delta = 0.
//   C.2 occlusion: triangles over the halfway pixel lattice, cell (x,y) split
//       into UL {(x,y),(x+1,y),(x,y+1)} and LR {(x+1,y),(x+1,y+1),(x,y+1)};
//       vertices projected by warp_position in 1/256-px fixed point; coverage
//       by int64 edge functions with a top-left tie rule; z = float(1/(|2s|+1e-3)),
//       flat per triangle (min of its vertices); z-buffer key (z bits, tri id),
//       min-reduced (order independent). Pixel x is visible in view e iff its
//       UL triangle is not degenerate and the front-most triangle at
//       round(P_e(x)) is one of the six triangles incident to x, or is not
//       nearer than z(x) by more than 1e-4. Degenerate: area <= 0, non-finite
//       flow, or a bounding box wider/taller than 8 px (a rubber-sheet triangle
//       spanning a flow discontinuity of > 8 px per lattice cell is not a surface:
//       it would over-occlude the band beside a foreground edge).
//   C.3 vis4 bit e = that per-view visibility; V_k = AND of endpoints
//       (energy.hpp:65-68). Mask prolongation: bilinear of the 0/1 plane at
//       x/2 (image.cpp sample semantics), visible iff >= 0.5.
//   C.4 illumination uses raw intensities and replaces (does not accumulate)
//       the coarser maps; box upsample = 2x2 replication.
//   C.5 levels auto-reduced until the coarsest short side is >= 16 px.
//   C.6 coarsest level: V all visible, no illumination, base = 0 (+coarse_s_offset).
//   C.7 FlowResult: WarpGrid::interpolate of the finest total grid, disparity 2 s_x.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "backend.hpp"
#include "ctx.hpp"
#include "hierarchy.hpp"
#include "hwflow_c.h"

// Per-pair delta hierarchy + accumulated grids (SPEC.md:396 `prev`).
struct hwf_state {
  int n = 0, w = 0, h = 0, L = 0, step = 0;
  bool valid = false;
  std::vector<std::vector<std::vector<double>>> delta, total;  // [pair][level][6G]
};

namespace orc {
namespace {

constexpr int kZbufSpanPx = 8;
constexpr double kDepthTol = 1e-4;
constexpr double kIllumSigma = 3.2;

}  // namespace

std::vector<std::vector<double>> load_frames(const hwf_frame4* f) {
  if (!f || f->width < 1 || f->height < 1) throw std::invalid_argument("bad frame dims");
  const size_t N = static_cast<size_t>(f->width) * f->height;
  std::vector<std::vector<double>> out(4, std::vector<double>(N));
  for (int e = 0; e < 4; ++e) {
    if (!f->plane[e]) throw std::invalid_argument("null image plane");
    if (f->dtype == HWF_DTYPE_U8) {
      const uint8_t* p = static_cast<const uint8_t*>(f->plane[e]);
      for (size_t i = 0; i < N; ++i) out[e][i] = p[i] / 255.0;
    } else if (f->dtype == HWF_DTYPE_F64) {
      const double* p = static_cast<const double*>(f->plane[e]);
      for (size_t i = 0; i < N; ++i) out[e][i] = std::min(1.0, std::max(0.0, p[i]));
    } else {
      throw std::invalid_argument("unknown dtype");
    }
  }
  return out;
}

// ---- occlusion (pins C.2/C.3) -------------------------------
void occlusion(int w, int h, int step, const double* total, uint8_t* vis4) {
  const GridDims g = grid_dims(w, h, step);
  const int N = w * h;
  std::vector<int32_t> qx(4 * static_cast<size_t>(N)), qy(4 * static_cast<size_t>(N));
  std::vector<float> Z(N);
  std::vector<uint8_t> bad(N, 0);
  for (int pix = 0; pix < N; ++pix) {
    const int px = pix % w, py = pix / w;
    double fl[6];
    interpolate(g, total, px, py, fl);
    const double s2x = 2.0 * fl[0], s2y = 2.0 * fl[1];
    const double z = 1.0 / (std::sqrt(s2x * s2x + s2y * s2y) + 1e-3);
    Z[pix] = static_cast<float>(z);
    bool ok = std::isfinite(z);
    for (int e = 0; e < 4; ++e) {
      double wx, wy;
      warp_position(px, py, fl, e & 1, e >> 1, &wx, &wy);
      const double fx = wx * 256.0, fy = wy * 256.0;
      ok = ok && std::isfinite(fx) && std::isfinite(fy) && std::abs(fx) < 1073741824.0 &&
           std::abs(fy) < 1073741824.0;
      qx[4 * pix + e] = ok ? static_cast<int32_t>(std::llrint(fx)) : 0;
      qy[4 * pix + e] = ok ? static_cast<int32_t>(std::llrint(fy)) : 0;
    }
    bad[pix] = ok ? 0 : 1;
  }
  std::memset(vis4, 0, N);
  if (w < 2 || h < 2) {
    for (int pix = 0; pix < N; ++pix) vis4[pix] = bad[pix] ? 0 : 0x0F;
    return;
  }
  std::vector<uint64_t> zbuf(N);
  std::vector<uint8_t> degen(N);
  const int cw = w - 1;
  for (int e = 0; e < 4; ++e) {
    std::fill(zbuf.begin(), zbuf.end(), ~0ull);
    std::fill(degen.begin(), degen.end(), 0);
    for (int cy = 0; cy < h - 1; ++cy)
      for (int cx = 0; cx < cw; ++cx)
        for (int t = 0; t < 2; ++t) {
          const int v[3] = {t == 0 ? cy * w + cx : cy * w + cx + 1,
                            t == 0 ? cy * w + cx + 1 : (cy + 1) * w + cx + 1, (cy + 1) * w + cx};
          int64_t X[3], Y[3];
          bool deg = false;
          for (int i = 0; i < 3; ++i) {
            X[i] = qx[4 * v[i] + e];
            Y[i] = qy[4 * v[i] + e];
            deg = deg || bad[v[i]];
          }
          const int64_t area = (X[1] - X[0]) * (Y[2] - Y[0]) - (Y[1] - Y[0]) * (X[2] - X[0]);
          const int64_t mnx = std::min({X[0], X[1], X[2]}), mxx = std::max({X[0], X[1], X[2]});
          const int64_t mny = std::min({Y[0], Y[1], Y[2]}), mxy = std::max({Y[0], Y[1], Y[2]});
          deg = deg || area <= 0 || (mxx - mnx) > kZbufSpanPx * 256 || (mxy - mny) > kZbufSpanPx * 256;
          if (deg) {
            if (t == 0) degen[cy * w + cx] = 1;
            continue;
          }
          const float zf = std::min({Z[v[0]], Z[v[1]], Z[v[2]]});
          uint32_t zb;
          std::memcpy(&zb, &zf, 4);
          const uint64_t key = (static_cast<uint64_t>(zb) << 32) |
                               static_cast<uint32_t>(2 * (cy * cw + cx) + t);
          const int64_t x0 = std::max<int64_t>(0, -((-mnx) >> 8)), x1 = std::min<int64_t>(w - 1, mxx >> 8);
          const int64_t y0 = std::max<int64_t>(0, -((-mny) >> 8)), y1 = std::min<int64_t>(h - 1, mxy >> 8);
          for (int64_t yy = y0; yy <= y1; ++yy)
            for (int64_t xx = x0; xx <= x1; ++xx) {
              const int64_t Px = xx * 256, Py = yy * 256;
              bool in = true;
              for (int i = 0; i < 3 && in; ++i) {
                const int j = (i + 1) % 3;
                const int64_t dx = X[j] - X[i], dy = Y[j] - Y[i];
                const int64_t E = dx * (Py - Y[i]) - dy * (Px - X[i]);
                in = E > 0 || (E == 0 && (dy > 0 || (dy == 0 && dx < 0)));
              }
              if (in) {
                uint64_t& zref = zbuf[yy * w + xx];
                zref = std::min(zref, key);
              }
            }
        }
    for (int pix = 0; pix < N; ++pix) {
      const int px = pix % w, py = pix / w;
      bool vis = !bad[pix];
      if (vis && px < w - 1 && py < h - 1 && degen[pix]) vis = false;
      if (vis) {
        const int64_t rx = (static_cast<int64_t>(qx[4 * pix + e]) + 128) >> 8;
        const int64_t ry = (static_cast<int64_t>(qy[4 * pix + e]) + 128) >> 8;
        if (rx >= 0 && rx < w && ry >= 0 && ry < h) {
          const uint64_t key = zbuf[ry * w + rx];
          if (key != ~0ull) {
            const uint32_t tri = static_cast<uint32_t>(key & 0xffffffffu);
            const int tt = tri & 1, cell = tri >> 1, ccx = cell % cw, ccy = cell / cw;
            const bool ring =
                tt == 0 ? ((ccx == px && ccy == py) || (ccx == px - 1 && ccy == py) ||
                           (ccx == px && ccy == py - 1))
                        : ((ccx == px - 1 && ccy == py) || (ccx == px - 1 && ccy == py - 1) ||
                           (ccx == px && ccy == py - 1));
            if (!ring) {
              const uint32_t zb = static_cast<uint32_t>(key >> 32);
              float zf;
              std::memcpy(&zf, &zb, 4);
              if (static_cast<double>(Z[pix]) - kDepthTol > static_cast<double>(zf)) vis = false;
            }
          }
        }
      }
      if (vis) vis4[pix] |= static_cast<uint8_t>(1u << e);
    }
  }
}

// ---- illumination (pin C.4) ---------------------------------
void illumination(int w, int h, int step, const double* const images[4], const double* total,
                  const uint8_t* vis4, double* half_maps) {
  const GridDims g = grid_dims(w, h, step);
  const int N = w * h;
  std::vector<double> r(N), b;
  for (int t = 0; t < 2; ++t) {
    const int e1 = 1 + 2 * t, e0 = 2 * t;
    const Raster I1{w, h, images[e1]}, I0{w, h, images[e0]};
    for (int pix = 0; pix < N; ++pix) {
      r[pix] = 0.0;
      if (!((vis4[pix] >> e1) & 1) || !((vis4[pix] >> e0) & 1)) continue;
      const int px = pix % w, py = pix / w;
      double fl[6], x1, y1, x0, y0;
      interpolate(g, total, px, py, fl);
      warp_position(px, py, fl, 1, t, &x1, &y1);
      warp_position(px, py, fl, 0, t, &x0, &y0);
      r[pix] = sample(I1, x1, y1, nullptr, nullptr) - sample(I0, x0, y0, nullptr, nullptr);
    }
    gaussian_blur(Raster{w, h, r.data()}, kIllumSigma, b);
    for (int pix = 0; pix < N; ++pix) half_maps[static_cast<size_t>(t) * N + pix] = 0.5 * b[pix];
  }
}

// ---- prolongation (pins C.1/C.3/C.4) ------------------------
void prolongate(int wc, int hc, int wf, int hf, int step, const double* total_c,
                const uint8_t* vis_c, const double* hm_c, double* base_f, uint8_t* vis_f,
                double* hm_f) {
  const GridDims gc = grid_dims(wc, hc, step), gf = grid_dims(wf, hf, step);
  const double xmax = static_cast<double>(gc.gw - 1) * step, ymax = static_cast<double>(gc.gh - 1) * step;
  for (int k = 0; k < gf.nodes(); ++k) {
    const double x = std::min(static_cast<double>((k % gf.gw) * step) / 2.0, xmax);
    const double y = std::min(static_cast<double>((k / gf.gw) * step) / 2.0, ymax);
    double fl[6];
    interpolate(gc, total_c, x, y, fl);
    for (int c = 0; c < 6; ++c) base_f[6 * k + c] = 2.0 * fl[c];
  }
  if (vis_c && vis_f) {
    const size_t Nc = static_cast<size_t>(wc) * hc;
    std::vector<double> plane(Nc);
    std::memset(vis_f, 0, static_cast<size_t>(wf) * hf);
    for (int e = 0; e < 4; ++e) {
      for (size_t i = 0; i < Nc; ++i) plane[i] = (vis_c[i] >> e) & 1 ? 1.0 : 0.0;
      const Raster R{wc, hc, plane.data()};
      for (int y = 0; y < hf; ++y)
        for (int x = 0; x < wf; ++x)
          if (sample(R, x / 2.0, y / 2.0, nullptr, nullptr) >= 0.5)
            vis_f[static_cast<size_t>(y) * wf + x] |= static_cast<uint8_t>(1u << e);
    }
  }
  if (hm_c && hm_f) {
    const size_t Nc = static_cast<size_t>(wc) * hc, Nf = static_cast<size_t>(wf) * hf;
    for (int t = 0; t < 2; ++t)
      for (int y = 0; y < hf; ++y)
        for (int x = 0; x < wf; ++x)
          hm_f[t * Nf + static_cast<size_t>(y) * wf + x] =
              hm_c[t * Nc + static_cast<size_t>(std::min(y / 2, hc - 1)) * wc + std::min(x / 2, wc - 1)];
  }
}

// ---- temporal propagation (pin: pull-back along the previous
// frame's accumulated motion at the node, p - 2 m(p), bilinear WarpGrid sample of
// the previous delta, all six components zero outside the lattice coverage)
void propagate(int w, int h, int step, const double* prev_delta, const double* prev_total, double* next_delta) {
  const GridDims g = grid_dims(w, h, step);
  const double xmax = static_cast<double>(g.gw - 1) * step, ymax = static_cast<double>(g.gh - 1) * step;
  for (int k = 0; k < g.nodes(); ++k) {
    const double px = static_cast<double>((k % g.gw) * step), py = static_cast<double>((k / g.gw) * step);
    const double qx = px - 2.0 * prev_total[6 * k + 2], qy = py - 2.0 * prev_total[6 * k + 3];
    if (qx >= 0.0 && qy >= 0.0 && qx <= xmax && qy <= ymax) {
      interpolate(g, prev_delta, qx, qy, next_delta + 6 * k);
    } else {
      for (int c = 0; c < 6; ++c) next_delta[6 * k + c] = 0.0;
    }
  }
}

int gn_for_level(const hwf_schedule* S, int l) {  // solver.hpp:30-34
  if (S->n_gn_per_level > 0) return S->gn_per_level[std::min(l, S->n_gn_per_level - 1)];
  return l <= 1 ? 2 : 5;
}

namespace {

// Algorithm 1.
void run_scene_flow(Backend* B, const hwf_frame4* fr, const hwf_energy_params* P,
                    const hwf_schedule* S, const double* F, hwf_result* out, hwf_stats* stats,
                    const hwf_state* prev = nullptr, hwf_state* next = nullptr, int pair = 0) {
  if (hwf_validate_params(P) != HWF_OK) throw std::invalid_argument("energy weights must be >= 0");
  if (P->w_epi > 0.0 && !F) throw std::invalid_argument("epipolar term enabled without a fundamental matrix");
  const auto imgs = load_frames(fr);
  int L = 0, dims[4 * HWF_MAX_LEVELS];
  if (hwf_level_dims(fr->width, fr->height, S->levels, S->grid_step, &L, dims) != HWF_OK)
    throw std::invalid_argument("bad level dims");
  size_t pyr_size = 0;
  for (int l = 0; l < L; ++l) pyr_size += 4ull * dims[4 * l] * dims[4 * l + 1];
  std::vector<double> pyr(pyr_size);
  B->pyramid(imgs, fr->width, fr->height, L, pyr.data());
  std::vector<size_t> off(L + 1, 0);
  for (int l = 0; l < L; ++l) off[l + 1] = off[l] + 4ull * dims[4 * l] * dims[4 * l + 1];

  std::vector<double> total_prev, hm_prev;
  std::vector<uint8_t> vis_prev;
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->levels_used = L;
  }
  for (int l = L - 1; l >= 0; --l) {
    const int w = dims[4 * l], h = dims[4 * l + 1], N = w * h;
    const int G = dims[4 * l + 2] * dims[4 * l + 3];
    std::vector<double> base(6 * static_cast<size_t>(G), 0.0), delta(6 * static_cast<size_t>(G), 0.0);
    if (prev && prev->valid)  // warm start; first frame: zero deltas
      propagate(w, h, S->grid_step, prev->delta[pair][l].data(), prev->total[pair][l].data(), delta.data());
    std::vector<uint8_t> vis(N, 0x0F), outl(N, 1);
    std::vector<double> node_w(G, 1.0), hm;
    if (l == L - 1) {
      for (int k = 0; k < G; ++k) {
        base[6 * k] += S->coarse_s_offset[0];
        base[6 * k + 1] += S->coarse_s_offset[1];
      }
    } else {
      hm.assign(2 * static_cast<size_t>(N), 0.0);
      prolongate(dims[4 * (l + 1)], dims[4 * (l + 1) + 1], w, h, S->grid_step, total_prev.data(),
                 vis_prev.data(), hm_prev.data(), base.data(), vis.data(), hm.data());
    }
    std::vector<double> illum;
    hwf_level lv{};
    lv.width = w;
    lv.height = h;
    lv.grid_step = S->grid_step;
    for (int e = 0; e < 4; ++e) lv.images[e] = pyr.data() + off[l] + static_cast<size_t>(e) * N;
    if (!hm.empty()) {
      illum.resize(4 * static_cast<size_t>(N));
      for (int e = 0; e < 4; ++e) {
        const double* src = hm.data() + static_cast<size_t>(e >> 1) * N;
        for (int i = 0; i < N; ++i) illum[static_cast<size_t>(e) * N + i] = (e & 1) ? -src[i] : src[i];
        lv.illum[e] = illum.data() + static_cast<size_t>(e) * N;
      }
    }
    lv.total = base.data();  // rebound inside gauss_newton to base + delta
    lv.delta = delta.data();
    lv.vis4 = vis.data();
    lv.outlier = outl.data();
    lv.node_w = node_w.data();
    lv.fundamental = F;
    std::vector<double> eb, ea;
    B->gn_level(&lv, base.data(), delta.data(), outl.data(), node_w.data(), P, S,
                gn_for_level(S, l), &eb, &ea);
    if (stats) {
      stats->gn_iters[l] = static_cast<int>(eb.size());
      for (size_t i = 0; i < eb.size() && i < HWF_MAX_GN; ++i) {
        stats->energy_before[l][i] = eb[i];
        stats->energy_after[l][i] = ea[i];
      }
    }
    std::vector<double> total(base.size());
    for (size_t i = 0; i < total.size(); ++i) total[i] = base[i] + delta[i];
    if (next) {
      next->delta[pair][l] = delta;
      next->total[pair][l] = total;
    }
    std::vector<uint8_t> vis_new(N);
    occlusion(w, h, S->grid_step, total.data(), vis_new.data());
    if (l > 0) {
      hm_prev.assign(2 * static_cast<size_t>(N), 0.0);
      illumination(w, h, S->grid_step, lv.images, total.data(), vis_new.data(), hm_prev.data());
    }
    total_prev.swap(total);
    vis_prev.swap(vis_new);
  }
  // FlowResult (geometry.hpp:26-37) via WarpGrid::interpolate (warp_grid.cpp:56-65).
  const int w = fr->width, h = fr->height;
  const GridDims g0 = grid_dims(w, h, S->grid_step);
  for (int pix = 0; pix < w * h; ++pix) {
    double fl[6];
    interpolate(g0, total_prev.data(), pix % w, pix / w, fl);
    if (out->s) { out->s[2 * pix] = fl[0]; out->s[2 * pix + 1] = fl[1]; }
    if (out->m) { out->m[2 * pix] = fl[2]; out->m[2 * pix + 1] = fl[3]; }
    if (out->d) { out->d[2 * pix] = fl[4]; out->d[2 * pix + 1] = fl[5]; }
    if (out->disparity) out->disparity[pix] = 2.0 * fl[0];
    if (out->vis4) out->vis4[pix] = vis_prev[pix];
  }
  if (out->grid_total) std::memcpy(out->grid_total, total_prev.data(), total_prev.size() * sizeof(double));
}

template <class Fn>
int guard(hwf_ctx* ctx, Fn&& fn) {
  try {
    fn();
    return HWF_OK;
  } catch (const Divergence& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EDIVERGED;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EINVAL;
  }
}

}  // namespace
}  // namespace orc

// ============================== C-ABI =========================================
extern "C" {

int hwf_create(int /*device*/, hwf_ctx** out) {
  if (!out) return HWF_EINVAL;
  *out = new hwf_ctx();
  return HWF_OK;
}
void hwf_destroy(hwf_ctx* ctx) { delete ctx; }
const char* hwf_last_error(const hwf_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
const char* hwf_backend(void) { return orc::backend()->name(); }

void hwf_default_params(hwf_energy_params* p) {  // energy.hpp:17-27 (live)
  *p = hwf_energy_params{1.0, 1.0, 2.0, 0.0, 1.0, 1.0, 5.0, 5.0, 0.5, 5.0, 100.0, 1000.0, 0.001, 0.2};
}
int hwf_preset_params(const char* name, hwf_energy_params* p) {  // energy.cpp:9-41
  hwf_default_params(p);
  const std::string n = name ? name : "";
  if (n == "live") return HWF_OK;
  if (n == "facial") {
    p->w_reg = 0.5; p->w_photo = 0.5; p->w_grad = 5.0; p->w_epi = 0.5;
    p->w_s = 0.75; p->w_m = 0.5; p->w_d = 0.01; p->m_s = 0.5; p->m_m = 10.0; p->m_d = 100.0;
    return HWF_OK;
  }
  if (n == "stereo-hq") {
    p->w_reg = 5.0; p->w_photo = 1.0; p->w_grad = 5.0; p->w_epi = 0.5;
    p->w_s = 0.5; p->w_m = 1.0; p->w_d = 1.0; p->m_s = 0.1; p->m_m = 10000.0; p->m_d = 10000.0;
    return HWF_OK;
  }
  return HWF_EINVAL;
}
int hwf_validate_params(const hwf_energy_params* p) {  // energy.cpp:43-50
  const double ws[] = {p->w_reg, p->w_photo, p->w_grad, p->w_epi, p->w_smooth, p->w_mag,
                       p->w_s,   p->w_m,     p->w_d,    p->m_s,   p->m_m,      p->m_d};
  for (double w : ws)
    if (!(w >= 0.0)) return HWF_EINVAL;
  return (p->eps_huber > 0.0) ? HWF_OK : HWF_EINVAL;
}
void hwf_default_schedule(hwf_schedule* s) {  // solver.hpp:14-28
  std::memset(s, 0, sizeof(*s));
  s->levels = 5;
  s->pcg_iters = 5;
  s->patch_iters = 5;
  s->subdomain_px = 16;
  s->boundary_px = 2;
  s->grid_step = 2;
  s->threads = 1;
  s->active_fields = 7;
}
int hwf_level_dims(int width, int height, int levels, int grid_step, int* levels_used, int* dims) {
  if (width < 1 || height < 1 || grid_step < 1 || levels < 1) return HWF_EINVAL;
  int L = std::min(levels, HWF_MAX_LEVELS);
  int w = width, h = height;
  for (int l = 0; l < L; ++l) {
    if (l > 0 && std::min(w, h) < 16) {  // SPEC.md:450 (pin C.5)
      L = l;
      break;
    }
    dims[4 * l] = w;
    dims[4 * l + 1] = h;
    dims[4 * l + 2] = std::max((w - 1 + grid_step - 1) / grid_step + 1, 2);
    dims[4 * l + 3] = std::max((h - 1 + grid_step - 1) / grid_step + 1, 2);
    if (l + 1 < L) {
      const int nw = (w + 1) / 2, nh = (h + 1) / 2;
      if (std::min(nw, nh) < 16) {
        L = l + 1;
        break;
      }
      w = nw;
      h = nh;
    }
  }
  *levels_used = L;
  return HWF_OK;
}

int hwf_solve_pair(hwf_ctx* ctx, const hwf_frame4* frames, const hwf_energy_params* params,
                   const hwf_schedule* sched, const double* F, hwf_result* out, hwf_stats* stats) {
  return orc::guard(ctx, [&] { orc::run_scene_flow(orc::backend(), frames, params, sched, F, out, stats); });
}
int hwf_solve_batch(hwf_ctx* ctx, int n, const hwf_frame4* frames, const hwf_energy_params* params,
                    const hwf_schedule* sched, const double* F, hwf_result* out, hwf_stats* stats) {
  for (int i = 0; i < n; ++i) {
    const int rc = hwf_solve_pair(ctx, frames + i, params, sched, F, out + i, stats ? stats + i : nullptr);
    if (rc != HWF_OK) return rc;
  }
  return HWF_OK;
}
int hwf_state_create(hwf_ctx* ctx, int n, int w, int h, int levels, int step, hwf_state** out) {
  return orc::guard(ctx, [&] {
    int L = 0, dims[4 * HWF_MAX_LEVELS];
    if (n < 1 || hwf_level_dims(w, h, levels, step, &L, dims) != HWF_OK) throw std::invalid_argument("bad state dims");
    auto* st = new hwf_state();
    st->n = n;
    st->w = w;
    st->h = h;
    st->L = L;
    st->step = step;
    st->delta.assign(n, std::vector<std::vector<double>>(L));
    st->total.assign(n, std::vector<std::vector<double>>(L));
    for (int i = 0; i < n; ++i)
      for (int l = 0; l < L; ++l) {
        st->delta[i][l].assign(6ull * dims[4 * l + 2] * dims[4 * l + 3], 0.0);
        st->total[i][l].assign(6ull * dims[4 * l + 2] * dims[4 * l + 3], 0.0);
      }
    *out = st;
  });
}
void hwf_state_destroy(hwf_state* st) { delete st; }
int hwf_state_read(hwf_ctx* ctx, const hwf_state* st, int pair, double* delta, double* total) {
  return orc::guard(ctx, [&] {
    if (!st || pair < 0 || pair >= st->n) throw std::invalid_argument("bad state/pair");
    size_t off = 0;
    for (int l = 0; l < st->L; ++l) {
      const auto& d = st->delta[pair][l];
      if (delta) std::memcpy(delta + off, d.data(), d.size() * sizeof(double));
      if (total) std::memcpy(total + off, st->total[pair][l].data(), d.size() * sizeof(double));
      off += d.size();
    }
  });
}
int hwf_solve_batch_seq(hwf_ctx* ctx, int n, const hwf_frame4* frames, const hwf_energy_params* params,
                        const hwf_schedule* sched, const double* F, const hwf_state* prev, hwf_state* next,
                        hwf_result* out, hwf_stats* stats) {
  return orc::guard(ctx, [&] {
    int L = 0, dims[4 * HWF_MAX_LEVELS];
    if (hwf_level_dims(frames[0].width, frames[0].height, sched->levels, sched->grid_step, &L, dims) != HWF_OK)
      throw std::invalid_argument("bad dims");
    for (const hwf_state* st : {prev, static_cast<const hwf_state*>(next)})
      if (st && (st->n != n || st->w != frames[0].width || st->h != frames[0].height || st->L != L ||
                 st->step != sched->grid_step))
        throw std::invalid_argument("state does not match the batch (pairs, size, levels, grid step)");
    for (int i = 0; i < n; ++i)
      orc::run_scene_flow(orc::backend(), frames + i, params, sched, F, out + i, stats ? stats + i : nullptr, prev,
                          next, i);
    if (next) next->valid = true;
  });
}
int hwf_propagate_temporal(hwf_ctx* ctx, int w, int h, int step, const double* pd, const double* pt, double* nd) {
  return orc::guard(ctx, [&] { orc::propagate(w, h, step, pd, pt, nd); });
}

int hwf_pyramid(hwf_ctx* ctx, const hwf_frame4* frames, int levels, double* out) {
  return orc::guard(ctx, [&] {
    if (levels < 1) throw std::invalid_argument("pyramid needs >= 1 level");
    orc::backend()->pyramid(orc::load_frames(frames), frames->width, frames->height, levels, out);
  });
}
int hwf_eval_energy(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* p, hwf_energy* out,
                    double* residuals) {
  return orc::guard(ctx, [&] { *out = orc::backend()->eval_energy(lv, p, residuals, ctx ? ctx->threads : 1); });
}
int hwf_refresh_weights(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* p,
                        uint8_t* outlier_out, double* node_w_out) {
  return orc::guard(ctx, [&] { orc::backend()->refresh(lv, p, outlier_out, node_w_out, ctx ? ctx->threads : 1); });
}
int hwf_linearize(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* p, uint32_t active,
                  double lm, double* blocks, double* rhs, double* precond) {
  return orc::guard(ctx, [&] {
    orc::backend()->linearize(lv, p, active, lm, blocks, rhs, precond, ctx ? ctx->threads : 1);
  });
}
int hwf_assemble_jacobian(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* p, uint32_t active,
                          int negate_field, double* residuals, int* rows, int* cols, double* vals, long long cap,
                          long long* nnz) {
  return orc::guard(ctx, [&] {
    if (!lv || !p || !nnz || negate_field < -1 || negate_field > 2) throw std::invalid_argument("bad jacobian query");
    std::vector<double> R;
    std::vector<orc::JacEntry> e;
    orc::backend()->jacobian(lv, p, active, negate_field, R, e, 1);
    *nnz = static_cast<long long>(e.size());
    if (residuals) std::memcpy(residuals, R.data(), R.size() * sizeof(double));
    if (cap > 0 || rows || cols || vals) {
      if (cap < *nnz || !rows || !cols || !vals) throw std::invalid_argument("jacobian triplet buffers too small");
      for (size_t i = 0; i < e.size(); ++i) {
        rows[i] = e[i].row;
        cols[i] = e[i].col;
        vals[i] = e[i].value;
      }
    }
  });
}

int hwf_normal_dense(int gw, int gh, const double* blocks, double* dense) {  // solver.cpp:89-98
  if (gw < 1 || gh < 1 || !blocks || !dense) return HWF_EINVAL;
  const long long G = static_cast<long long>(gw) * gh, D = 6 * G;
  std::fill(dense, dense + D * D, 0.0);
  for (long long n = 0; n < G; ++n)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const long long a = n % gw + dx, b = n / gw + dy;
        if (a < 0 || a >= gw || b < 0 || b >= gh) continue;
        const long long nb = b * gw + a;
        const double* B = blocks + (n * 9 + (dy + 1) * 3 + (dx + 1)) * 36;
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) dense[(6 * n + i) * D + 6 * nb + j] = B[6 * i + j];
      }
  return HWF_OK;
}

int hwf_pcg(hwf_ctx* ctx, int gw, int gh, const double* blocks, const double* rhs, int iters,
            double* x, double* trace) {
  return orc::guard(ctx, [&] { orc::backend()->pcg(gw, gh, blocks, rhs, iters, x, trace); });
}
int hwf_schwarz(hwf_ctx* ctx, int gw, int gh, int step, int tile, int boundary, const double* blocks,
                const double* rhs, int patch_iters, int pcg_iters, double* x) {
  return orc::guard(ctx, [&] {
    orc::backend()->schwarz(gw, gh, step, tile, boundary, blocks, rhs, patch_iters, pcg_iters, x);
  });
}
int hwf_gn_level_trace(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta,
                       uint8_t* outlier, double* node_w, const hwf_energy_params* p,
                       const hwf_schedule* sched, int gn_iters, double* eb, double* ea, double* pcg_trace) {
  return orc::guard(ctx, [&] {
    std::vector<double> b, a;
    std::vector<std::vector<double>> tr;
    orc::backend()->gn_level(lv, base, delta, outlier, node_w, p, sched, gn_iters, &b, &a,
                             pcg_trace && sched->subdomain_px <= 0 ? &tr : nullptr);
    if (eb) std::memcpy(eb, b.data(), b.size() * sizeof(double));
    if (ea) std::memcpy(ea, a.data(), a.size() * sizeof(double));
    const size_t row = static_cast<size_t>(sched->pcg_iters) + 1;
    for (size_t it = 0; it < tr.size(); ++it)
      for (size_t k = 0; k < tr[it].size() && k < row; ++k) pcg_trace[it * row + k] = tr[it][k];
  });
}
int hwf_gn_level(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta,
                 uint8_t* outlier, double* node_w, const hwf_energy_params* p,
                 const hwf_schedule* sched, int gn_iters, double* eb, double* ea) {
  return hwf_gn_level_trace(ctx, lv, base, delta, outlier, node_w, p, sched, gn_iters, eb, ea, nullptr);
}
int hwf_occlusion(hwf_ctx* ctx, int w, int h, int step, const double* total, uint8_t* vis4) {
  return orc::guard(ctx, [&] { orc::occlusion(w, h, step, total, vis4); });
}
int hwf_illumination(hwf_ctx* ctx, int w, int h, int step, const double* images[4],
                     const double* total, const uint8_t* vis4, double* hm) {
  return orc::guard(ctx, [&] { orc::illumination(w, h, step, images, total, vis4, hm); });
}
int hwf_prolongate(hwf_ctx* ctx, int wc, int hc, int wf, int hf, int step, const double* total_c,
                   const uint8_t* vis_c, const double* hm_c, double* base_f, uint8_t* vis_f,
                   double* hm_f) {
  return orc::guard(ctx, [&] {
    orc::prolongate(wc, hc, wf, hf, step, total_c, vis_c, hm_c, base_f, vis_f, hm_f);
  });
}

}  // extern "C"
