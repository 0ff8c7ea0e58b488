// oracle/core.cpp — TEST INFRASTRUCTURE ONLY (parity checker; see core.hpp).
// Restatement of /root/reference/proj/src/{image,warp_grid,energy,solver}.cpp
// in plain arrays. Compiled with -ffp-contract=off so that the bit-exact
// stages (pyramid, flow interpolation feeding the occlusion raster) round
// exactly like the reference build and like the device code's explicit
// __dadd_rn/__dmul_rn sequences.
#include "core.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace orc {

// ---------------------------------------------------------------- image.cpp
namespace {
struct CellC {
  int i0;
  double f;
  bool clamped;
};
// image.cpp:19-31
CellC cell_coord(double v, int n) {
  CellC c;
  if (v <= 0.0) {
    c = {0, 0.0, true};
  } else if (v >= n - 1) {
    c = {n >= 2 ? n - 2 : 0, 1.0, true};
  } else {
    const double fl = std::floor(v);
    c = {static_cast<int>(fl), v - fl, false};
  }
  if (n == 1) c = {0, 0.0, true};
  return c;
}
}  // namespace

// image.cpp:37-54
double sample(const Raster& im, double x, double y, double* ddx, double* ddy) {
  const CellC cx = cell_coord(x, im.w), cy = cell_coord(y, im.h);
  const int x1 = std::min(cx.i0 + 1, im.w - 1), y1 = std::min(cy.i0 + 1, im.h - 1);
  const double v00 = im.at(cx.i0, cy.i0), v10 = im.at(x1, cy.i0);
  const double v01 = im.at(cx.i0, y1), v11 = im.at(x1, y1);
  const double fx = cx.f, fy = cy.f;
  const double v = (1 - fx) * (1 - fy) * v00 + fx * (1 - fy) * v10 + (1 - fx) * fy * v01 +
                   fx * fy * v11;
  if (ddx) {
    const double dx = (1 - fy) * (v10 - v00) + fy * (v11 - v01);
    const double dy = (1 - fx) * (v01 - v00) + fx * (v11 - v10);
    *ddx = cx.clamped ? 0.0 : dx;
    *ddy = cy.clamped ? 0.0 : dy;
  }
  return v;
}

// image.cpp:56-77
void pixel_grad(const Raster& im, int x, int y, double g[2]) {
  if (im.w == 1)
    g[0] = 0.0;
  else if (x == 0)
    g[0] = im.at(1, y) - im.at(0, y);
  else if (x == im.w - 1)
    g[0] = im.at(im.w - 1, y) - im.at(im.w - 2, y);
  else
    g[0] = 0.5 * (im.at(x + 1, y) - im.at(x - 1, y));
  if (im.h == 1)
    g[1] = 0.0;
  else if (y == 0)
    g[1] = im.at(x, 1) - im.at(x, 0);
  else if (y == im.h - 1)
    g[1] = im.at(x, im.h - 1) - im.at(x, im.h - 2);
  else
    g[1] = 0.5 * (im.at(x, y + 1) - im.at(x, y - 1));
}

// image.cpp:81-98
void grad_at(const Raster& im, double x, double y, double g[2], double D[2][2]) {
  const CellC cx = cell_coord(x, im.w), cy = cell_coord(y, im.h);
  const int x1 = std::min(cx.i0 + 1, im.w - 1), y1 = std::min(cy.i0 + 1, im.h - 1);
  double g00[2], g10[2], g01[2], g11[2];
  pixel_grad(im, cx.i0, cy.i0, g00);
  pixel_grad(im, x1, cy.i0, g10);
  pixel_grad(im, cx.i0, y1, g01);
  pixel_grad(im, x1, y1, g11);
  const double fx = cx.f, fy = cy.f;
  const double a = (1 - fx) * (1 - fy), b = fx * (1 - fy), c = (1 - fx) * fy, d = fx * fy;
  for (int k = 0; k < 2; ++k) g[k] = a * g00[k] + b * g10[k] + c * g01[k] + d * g11[k];
  if (D) {
    for (int k = 0; k < 2; ++k) {
      const double dgx = (1 - fy) * (g10[k] - g00[k]) + fy * (g11[k] - g01[k]);
      const double dgy = (1 - fx) * (g01[k] - g00[k]) + fx * (g11[k] - g10[k]);
      D[k][0] = cx.clamped ? 0.0 : dgx;
      D[k][1] = cy.clamped ? 0.0 : dgy;
    }
  }
}

// image.cpp:100-122 — 2x2 block mean, fixed order (dy-major), sum/cnt.
void downsample(const Raster& im, std::vector<double>& out, int* ow, int* oh) {
  if (im.w == 0 || im.h == 0) throw std::invalid_argument("downsample of empty image");
  *ow = (im.w + 1) / 2;
  *oh = (im.h + 1) / 2;
  out.assign(static_cast<size_t>(*ow) * *oh, 0.0);
  for (int y = 0; y < *oh; ++y)
    for (int x = 0; x < *ow; ++x) {
      double sum = 0.0;
      int cnt = 0;
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const int sx = 2 * x + dx, sy = 2 * y + dy;
          if (sx < im.w && sy < im.h) {
            sum += im.at(sx, sy);
            ++cnt;
          }
        }
      out[static_cast<size_t>(y) * *ow + x] = sum / cnt;
    }
}

// image.cpp:124-155 — separable normalized Gaussian, radius ceil(3 sigma).
void gaussian_blur(const Raster& im, double sigma, std::vector<double>& out) {
  if (sigma <= 0.0) throw std::invalid_argument("gaussian_blur: sigma must be > 0");
  const int r = static_cast<int>(std::ceil(3.0 * sigma));
  std::vector<double> k(2 * r + 1);
  double sum = 0.0;
  for (int i = -r; i <= r; ++i) {
    k[i + r] = std::exp(-0.5 * (i * i) / (sigma * sigma));
    sum += k[i + r];
  }
  for (auto& v : k) v /= sum;
  std::vector<double> tmp(static_cast<size_t>(im.w) * im.h);
  for (int y = 0; y < im.h; ++y)
    for (int x = 0; x < im.w; ++x) {
      double acc = 0.0;
      for (int i = -r; i <= r; ++i) acc += k[i + r] * im.at_clamped(x + i, y);
      tmp[static_cast<size_t>(y) * im.w + x] = acc;
    }
  const Raster t{im.w, im.h, tmp.data()};
  out.assign(tmp.size(), 0.0);
  for (int y = 0; y < im.h; ++y)
    for (int x = 0; x < im.w; ++x) {
      double acc = 0.0;
      for (int i = -r; i <= r; ++i) acc += k[i + r] * t.at_clamped(x, y + i);
      out[static_cast<size_t>(y) * im.w + x] = acc;
    }
}

// image.cpp:157-175 — lambda_min of the 3x3 structure tensor.
double structure_weight(const Raster& im, int cx, int cy, double delta, double w_max) {
  double a = 0.0, b = 0.0, c = 0.0;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int x = std::clamp(cx + dx, 0, im.w - 1);
      const int y = std::clamp(cy + dy, 0, im.h - 1);
      double g[2];
      pixel_grad(im, x, y, g);
      a += g[0] * g[0];
      b += g[0] * g[1];
      c += g[1] * g[1];
    }
  const double tr = a + c;
  const double disc = std::sqrt(std::max(0.0, 0.25 * (a - c) * (a - c) + b * b));
  const double lmin = 0.5 * tr - disc;
  const double w = 1.0 / (std::max(lmin, 0.0) + delta);
  return std::clamp(w, 1.0, w_max);
}

// ------------------------------------------------------------ warp_grid.cpp
// warp_grid.cpp:8-17
GridDims grid_dims(int image_w, int image_h, int step) {
  if (image_w < 1 || image_h < 1 || step < 1)
    throw std::invalid_argument("WarpGrid: bad dimensions or step");
  GridDims g;
  g.gw = std::max((image_w - 1 + step - 1) / step + 1, 2);
  g.gh = std::max((image_h - 1 + step - 1) / step + 1, 2);
  g.step = step;
  return g;
}

// warp_grid.cpp:35-54
Support support(const GridDims& g, double x, double y) {
  if (!(x >= 0.0 && y >= 0.0 && x <= static_cast<double>(g.gw - 1) * g.step &&
        y <= static_cast<double>(g.gh - 1) * g.step))
    throw std::out_of_range("WarpGrid: position outside lattice");
  const double u = x / g.step, v = y / g.step;
  const int a0 = std::clamp(static_cast<int>(std::floor(u)), 0, g.gw - 2);
  const int b0 = std::clamp(static_cast<int>(std::floor(v)), 0, g.gh - 2);
  const double fu = std::clamp(u - a0, 0.0, 1.0), fv = std::clamp(v - b0, 0.0, 1.0);
  Support s;
  s.node[0] = b0 * g.gw + a0;
  s.node[1] = b0 * g.gw + a0 + 1;
  s.node[2] = (b0 + 1) * g.gw + a0;
  s.node[3] = (b0 + 1) * g.gw + a0 + 1;
  s.wt[0] = (1 - fu) * (1 - fv);
  s.wt[1] = fu * (1 - fv);
  s.wt[2] = (1 - fu) * fv;
  s.wt[3] = fu * fv;
  return s;
}

// warp_grid.cpp:56-65 — accumulation from zero in corner order.
void interpolate(const GridDims& g, const double* nodes6, double x, double y, double out[6]) {
  const Support sp = support(g, x, y);
  for (int c = 0; c < 6; ++c) {
    double acc = 0.0;
    for (int i = 0; i < 4; ++i) acc += sp.wt[i] * nodes6[6 * sp.node[i] + c];
    out[c] = acc;
  }
}

// --------------------------------------------------------------- energy.cpp
namespace {
inline double phi(double x, double eps) { return std::sqrt(x * x + eps * eps); }  // energy.hpp:41
inline double dphi(double x, double eps) { return x / phi(x, eps); }              // energy.hpp:46
double smooth_w(const hwf_energy_params& P, int f) { return f == 0 ? P.w_s : (f == 1 ? P.w_m : P.w_d); }
double mag_w(const hwf_energy_params& P, int f) { return f == 0 ? P.m_s : (f == 1 ? P.m_m : P.m_d); }
}  // namespace

Level make_level(const hwf_level* lv, const hwf_energy_params* P, int threads) {
  Level L;
  L.w = lv->width;
  L.h = lv->height;
  L.g = grid_dims(lv->width, lv->height, lv->grid_step);
  for (int e = 0; e < 4; ++e) {
    L.img[e] = Raster{lv->width, lv->height, lv->images[e]};
    L.illum[e] = lv->illum[e];
  }
  L.total = lv->total;
  L.delta = lv->delta;
  L.vis4 = lv->vis4;
  L.outlier = lv->outlier;
  L.node_w = lv->node_w;
  L.F = lv->fundamental;
  L.P = *P;
  L.threads = threads;
  return L;
}

// energy.cpp:62-129
PixelEval eval_pixel(const Level& L, int px, int py, bool derivs) {
  const hwf_energy_params& P = L.P;
  const int pix = py * L.w + px;
  double fl[6];
  interpolate(L.g, L.total, px, py, fl);
  double val[4], dv[4][2], gv[4][2], dg[4][2][2];
  for (int e = 0; e < 4; ++e) {
    double wx, wy;
    warp_position(px, py, fl, e & 1, e >> 1, &wx, &wy);
    val[e] = sample(L.img[e], wx, wy, derivs ? &dv[e][0] : nullptr, derivs ? &dv[e][1] : nullptr);
    if (L.illum[e]) val[e] += L.illum[e][pix];
    grad_at(L.img[e], wx, wy, gv[e], derivs ? dg[e] : nullptr);
  }
  PixelEval out;
  const bool W = L.outlier[pix] != 0;
  double pc[4] = {0, 0, 0, 0};
  double gc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int k = 0; k < 6; ++k) {
    if (!W || !L.check_visible(pix, k)) continue;
    const int a = kCheckA[k], b = kCheckB[k];
    const double dk = val[a] - val[b];
    out.e_photo += phi(dk, P.eps_huber);
    const double gk0 = gv[a][0] - gv[b][0], gk1 = gv[a][1] - gv[b][1];
    const double gn2 = gk0 * gk0 + gk1 * gk1;
    out.e_grad += phi(gn2, P.eps_huber);
    if (derivs) {
      const double d = dphi(dk, P.eps_huber);
      pc[a] += d;
      pc[b] -= d;
      const double s2 = 2.0 * dphi(gn2, P.eps_huber);
      const double q0 = s2 * gk0, q1 = s2 * gk1;
      gc[a][0] += q0;
      gc[a][1] += q1;
      gc[b][0] -= q0;
      gc[b][1] -= q1;
    }
  }
  out.r_photo = std::sqrt(P.w_photo * out.e_photo);
  out.r_grad = std::sqrt(P.w_grad * out.e_grad);
  if (derivs) {
    if (out.r_photo > 0.0) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      for (int e = 0; e < 4; ++e) {
        if (pc[e] == 0.0) continue;
        const double sc = sgn(e & 1), st = sgn(e >> 1), sg[3] = {sc, st, sc * st};
        const double c0 = pc[e] * dv[e][0], c1 = pc[e] * dv[e][1];
        for (int f = 0; f < 3; ++f) {
          acc[2 * f] += sg[f] * c0;
          acc[2 * f + 1] += sg[f] * c1;
        }
      }
      const double s = P.w_photo / (2.0 * out.r_photo);
      for (int j = 0; j < 6; ++j) out.jp[j] = s * acc[j];
    }
    if (out.r_grad > 0.0) {
      double acc[6] = {0, 0, 0, 0, 0, 0};
      for (int e = 0; e < 4; ++e) {
        if (gc[e][0] == 0.0 && gc[e][1] == 0.0) continue;
        const double sc = sgn(e & 1), st = sgn(e >> 1), sg[3] = {sc, st, sc * st};
        // c = dgrad^T * coef  (energy.cpp:122)
        const double c0 = dg[e][0][0] * gc[e][0] + dg[e][1][0] * gc[e][1];
        const double c1 = dg[e][0][1] * gc[e][0] + dg[e][1][1] * gc[e][1];
        for (int f = 0; f < 3; ++f) {
          acc[2 * f] += sg[f] * c0;
          acc[2 * f + 1] += sg[f] * c1;
        }
      }
      const double s = P.w_grad / (2.0 * out.r_grad);
      for (int j = 0; j < 6; ++j) out.jg[j] = s * acc[j];
    }
  }
  return out;
}

// energy.cpp:131-206
NodeEval eval_node(const Level& L, int node, bool derivs) {
  const hwf_energy_params& P = L.P;
  const int gw = L.g.gw, gh = L.g.gh, a = node % gw, b = node / gw;
  NodeEval out;
  out.right = (a + 1 < gw) ? node + 1 : -1;
  out.down = (b + 1 < gh) ? node + gw : -1;
  const double* T = L.total;
  const double wi = L.node_w[node];
  for (int f = 0; f < 3; ++f) {
    const double wf = smooth_w(P, f);
    const double w = P.w_smooth * P.w_reg * wi * wf;
    for (int c = 0; c < 2; ++c) {
      const int row = 2 * f + c;
      double dr = 0.0, dd = 0.0, q = 0.0;
      if (out.right >= 0) {
        dr = T[6 * node + row] - T[6 * out.right + row];
        q += dr * dr;
      }
      if (out.down >= 0) {
        dd = T[6 * node + row] - T[6 * out.down + row];
        q += dd * dd;
      }
      out.e_smooth += wi * wf * q;
      out.smooth_r[row] = std::sqrt(w * q);
      if (derivs && q > 0.0) {
        const double coef = std::sqrt(w) / std::sqrt(q);
        out.jc[row] = coef * (dr + dd);
        out.jr[row] = -coef * dr;
        out.jd[row] = -coef * dd;
      }
    }
  }
  if (P.w_epi > 0.0) {  // energy.cpp:169-192 with warp_grid.cpp:95-112 positions
    if (!L.F) throw std::invalid_argument("epipolar term enabled without a fundamental matrix");
    const double* F = L.F;
    const double gx = static_cast<double>(a) * L.g.step, gy = static_cast<double>(b) * L.g.step;
    const double* n6 = T + 6 * node;
    const double s0 = n6[0], s1 = n6[1], m0 = n6[2], m1 = n6[3], d0 = n6[4], d1 = n6[5];
    const double pos[4][3] = {{gx - s0 - m0 + d0, gy - s1 - m1 + d1, 1.0},
                              {gx + s0 - m0 - d0, gy + s1 - m1 - d1, 1.0},
                              {gx - s0 + m0 - d0, gy - s1 + m1 - d1, 1.0},
                              {gx + s0 + m0 + d0, gy + s1 + m1 + d1, 1.0}};
    const double sw = std::sqrt(P.w_epi * P.w_reg);
    for (int t = 0; t < 2; ++t) {
      const double* l = pos[2 * t];
      const double* r = pos[2 * t + 1];
      double Fr[3], Ftl[3];
      for (int i = 0; i < 3; ++i) {
        Fr[i] = F[3 * i] * r[0] + F[3 * i + 1] * r[1] + F[3 * i + 2] * r[2];
        Ftl[i] = F[i] * l[0] + F[3 + i] * l[1] + F[6 + i] * l[2];
      }
      const double e = l[0] * Fr[0] + l[1] * Fr[1] + l[2] * Fr[2];
      out.e_epi += e * e;
      out.epi_r[t] = sw * e;
      if (derivs) {
        const double st = sgn(t);
        const double u0 = Fr[0], u1 = Fr[1], v0 = Ftl[0], v1 = Ftl[1];
        const double j[6] = {v0 - u0, v1 - u1, st * (u0 + v0), st * (u1 + v1), st * (v0 - u0),
                             st * (v1 - u1)};
        for (int c = 0; c < 6; ++c) out.epi_j[t][c] = sw * j[c];
      }
    }
  }
  const double* D = L.delta;
  for (int f = 0; f < 3; ++f) {
    const double mf = mag_w(P, f);
    const double sw = std::sqrt(P.w_mag * P.w_reg * mf);
    const double x = D[6 * node + 2 * f], y = D[6 * node + 2 * f + 1];
    out.e_mag += mf * (x * x + y * y);
    out.mag_r[2 * f] = sw * x;
    out.mag_r[2 * f + 1] = sw * y;
    out.mag_j[2 * f] = sw;
    out.mag_j[2 * f + 1] = sw;
  }
  return out;
}

// energy.cpp:208-251: stacked residuals (photo N, grad N, smooth 6G, epi 2G,
// mag 6G) and the unweighted breakdown; serial sums in index order.
hwf_energy energy(const Level& L, double* R) {
  const int N = L.N(), G = L.G();
  std::vector<double> ep(N), eg(N), rp(N), rg(N);
#pragma omp parallel for num_threads(L.threads) schedule(static)
  for (int pix = 0; pix < N; ++pix) {
    const PixelEval ev = eval_pixel(L, pix % L.w, pix / L.w, false);
    ep[pix] = ev.e_photo;
    eg[pix] = ev.e_grad;
    rp[pix] = ev.r_photo;
    rg[pix] = ev.r_grad;
  }
  hwf_energy out{};
  out.residual_count = 2LL * N + 14LL * G;
  double tot = 0.0;
  for (int i = 0; i < N; ++i) {
    out.photo += ep[i];
    out.grad += eg[i];
    tot += rp[i] * rp[i] + rg[i] * rg[i];
    if (R) {
      R[i] = rp[i];
      R[N + i] = rg[i];
    }
  }
  for (int k = 0; k < G; ++k) {
    const NodeEval ev = eval_node(L, k, false);
    out.smooth += ev.e_smooth;
    out.epi += ev.e_epi;
    out.mag += ev.e_mag;
    for (int j = 0; j < 6; ++j) tot += ev.smooth_r[j] * ev.smooth_r[j] + ev.mag_r[j] * ev.mag_r[j];
    tot += ev.epi_r[0] * ev.epi_r[0] + ev.epi_r[1] * ev.epi_r[1];
    if (R) {
      for (int j = 0; j < 6; ++j) R[2 * N + 6 * k + j] = ev.smooth_r[j];
      for (int t = 0; t < 2; ++t) R[2 * N + 6 * G + 2 * k + t] = ev.epi_r[t];
      for (int j = 0; j < 6; ++j) R[2 * N + 8 * G + 6 * k + j] = ev.mag_r[j];
    }
  }
  if (!std::isfinite(tot)) throw Divergence("non-finite residuals in energy assembly");
  out.total = tot;
  return out;
}

// energy.cpp:253-271
void refresh_outlier(const Level& L, uint8_t* outlier) {
  const int N = L.N();
#pragma omp parallel for num_threads(L.threads) schedule(static)
  for (int pix = 0; pix < N; ++pix) {
    const int px = pix % L.w, py = pix / L.w;
    double fl[6];
    interpolate(L.g, L.total, px, py, fl);
    double val[4];
    for (int e = 0; e < 4; ++e) {
      double wx, wy;
      warp_position(px, py, fl, e & 1, e >> 1, &wx, &wy);
      val[e] = sample(L.img[e], wx, wy, nullptr, nullptr) + (L.illum[e] ? L.illum[e][pix] : 0.0);
    }
    double sum = 0.0;
    int cnt = 0;
    for (int k = 0; k < 6; ++k) {
      if (!L.check_visible(pix, k)) continue;
      sum += std::abs(val[kCheckA[k]] - val[kCheckB[k]]);
      ++cnt;
    }
    outlier[pix] = (cnt == 0 || sum / cnt < L.P.eps_color) ? 1 : 0;
  }
}

// energy.cpp:273-293 — w_i from the halfway image's structure tensor.
void refresh_node_w(const Level& L, double* node_w) {
  const int N = L.N();
  std::vector<double> half(N);
#pragma omp parallel for num_threads(L.threads) schedule(static)
  for (int pix = 0; pix < N; ++pix) {
    const int px = pix % L.w, py = pix / L.w;
    double fl[6];
    interpolate(L.g, L.total, px, py, fl);
    double acc = 0.0;
    for (int e = 0; e < 4; ++e) {
      double wx, wy;
      warp_position(px, py, fl, e & 1, e >> 1, &wx, &wy);
      acc += sample(L.img[e], wx, wy, nullptr, nullptr);
      if (L.illum[e]) acc += L.illum[e][pix];
    }
    half[pix] = 0.25 * acc;
  }
  const Raster hr{L.w, L.h, half.data()};
  for (int k = 0; k < L.G(); ++k) {
    const int cx = std::min((k % L.g.gw) * L.g.step, L.w - 1);
    const int cy = std::min((k / L.g.gw) * L.g.step, L.h - 1);
    node_w[k] = structure_weight(hr, cx, cy);
  }
}

// --------------------------------------------------------------- solver.cpp
int System::neighbor(int n, int dx, int dy) const {  // solver.cpp:41-46
  const int a = n % gw + dx, b = n / gw + dy;
  if (a < 0 || a >= gw || b < 0 || b >= gh) return -1;
  return b * gw + a;
}

// solver.cpp:48-62 — 9-slot block SpMV.
void System::apply(const std::vector<double>& x, std::vector<double>& y) const {
  y.assign(6 * static_cast<size_t>(G()), 0.0);
  for (int n = 0; n < G(); ++n) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int nb = neighbor(n, dx, dy);
        if (nb < 0) continue;
        const double* B = block(n, slot(dx, dy));
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) acc[i] += B[6 * i + j] * x[6 * nb + j];
      }
    for (int i = 0; i < 6; ++i) y[6 * n + i] = acc[i];
  }
}

// solver.cpp:64-78 — inverted 2x2 diagonal field blocks, identity if singular.
void System::build_preconditioner() {
  pre.assign(static_cast<size_t>(G()) * 12, 0.0);
  for (int n = 0; n < G(); ++n) {
    const double* D = block(n, slot(0, 0));
    for (int f = 0; f < 3; ++f) {
      double* M = &pre[(static_cast<size_t>(n) * 3 + f) * 4];
      const double m00 = D[6 * (2 * f) + 2 * f], m01 = D[6 * (2 * f) + 2 * f + 1];
      const double m10 = D[6 * (2 * f + 1) + 2 * f], m11 = D[6 * (2 * f + 1) + 2 * f + 1];
      const double det = m00 * m11 - m01 * m10;
      if (std::abs(det) > 1e-300) {
        M[0] = m11 / det;
        M[1] = -m01 / det;
        M[2] = -m10 / det;
        M[3] = m00 / det;
      } else {
        M[0] = 1.0;
        M[1] = 0.0;
        M[2] = 0.0;
        M[3] = 1.0;
      }
    }
  }
}

// solver.cpp:80-87
void System::precondition(const std::vector<double>& r, std::vector<double>& z) const {
  z.assign(r.size(), 0.0);
  for (int n = 0; n < G(); ++n)
    for (int f = 0; f < 3; ++f) {
      const double* M = &pre[(static_cast<size_t>(n) * 3 + f) * 4];
      const size_t o = 6 * static_cast<size_t>(n) + 2 * f;
      z[o] = M[0] * r[o] + M[1] * r[o + 1];
      z[o + 1] = M[2] * r[o] + M[3] * r[o + 1];
    }
}

namespace {
inline bool forward_offset(int dx, int dy) { return dy > 0 || (dy == 0 && dx >= 0); }  // solver.cpp:15
inline void cell_range(int a0, int step, int extent, int cells, int* lo, int* hi) {     // solver.cpp:21
  *lo = a0 * step;
  *hi = (a0 == cells - 1) ? extent : std::min(extent, (a0 + 1) * step);
}
inline void mask6(double* v, uint32_t active) {  // solver.cpp:27-31
  for (int f = 0; f < 3; ++f)
    if (!((active >> f) & 1)) v[2 * f] = v[2 * f + 1] = 0.0;
}
}  // namespace

// solver.cpp:247-314 (assemble_jacobian): residual rows photo [0, N), grad [N, 2N), smooth [2N, 2N+6G),
// epi [2N+6G, 2N+8G), mag [2N+8G, 2N+14G); entries in the reference's loop order.
void assemble_jacobian(const Level& L, uint32_t active, int negate_field, std::vector<double>& R,
                       std::vector<JacTriplet>& out) {
  const int N = L.N(), G = L.G();
  R.assign(static_cast<size_t>(2) * N + 14 * static_cast<size_t>(G), 0.0);
  out.clear();
  auto hooks = [&](double* v) {
    mask6(v, active);
    if (negate_field >= 0) {
      v[2 * negate_field] *= -1.0;
      v[2 * negate_field + 1] *= -1.0;
    }
  };
  for (int pix = 0; pix < N; ++pix) {
    const int px = pix % L.w, py = pix / L.w;
    const PixelEval ev = eval_pixel(L, px, py, true);
    R[pix] = ev.r_photo;
    R[N + pix] = ev.r_grad;
    const Support sp = support(L.g, px, py);
    double jp[6], jg[6];
    std::copy(ev.jp, ev.jp + 6, jp);
    std::copy(ev.jg, ev.jg + 6, jg);
    hooks(jp);
    hooks(jg);
    for (int i = 0; i < 4; ++i) {
      if (sp.wt[i] == 0.0) continue;
      for (int j = 0; j < 6; ++j) {
        const int col = 6 * sp.node[i] + j;
        if (jp[j] != 0.0) out.push_back({pix, col, sp.wt[i] * jp[j]});
        if (jg[j] != 0.0) out.push_back({N + pix, col, sp.wt[i] * jg[j]});
      }
    }
  }
  for (int n = 0; n < G; ++n) {
    const NodeEval ev = eval_node(L, n, true);
    for (int row = 0; row < 6; ++row) {
      const int r = 2 * N + 6 * n + row;
      R[r] = ev.smooth_r[row];
      const int f = row / 2;
      if (!((active >> f) & 1)) continue;
      const double sgn = f == negate_field ? -1.0 : 1.0;
      if (ev.jc[row] != 0.0) out.push_back({r, 6 * n + row, sgn * ev.jc[row]});
      if (ev.right >= 0 && ev.jr[row] != 0.0) out.push_back({r, 6 * ev.right + row, sgn * ev.jr[row]});
      if (ev.down >= 0 && ev.jd[row] != 0.0) out.push_back({r, 6 * ev.down + row, sgn * ev.jd[row]});
    }
    for (int t = 0; t < 2; ++t) {
      const int r = 2 * N + 6 * G + 2 * n + t;
      R[r] = ev.epi_r[t];
      double j[6];
      std::copy(ev.epi_j[t], ev.epi_j[t] + 6, j);
      hooks(j);
      for (int c = 0; c < 6; ++c)
        if (j[c] != 0.0) out.push_back({r, 6 * n + c, j[c]});
    }
    for (int row = 0; row < 6; ++row) {
      const int r = 2 * N + 8 * G + 6 * n + row;
      R[r] = ev.mag_r[row];
      const int f = row / 2;
      if (!((active >> f) & 1)) continue;
      const double sgn = f == negate_field ? -1.0 : 1.0;
      if (ev.mag_j[row] != 0.0) out.push_back({r, 6 * n + row, sgn * ev.mag_j[row]});
    }
  }
}

// solver.cpp:100-245
System build_normal_system(const Level& L, uint32_t active, double lm_lambda) {
  const int gw = L.g.gw, gh = L.g.gh, step = L.g.step, N = L.N(), G = L.G();
  System S;
  S.gw = gw;
  S.gh = gh;
  S.blk.assign(static_cast<size_t>(G) * 9 * 36, 0.0);
  S.rhs.assign(6 * static_cast<size_t>(G), 0.0);
  struct PJ {
    double jp[6], jg[6], rp, rg;
  };
  std::vector<PJ> pj(N);
  int bad = -1;
#pragma omp parallel for num_threads(L.threads) schedule(static)
  for (int pix = 0; pix < N; ++pix) {  // pass 1 (solver.cpp:114-121)
    const PixelEval ev = eval_pixel(L, pix % L.w, pix / L.w, true);
    bool fin = true;
    for (int j = 0; j < 6; ++j) fin = fin && std::isfinite(ev.jp[j]) && std::isfinite(ev.jg[j]);
    if (!fin) {
#pragma omp critical
      bad = (bad < 0 || pix < bad) ? pix : bad;
    }
    PJ& p = pj[pix];
    for (int j = 0; j < 6; ++j) {
      p.jp[j] = ev.jp[j];
      p.jg[j] = ev.jg[j];
    }
    mask6(p.jp, active);
    mask6(p.jg, active);
    p.rp = ev.r_photo;
    p.rg = ev.r_grad;
  }
  if (bad >= 0) throw Divergence("non-finite Jacobian at pixel residual " + std::to_string(bad));

  const int cx = gw - 1, cy = gh - 1;
#pragma omp parallel for num_threads(L.threads) schedule(static)
  for (int n = 0; n < G; ++n) {  // pass 2 gather (solver.cpp:126-160)
    const int a = n % gw, b = n / gw;
    double racc[6] = {0, 0, 0, 0, 0, 0};
    for (int b0 = std::max(0, b - 1); b0 <= std::min(b, cy - 1); ++b0)
      for (int a0 = std::max(0, a - 1); a0 <= std::min(a, cx - 1); ++a0) {
        int xl, xh, yl, yh;
        cell_range(a0, step, L.w, cx, &xl, &xh);
        cell_range(b0, step, L.h, cy, &yl, &yh);
        const int corner = (a - a0) + 2 * (b - b0);
        for (int py = yl; py < yh; ++py)
          for (int px = xl; px < xh; ++px) {
            const double fu = std::clamp(static_cast<double>(px) / step - a0, 0.0, 1.0);
            const double fv = std::clamp(static_cast<double>(py) / step - b0, 0.0, 1.0);
            const double al[4] = {(1 - fu) * (1 - fv), fu * (1 - fv), (1 - fu) * fv, fu * fv};
            const double wn = al[corner];
            if (wn == 0.0) continue;
            const PJ& p = pj[static_cast<size_t>(py) * L.w + px];
            for (int i = 0; i < 6; ++i) racc[i] -= wn * (p.jp[i] * p.rp + p.jg[i] * p.rg);
            double outer[36];
            for (int i = 0; i < 6; ++i)
              for (int j = 0; j < 6; ++j) outer[6 * i + j] = p.jp[i] * p.jp[j] + p.jg[i] * p.jg[j];
            for (int cj = 0; cj < 4; ++cj) {
              const int da = (a0 + cj % 2) - a, db = (b0 + cj / 2) - b;
              if (!forward_offset(da, db)) continue;
              double* B = S.block(n, slot(da, db));
              const double s = wn * al[cj];
              for (int i = 0; i < 36; ++i) B[i] += s * outer[i];
            }
          }
      }
    for (int i = 0; i < 6; ++i) S.rhs[6 * n + i] = racc[i];
  }

  // Regularizers (solver.cpp:164-211), forward placement then mirrored.
  auto add_pair = [&](int ni, int ci, int nj, int cj, double v) {
    const int da = nj % gw - ni % gw, db = nj / gw - ni / gw;
    if (forward_offset(da, db))
      S.block(ni, slot(da, db))[6 * ci + cj] += v;
    else
      S.block(nj, slot(-da, -db))[6 * cj + ci] += v;
  };
  for (int n = 0; n < G; ++n) {
    const NodeEval ev = eval_node(L, n, true);
    for (int row = 0; row < 6; ++row) {
      if (!((active >> (row / 2)) & 1)) continue;
      const int sn[3] = {n, ev.right, ev.down};
      const double sc[3] = {ev.jc[row], ev.jr[row], ev.jd[row]};
      for (int i = 0; i < 3; ++i) {
        if (sn[i] < 0 || sc[i] == 0.0) continue;
        S.rhs[6 * sn[i] + row] -= sc[i] * ev.smooth_r[row];
        for (int j = 0; j < 3; ++j) {
          if (sn[j] < 0 || sc[j] == 0.0) continue;
          if (sn[j] < sn[i]) continue;
          if (sn[i] == sn[j])
            S.block(sn[i], slot(0, 0))[6 * row + row] += sc[i] * sc[j];
          else
            add_pair(sn[i], row, sn[j], row, sc[i] * sc[j]);
        }
      }
    }
    for (int t = 0; t < 2; ++t) {
      if (ev.epi_r[t] == 0.0 && L.P.w_epi == 0.0) continue;
      double j[6];
      for (int c = 0; c < 6; ++c) j[c] = ev.epi_j[t][c];
      mask6(j, active);
      double* B = S.block(n, slot(0, 0));
      for (int r = 0; r < 6; ++r) {
        S.rhs[6 * n + r] -= j[r] * ev.epi_r[t];
        for (int c = 0; c < 6; ++c) B[6 * r + c] += j[r] * j[c];
      }
    }
    for (int row = 0; row < 6; ++row) {
      if (!((active >> (row / 2)) & 1)) continue;
      S.rhs[6 * n + row] -= ev.mag_j[row] * ev.mag_r[row];
      S.block(n, slot(0, 0))[6 * row + row] += ev.mag_j[row] * ev.mag_j[row];
    }
  }
  // Pin inactive fields / LM boost (solver.cpp:213-226).
  for (int n = 0; n < G; ++n) {
    double* D = S.block(n, slot(0, 0));
    for (int f = 0; f < 3; ++f) {
      if (!((active >> f) & 1)) {
        D[6 * (2 * f) + 2 * f] = 1.0;
        D[6 * (2 * f) + 2 * f + 1] = 0.0;
        D[6 * (2 * f + 1) + 2 * f] = 0.0;
        D[6 * (2 * f + 1) + 2 * f + 1] = 1.0;
        S.rhs[6 * n + 2 * f] = S.rhs[6 * n + 2 * f + 1] = 0.0;
      } else if (lm_lambda > 0.0) {
        for (int c = 0; c < 2; ++c) D[6 * (2 * f + c) + 2 * f + c] *= 1.0 + lm_lambda;
      }
    }
  }
  // Mirror backward slots (solver.cpp:228-241).
  for (int n = 0; n < G; ++n)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        if (forward_offset(dx, dy)) continue;
        const int nb = S.neighbor(n, dx, dy);
        if (nb < 0) continue;
        double* B = S.block(n, slot(dx, dy));
        const double* Fb = S.block(nb, slot(-dx, -dy));
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) B[6 * i + j] = Fb[6 * j + i];
      }
  S.build_preconditioner();
  return S;
}

namespace {
double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
using Op = std::function<void(const std::vector<double>&, std::vector<double>&)>;
// solver.cpp:320-361
std::vector<double> pcg_impl(const Op& apply, const Op& precond, const std::vector<double>& b,
                             const std::vector<double>& x0, int iters,
                             std::vector<double>* trace) {
  std::vector<double> x = x0, r = b, tmp, z, p;
  bool zero = true;
  for (double v : x) zero = zero && v == 0.0;
  if (!zero) {
    apply(x, tmp);
    for (size_t i = 0; i < r.size(); ++i) r[i] -= tmp[i];
  }
  if (trace) trace->push_back(std::sqrt(dot(r, r)));
  precond(r, z);
  double rz = dot(r, z);
  const double rz0 = std::abs(rz);
  if (rz0 == 0.0) {
    if (trace)
      for (int it = 0; it < iters; ++it) trace->push_back(0.0);
    return x;
  }
  p = z;
  for (int it = 0; it < iters; ++it) {
    apply(p, tmp);
    const double pAp = dot(p, tmp);
    if (pAp <= 0.0) throw Divergence("PCG: non-positive curvature, system not SPD");
    const double alpha = rz / pAp;
    for (size_t i = 0; i < x.size(); ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * tmp[i];
    }
    if (trace) trace->push_back(std::sqrt(dot(r, r)));
    precond(r, z);
    const double rzn = dot(r, z);
    if (std::abs(rzn) > 100.0 * rz0)
      throw Divergence("PCG: preconditioned residual grew by more than 10x");
    const double beta = rzn / rz;
    rz = rzn;
    for (size_t i = 0; i < p.size(); ++i) p[i] = z[i] + beta * p[i];
  }
  return x;
}
}  // namespace

// solver.cpp:365-380
std::vector<double> pcg_solve(const System& S, int iters, std::vector<double>* trace) {
  return pcg_impl([&](const std::vector<double>& x, std::vector<double>& y) { S.apply(x, y); },
                  [&](const std::vector<double>& r, std::vector<double>& z) { S.precondition(r, z); },
                  S.rhs, std::vector<double>(S.rhs.size(), 0.0), iters, trace);
}

// solver.cpp:382-412 (the boundary ring is built but never read by the
// reference solver, so it is not restated).
std::vector<Subdomain> build_subdomains(int gw, int gh, int step, int tile_px) {
  if (tile_px <= 0) throw std::invalid_argument("subdomain tile must be > 0");
  const int tx_n = ((gw - 1) * step) / tile_px + 1, ty_n = ((gh - 1) * step) / tile_px + 1;
  std::vector<Subdomain> out(static_cast<size_t>(tx_n) * ty_n);
  for (int b = 0; b < gh; ++b)
    for (int a = 0; a < gw; ++a)
      out[static_cast<size_t>((b * step) / tile_px) * tx_n + (a * step) / tile_px].interior.push_back(
          b * gw + a);
  std::vector<Subdomain> kept;
  for (auto& s : out)
    if (!s.interior.empty()) kept.push_back(std::move(s));
  return kept;
}

// One sweep of schwarz_iterate (solver.cpp:430-480) over the subdomains s with take[s]
// (all when take is null): each local PCG is warm-started from pub, with its off-subdomain
// neighbours frozen at pub; the local solutions go to next.
void schwarz_sweep(const System& S, const std::vector<Subdomain>& subs, const std::vector<int>& owner,
                   const std::vector<int>& loc, const std::vector<double>& pub, std::vector<double>& next,
                   int pcg_iters, const std::vector<char>* take) {
  for (size_t s = 0; s < subs.size(); ++s) {
    if (take && !(*take)[s]) continue;
    const auto& in = subs[s].interior;
    const int ln = static_cast<int>(in.size());
    std::vector<double> b(6 * ln), x0(6 * ln);
    for (int i = 0; i < ln; ++i) {
      const int g = in[i];
      double bi[6];
      for (int c = 0; c < 6; ++c) bi[c] = S.rhs[6 * g + c];
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (dx == 0 && dy == 0) continue;
          const int nb = S.neighbor(g, dx, dy);
          if (nb < 0 || owner[nb] == static_cast<int>(s)) continue;
          const double* B = S.block(g, slot(dx, dy));
          for (int r = 0; r < 6; ++r)
            for (int c = 0; c < 6; ++c) bi[r] -= B[6 * r + c] * pub[6 * nb + c];
        }
      for (int c = 0; c < 6; ++c) {
        b[6 * i + c] = bi[c];
        x0[6 * i + c] = pub[6 * g + c];
      }
    }
    auto apply = [&](const std::vector<double>& x, std::vector<double>& y) {
      y.assign(6 * ln, 0.0);
      for (int i = 0; i < ln; ++i) {
        const int g = in[i];
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int nb = S.neighbor(g, dx, dy);
            if (nb < 0 || owner[nb] != static_cast<int>(s)) continue;
            const double* B = S.block(g, slot(dx, dy));
            for (int r = 0; r < 6; ++r)
              for (int c = 0; c < 6; ++c) y[6 * i + r] += B[6 * r + c] * x[6 * loc[nb] + c];
          }
      }
    };
    auto precond = [&](const std::vector<double>& r, std::vector<double>& z) {
      z.assign(6 * ln, 0.0);
      for (int i = 0; i < ln; ++i)
        for (int f = 0; f < 3; ++f) {
          const double* M = &S.pre[(static_cast<size_t>(in[i]) * 3 + f) * 4];
          const int o = 6 * i + 2 * f;
          z[o] = M[0] * r[o] + M[1] * r[o + 1];
          z[o + 1] = M[2] * r[o] + M[3] * r[o + 1];
        }
    };
    const std::vector<double> xl = pcg_impl(apply, precond, b, x0, pcg_iters, nullptr);
    for (int i = 0; i < ln; ++i)
      for (int c = 0; c < 6; ++c) next[6 * in[i] + c] = xl[6 * i + c];
  }
}

void subdomain_owner(const std::vector<Subdomain>& subs, int G, std::vector<int>& owner, std::vector<int>& loc) {
  owner.assign(G, -1);
  loc.assign(G, 0);
  for (size_t s = 0; s < subs.size(); ++s)
    for (size_t i = 0; i < subs[s].interior.size(); ++i) {
      owner[subs[s].interior[i]] = static_cast<int>(s);
      loc[subs[s].interior[i]] = static_cast<int>(i);
    }
}

// solver.cpp:414-482 — non-overlapping block-Jacobi sweeps with warm start.
std::vector<double> schwarz(const System& S, const std::vector<Subdomain>& subs, int patch_iters,
                            int pcg_iters) {
  const int G = S.G();
  std::vector<double> pub(6 * static_cast<size_t>(G), 0.0);
  std::vector<int> owner, loc;
  subdomain_owner(subs, G, owner, loc);
  for (int sweep = 0; sweep < patch_iters; ++sweep) {
    std::vector<double> next = pub;
    schwarz_sweep(S, subs, owner, loc, pub, next, pcg_iters, nullptr);
    pub = next;
  }
  return pub;
}

// solver.cpp:484-532
void gauss_newton(Level L, const double* base, double* delta, uint8_t* outlier, double* node_w,
                  const hwf_schedule& S, int gn_iters, std::vector<double>* e_before,
                  std::vector<double>* e_after, std::vector<std::vector<double>>* pcg_trace) {
  const int G = L.G();
  std::vector<Subdomain> subs;
  if (S.subdomain_px > 0) subs = build_subdomains(L.g.gw, L.g.gh, L.g.step, S.subdomain_px);
  std::vector<double> total(6 * static_cast<size_t>(G));
  for (int it = 0; it < gn_iters; ++it) {
    for (size_t i = 0; i < total.size(); ++i) total[i] = base[i] + delta[i];
    L.total = total.data();
    L.delta = delta;
    L.outlier = outlier;
    L.node_w = node_w;
    refresh_outlier(L, outlier);
    refresh_node_w(L, node_w);
    const double eb = energy(L, nullptr).total;
    if (e_before) e_before->push_back(eb);
    const System sys = build_normal_system(L, S.active_fields, S.lm_lambda);
    std::vector<double> step;
    if (S.subdomain_px > 0) {
      step = schwarz(sys, subs, S.patch_iters, S.pcg_iters);
    } else {  // solver.cpp:508-513
      std::vector<double> trace;
      step = pcg_solve(sys, S.pcg_iters, pcg_trace ? &trace : nullptr);
      if (pcg_trace) pcg_trace->push_back(std::move(trace));
    }
    for (double v : step)
      if (!std::isfinite(v)) throw Divergence("non-finite Gauss-Newton update");
    for (int n = 0; n < G; ++n)
      for (int f = 0; f < 3; ++f)
        if ((S.active_fields >> f) & 1) {
          delta[6 * n + 2 * f] += step[6 * n + 2 * f];
          delta[6 * n + 2 * f + 1] += step[6 * n + 2 * f + 1];
        }
    for (size_t i = 0; i < total.size(); ++i) total[i] = base[i] + delta[i];
    const double ea = energy(L, nullptr).total;
    if (!std::isfinite(ea)) throw Divergence("non-finite energy after Gauss-Newton step");
    if (e_after) e_after->push_back(ea);
  }
}

}  // namespace orc
