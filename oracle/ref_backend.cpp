// oracle/ref_backend.cpp — TEST INFRASTRUCTURE ONLY. Backend over the
// reference's own shipped sources (/root/reference/proj/src/*.cpp, compiled
// verbatim against oracle/eigen_shim by oracle/Makefile into oracle/_ref/).
// Only glue lives here: copying hwf_* buffers into the reference's value
// types and back, and mapping hwflow::SolverDivergence to orc::Divergence.
#include <cstring>

#include "backend.hpp"
#include "hwflow/energy.hpp"
#include "hwflow/image.hpp"
#include "hwflow/solver.hpp"
#include "hwflow/warp_grid.hpp"

namespace orc {
namespace {

using hwflow::Image;
using hwflow::WarpGrid;

Image to_image(int w, int h, const double* p) {
  Image im(w, h);
  std::memcpy(im.data().data(), p, sizeof(double) * static_cast<size_t>(w) * h);
  return im;
}

WarpGrid to_grid(int w, int h, int step, const double* v6) {
  WarpGrid g(w, h, step);
  if (v6)
    for (int k = 0; k < g.node_count(); ++k)
      for (int f = 0; f < 3; ++f) g.node(f, k) = hwflow::Vec2(v6[6 * k + 2 * f], v6[6 * k + 2 * f + 1]);
  return g;
}

void from_grid(const WarpGrid& g, double* v6) {
  for (int k = 0; k < g.node_count(); ++k)
    for (int f = 0; f < 3; ++f) {
      v6[6 * k + 2 * f] = g.node(f, k).x();
      v6[6 * k + 2 * f + 1] = g.node(f, k).y();
    }
}

hwflow::EnergyParams to_params(const hwf_energy_params* P) {
  hwflow::EnergyParams p;
  p.w_reg = P->w_reg;
  p.w_photo = P->w_photo;
  p.w_grad = P->w_grad;
  p.w_epi = P->w_epi;
  p.w_smooth = P->w_smooth;
  p.w_mag = P->w_mag;
  p.w_s = P->w_s;
  p.w_m = P->w_m;
  p.w_d = P->w_d;
  p.m_s = P->m_s;
  p.m_m = P->m_m;
  p.m_d = P->m_d;
  p.eps_huber = P->eps_huber;
  p.eps_color = P->eps_color;
  return p;
}

// Owns the value types an EnergyContext points at.
struct RefLevel {
  std::vector<Image> img, ill;
  WarpGrid total, delta;
  hwflow::PixelWeights wts;
  hwflow::Mat3 F = hwflow::Mat3::Zero();
  hwflow::EnergyContext ctx;
  RefLevel(const hwf_level* lv, const hwf_energy_params* P, int threads) {
    const int w = lv->width, h = lv->height, N = w * h;
    for (int e = 0; e < 4; ++e) img.push_back(to_image(w, h, lv->images[e]));
    for (int e = 0; e < 4; ++e) ill.push_back(lv->illum[e] ? to_image(w, h, lv->illum[e]) : Image());
    total = to_grid(w, h, lv->grid_step, lv->total);
    delta = to_grid(w, h, lv->grid_step, lv->delta);
    const int G = total.node_count();
    wts.init_all_visible(N, G);
    if (lv->vis4) wts.vis4.assign(lv->vis4, lv->vis4 + N);
    if (lv->outlier) wts.outlier.assign(lv->outlier, lv->outlier + N);
    if (lv->node_w) wts.node_w.assign(lv->node_w, lv->node_w + G);
    if (lv->fundamental)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) F(i, j) = lv->fundamental[3 * i + j];
    for (int e = 0; e < 4; ++e) {
      ctx.images[e] = &img[e];
      ctx.illum[e] = lv->illum[e] ? &ill[e] : nullptr;
    }
    ctx.total = &total;
    ctx.delta = &delta;
    ctx.weights = &wts;
    ctx.fundamental = lv->fundamental ? &F : nullptr;
    ctx.params = to_params(P);
    ctx.width = w;
    ctx.height = h;
    ctx.threads = threads;
  }
};

hwflow::NormalSystem load_system(int gw, int gh, const double* blocks, const double* rhs) {
  hwflow::NormalSystem S(gw, gh);
  for (int n = 0; n < gw * gh; ++n)
    for (int s = 0; s < 9; ++s) {
      hwflow::Mat6& B = S.block(n, s);
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) B(i, j) = blocks[(static_cast<size_t>(n) * 9 + s) * 36 + 6 * i + j];
    }
  for (int i = 0; i < 6 * gw * gh; ++i) S.rhs()(i) = rhs[i];
  S.build_preconditioner();
  return S;
}

template <class Fn>
auto guard(Fn&& fn) {
  try {
    return fn();
  } catch (const hwflow::SolverDivergence& e) {
    throw Divergence(e.what());
  }
}

struct Ref final : Backend {
  const char* name() const override { return "reference"; }
  void pyramid(const std::vector<std::vector<double>>& images, int w, int h, int levels,
               double* out) override {
    std::vector<hwflow::Pyramid> pyr;
    for (int e = 0; e < 4; ++e) pyr.push_back(hwflow::build_pyramid(to_image(w, h, images[e].data()), levels));
    size_t off = 0;
    for (int l = 0; l < levels; ++l)
      for (int e = 0; e < 4; ++e) {
        const auto& d = pyr[e].levels[l].data();
        std::memcpy(out + off, d.data(), d.size() * sizeof(double));
        off += d.size();
      }
  }
  hwf_energy eval_energy(const hwf_level* lv, const hwf_energy_params* P, double* R,
                         int threads) override {
    return guard([&] {
      RefLevel L(lv, P, threads);
      const auto br = hwflow::energy_breakdown(L.ctx);
      const Eigen::VectorXd r = hwflow::assemble_residuals(L.ctx);
      hwf_energy out{};
      out.photo = br.photo;
      out.grad = br.grad;
      out.smooth = br.smooth;
      out.epi = br.epi;
      out.mag = br.mag;
      out.total = r.squaredNorm();
      out.residual_count = L.ctx.residual_count();
      if (R) std::memcpy(R, r.data(), sizeof(double) * r.size());
      return out;
    });
  }
  void refresh(const hwf_level* lv, const hwf_energy_params* P, uint8_t* outlier, double* node_w,
               int threads) override {
    RefLevel L(lv, P, threads);
    hwflow::refresh_outlier_bits(L.ctx, L.wts);
    hwflow::refresh_feature_weights(L.ctx, L.wts);
    std::memcpy(outlier, L.wts.outlier.data(), L.wts.outlier.size());
    std::memcpy(node_w, L.wts.node_w.data(), L.wts.node_w.size() * sizeof(double));
  }
  void jacobian(const hwf_level* lv, const hwf_energy_params* P, uint32_t active, int negate_field,
                std::vector<double>& R, std::vector<JacEntry>& entries, int threads) override {
    guard([&] {
      RefLevel L(lv, P, threads);
      const hwflow::JacobianRows J = hwflow::assemble_jacobian(L.ctx, static_cast<uint8_t>(active), negate_field);
      R.resize(J.rows);
      for (int i = 0; i < J.rows; ++i) R[i] = J.residuals(i);
      entries.resize(J.entries.size());
      for (size_t i = 0; i < J.entries.size(); ++i)
        entries[i] = {J.entries[i].row, J.entries[i].col, J.entries[i].value};
      return 0;
    });
  }
  void linearize(const hwf_level* lv, const hwf_energy_params* P, uint32_t active, double lm,
                 double* blocks, double* rhs, double* precond, int threads) override {
    guard([&] {
      RefLevel L(lv, P, threads);
      hwflow::SolveSchedule s;
      s.active_fields = static_cast<uint8_t>(active);
      s.lm_lambda = lm;
      s.threads = threads;
      const hwflow::NormalSystem S = hwflow::build_normal_system(L.ctx, s);
      const int G = S.node_count();
      for (int n = 0; n < G; ++n) {
        for (int sl = 0; sl < 9; ++sl)
          for (int i = 0; i < 6; ++i)
            for (int j = 0; j < 6; ++j)
              blocks[(static_cast<size_t>(n) * 9 + sl) * 36 + 6 * i + j] = S.block(n, sl)(i, j);
        for (int i = 0; i < 6; ++i) rhs[6 * n + i] = S.rhs()(6 * n + i);
        if (precond)
          for (int f = 0; f < 3; ++f) {
            const hwflow::Mat2& M = S.precond_block(n, f);
            double* o = precond + (static_cast<size_t>(n) * 3 + f) * 4;
            o[0] = M(0, 0);
            o[1] = M(0, 1);
            o[2] = M(1, 0);
            o[3] = M(1, 1);
          }
      }
      return 0;
    });
  }
  void pcg(int gw, int gh, const double* blocks, const double* rhs, int iters, double* x,
           double* trace) override {
    guard([&] {
      const hwflow::NormalSystem S = load_system(gw, gh, blocks, rhs);
      std::vector<double> tr;
      const Eigen::VectorXd r = hwflow::pcg_solve(S, iters, 1, trace ? &tr : nullptr);
      std::memcpy(x, r.data(), sizeof(double) * r.size());
      if (trace) std::memcpy(trace, tr.data(), tr.size() * sizeof(double));
      return 0;
    });
  }
  void schwarz(int gw, int gh, int step, int tile, int boundary, const double* blocks,
               const double* rhs, int patch_iters, int pcg_iters, double* x) override {
    guard([&] {
      const hwflow::NormalSystem S = load_system(gw, gh, blocks, rhs);
      const auto subs = hwflow::build_subdomains(gw, gh, step, tile, boundary);
      const Eigen::VectorXd r = hwflow::schwarz_iterate(S, subs, patch_iters, pcg_iters, 1);
      std::memcpy(x, r.data(), sizeof(double) * r.size());
      return 0;
    });
  }
  void gn_level(const hwf_level* lv, const double* base, double* delta, uint8_t* outlier,
                double* node_w, const hwf_energy_params* P, const hwf_schedule* S, int gn_iters,
                std::vector<double>* eb, std::vector<double>* ea,
                std::vector<std::vector<double>>* trace) override {
    guard([&] {
      const int threads = S->threads > 0 ? S->threads : 1;
      RefLevel L(lv, P, threads);
      const WarpGrid b = to_grid(lv->width, lv->height, lv->grid_step, base);
      WarpGrid d = to_grid(lv->width, lv->height, lv->grid_step, delta);
      L.wts.outlier.assign(outlier, outlier + static_cast<size_t>(lv->width) * lv->height);
      L.wts.node_w.assign(node_w, node_w + b.node_count());
      hwflow::SolveSchedule s;
      s.pcg_iters = S->pcg_iters;
      s.patch_iters = S->patch_iters;
      s.subdomain_px = S->subdomain_px;
      s.boundary_px = S->boundary_px;
      s.grid_step = S->grid_step;
      s.threads = threads;
      s.lm_lambda = S->lm_lambda;
      s.active_fields = static_cast<uint8_t>(S->active_fields);
      s.pcg_trace = trace;  // solver.hpp:28
      const hwflow::GnStats st = hwflow::gauss_newton(L.ctx, b, d, L.wts, s, gn_iters);
      from_grid(d, delta);
      std::memcpy(outlier, L.wts.outlier.data(), L.wts.outlier.size());
      std::memcpy(node_w, L.wts.node_w.data(), L.wts.node_w.size() * sizeof(double));
      if (eb) *eb = st.energy_before;
      if (ea) *ea = st.energy_after;
      return 0;
    });
  }
};

}  // namespace

Backend* backend() {
  static Ref r;
  return &r;
}

}  // namespace orc
