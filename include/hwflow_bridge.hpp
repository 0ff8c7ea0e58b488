// hwflow_bridge.hpp — drop-in adapter from the reference's hwflow:: C++ API
// (/root/reference/proj/include/hwflow/*.hpp) onto the C-ABI in hwflow_c.h.
//
// A maintainer of the reference includes this header next to the hwflow
// headers and links libhwflow_cuda.so; the per-level seam and the per-frame
// entry then run on the B200:
//   hwflow::b200::gauss_newton(...)   replaces hwflow::gauss_newton   (solver.hpp:152-154)
//   hwflow::b200::run_scene_flow(...) is run_scene_flow
//   hwflow::b200::build_pyramid(...)  replaces hwflow::build_pyramid  (image.hpp:83)
//   hwflow::b200::assemble_jacobian(...) replaces hwflow::assemble_jacobian (solver.hpp:106-111)
//   hwflow::b200::{validate, triangulate_dlt, compute_scene_points, export_mesh_obj}
//                                      are the geometry.hpp:20-59 declarations
// Same argument meaning; SolverDivergence / std::invalid_argument are thrown
// where the reference throws them (core.hpp:19, energy.cpp:40-50).
#pragma once

#include <array>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hwflow/core.hpp"
#include "hwflow/energy.hpp"
#include "hwflow/geometry.hpp"
#include "hwflow/image.hpp"
#include "hwflow/solver.hpp"
#include "hwflow/warp_grid.hpp"
#include "hwflow_c.h"

namespace hwflow::b200 {

inline void check(hwf_ctx* ctx, int rc) {
  if (rc == HWF_OK) return;
  const std::string msg = hwf_last_error(ctx);
  if (rc == HWF_EDIVERGED) throw SolverDivergence(msg);
  if (rc == HWF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("hwflow CUDA error: " + msg);
}

// One device context (create once per GPU, reuse across frames).
class Device {
 public:
  explicit Device(int device = 0) {
    if (hwf_create(device, &ctx_) != HWF_OK) throw std::runtime_error("hwf_create failed (no usable B200)");
  }
  ~Device() { hwf_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  hwf_ctx* get() const { return ctx_; }

 private:
  hwf_ctx* ctx_ = nullptr;
};

inline hwf_energy_params to_c(const EnergyParams& p) {  // energy.hpp:17-27, same order
  return hwf_energy_params{p.w_reg, p.w_photo, p.w_grad, p.w_epi, p.w_smooth, p.w_mag, p.w_s,
                           p.w_m,   p.w_d,     p.m_s,    p.m_m,   p.m_d,      p.eps_huber, p.eps_color};
}

inline hwf_schedule to_c(const SolveSchedule& s) {  // solver.hpp:14-28
  hwf_schedule c{};
  c.levels = s.levels;
  c.n_gn_per_level = static_cast<int>(std::min<size_t>(s.gn_per_level.size(), HWF_MAX_LEVELS));
  for (int i = 0; i < c.n_gn_per_level; ++i) c.gn_per_level[i] = s.gn_per_level[i];
  c.pcg_iters = s.pcg_iters;
  c.patch_iters = s.patch_iters;
  c.subdomain_px = s.subdomain_px;
  c.boundary_px = s.boundary_px;
  c.grid_step = s.grid_step;
  c.threads = s.threads;
  c.lm_lambda = s.lm_lambda;
  c.active_fields = s.active_fields;
  c.coarse_s_offset[0] = s.coarse_s_offset.x();
  c.coarse_s_offset[1] = s.coarse_s_offset.y();
  return c;
}

inline std::vector<double> grid_to_c(const WarpGrid& g) {
  std::vector<double> v(6 * static_cast<size_t>(g.node_count()));
  for (int k = 0; k < g.node_count(); ++k)
    for (int f = 0; f < 3; ++f) {
      v[6 * k + 2 * f] = g.node(f, k).x();
      v[6 * k + 2 * f + 1] = g.node(f, k).y();
    }
  return v;
}

inline void grid_from_c(const std::vector<double>& v, WarpGrid& g) {
  for (int k = 0; k < g.node_count(); ++k)
    for (int f = 0; f < 3; ++f) g.node(f, k) = Vec2(v[6 * k + 2 * f], v[6 * k + 2 * f + 1]);
}

// gauss_newton (solver.cpp:484-532) on the device: same contract — mutates
// delta and the refreshable parts of weights, returns per-iteration energies.
inline GnStats gauss_newton(const Device& dev, EnergyContext& ctx, const WarpGrid& base, WarpGrid& delta,
                            PixelWeights& weights, const SolveSchedule& sched, int gn_iters) {
  hwf_level lv{};
  lv.width = ctx.width;
  lv.height = ctx.height;
  lv.grid_step = base.step();
  for (int e = 0; e < 4; ++e) {
    lv.images[e] = ctx.images[e]->data().data();
    lv.illum[e] = ctx.illum[e] ? ctx.illum[e]->data().data() : nullptr;
  }
  const std::vector<double> b = grid_to_c(base);
  std::vector<double> d = grid_to_c(delta);
  lv.vis4 = weights.vis4.data();
  lv.fundamental = nullptr;
  double F[9];
  if (ctx.fundamental) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[3 * i + j] = (*ctx.fundamental)(i, j);
    lv.fundamental = F;
  }
  const hwf_energy_params p = to_c(ctx.params);
  const hwf_schedule s = to_c(sched);
  std::vector<double> eb(gn_iters), ea(gn_iters);
  const bool traced = sched.pcg_trace && sched.subdomain_px <= 0;  // solver.cpp:508-513
  const size_t row = static_cast<size_t>(sched.pcg_iters) + 1;
  std::vector<double> tr(traced ? row * gn_iters : 0);
  check(dev.get(), hwf_gn_level_trace(dev.get(), &lv, b.data(), d.data(), weights.outlier.data(),
                                      weights.node_w.data(), &p, &s, gn_iters, eb.data(), ea.data(),
                                      traced ? tr.data() : nullptr));
  if (traced)
    for (int it = 0; it < gn_iters; ++it) sched.pcg_trace->emplace_back(tr.begin() + it * row, tr.begin() + (it + 1) * row);
  grid_from_c(d, delta);
  GnStats st;
  st.energy_before = eb;
  st.energy_after = ea;
  return st;
}

// assemble_jacobian (solver.hpp:106-111): the derivative checker's rows, evaluated on the device.
inline JacobianRows assemble_jacobian(const Device& dev, const EnergyContext& ctx, uint8_t active_fields = 0b111,
                                      int negate_field = -1) {
  hwf_level lv{};
  lv.width = ctx.width;
  lv.height = ctx.height;
  lv.grid_step = ctx.total->step();
  for (int e = 0; e < 4; ++e) {
    lv.images[e] = ctx.images[e]->data().data();
    lv.illum[e] = ctx.illum[e] ? ctx.illum[e]->data().data() : nullptr;
  }
  const std::vector<double> t = grid_to_c(*ctx.total), d = grid_to_c(*ctx.delta);
  lv.total = t.data();
  lv.delta = d.data();
  lv.vis4 = ctx.weights->vis4.data();
  lv.outlier = ctx.weights->outlier.data();
  lv.node_w = ctx.weights->node_w.data();
  double F[9];
  if (ctx.fundamental) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[3 * i + j] = (*ctx.fundamental)(i, j);
    lv.fundamental = F;
  }
  const hwf_energy_params p = to_c(ctx.params);
  long long nnz = 0;
  check(dev.get(), hwf_assemble_jacobian(dev.get(), &lv, &p, active_fields, negate_field, nullptr, nullptr, nullptr,
                                         nullptr, 0, &nnz));
  JacobianRows out;
  out.rows = ctx.residual_count();
  out.cols = 6 * ctx.node_count();
  std::vector<double> R(out.rows), v(nnz);
  std::vector<int> r(nnz), c(nnz);
  check(dev.get(), hwf_assemble_jacobian(dev.get(), &lv, &p, active_fields, negate_field, R.data(), r.data(), c.data(),
                                         v.data(), nnz, &nnz));
  out.residuals.resize(out.rows);
  for (int i = 0; i < out.rows; ++i) out.residuals(i) = R[i];
  out.entries.resize(nnz);
  for (long long i = 0; i < nnz; ++i) out.entries[i] = {r[i], c[i], v[i]};
  return out;
}

// build_pyramid for the four inputs at once (image.cpp:177-185, bit-exact).
inline std::array<Pyramid, 4> build_pyramid(const Device& dev, const std::array<Image, 4>& images, int levels) {
  hwf_frame4 f{images[0].width(), images[0].height(), HWF_DTYPE_F64, {}};
  size_t total = 0;
  for (int e = 0; e < 4; ++e) f.plane[e] = images[e].data().data();
  std::vector<std::pair<int, int>> dims;
  for (int l = 0, w = f.width, h = f.height; l < levels; ++l, w = (w + 1) / 2, h = (h + 1) / 2) {
    dims.emplace_back(w, h);
    total += 4ull * w * h;
  }
  std::vector<double> out(total);
  check(dev.get(), hwf_pyramid(dev.get(), &f, levels, out.data()));
  std::array<Pyramid, 4> pyr;
  size_t off = 0;
  for (const auto& [w, h] : dims)
    for (int e = 0; e < 4; ++e) {
      Image im(w, h);
      std::memcpy(im.data().data(), out.data() + off, sizeof(double) * w * h);
      off += static_cast<size_t>(w) * h;
      pyr[e].levels.push_back(std::move(im));
    }
  return pyr;
}

// run_scene_flow: images by image_index(c,t) = c + 2t.
inline FlowResult run_scene_flow(const Device& dev, const std::array<Image, 4>& images, const EnergyParams& params,
                                 const SolveSchedule& sched, const Mat3* fundamental = nullptr,
                                 GnStats* finest_stats = nullptr) {
  const int w = images[0].width(), h = images[0].height();
  hwf_frame4 f{w, h, HWF_DTYPE_F64, {}};
  for (int e = 0; e < 4; ++e) f.plane[e] = images[e].data().data();
  const size_t N = static_cast<size_t>(w) * h;
  std::vector<double> s(2 * N), m(2 * N), d(2 * N);
  FlowResult r;
  r.width = w;
  r.height = h;
  r.disparity.resize(N);
  r.vis4.resize(N);
  hwf_result out{s.data(), m.data(), d.data(), r.disparity.data(), r.vis4.data(), nullptr};
  double F[9];
  if (fundamental)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[3 * i + j] = (*fundamental)(i, j);
  const hwf_energy_params p = to_c(params);
  const hwf_schedule sc = to_c(sched);
  hwf_stats st{};
  check(dev.get(), hwf_solve_pair(dev.get(), &f, &p, &sc, fundamental ? F : nullptr, &out, &st));
  r.s.resize(N);
  r.m.resize(N);
  r.d.resize(N);
  for (size_t i = 0; i < N; ++i) {
    r.s[i] = Vec2(s[2 * i], s[2 * i + 1]);
    r.m[i] = Vec2(m[2 * i], m[2 * i + 1]);
    r.d[i] = Vec2(d[2 * i], d[2 * i + 1]);
  }
  if (finest_stats) {
    finest_stats->energy_before.assign(st.energy_before[0], st.energy_before[0] + st.gn_iters[0]);
    finest_stats->energy_after.assign(st.energy_after[0], st.energy_after[0] + st.gn_iters[0]);
  }
  return r;
}

// ---- geometry (geometry.hpp:14-59; the reference declares these, geometry.cpp is not shipped) ----
inline hwf_rig rig_to_c(const StereoRig& rig) {
  hwf_rig c{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c.F[3 * i + j] = rig.F(i, j);
  c.has_projections = rig.has_projections() ? 1 : 0;
  if (rig.has_projections())
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 4; ++j) {
        c.P0[4 * i + j] = (*rig.P0)(i, j);
        c.P1[4 * i + j] = (*rig.P1)(i, j);
      }
  return c;
}

// StereoRig::validate (geometry.hpp:20-22): throws std::invalid_argument.
inline void validate(const Device& dev, const StereoRig& rig) {
  const hwf_rig c = rig_to_c(rig);
  check(dev.get(), hwf_validate_rig(dev.get(), &c));
}

// triangulate_dlt (geometry.hpp:45-48).
inline Triangulation triangulate_dlt(const Device& dev, const Mat34& P0, const Mat34& P1, const Vec2& x0,
                                     const Vec2& x1) {
  double p0[12], p1[12], a[2] = {x0.x(), x0.y()}, b[2] = {x1.x(), x1.y()}, X[3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) {
      p0[4 * i + j] = P0(i, j);
      p1[4 * i + j] = P1(i, j);
    }
  uint8_t ok = 0;
  check(dev.get(), hwf_triangulate(dev.get(), 1, p0, p1, a, b, X, &ok));
  Triangulation t;
  t.point = Vec3(X[0], X[1], X[2]);
  t.valid = ok != 0;
  return t;
}

// compute_scene_points (geometry.hpp:54): fills points0/points1/scene_flow/point_valid.
inline void compute_scene_points(const Device& dev, FlowResult& r, const StereoRig& rig) {
  const size_t N = static_cast<size_t>(r.width) * r.height;
  std::vector<double> s(2 * N), m(2 * N), d(2 * N), p0(3 * N), p1(3 * N), sf(3 * N);
  for (size_t i = 0; i < N; ++i)
    for (int k = 0; k < 2; ++k) {
      s[2 * i + k] = r.s[i](k);
      m[2 * i + k] = r.m[i](k);
      d[2 * i + k] = r.d[i](k);
    }
  r.point_valid.assign(N, 0);
  const hwf_rig c = rig_to_c(rig);
  check(dev.get(), hwf_scene_points(dev.get(), r.width, r.height, s.data(), m.data(), d.data(), &c, p0.data(),
                                    p1.data(), sf.data(), r.point_valid.data()));
  r.points0.resize(N);
  r.points1.resize(N);
  r.scene_flow.resize(N);
  for (size_t i = 0; i < N; ++i) {
    r.points0[i] = Vec3(p0[3 * i], p0[3 * i + 1], p0[3 * i + 2]);
    r.points1[i] = Vec3(p1[3 * i], p1[3 * i + 1], p1[3 * i + 2]);
    r.scene_flow[i] = Vec3(sf[3 * i], sf[3 * i + 1], sf[3 * i + 2]);
  }
  r.has_points = true;
}

// export_mesh_obj (geometry.hpp:56-59).
inline void export_mesh_obj(const Device& dev, const FlowResult& r, const std::string& path) {
  const size_t N = static_cast<size_t>(r.width) * r.height;
  std::vector<double> p0;
  if (r.has_points) {
    p0.resize(3 * N);
    for (size_t i = 0; i < N; ++i)
      for (int k = 0; k < 3; ++k) p0[3 * i + k] = r.points0[i](k);
  }
  check(dev.get(), hwf_export_mesh_obj(dev.get(), r.width, r.height, r.disparity.data(), r.vis4.data(),
                                       r.has_points ? p0.data() : nullptr,
                                       r.has_points ? r.point_valid.data() : nullptr, path.c_str()));
}

}  // namespace hwflow::b200
