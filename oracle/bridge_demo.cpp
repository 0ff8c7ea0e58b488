// oracle/bridge_demo.cpp — TEST INFRASTRUCTURE ONLY.
//
// What a maintainer of the reference gets by adding include/hwflow_bridge.hpp: this program is written
// against the reference's own C++ API (/root/reference/proj/include/hwflow/*.hpp, value types Image,
// WarpGrid, PixelWeights, EnergyContext, SolveSchedule, GnStats) and is linked with BOTH the reference's
// sources (compiled verbatim by oracle/Makefile, CPU) and libhwflow_cuda.so (the product, through the C-ABI).
// It runs the same calls on both sides and prints one JSON line; tests/test_bridge.py (-m gpu) runs it on
// the B200 and checks the numbers:
//   1. build_pyramid (image.cpp:177-185)    hwflow::build_pyramid  vs hwflow::b200::build_pyramid: bit-exact
//   2. gauss_newton (solver.cpp:484-532)    hwflow::gauss_newton   vs hwflow::b200::gauss_newton, 3 GN x
//      5 global PCG with pcg_trace, from the reference's own EnergyContext/PixelWeights: delta, W, w_i, energies
//   3. run_scene_flow     hwflow::b200::run_scene_flow; the 4 images and the FlowResult
//      are written to argv[1]
//      (the test compares it with the oracle's Algorithm 1)
//   4. SolverDivergence (core.hpp:19)       thrown by both sides on the same degenerate level
//   5. std::invalid_argument                thrown by both sides for a negative weight (energy.cpp:43-50)
//   6. assemble_jacobian (solver.cpp:247-314) hwflow:: vs hwflow::b200::, with the negate_field hook: same triplets
#include <cmath>
#include <cstdio>
#include <fstream>
#include <stdexcept>

#include "hwflow_bridge.hpp"

using namespace hwflow;

namespace {

// A smooth texture T and the four images I_c^t(x) = T(x - sc*s - st*m) (warp_grid.hpp:73-77).
double texture(double x, double y) {
  return 0.5 + 0.18 * std::sin(0.37 * x + 0.11 * y) + 0.12 * std::cos(0.21 * x - 0.29 * y) +
         0.08 * std::sin(0.73 * x * 0.5 + 0.61 * y * 0.5 + 1.3) + 0.05 * std::cos(1.1 * x - 0.9 * y);
}

std::array<Image, 4> make_images(int w, int h, Vec2 s, Vec2 m) {
  std::array<Image, 4> im;
  for (int t = 0; t < 2; ++t)
    for (int c = 0; c < 2; ++c) {
      const double sc = c ? 1.0 : -1.0, st = t ? 1.0 : -1.0;
      Image I(w, h);
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
          I.at(x, y) = std::min(1.0, std::max(0.0, texture(x - sc * s.x() - st * m.x(), y - sc * s.y() - st * m.y())));
      im[image_index(c, t)] = std::move(I);
    }
  return im;
}

template <class Fn>
int throws_kind(Fn&& fn) {  // 0 none, 1 SolverDivergence, 2 invalid_argument, 3 other
  try {
    fn();
  } catch (const SolverDivergence&) {
    return 1;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (...) {
    return 3;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const int w = 96, h = 72;
  const auto images = make_images(w, h, Vec2(1.25, 0.0), Vec2(0.5, -0.375));
  b200::Device dev;

  // 1. pyramid
  const auto pd = b200::build_pyramid(dev, images, 3);
  bool pyr_exact = true;
  for (int e = 0; e < 4; ++e) {
    const Pyramid pr = build_pyramid(images[e], 3);
    for (int l = 0; l < 3; ++l) pyr_exact = pyr_exact && pr.levels[l].data() == pd[e].levels[l].data();
  }

  // 2. one level of Gauss-Newton on the finest images, the reference's own value types on both sides
  SolveSchedule sched;
  sched.grid_step = 8;
  sched.subdomain_px = 0;
  sched.pcg_iters = 5;
  std::vector<std::vector<double>> trace_ref, trace_dev;
  WarpGrid base(w, h, sched.grid_step), delta_ref(w, h, sched.grid_step), delta_dev(w, h, sched.grid_step);
  for (int k = 0; k < base.node_count(); ++k) base.node(0, k) = Vec2(1.0, 0.0);
  PixelWeights wr, wd;
  wr.init_all_visible(w * h, base.node_count());
  wd.init_all_visible(w * h, base.node_count());
  EnergyContext cr, cd;
  for (int e = 0; e < 4; ++e) cr.images[e] = cd.images[e] = &images[e];
  cr.params = cd.params = EnergyParams{};
  cr.width = cd.width = w;
  cr.height = cd.height = h;
  sched.pcg_trace = &trace_ref;
  const GnStats sr = gauss_newton(cr, base, delta_ref, wr, sched, 3);
  sched.pcg_trace = &trace_dev;
  const GnStats sd = b200::gauss_newton(dev, cd, base, delta_dev, wd, sched, 3);
  sched.pcg_trace = nullptr;
  double dmax = 0.0, emax = 0.0, nwmax = 0.0, trmax = 0.0;
  for (int k = 0; k < base.node_count(); ++k)
    for (int f = 0; f < 3; ++f) dmax = std::max(dmax, (delta_ref.node(f, k) - delta_dev.node(f, k)).norm());
  for (int i = 0; i < 3; ++i) {
    emax = std::max(emax, std::abs(sr.energy_after[i] - sd.energy_after[i]) / sr.energy_after[i]);
    emax = std::max(emax, std::abs(sr.energy_before[i] - sd.energy_before[i]) / sr.energy_before[i]);
  }
  for (size_t k = 0; k < wr.node_w.size(); ++k) nwmax = std::max(nwmax, std::abs(wr.node_w[k] - wd.node_w[k]) / wr.node_w[k]);
  const bool w_exact = wr.outlier == wd.outlier;
  const bool trace_shape = trace_ref.size() == trace_dev.size() && trace_dev.size() == 3;
  for (size_t i = 0; trace_shape && i < trace_ref.size(); ++i)
    for (size_t j = 0; j < trace_ref[i].size() && j < trace_dev[i].size(); ++j)
      trmax = std::max(trmax, std::abs(trace_ref[i][j] - trace_dev[i][j]) / std::max(1e-300, trace_ref[i][0]));

  // 2b. assemble_jacobian (solver.cpp:247-314) on the reference's EnergyContext at the state GN left behind
  WarpGrid tot = base.plus(delta_ref);
  cr.total = &tot;
  cr.delta = &delta_ref;
  cr.weights = &wr;
  const JacobianRows jr = assemble_jacobian(cr, 0b111, 1), jd = b200::assemble_jacobian(dev, cr, 0b111, 1);
  bool jac_same_entries = jr.entries.size() == jd.entries.size() && jr.rows == jd.rows && jr.cols == jd.cols;
  // max |difference| over max |value|, for the Jacobian values and the residuals separately
  double jdiff = 0.0, jmax = 0.0, rdiff = 0.0, rmax = 0.0;
  for (size_t i = 0; jac_same_entries && i < jr.entries.size(); ++i) {
    jac_same_entries = jr.entries[i].row == jd.entries[i].row && jr.entries[i].col == jd.entries[i].col;
    jdiff = std::max(jdiff, std::abs(jr.entries[i].value - jd.entries[i].value));
    jmax = std::max(jmax, std::abs(jr.entries[i].value));
  }
  for (int i = 0; jac_same_entries && i < jr.rows; ++i) {
    rdiff = std::max(rdiff, std::abs(jr.residuals(i) - jd.residuals(i)));
    rmax = std::max(rmax, std::abs(jr.residuals(i)));
  }
  const double jac_rel = std::max(jdiff / std::max(jmax, 1e-300), rdiff / std::max(rmax, 1e-300));
  cr.total = nullptr;

  // 3. Algorithm 1 on the device through the bridge; images (4 x f64 planes), then the FlowResult (s, m, d,
  //    disparity as f64, vis4 u8) to argv[1]
  SolveSchedule full;
  full.levels = 3;
  full.grid_step = 8;
  full.subdomain_px = 0;
  full.pcg_iters = 5;
  GnStats finest;
  const FlowResult fr = b200::run_scene_flow(dev, images, EnergyParams{}, full, nullptr, &finest);
  if (argc > 1) {
    std::ofstream o(argv[1], std::ios::binary);
    for (const Image& I : images) o.write(reinterpret_cast<const char*>(I.data().data()), sizeof(double) * I.size());
    for (const auto* v : {&fr.s, &fr.m, &fr.d})
      for (const Vec2& p : *v) {
        const double xy[2] = {p.x(), p.y()};
        o.write(reinterpret_cast<const char*>(xy), sizeof(xy));
      }
    o.write(reinterpret_cast<const char*>(fr.disparity.data()), sizeof(double) * fr.disparity.size());
    o.write(reinterpret_cast<const char*>(fr.vis4.data()), fr.vis4.size());
  }

  // 4. divergence: flat images, no Tikhonov/magnitude terms -> singular J^T J; both sides must throw
  //    SolverDivergence (solver.cpp:345 pAp <= 0 or :515 non-finite update) or both must not.
  std::array<Image, 4> flat;
  for (auto& I : flat) I = Image(32, 24, 0.5);
  EnergyParams degenerate;
  degenerate.m_s = degenerate.m_m = degenerate.m_d = 0.0;
  degenerate.w_reg = 0.0;
  auto run_div = [&](bool on_dev) {
    WarpGrid b(32, 24, 8), d(32, 24, 8);
    PixelWeights pw;
    pw.init_all_visible(32 * 24, b.node_count());
    EnergyContext c;
    for (int e = 0; e < 4; ++e) c.images[e] = &flat[e];
    c.params = degenerate;
    c.width = 32;
    c.height = 24;
    SolveSchedule s1;
    s1.grid_step = 8;
    s1.subdomain_px = 0;
    if (on_dev)
      b200::gauss_newton(dev, c, b, d, pw, s1, 1);
    else
      gauss_newton(c, b, d, pw, s1, 1);
  };
  const int div_ref = throws_kind([&] { run_div(false); });
  const int div_dev = throws_kind([&] { run_div(true); });

  // 5. invalid parameters (energy.cpp:43-50 validate): negative weight
  EnergyParams bad;
  bad.w_photo = -1.0;
  const int inv_ref = throws_kind([&] { bad.validate(); });
  const int inv_dev = throws_kind([&] { b200::run_scene_flow(dev, images, bad, full); });

  std::printf(
      "{\"pyramid_bit_exact\": %s, \"gn_delta_max\": %.3e, \"gn_energy_rel\": %.3e, \"gn_node_w_rel\": %.3e, "
      "\"gn_W_exact\": %s, \"pcg_trace_shape\": %s, \"pcg_trace_rel\": %.3e, \"solve_width\": %d, \"solve_height\": %d, "
      "\"finest_gn_iters\": %zu, \"divergence_ref\": %d, \"divergence_dev\": %d, \"invalid_ref\": %d, \"invalid_dev\": %d, "
      "\"jacobian_same_entries\": %s, \"jacobian_rel\": %.3e, \"jacobian_nnz\": %zu}\n",
      pyr_exact ? "true" : "false", dmax, emax, nwmax, w_exact ? "true" : "false", trace_shape ? "true" : "false", trmax,
      fr.width, fr.height, finest.energy_after.size(), div_ref, div_dev, inv_ref, inv_dev,
      jac_same_entries ? "true" : "false", jac_rel, jr.entries.size());
  return 0;
}
