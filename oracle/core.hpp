// oracle/core.hpp — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
//
// Plain-C++ restatement of the reference's per-level algorithm
// (/root/reference/proj/src/{image,warp_grid,energy,solver}.cpp). Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg may load the library
// built from this file. Every function cites the reference file:line it follows.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hwflow_c.h"

namespace orc {

struct Divergence : std::runtime_error {  // core.hpp:19-21 SolverDivergence
  explicit Divergence(const std::string& m) : std::runtime_error(m) {}
};

// ---- rasters (image.hpp:12-61) ---------------------------------------------
struct Raster {
  int w = 0, h = 0;
  const double* p = nullptr;
  double at(int x, int y) const { return p[static_cast<size_t>(y) * w + x]; }
  double at_clamped(int x, int y) const {  // image.hpp:28-32
    x = x < 0 ? 0 : (x >= w ? w - 1 : x);
    y = y < 0 ? 0 : (y >= h ? h - 1 : y);
    return at(x, y);
  }
};

double sample(const Raster& im, double x, double y, double* ddx, double* ddy);
void pixel_grad(const Raster& im, int x, int y, double g[2]);
void grad_at(const Raster& im, double x, double y, double g[2], double D[2][2] /*nullable*/);
void downsample(const Raster& im, std::vector<double>& out, int* ow, int* oh);
void gaussian_blur(const Raster& im, double sigma, std::vector<double>& out);
double structure_weight(const Raster& im, int cx, int cy, double delta = 1e-4,
                        double w_max = 100.0);

// ---- warp grid (warp_grid.hpp:25-71) ---------------------------------------
struct GridDims {
  int gw = 0, gh = 0, step = 1;
  int nodes() const { return gw * gh; }
};
GridDims grid_dims(int image_w, int image_h, int step);
struct Support {
  int node[4];
  double wt[4];
};
Support support(const GridDims& g, double x, double y);
void interpolate(const GridDims& g, const double* nodes6, double x, double y, double out[6]);

inline double sgn(int idx) { return idx == 0 ? -1.0 : 1.0; }  // core.hpp:24
// warp_grid.hpp:74-77: x + sc*s + st*m + sc*st*d
inline void warp_position(double x, double y, const double f[6], int cam, int time,
                          double* wx, double* wy) {
  const double sc = sgn(cam), st = sgn(time), scst = sc * st;
  *wx = x + sc * f[0] + st * f[2] + scst * f[4];
  *wy = y + sc * f[1] + st * f[3] + scst * f[5];
}
constexpr int kCheckA[6] = {1, 3, 2, 3, 3, 2};  // warp_grid.hpp:85-87
constexpr int kCheckB[6] = {0, 2, 0, 1, 0, 1};

// ---- energy (energy.hpp / energy.cpp) --------------------------------------
struct Level {
  int w = 0, h = 0;
  GridDims g;
  Raster img[4];
  const double* illum[4] = {nullptr, nullptr, nullptr, nullptr};
  const double* total = nullptr;
  const double* delta = nullptr;
  const uint8_t* vis4 = nullptr;
  const uint8_t* outlier = nullptr;
  const double* node_w = nullptr;
  const double* F = nullptr;
  hwf_energy_params P{};
  int threads = 1;
  int N() const { return w * h; }
  int G() const { return g.nodes(); }
  bool check_visible(int pix, int k) const {  // energy.hpp:65-68
    const uint8_t v = vis4[pix];
    return ((v >> kCheckA[k]) & 1) && ((v >> kCheckB[k]) & 1);
  }
};

Level make_level(const hwf_level* lv, const hwf_energy_params* P, int threads);

struct PixelEval {  // energy.hpp:92-97
  double r_photo = 0, r_grad = 0, e_photo = 0, e_grad = 0;
  double jp[6] = {0, 0, 0, 0, 0, 0}, jg[6] = {0, 0, 0, 0, 0, 0};
};
PixelEval eval_pixel(const Level& L, int px, int py, bool derivs);

struct NodeEval {  // energy.hpp:103-115
  double smooth_r[6] = {}, epi_r[2] = {}, mag_r[6] = {};
  double e_smooth = 0, e_epi = 0, e_mag = 0;
  double jc[6] = {}, jr[6] = {}, jd[6] = {};
  double epi_j[2][6] = {};
  double mag_j[6] = {};
  int right = -1, down = -1;
};
NodeEval eval_node(const Level& L, int node, bool derivs);

hwf_energy energy(const Level& L, double* residuals /*nullable*/);
void refresh_outlier(const Level& L, uint8_t* outlier);
void refresh_node_w(const Level& L, double* node_w);

// ---- solver (solver.hpp / solver.cpp) --------------------------------------
struct System {  // solver.hpp:41-87
  int gw = 0, gh = 0;
  std::vector<double> blk;  // [G*9][36]
  std::vector<double> rhs;  // 6G
  std::vector<double> pre;  // [G*3][4]
  int G() const { return gw * gh; }
  double* block(int n, int s) { return &blk[(static_cast<size_t>(n) * 9 + s) * 36]; }
  const double* block(int n, int s) const { return &blk[(static_cast<size_t>(n) * 9 + s) * 36]; }
  int neighbor(int n, int dx, int dy) const;
  void apply(const std::vector<double>& x, std::vector<double>& y) const;
  void precondition(const std::vector<double>& r, std::vector<double>& z) const;
  void build_preconditioner();
};
inline int slot(int dx, int dy) { return (dy + 1) * 3 + (dx + 1); }

System build_normal_system(const Level& L, uint32_t active, double lm_lambda);
struct JacTriplet {
  int row, col;
  double value;
};
void assemble_jacobian(const Level& L, uint32_t active, int negate_field, std::vector<double>& R,
                       std::vector<JacTriplet>& out);  // solver.cpp:247-314
std::vector<double> pcg_solve(const System& S, int iters, std::vector<double>* trace);
struct Subdomain {
  std::vector<int> interior;
};
std::vector<Subdomain> build_subdomains(int gw, int gh, int step, int tile_px);
std::vector<double> schwarz(const System& S, const std::vector<Subdomain>& subs, int patch_iters,
                            int pcg_iters);
void subdomain_owner(const std::vector<Subdomain>& subs, int G, std::vector<int>& owner, std::vector<int>& loc);
void schwarz_sweep(const System& S, const std::vector<Subdomain>& subs, const std::vector<int>& owner,
                   const std::vector<int>& loc, const std::vector<double>& pub, std::vector<double>& next,
                   int pcg_iters, const std::vector<char>* take);

// gauss_newton (solver.cpp:484-532). Level's total/delta/outlier/node_w are
// rebound internally; delta, outlier and node_w are updated in place.
void gauss_newton(Level L, const double* base, double* delta, uint8_t* outlier, double* node_w,
                  const hwf_schedule& S, int gn_iters, std::vector<double>* e_before,
                  std::vector<double>* e_after, std::vector<std::vector<double>>* pcg_trace = nullptr);

}  // namespace orc
