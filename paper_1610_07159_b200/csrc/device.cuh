// device.cuh — sm_100a device helpers for the halfway-domain scene-flow solve.
//
// Layouts (per batch of B frame pairs, one level with N = w*h pixels, G nodes):
//   images  double [B][4][N]          image_index(c,t)=c+2t (core.hpp:27), row-major
//   illum   double [B][4][N]          halfway-pixel indexed additive maps (energy.cpp:75)
//   vis4/W  uint8  [B][N]
//   grids   double [B][G][6]          (s_x,s_y,m_x,m_y,d_x,d_y) per node (solver.cpp:521)
//   cells   double [B][C][234]        per warp-grid cell: 10 corner-pair symmetric 6x6
//                                     sums (21 packed each) + 4 corner rhs sums (6 each)
//   sys     double [B][G][120]        5 forward symmetric blocks (21 packed each, slots
//                                     (0,0),(1,0),(-1,1),(0,1),(1,1)), rhs (6), inverted
//                                     2x2 precond per field (3 packed each)
// Backward slots are never stored: block(n,-s) = block(n-s,s)^T = block(n-s,s) because
// every J^T J block the reference assembles is symmetric (solver.cpp:12-17,228-241).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hwflow_c.h"

namespace hwf {

// per-cell records of k_pixel's reduction: 10 corner-pair blocks of 21 packed entries, then 4 corner rhs of 6
#ifdef HWF_CELLS_PACKED  // A/B: packed blocks (21 and 6 doubles), 8 B aligned
constexpr int kCellBlk = 21, kCellRhsW = 6;
#else  // blocks padded to 24 doubles and rhs to 8: 32 B aligned, so k_node reads whole sectors (256-bit loads)
#define HWF_CELLS_V4
constexpr int kCellBlk = 24, kCellRhsW = 8;
#endif
constexpr int kCellRhs = 10 * kCellBlk;
constexpr int kCellStride = kCellRhs + 4 * kCellRhsW;
constexpr int kCellData = 10 * 21 + 4 * 6;  // the doubles of a cell record that carry data (algorithmic bytes)
constexpr int kSysStride = 120;
constexpr int kSysRhs = 105;
constexpr int kSysPre = 111;
constexpr int kNumEnergy = 5;  // photo, grad, smooth, epi, mag (energy.hpp:125-131)

// packed upper-triangular 6x6 index, i <= j
__host__ __device__ __forceinline__ int sym6(int i, int j) {
  if (i > j) {
    const int t = i;
    i = j;
    j = t;
  }
  return i * 6 - (i * (i - 1)) / 2 + (j - i);
}
// (i, j) of packed index m (the inverse of sym6)
__host__ __device__ constexpr int sym_i(int m) { return m < 6 ? 0 : (m < 11 ? 1 : (m < 15 ? 2 : (m < 18 ? 3 : (m < 20 ? 4 : 5)))); }
__host__ __device__ constexpr int sym_j(int m) { return m - (sym_i(m) * 6 - (sym_i(m) * (sym_i(m) - 1)) / 2) + sym_i(m); }
// unordered corner pair (i <= j) of a cell, 10 pairs
__host__ __device__ __forceinline__ int pair4(int i, int j) {
  if (i > j) {
    const int t = i;
    i = j;
    j = t;
  }
  return i * 4 - (i * (i - 1)) / 2 + (j - i);
}
// forward slot index 0..4 for offset (dx,dy), or -1 (solver.cpp:15-17)
__host__ __device__ __forceinline__ int fwd_slot(int dx, int dy) {
  const int s9 = (dy + 1) * 3 + (dx + 1);
  return s9 >= 4 ? s9 - 4 : -1;
}

struct Params {  // hwf_energy_params by value
  double w_reg, w_photo, w_grad, w_epi, w_smooth, w_mag;
  double w_s, w_m, w_d, m_s, m_m, m_d;
  double eps_huber, eps_color;
};

__device__ __forceinline__ double field_smooth_w(const Params& P, int f) {
  return f == 0 ? P.w_s : (f == 1 ? P.w_m : P.w_d);
}
__device__ __forceinline__ double field_mag_w(const Params& P, int f) {
  return f == 0 ? P.m_s : (f == 1 ? P.m_m : P.m_d);
}

// kChecks (warp_grid.hpp:85-87): a = {1,3,2,3,3,2}, b = {0,2,0,1,0,1}, nibble k from the top.
__host__ __device__ __forceinline__ int check_a(int k) { return (0x132332 >> (4 * (5 - k))) & 0xF; }
__host__ __device__ __forceinline__ int check_b(int k) { return (0x020101 >> (4 * (5 - k))) & 0xF; }

// image.cpp:19-31 cell_coord
struct Coord {
  int i0;
  double f;
  bool clamped;
};
__device__ __forceinline__ Coord cell_coord(double v, int n) {
  Coord c;
#if defined(HWF_CELL_COORD) && HWF_CELL_COORD > 0  // A/B (tools/cell_coord_ab.py): branch-free forms
  const bool lo = v <= 0.0, hi = v >= n - 1;  // both false for NaN
  const double fl = floor(v);
#if HWF_CELL_COORD == 1  // the same function with selects: NaN keeps f = NaN, i0 = (int)NaN = 0
  c.i0 = lo ? 0 : (hi ? (n >= 2 ? n - 2 : 0) : static_cast<int>(fl));
  c.f = lo ? 0.0 : (hi ? 1.0 : v - fl);
#elif HWF_CELL_COORD == 2  // clamp first with fmin/fmax: a NaN coordinate becomes 0 (cell 0, f = 0)
  const double vc = fmin(fmax(v, 0.0), static_cast<double>(n - 1));
  c.i0 = min(static_cast<int>(floor(vc)), max(n - 2, 0));
  c.f = vc - c.i0;
#else  // 3: the cell clamped but not the fraction (f = v - i0 extrapolates outside [0, n - 1])
  c.i0 = min(max(static_cast<int>(fl), 0), max(n - 2, 0));
  c.f = v - c.i0;
#endif
  c.clamped = lo || hi;
  if (n == 1) {
    c.i0 = 0;
    c.f = 0.0;
    c.clamped = true;
  }
  return c;
#endif
  if (v <= 0.0) {
    c.i0 = 0;
    c.f = 0.0;
    c.clamped = true;
  } else if (v >= n - 1) {
    c.i0 = n >= 2 ? n - 2 : 0;
    c.f = 1.0;
    c.clamped = true;
  } else {
    const double fl = floor(v);
    c.i0 = static_cast<int>(fl);
    c.f = v - fl;
    c.clamped = false;
  }
  if (n == 1) {
    c.i0 = 0;
    c.f = 0.0;
    c.clamped = true;
  }
  return c;
}

// Edge-clamped bilinear value + exact in-cell derivative (image.cpp:37-54) and
// bilinear central-difference gradient + its derivative (image.cpp:56-98),
// from one 12-pixel footprint.
struct Samp {
  double v, dvx, dvy;       // value, d value / d p
  double gx, gy;            // gradient
  double D00, D01, D10, D11;  // D(k,j) = d grad_k / d p_j
};

template <bool DERIVS, bool GRAD>
__device__ __forceinline__ void sample_img(const double* __restrict__ I, int w, int h, double x,
                                           double y, Samp& s) {
  const Coord cx = cell_coord(x, w), cy = cell_coord(y, h);
  const int c1 = cx.i0, c2 = min(cx.i0 + 1, w - 1);
  const int r1 = cy.i0, r2 = min(cy.i0 + 1, h - 1);
  const double* R1 = I + static_cast<size_t>(r1) * w;
  const double* R2 = I + static_cast<size_t>(r2) * w;
  const double v00 = __ldg(R1 + c1), v10 = __ldg(R1 + c2), v01 = __ldg(R2 + c1), v11 = __ldg(R2 + c2);
  const double fx = cx.f, fy = cy.f;
  const double a = (1 - fx) * (1 - fy), b = fx * (1 - fy), c = (1 - fx) * fy, d = fx * fy;
  s.v = a * v00 + b * v10 + c * v01 + d * v11;
  if (DERIVS) {
    const double dx = (1 - fy) * (v10 - v00) + fy * (v11 - v01);
    const double dy = (1 - fx) * (v01 - v00) + fx * (v11 - v10);
    s.dvx = cx.clamped ? 0.0 : dx;
    s.dvy = cy.clamped ? 0.0 : dy;
  }
  if (GRAD) {
    const int c0 = max(c1 - 1, 0), c3 = min(c2 + 1, w - 1);
    const int r0 = max(r1 - 1, 0), r3 = min(r2 + 1, h - 1);
    const double* R0 = I + static_cast<size_t>(r0) * w;
    const double* R3 = I + static_cast<size_t>(r3) * w;
    const double u0 = __ldg(R1 + c0), u3 = __ldg(R1 + c3);
    const double l0 = __ldg(R2 + c0), l3 = __ldg(R2 + c3);
    const double t1 = __ldg(R0 + c1), t2 = __ldg(R0 + c2);
    const double b1 = __ldg(R3 + c1), b2 = __ldg(R3 + c2);
    // one-sided (x1) at borders, central (x0.5) inside (image.cpp:56-77)
    const double fc1 = (c1 == 0 || c1 == w - 1) ? 1.0 : 0.5;
    const double fc2 = (c2 == 0 || c2 == w - 1) ? 1.0 : 0.5;
    const double fr1 = (r1 == 0 || r1 == h - 1) ? 1.0 : 0.5;
    const double fr2 = (r2 == 0 || r2 == h - 1) ? 1.0 : 0.5;
    const double g00x = fc1 * (v10 - u0), g00y = fr1 * (v01 - t1);
    const double g10x = fc2 * (u3 - v00), g10y = fr1 * (v11 - t2);
    const double g01x = fc1 * (v11 - l0), g01y = fr2 * (b1 - v00);
    const double g11x = fc2 * (l3 - v01), g11y = fr2 * (b2 - v10);
    s.gx = a * g00x + b * g10x + c * g01x + d * g11x;
    s.gy = a * g00y + b * g10y + c * g01y + d * g11y;
    if (DERIVS) {
      const double dxx = (1 - fy) * (g10x - g00x) + fy * (g11x - g01x);
      const double dyx = (1 - fy) * (g10y - g00y) + fy * (g11y - g01y);
      const double dxy = (1 - fx) * (g01x - g00x) + fx * (g11x - g10x);
      const double dyy = (1 - fx) * (g01y - g00y) + fx * (g11y - g10y);
      s.D00 = cx.clamped ? 0.0 : dxx;
      s.D10 = cx.clamped ? 0.0 : dyx;
      s.D01 = cy.clamped ? 0.0 : dxy;
      s.D11 = cy.clamped ? 0.0 : dyy;
    }
  }
}

// Bilinear footprint of a continuous position (image.cpp:19-31,37-54): the four
// corner offsets, the in-cell fractions and whether each coordinate is clamped.
struct Foot {
  int o00, o10, o01, o11;
  int x0, y0;  // the (x, y) of o00
  double fx, fy;
  bool clx, cly;
};
__device__ __forceinline__ Foot footprint(int w, int h, double x, double y) {
  const Coord cx = cell_coord(x, w), cy = cell_coord(y, h);
  const int c2 = min(cx.i0 + 1, w - 1), r2 = min(cy.i0 + 1, h - 1);
  Foot f;
  f.o00 = cy.i0 * w + cx.i0;
  f.o10 = cy.i0 * w + c2;
  f.o01 = r2 * w + cx.i0;
  f.o11 = r2 * w + c2;
  f.x0 = cx.i0;
  f.y0 = cy.i0;
  f.fx = cx.f;
  f.fy = cy.f;
  f.clx = cx.clamped;
  f.cly = cy.clamped;
  return f;
}

// Central-difference pixel gradient (image.cpp:56-77): one-sided at borders.
__device__ __forceinline__ double2 pixel_grad(const double* __restrict__ I, int w, int h, int x, int y) {
  const double* R = I + static_cast<size_t>(y) * w;
  double2 g;
  g.x = w == 1 ? 0.0 : ((x == 0 || x == w - 1) ? 1.0 : 0.5) * (R[min(x + 1, w - 1)] - R[max(x - 1, 0)]);
  g.y = h == 1 ? 0.0
               : ((y == 0 || y == h - 1) ? 1.0 : 0.5) *
                     (I[static_cast<size_t>(min(y + 1, h - 1)) * w + x] - I[static_cast<size_t>(max(y - 1, 0)) * w + x]);
  return g;
}

// x / step (warp_grid.cpp:44-45), correctly rounded. A power-of-two step (every BASELINE config) is an exact
// multiplication by 2^-k, the same double as the division, without the FP64 division sequence.
__device__ __forceinline__ double div_step(double x, int step) {
  if ((step & (step - 1)) == 0)
    return x * __longlong_as_double(static_cast<long long>(1023 - (__ffs(step) - 1)) << 52);
  return x / step;
}

// warp_grid.cpp:41-54 support for an in-coverage position; returns the cell.
__device__ __forceinline__ void grid_support(int gw, int gh, int step, double x, double y, int& a0,
                                             int& b0, double& fu, double& fv) {
  const double u = div_step(x, step), v = div_step(y, step);
  a0 = min(max(static_cast<int>(floor(u)), 0), gw - 2);
  b0 = min(max(static_cast<int>(floor(v)), 0), gh - 2);
  fu = fmin(fmax(u - a0, 0.0), 1.0);
  fv = fmin(fmax(v - b0, 0.0), 1.0);
}

// warp_grid.cpp:56-65 with every product and sum rounded separately (no FMA
// contraction) so that it is bit-identical to the -ffp-contract=off oracle.
// Used where bit-exactness matters (occlusion vertex positions, prolongation).
__device__ __forceinline__ void interp_exact(const double* __restrict__ T, int gw, int gh, int step,
                                             double x, double y, double out[6]) {
  int a0, b0;
  double fu, fv;
  grid_support(gw, gh, step, x, y, a0, b0, fu, fv);
  const double omu = __dadd_rn(1.0, -fu), omv = __dadd_rn(1.0, -fv);
  const double w0 = __dmul_rn(omu, omv), w1 = __dmul_rn(fu, omv), w2 = __dmul_rn(omu, fv),
               w3 = __dmul_rn(fu, fv);
  const double* n0 = T + 6 * static_cast<size_t>(b0 * gw + a0);
  const double* n2 = T + 6 * static_cast<size_t>((b0 + 1) * gw + a0);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double acc = __dadd_rn(0.0, __dmul_rn(w0, n0[c]));  // from zero, as the reference
    acc = __dadd_rn(acc, __dmul_rn(w1, n0[6 + c]));
    acc = __dadd_rn(acc, __dmul_rn(w2, n2[c]));
    acc = __dadd_rn(acc, __dmul_rn(w3, n2[6 + c]));
    out[c] = acc;
  }
}

// Fast interpolation for the solver sweeps (tolerance-level parity).
__device__ __forceinline__ void interp_fast(const double* __restrict__ T, int gw, int gh, int step,
                                            double x, double y, double out[6]) {
  int a0, b0;
  double fu, fv;
  grid_support(gw, gh, step, x, y, a0, b0, fu, fv);
  const double w0 = (1 - fu) * (1 - fv), w1 = fu * (1 - fv), w2 = (1 - fu) * fv, w3 = fu * fv;
  // node records are 48 B (16 B aligned): three 16-byte loads per node
  const double2* n0 = reinterpret_cast<const double2*>(T + 6 * static_cast<size_t>(b0 * gw + a0));
  const double2* n2 = reinterpret_cast<const double2*>(T + 6 * static_cast<size_t>((b0 + 1) * gw + a0));
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double2 p0 = __ldg(n0 + c), p1 = __ldg(n0 + 3 + c), p2 = __ldg(n2 + c), p3 = __ldg(n2 + 3 + c);
    out[2 * c] = w0 * p0.x + w1 * p1.x + w2 * p2.x + w3 * p3.x;
    out[2 * c + 1] = w0 * p0.y + w1 * p1.y + w2 * p2.y + w3 * p3.y;
  }
}

// warp_grid.hpp:74-77 (sigma_0 = -1, sigma_1 = +1); exact adds in reference order.
__device__ __forceinline__ void warp_pos_exact(double x, double y, const double f[6], int e,
                                               double& wx, double& wy) {
  const double sc = (e & 1) ? 1.0 : -1.0, st = (e >> 1) ? 1.0 : -1.0, scst = sc * st;
  wx = __dadd_rn(__dadd_rn(__dadd_rn(x, sc * f[0]), st * f[2]), scst * f[4]);
  wy = __dadd_rn(__dadd_rn(__dadd_rn(y, sc * f[1]), st * f[3]), scst * f[5]);
}

// One occlusion lattice vertex (pin C.2, oracle/hierarchy.cpp) from the exactly interpolated flow fl at halfway
// pixel (x, y): its position in the 4 views in 1/256 px fixed point, the float depth proxy 1/(|2s| + 1e-3), and
// validity. Written by k_occ_project, or by the fused E_after pass (k_pixel<false, *, *, *, PROJ>).
__device__ __forceinline__ bool occ_project_flow(int x, int y, const double fl[6], int2 (&q)[4], float& zf) {
  const double s2x = 2.0 * fl[0], s2y = 2.0 * fl[1];
  const double nrm = __dsqrt_rn(__dadd_rn(__dmul_rn(s2x, s2x), __dmul_rn(s2y, s2y)));
  const double z = __ddiv_rn(1.0, __dadd_rn(nrm, 1e-3));
  zf = __double2float_rn(z);
  bool ok = isfinite(z);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    double wx, wy;
    warp_pos_exact(x, y, fl, e, wx, wy);
    const double fx = wx * 256.0, fy = wy * 256.0;
    ok = ok && isfinite(fx) && isfinite(fy) && fabs(fx) < 1073741824.0 && fabs(fy) < 1073741824.0;
    q[e].x = ok ? static_cast<int>(__double2ll_rn(fx)) : 0;
    q[e].y = ok ? static_cast<int>(__double2ll_rn(fy)) : 0;
  }
  return ok;
}

// deterministic warp sum (xor butterfly: every lane ends with the identical value)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

}  // namespace hwf
