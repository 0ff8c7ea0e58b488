// oracle/geometry.cpp — TEST INFRASTRUCTURE ONLY (parity checker).
//
// Restatement of the reference's geometry module (include/hwflow/geometry.hpp:14-59;
// SPEC.md:466-512). The header ships, geometry.cpp does not (CMakeLists.txt lists
// it; absent), so parity is pinned by SPEC.md's examples only. Pins:
//   G.1 triangulate_dlt: A = [x0 P0_2 - P0_0; y0 P0_2 - P0_1; x1 P1_2 - P1_0;
//       y1 P1_2 - P1_1], each row scaled to unit L2 norm (a zero row stays zero).
//       Null vector from a one-sided (Hestenes) Jacobi SVD of A: cyclic column
//       pairs (0,1),(0,2),(0,3),(1,2),(1,3),(2,3); a rotation is skipped when
//       |g| <= 1e-15 sqrt(a b) (a, b = squared column norms, g = their dot);
//       at most 30 sweeps; X_h = the column of V whose column of AV has the
//       smallest norm (lowest index on ties).
//   G.2 "near-parallel rays (condition number > 1e8) flagged invalid"
//       (SPEC.md:484): valid iff X_h is finite and |W| > 1e-8 ||X_h||, i.e. the
//       dehomogenisation condition ||X_h|| / |W| <= 1e8. Invalid points are 0.
//   G.3 triangulate_pixel(x, f, t): the correspondence (warp_position(x,f,0,t),
//       warp_position(x,f,1,t)) (warp_grid.hpp:74-77).
//   G.4 compute_scene_points: per pixel (x, y) of the dense flows; scene_flow =
//       points1 - points0; point_valid = valid(t=0) && valid(t=1); 0 if invalid.
//   G.5 StereoRig::validate: singular values of F (same Jacobi SVD) s1 >= s2 >=
//       s3: s1 > 0, s3 <= 1e-6 s1 and s2 > 1e-6 s1. With projections, the 8 test
//       points (+-1, +-1, 4 | 6) are projected by both cameras; a point with
//       |z_c| <= 1e-12 or an undefined epipolar line is skipped; the distance of
//       x0 to the line F x1 must be < 1e-6 px (x_0^T F x_1 = 0: energy.cpp:176-178).
//   G.6 export_mesh_obj: vertex for pixel p iff vis4[p] == 0xF and, with points,
//       point_valid[p] (else disparity[p] finite); position points0[p] or
//       (x, y, disparity[p]); vertices pixel-major; per lattice cell (row-major)
//       the UL {p(x,y), p(x+1,y), p(x,y+1)} and LR {p(x+1,y), p(x+1,y+1), p(x,y+1)}
//       triangles (occlusion's split, hierarchy.cpp C.2) when all three vertices exist.
//       Format: "v %.17g %.17g %.17g" and 1-based "f a b c".
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ctx.hpp"
#include "hwflow_c.h"

namespace {

void jacobi_svd4(double A[4][4], double V[4][4]) {  // G.1 (columns of A become A V)
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  static const int kp[6] = {0, 0, 0, 1, 1, 2}, kq[6] = {1, 2, 3, 2, 3, 3};
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int k = 0; k < 6; ++k) {
      const int p = kp[k], q = kq[k];
      double a = 0.0, b = 0.0, g = 0.0;
      for (int i = 0; i < 4; ++i) {
        a += A[i][p] * A[i][p];
        b += A[i][q] * A[i][q];
        g += A[i][p] * A[i][q];
      }
      if (std::fabs(g) <= 1e-15 * std::sqrt(a * b)) continue;
      rotated = true;
      const double zeta = (b - a) / (2.0 * g);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
      for (int i = 0; i < 4; ++i) {
        const double up = A[i][p], uq = A[i][q];
        A[i][p] = c * up - s * uq;
        A[i][q] = s * up + c * uq;
        const double vp = V[i][p], vq = V[i][q];
        V[i][p] = c * vp - s * vq;
        V[i][q] = s * vp + c * vq;
      }
    }
    if (!rotated) break;
  }
}

bool dlt(const double* P0, const double* P1, const double* x0, const double* x1, double X[3]) {
  double A[4][4];
  const double* Ps[2] = {P0, P1};
  const double* xs[2] = {x0, x1};
  for (int v = 0; v < 2; ++v)
    for (int k = 0; k < 2; ++k) {
      double* row = A[2 * v + k];
      double n2 = 0.0;
      for (int j = 0; j < 4; ++j) {
        row[j] = xs[v][k] * Ps[v][8 + j] - Ps[v][4 * k + j];
        n2 += row[j] * row[j];
      }
      if (n2 > 0.0) {
        const double inv = 1.0 / std::sqrt(n2);
        for (int j = 0; j < 4; ++j) row[j] *= inv;
      }
    }
  double V[4][4];
  jacobi_svd4(A, V);
  int best = 0;
  double bn = 0.0;
  for (int j = 0; j < 4; ++j) {
    double n2 = 0.0;
    for (int i = 0; i < 4; ++i) n2 += A[i][j] * A[i][j];
    if (j == 0 || n2 < bn) {
      bn = n2;
      best = j;
    }
  }
  double h[4], hn = 0.0;
  bool fin = true;
  for (int i = 0; i < 4; ++i) {
    h[i] = V[i][best];
    hn += h[i] * h[i];
    fin = fin && std::isfinite(h[i]);
  }
  hn = std::sqrt(hn);
  if (!fin || !(std::fabs(h[3]) > 1e-8 * hn)) {  // G.2
    X[0] = X[1] = X[2] = 0.0;
    return false;
  }
  for (int i = 0; i < 3; ++i) X[i] = h[i] / h[3];
  return std::isfinite(X[0]) && std::isfinite(X[1]) && std::isfinite(X[2]);
}

void singular_values3(const double* F, double s[3]) {  // G.5: same Jacobi on [F | 0]
  double A[4][4] = {};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[i][j] = F[3 * i + j];
  double V[4][4];
  jacobi_svd4(A, V);
  for (int j = 0; j < 3; ++j) {
    double n2 = 0.0;
    for (int i = 0; i < 4; ++i) n2 += A[i][j] * A[i][j];
    s[j] = std::sqrt(n2);
  }
  for (int i = 0; i < 3; ++i)  // descending
    for (int j = i + 1; j < 3; ++j)
      if (s[j] > s[i]) std::swap(s[i], s[j]);
}

void validate(const hwf_rig* rig) {
  if (!rig) throw std::invalid_argument("null rig");
  double s[3];
  singular_values3(rig->F, s);
  if (!(s[0] > 0.0) || !(s[2] <= 1e-6 * s[0]) || !(s[1] > 1e-6 * s[0]))
    throw std::invalid_argument("fundamental matrix must have rank 2");
  if (!rig->has_projections) return;
  for (int k = 0; k < 8; ++k) {
    const double X[4] = {(k & 1) ? 1.0 : -1.0, (k & 2) ? 1.0 : -1.0, (k & 4) ? 6.0 : 4.0, 1.0};
    double x[2][3];
    bool ok = true;
    for (int c = 0; c < 2; ++c) {
      const double* P = c ? rig->P1 : rig->P0;
      double h[3];
      for (int i = 0; i < 3; ++i) h[i] = P[4 * i] * X[0] + P[4 * i + 1] * X[1] + P[4 * i + 2] * X[2] + P[4 * i + 3] * X[3];
      if (std::fabs(h[2]) <= 1e-12) ok = false;
      x[c][0] = h[0] / h[2];
      x[c][1] = h[1] / h[2];
      x[c][2] = 1.0;
    }
    if (!ok) continue;
    double l[3];  // F x1
    for (int i = 0; i < 3; ++i) l[i] = rig->F[3 * i] * x[1][0] + rig->F[3 * i + 1] * x[1][1] + rig->F[3 * i + 2];
    const double ln = std::sqrt(l[0] * l[0] + l[1] * l[1]);
    if (!(ln > 0.0)) continue;
    const double dist = std::fabs(x[0][0] * l[0] + x[0][1] * l[1] + l[2]) / ln;
    if (!(dist < 1e-6)) throw std::invalid_argument("fundamental matrix inconsistent with the projections");
  }
}

template <class Fn>
int guard(hwf_ctx* ctx, Fn&& fn) {
  try {
    fn();
    return HWF_OK;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EINVAL;
  }
}

}  // namespace

extern "C" {

int hwf_validate_rig(hwf_ctx* ctx, const hwf_rig* rig) {
  return guard(ctx, [&] { validate(rig); });
}

int hwf_triangulate(hwf_ctx* ctx, int n, const double P0[12], const double P1[12], const double* x0,
                    const double* x1, double* X, uint8_t* valid) {
  return guard(ctx, [&] {
    if (n < 0 || !P0 || !P1 || (n > 0 && (!x0 || !x1 || !X))) throw std::invalid_argument("bad triangulation args");
    for (int i = 0; i < n; ++i) {
      const bool ok = dlt(P0, P1, x0 + 2 * i, x1 + 2 * i, X + 3 * i);
      if (valid) valid[i] = ok ? 1 : 0;
    }
  });
}

int hwf_scene_points(hwf_ctx* ctx, int w, int h, const double* s, const double* m, const double* d,
                     const hwf_rig* rig, double* points0, double* points1, double* scene_flow,
                     uint8_t* point_valid) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || !s || !m || !d || !rig) throw std::invalid_argument("bad scene-point args");
    if (!rig->has_projections) throw std::invalid_argument("scene points need projection matrices");
    const long long N = static_cast<long long>(w) * h;
    for (long long p = 0; p < N; ++p) {
      const double px = static_cast<double>(p % w), py = static_cast<double>(p / w);
      double pt[2][3];
      bool ok = true;
      for (int t = 0; t < 2; ++t) {  // G.3: warp_position, sigma_c = -1 for c = 0, sigma_t = -1 for t = 0
        const double st = t ? 1.0 : -1.0;
        const double x0[2] = {px - s[2 * p] + st * m[2 * p] - st * d[2 * p],
                              py - s[2 * p + 1] + st * m[2 * p + 1] - st * d[2 * p + 1]};
        const double x1[2] = {px + s[2 * p] + st * m[2 * p] + st * d[2 * p],
                              py + s[2 * p + 1] + st * m[2 * p + 1] + st * d[2 * p + 1]};
        ok = dlt(rig->P0, rig->P1, x0, x1, pt[t]) && ok;
      }
      for (int i = 0; i < 3; ++i) {
        if (!ok) pt[0][i] = pt[1][i] = 0.0;
        if (points0) points0[3 * p + i] = pt[0][i];
        if (points1) points1[3 * p + i] = pt[1][i];
        if (scene_flow) scene_flow[3 * p + i] = pt[1][i] - pt[0][i];
      }
      if (point_valid) point_valid[p] = ok ? 1 : 0;
    }
  });
}

int hwf_export_mesh_obj(hwf_ctx* ctx, int w, int h, const double* disparity, const uint8_t* vis4,
                        const double* points0, const uint8_t* point_valid, const char* path) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || !vis4 || !path) throw std::invalid_argument("bad mesh args");
    const bool pts = points0 && point_valid;
    if (!pts && !disparity) throw std::invalid_argument("mesh needs points or a disparity");
    FILE* f = std::fopen(path, "w");
    if (!f) throw std::invalid_argument(std::string("cannot open ") + path);
    const long long N = static_cast<long long>(w) * h;
    std::vector<long long> id(N, 0);
    long long nv = 0;
    std::fprintf(f, "# hwflow mesh %d x %d\n", w, h);
    for (long long p = 0; p < N; ++p) {  // G.6
      if (vis4[p] != 0x0F) continue;
      double v[3];
      if (pts) {
        if (!point_valid[p]) continue;
        v[0] = points0[3 * p];
        v[1] = points0[3 * p + 1];
        v[2] = points0[3 * p + 2];
      } else {
        if (!std::isfinite(disparity[p])) continue;
        v[0] = static_cast<double>(p % w);
        v[1] = static_cast<double>(p / w);
        v[2] = disparity[p];
      }
      id[p] = ++nv;
      std::fprintf(f, "v %.17g %.17g %.17g\n", v[0], v[1], v[2]);
    }
    for (int y = 0; y + 1 < h; ++y)
      for (int x = 0; x + 1 < w; ++x) {
        const long long a = id[static_cast<long long>(y) * w + x], b = id[static_cast<long long>(y) * w + x + 1];
        const long long c = id[static_cast<long long>(y + 1) * w + x], e = id[static_cast<long long>(y + 1) * w + x + 1];
        if (a && b && c) std::fprintf(f, "f %lld %lld %lld\n", a, b, c);
        if (b && e && c) std::fprintf(f, "f %lld %lld %lld\n", b, e, c);
      }
    const bool bad = std::ferror(f) != 0;
    if (std::fclose(f) != 0 || bad) throw std::invalid_argument(std::string("write failed: ") + path);
  });
}

}  // extern "C"
