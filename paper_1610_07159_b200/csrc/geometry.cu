// geometry.cu — dense geometry outputs on the device (§8f rank 2).
//
// The reference declares the geometry module (include/hwflow/geometry.hpp:14-59)
// but ships no geometry.cpp; the pins (DLT row scaling, the one-sided Jacobi null
// vector, the 1e-8 dehomogenisation condition, the OBJ layout) are stated once in
// oracle/geometry.cpp (G.1-G.6) and followed here.
//   k_triangulate   — triangulate_dlt (geometry.hpp:45-48), thread per correspondence.
//   k_scene_points  — compute_scene_points (geometry.hpp:50-54): thread per pixel,
//                     triangulate_pixel at t = 0 and t = 1, scene flow = difference.
// StereoRig::validate and export_mesh_obj are host-side checks / serial I/O.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hwflow_c.h"
#include "host.h"

using namespace hwf_host;

namespace {

// One-sided (Hestenes) Jacobi SVD of a 4x4: A <- A V (G.1).
__host__ __device__ inline void jacobi_svd4(double A[4][4], double V[4][4]) {
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int k = 0; k < 6; ++k) {
      const int p = k < 3 ? 0 : (k < 5 ? 1 : 2);
      const int q = k < 3 ? k + 1 : (k < 5 ? k - 1 : 3);
      double a = 0.0, b = 0.0, g = 0.0;
      for (int i = 0; i < 4; ++i) {
        a += A[i][p] * A[i][p];
        b += A[i][q] * A[i][q];
        g += A[i][p] * A[i][q];
      }
      if (fabs(g) <= 1e-15 * sqrt(a * b)) continue;
      rotated = true;
      const double zeta = (b - a) / (2.0 * g);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
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

// triangulate_dlt with unit-norm rows (G.1) and the 1e-8 condition (G.2).
__device__ bool dlt(const double* P0, const double* P1, double x0x, double x0y, double x1x, double x1y,
                    double X[3]) {
  double A[4][4];
  const double xs[4] = {x0x, x0y, x1x, x1y};
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double* P = r < 2 ? P0 : P1;
    const int k = r & 1;
    double n2 = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      A[r][j] = xs[r] * P[8 + j] - P[4 * k + j];
      n2 += A[r][j] * A[r][j];
    }
    if (n2 > 0.0) {
      const double inv = 1.0 / sqrt(n2);
#pragma unroll
      for (int j = 0; j < 4; ++j) A[r][j] *= inv;
    }
  }
  double V[4][4];
  jacobi_svd4(A, V);
  int best = 0;
  double bn = 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double n2 = A[0][j] * A[0][j] + A[1][j] * A[1][j] + A[2][j] * A[2][j] + A[3][j] * A[3][j];
    if (j == 0 || n2 < bn) {
      bn = n2;
      best = j;
    }
  }
  double h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = best == 0 ? V[i][0] : best == 1 ? V[i][1] : best == 2 ? V[i][2] : V[i][3];
  const double hn = sqrt(h[0] * h[0] + h[1] * h[1] + h[2] * h[2] + h[3] * h[3]);
  const bool fin = isfinite(h[0]) && isfinite(h[1]) && isfinite(h[2]) && isfinite(h[3]);
  if (!fin || !(fabs(h[3]) > 1e-8 * hn)) {
    X[0] = X[1] = X[2] = 0.0;
    return false;
  }
  X[0] = h[0] / h[3];
  X[1] = h[1] / h[3];
  X[2] = h[2] / h[3];
  return isfinite(X[0]) && isfinite(X[1]) && isfinite(X[2]);
}

struct Cams {
  double P0[12], P1[12];
};

__global__ void k_triangulate(int n, const Cams C, const double* __restrict__ x0, const double* __restrict__ x1,
                              double* __restrict__ X, uint8_t* __restrict__ valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[3];
  const bool ok = dlt(C.P0, C.P1, x0[2 * i], x0[2 * i + 1], x1[2 * i], x1[2 * i + 1], p);
  X[3 * i] = p[0];
  X[3 * i + 1] = p[1];
  X[3 * i + 2] = p[2];
  valid[i] = ok ? 1 : 0;
}

// triangulate_pixel at t = 0, 1 (G.3, G.4): warp_position (warp_grid.hpp:74-77),
// sigma_c = -1 for c = 0, sigma_t = -1 for t = 0.
__global__ void k_scene_points(int w, long long N, const Cams C, const double* __restrict__ s,
                               const double* __restrict__ m, const double* __restrict__ d,
                               double* __restrict__ p0, double* __restrict__ p1, double* __restrict__ sf,
                               uint8_t* __restrict__ valid) {
  const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (p >= N) return;
  const double px = static_cast<double>(p % w), py = static_cast<double>(p / w);
  const double sx = s[2 * p], sy = s[2 * p + 1], mx = m[2 * p], my = m[2 * p + 1], dx = d[2 * p], dy = d[2 * p + 1];
  double pt[2][3];
  bool ok = true;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double st = t ? 1.0 : -1.0;
    ok = dlt(C.P0, C.P1, px - sx + st * mx - st * dx, py - sy + st * my - st * dy, px + sx + st * mx + st * dx,
             py + sy + st * my + st * dy, pt[t]) && ok;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a = ok ? pt[0][i] : 0.0, b = ok ? pt[1][i] : 0.0;
    p0[3 * p + i] = a;
    p1[3 * p + i] = b;
    sf[3 * p + i] = b - a;
  }
  valid[p] = ok ? 1 : 0;
}

void validate_rig(const hwf_rig* rig) {  // G.5
  if (!rig) throw InvalidArg("null rig");
  double A[4][4] = {}, V[4][4];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[i][j] = rig->F[3 * i + j];
  jacobi_svd4(A, V);
  double sv[3];
  for (int j = 0; j < 3; ++j) sv[j] = std::sqrt(A[0][j] * A[0][j] + A[1][j] * A[1][j] + A[2][j] * A[2][j] + A[3][j] * A[3][j]);
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (sv[j] > sv[i]) std::swap(sv[i], sv[j]);
  if (!(sv[0] > 0.0) || !(sv[2] <= 1e-6 * sv[0]) || !(sv[1] > 1e-6 * sv[0]))
    throw InvalidArg("fundamental matrix must have rank 2");
  if (!rig->has_projections) return;
  for (int k = 0; k < 8; ++k) {
    const double X[4] = {(k & 1) ? 1.0 : -1.0, (k & 2) ? 1.0 : -1.0, (k & 4) ? 6.0 : 4.0, 1.0};
    double x[2][2];
    bool ok = true;
    for (int c = 0; c < 2; ++c) {
      const double* P = c ? rig->P1 : rig->P0;
      double h[3];
      for (int i = 0; i < 3; ++i) h[i] = P[4 * i] * X[0] + P[4 * i + 1] * X[1] + P[4 * i + 2] * X[2] + P[4 * i + 3] * X[3];
      if (std::fabs(h[2]) <= 1e-12) ok = false;
      x[c][0] = h[0] / h[2];
      x[c][1] = h[1] / h[2];
    }
    if (!ok) continue;
    double l[3];  // epipolar line of x1 in view 0: F x1 (x_0^T F x_1 = 0)
    for (int i = 0; i < 3; ++i) l[i] = rig->F[3 * i] * x[1][0] + rig->F[3 * i + 1] * x[1][1] + rig->F[3 * i + 2];
    const double ln = std::sqrt(l[0] * l[0] + l[1] * l[1]);
    if (!(ln > 0.0)) continue;
    if (!(std::fabs(x[0][0] * l[0] + x[0][1] * l[1] + l[2]) / ln < 1e-6))
      throw InvalidArg("fundamental matrix inconsistent with the projections");
  }
}

Cams cams(const double* P0, const double* P1) {
  Cams c;
  for (int i = 0; i < 12; ++i) {
    c.P0[i] = P0[i];
    c.P1[i] = P1[i];
  }
  return c;
}

template <class T>
T* upload(DevMem& m, const T* host, size_t n) {
  T* d = m.alloc<T>(n);
  CK(cudaMemcpy(d, host, n * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

}  // namespace

extern "C" {

int hwf_validate_rig(hwf_ctx* ctx, const hwf_rig* rig) {
  return guard(ctx, [&] { validate_rig(rig); });
}

int hwf_triangulate(hwf_ctx* ctx, int n, const double P0[12], const double P1[12], const double* x0,
                    const double* x1, double* X, uint8_t* valid) {
  return guard(ctx, [&] {
    if (n < 0 || !P0 || !P1 || (n > 0 && (!x0 || !x1 || !X))) throw InvalidArg("bad triangulation args");
    if (n == 0) return;
    DevMem m;
    const double* d0 = upload(m, x0, 2 * static_cast<size_t>(n));
    const double* d1 = upload(m, x1, 2 * static_cast<size_t>(n));
    double* dX = m.alloc<double>(3 * static_cast<size_t>(n));
    uint8_t* dv = m.alloc<uint8_t>(n);
    k_triangulate<<<(n + 127) / 128, 128, 0, ctx->stream>>>(n, cams(P0, P1), d0, d1, dX, dv);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(X, dX, 3 * sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (valid) CK(cudaMemcpy(valid, dv, n, cudaMemcpyDeviceToHost));
  });
}

int hwf_scene_points(hwf_ctx* ctx, int w, int h, const double* s, const double* m, const double* d,
                     const hwf_rig* rig, double* points0, double* points1, double* scene_flow,
                     uint8_t* point_valid) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || !s || !m || !d || !rig) throw InvalidArg("bad scene-point args");
    if (!rig->has_projections) throw InvalidArg("scene points need projection matrices");
    const size_t N = static_cast<size_t>(w) * h;
    DevMem mem;
    const double* ds = upload(mem, s, 2 * N);
    const double* dm = upload(mem, m, 2 * N);
    const double* dd = upload(mem, d, 2 * N);
    double* o = mem.alloc<double>(9 * N);
    uint8_t* dv = mem.alloc<uint8_t>(N);
    k_scene_points<<<static_cast<unsigned>((N + 127) / 128), 128, 0, ctx->stream>>>(
        w, static_cast<long long>(N), cams(rig->P0, rig->P1), ds, dm, dd, o, o + 3 * N, o + 6 * N, dv);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    if (points0) CK(cudaMemcpy(points0, o, 3 * N * sizeof(double), cudaMemcpyDeviceToHost));
    if (points1) CK(cudaMemcpy(points1, o + 3 * N, 3 * N * sizeof(double), cudaMemcpyDeviceToHost));
    if (scene_flow) CK(cudaMemcpy(scene_flow, o + 6 * N, 3 * N * sizeof(double), cudaMemcpyDeviceToHost));
    if (point_valid) CK(cudaMemcpy(point_valid, dv, N, cudaMemcpyDeviceToHost));
  });
}

// Serial host I/O ("export is serial"); layout pinned in oracle/geometry.cpp G.6.
int hwf_export_mesh_obj(hwf_ctx* ctx, int w, int h, const double* disparity, const uint8_t* vis4,
                        const double* points0, const uint8_t* point_valid, const char* path) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || !vis4 || !path) throw InvalidArg("bad mesh args");
    const bool pts = points0 && point_valid;
    if (!pts && !disparity) throw InvalidArg("mesh needs points or a disparity");
    FILE* f = std::fopen(path, "w");
    if (!f) throw InvalidArg(std::string("cannot open ") + path);
    const size_t N = static_cast<size_t>(w) * h;
    std::vector<long long> id(N, 0);
    long long nv = 0;
    std::fprintf(f, "# hwflow mesh %d x %d\n", w, h);
    for (size_t p = 0; p < N; ++p) {
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
        const size_t r0 = static_cast<size_t>(y) * w + x, r1 = r0 + w;
        const long long a = id[r0], b = id[r0 + 1], c = id[r1], e = id[r1 + 1];
        if (a && b && c) std::fprintf(f, "f %lld %lld %lld\n", a, b, c);
        if (b && e && c) std::fprintf(f, "f %lld %lld %lld\n", b, e, c);
      }
    const bool bad = std::ferror(f) != 0;
    if (std::fclose(f) != 0 || bad) throw InvalidArg(std::string("write failed: ") + path);
  });
}

}  // extern "C"
