// maps.cu — pyramid, occlusion, illumination, prolongation, dense output and
// the deterministic energy reduction.
//
// Bit-exact stages (pyramid, occlusion) round every operation explicitly
// (__dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn) in the reference's order so that
// they match the -ffp-contract=off CPU oracle bit for bit.
#include <cmath>

#include "launch.h"

namespace hwf {
namespace {

constexpr int kThreads = 256;
constexpr int kZbufSpanPx = 8;    // oracle/hierarchy.cpp pin C.2
constexpr double kDepthTol = 1e-4;

// ---- pyramid (image.cpp:100-122, 177-185) -----------------
__global__ void k_pyr_in(const void* __restrict__ src, int dtype, double* __restrict__ dst, long long n) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if (dtype == HWF_DTYPE_U8) {
    dst[i] = __ddiv_rn(static_cast<double>(static_cast<const uint8_t*>(src)[i]), 255.0);
  } else {
    const double v = static_cast<const double*>(src)[i];
    dst[i] = fmin(1.0, fmax(0.0, v));
  }
}

// Level 1 straight from u8 frames: the level-0 values k/255 (k_pyr_in) are rebuilt in
// registers and averaged exactly as k_pyr_down does, so level 0 is never materialised.
__global__ void k_pyr_down_u8(const uint8_t* __restrict__ src, int w, int h, double* __restrict__ dst, int ow,
                              int oh) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  const int plane = blockIdx.z;
  if (x >= ow) return;
  const uint8_t* S = src + static_cast<size_t>(plane) * w * h;
  // k/255 correctly rounded as fma(k, hi, k * lo), exhaustively checked (pixel.cu u8val)
  auto u8v = [](int k8) {
    const double k = static_cast<double>(k8);
    return __fma_rn(k, 1.0 / 255.0, __dmul_rn(k, 5.4633625097902372e-20));
  };
  if (2 * x + 1 < w && 2 * y + 1 < h) {  // all four taps, in the loop's order (0,0), (1,0), (0,1), (1,1)
    const uint8_t* r0 = S + static_cast<size_t>(2 * y) * w + 2 * x;
    const uint8_t* r1 = r0 + w;
    const int a = r0[0], b = r0[1], c = r1[0], d = r1[1];
    dst[static_cast<size_t>(plane) * ow * oh + static_cast<size_t>(y) * ow + x] =
        __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, u8v(a)), u8v(b)), u8v(c)), u8v(d)), 0.25);
    return;
  }
  double sum = 0.0;
  int cnt = 0;
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const int sx = 2 * x + dx, sy = 2 * y + dy;
      if (sx < w && sy < h) {
        sum = __dadd_rn(sum, u8v(S[static_cast<size_t>(sy) * w + sx]));
        ++cnt;
      }
    }
  // cnt is 1, 2 or 4: dividing by it is an exact scaling
  dst[static_cast<size_t>(plane) * ow * oh + static_cast<size_t>(y) * ow + x] =
      __dmul_rn(sum, cnt == 4 ? 0.25 : (cnt == 2 ? 0.5 : 1.0));
}

__global__ void k_pyr_down(const double* __restrict__ src, int w, int h, double* __restrict__ dst,
                           int ow, int oh) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  const int plane = blockIdx.z;
  if (x >= ow) return;
  const double* S = src + static_cast<size_t>(plane) * w * h;
  if (2 * x + 1 < w && 2 * y + 1 < h) {  // all four taps, in the loop's order
    const double* r0 = S + static_cast<size_t>(2 * y) * w + 2 * x;
    const double* r1 = r0 + w;
    const double a = r0[0], b = r0[1], c = r1[0], d = r1[1];
    dst[static_cast<size_t>(plane) * ow * oh + static_cast<size_t>(y) * ow + x] =
        __dmul_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(0.0, a), b), c), d), 0.25);
    return;
  }
  double sum = 0.0;
  int cnt = 0;
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const int sx = 2 * x + dx, sy = 2 * y + dy;
      if (sx < w && sy < h) {
        sum = __dadd_rn(sum, S[static_cast<size_t>(sy) * w + sx]);
        ++cnt;
      }
    }
  // sum / cnt (image.cpp:117) with cnt in {1, 2, 4}: an exact power-of-two scaling
  dst[static_cast<size_t>(plane) * ow * oh + static_cast<size_t>(y) * ow + x] =
      __dmul_rn(sum, cnt == 4 ? 0.25 : (cnt == 2 ? 0.5 : 1.0));
}

__global__ void k_init_coarse(double* base, double* total, double* delta, long long n_nodes, double ox, double oy) {
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= 6 * n_nodes) return;
  const int c = static_cast<int>(t % 6);
  const double v = c == 0 ? __dadd_rn(0.0, ox) : (c == 1 ? __dadd_rn(0.0, oy) : 0.0);
  base[t] = v;
  total[t] = v;
  delta[t] = 0.0;
}

// ---- occlusion (pin C.2 in oracle/hierarchy.cpp) ---------
__global__ void k_occ_project(int w, int h, int gw, int gh, int step, const double* __restrict__ total,
                              int2* __restrict__ q, float* __restrict__ Z, uint8_t* __restrict__ bad) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, pair = blockIdx.z;
  if (x >= w) return;
  const size_t N = static_cast<size_t>(w) * h, G = static_cast<size_t>(gw) * gh;
  const size_t pix = static_cast<size_t>(y) * w + x;
  double fl[6];
  interp_exact(total + pair * G * 6, gw, gh, step, x, y, fl);
  int2 v[4];
  float zf;
  const bool ok = occ_project_flow(x, y, fl, v, zf);
  Z[pair * N + pix] = zf;
#pragma unroll
  for (int e = 0; e < 4; ++e) q[(pair * 4 + e) * N + pix] = v[e];  // view-major: a triangle's vertices are contiguous
  bad[pair * N + pix] = ok ? 0 : 1;
}

// Vertices in 1/256 px fixed point, |coordinate| < 2^30 (k_occ_project), so every box
// extent is exact as a 32-bit unsigned difference.
struct Tri {
  int X[3], Y[3];
  int mnx, mxx, mny, mxy;
};

// Vertices of triangle `tri` of the halfway lattice in view e (pin C.2).
__device__ __forceinline__ void tri_vertices(int w, long long tri, int& v0, int& v1, int& v2) {
  const int cw = w - 1, t = static_cast<int>(tri & 1);
  const int cell = static_cast<int>(tri >> 1), cx = cell % cw, cy = cell / cw;
  v0 = t == 0 ? cy * w + cx : cy * w + cx + 1;
  v1 = t == 0 ? cy * w + cx + 1 : (cy + 1) * w + cx + 1;
  v2 = (cy + 1) * w + cx;
}

__device__ __forceinline__ void make_tri(int2 p0, int2 p1, int2 p2, Tri& T) {
  T.X[0] = p0.x; T.X[1] = p1.x; T.X[2] = p2.x;
  T.Y[0] = p0.y; T.Y[1] = p1.y; T.Y[2] = p2.y;
  T.mnx = min(T.X[0], min(T.X[1], T.X[2]));
  T.mxx = max(T.X[0], max(T.X[1], T.X[2]));
  T.mny = min(T.Y[0], min(T.Y[1], T.Y[2]));
  T.mxy = max(T.Y[0], max(T.Y[1], T.Y[2]));
}

// Coverage of one pixel row, two exact forms of the same integer test (pin C.2):
// edge i is satisfied at pixel centre Px iff E_i = dx_i (Py - Y_i) - dy_i (Px - X_i)
// is > 0, or == 0 on a top-left edge (dy > 0, or dy == 0 and dx < 0). Inside a
// <= 8 px box, coordinates relative to the box origin keep every product and
// sum below 2^31, so int32 is exact.
//
// (a) small boxes: incremental E_i along the row, one test per pixel.
struct RowEdges {
  int E[3], step[3];
  bool tl[3];
};
__device__ __forceinline__ void raster_row_tests(const Tri& T, int yy, int x0, int x1, int w,
                                                 unsigned long long* zb, unsigned long long key) {
  RowEdges R;
  const int Px0 = x0 * 256, Py = yy * 256;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3;
    const int dx = T.X[j] - T.X[i], dy = T.Y[j] - T.Y[i];
    R.E[i] = dx * (Py - T.Y[i]) - dy * (Px0 - T.X[i]);
    R.step[i] = -256 * dy;
    R.tl[i] = dy > 0 || (dy == 0 && dx < 0);
  }
  unsigned long long* row = zb + static_cast<size_t>(yy) * w;
  for (int xx = x0; xx <= x1; ++xx) {
    bool in = true;
#pragma unroll
    for (int i = 0; i < 3; ++i) in = in && (R.E[i] > 0 || (R.E[i] == 0 && R.tl[i]));
#ifdef HWF_DIAG_RASTER_NO_ATOMIC  // diagnostic A/B only (wrong results): coverage without the z-buffer atomics
    if (in && key == 0) row[xx] = key;
#else
    if (in) atomicMin(row + xx, key);
#endif
#pragma unroll
    for (int i = 0; i < 3; ++i) R.E[i] += R.step[i];
  }
}

// (b) large boxes: solve each edge inequality for the covered x-interval, with
// xx' = xx - x0 and A'_i = dx_i (Py - Y_i) + dy_i (X_i - 256 x0):
//   dy > 0 (top-left):  E >= 0  <=>  xx' <= floor(A' / (256 dy))
//   dy < 0:             E >  0  <=>  xx' >= floor(-A' / (256 |dy|)) + 1
//   dy == 0:            row-constant test.
__device__ __forceinline__ int floordiv32(int a, int b) {  // b > 0
  int q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}
__device__ __forceinline__ void raster_row_span(const Tri& T, int yy, int x0, int x1, int w,
                                                unsigned long long* zb, unsigned long long key) {
  int lo = 0, hi = x1 - x0;
  const int Px0 = x0 * 256, Py = yy * 256;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3;
    const int dx = T.X[j] - T.X[i], dy = T.Y[j] - T.Y[i];
    const int A = dx * (Py - T.Y[i]) + dy * (T.X[i] - Px0);
    if (dy > 0) {
      hi = min(hi, floordiv32(A, 256 * dy));
    } else if (dy < 0) {
      lo = max(lo, floordiv32(-A, -256 * dy) + 1);
    } else if (!(A > 0 || (A == 0 && dx < 0))) {
      hi = lo - 1;
    }
  }
  unsigned long long* row = zb + static_cast<size_t>(yy) * w + x0;
  for (int k = lo; k <= hi; ++k) atomicMin(row + k, key);
}

constexpr int kSmallBoxPx = 16;  // triangles whose pixel box exceeds this go to the warp queue

// One triangle: degeneracy test, flat depth key, in-thread raster of small
// boxes, queue for large boxes. Returns whether the triangle is degenerate.
__device__ __forceinline__ bool raster_tri(int w, int h, const Tri& T, bool any_bad, float zf, unsigned int tri,
                                           unsigned long long* zb, unsigned long long* queue,
                                           unsigned int* qcount, unsigned long long qtag) {
  constexpr unsigned kSpan = kZbufSpanPx * 256;
  if (any_bad || static_cast<unsigned>(T.mxx - T.mnx) > kSpan || static_cast<unsigned>(T.mxy - T.mny) > kSpan)
    return true;
  // within an 8 px box every difference is <= 2^11, so the cross product is exact in int32
  const int area = (T.X[1] - T.X[0]) * (T.Y[2] - T.Y[0]) - (T.Y[1] - T.Y[0]) * (T.X[2] - T.X[0]);
  if (area <= 0) return true;
  const int x0 = max(0, -((-T.mnx) >> 8)), x1 = min(w - 1, T.mxx >> 8);
  const int y0 = max(0, -((-T.mny) >> 8)), y1 = min(h - 1, T.mxy >> 8);
  if (x1 < x0 || y1 < y0) return false;
  if ((x1 - x0 + 1) * (y1 - y0 + 1) > kSmallBoxPx) {
    queue[atomicAdd(qcount, 1u)] = qtag | tri;
    return false;
  }
  const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(zf)) << 32) | tri;
  for (int yy = y0; yy <= y1; ++yy) raster_row_tests(T, yy, x0, x1, w, zb, key);
  return false;
}

// One thread per (lattice cell, view, pair): both triangles of the cell (pin C.2),
// UL {(x,y),(x+1,y),(x,y+1)} then LR {(x+1,y),(x+1,y+1),(x,y+1)}, sharing 4 vertices.
// atomicMin on (depth bits, triangle id) makes the z-buffer order-independent.
__global__ void k_occ_raster(int w, int h, const int2* __restrict__ q, const float* __restrict__ Z,
                             const uint8_t* __restrict__ bad, unsigned long long* __restrict__ zbuf,
                             uint8_t* __restrict__ degen, unsigned long long* __restrict__ queue,
                             unsigned int* __restrict__ qcount) {
  const int cw = w - 1;
  const int cx = blockIdx.x * blockDim.x + threadIdx.x, cy = blockIdx.y, pair = blockIdx.z;
  if (cx >= cw) return;
  const size_t N = static_cast<size_t>(w) * h;
  const int i00 = cy * w + cx, i10 = i00 + 1, i01 = i00 + w, i11 = i01 + 1;
  const uint8_t* B = bad + pair * N;
  const float* ZZ = Z + pair * N;
  const bool b00 = B[i00], b10 = B[i10], b01 = B[i01], b11 = B[i11];
  const float z00 = ZZ[i00], z10 = ZZ[i10], z01 = ZZ[i01], z11 = ZZ[i11];
  const bool bad0 = b00 || b10 || b01, bad1 = b10 || b11 || b01;
  const float zf0 = fminf(z00, fminf(z10, z01)), zf1 = fminf(z10, fminf(z11, z01));  // flat depth per triangle
  const unsigned int tri0 = static_cast<unsigned int>(2 * (cy * cw + cx));
  // view e + 1's vertices load while view e rasterises (the compiler cannot move them above the
  // z-buffer atomics itself)
  const int2* Q0 = q + static_cast<size_t>(pair) * 4 * N;
  int2 n00 = Q0[i00], n10 = Q0[i10], n01 = Q0[i01], n11 = Q0[i11];
#pragma unroll 1
  for (int e = 0; e < 4; ++e) {  // the 4 views share the cell's depth and validity
    const int2 p00 = n00, p10 = n10, p01 = n01, p11 = n11;
    if (e < 3) {
      const int2* Qn = q + (static_cast<size_t>(pair) * 4 + e + 1) * N;
      n00 = Qn[i00];
      n10 = Qn[i10];
      n01 = Qn[i01];
      n11 = Qn[i11];
    }
    unsigned long long* zb = zbuf + (static_cast<size_t>(pair) * 4 + e) * N;
    const unsigned long long qtag =
        (static_cast<unsigned long long>(pair) << 34) | (static_cast<unsigned long long>(e) << 32);
    Tri T;
    make_tri(p00, p10, p01, T);
    const bool d0 = raster_tri(w, h, T, bad0, zf0, tri0, zb, queue, qcount, qtag);
    degen[(static_cast<size_t>(pair) * 4 + e) * N + i00] = d0 ? 1 : 0;
    make_tri(p10, p11, p01, T);
    raster_tri(w, h, T, bad1, zf1, tri0 + 1, zb, queue, qcount, qtag);
  }
}

// Thread per (queued large triangle, pixel row of its box): boxes are at most
// kZbufSpanPx + 1 rows tall (larger ones are degenerate), so a triangle's rows
// are consecutive work items.
__global__ void k_occ_raster_big(int w, int h, const int2* __restrict__ q, const float* __restrict__ Z,
                                 unsigned long long* __restrict__ zbuf, const unsigned long long* __restrict__ queue,
                                 const unsigned int* __restrict__ qcount) {
  constexpr int kRows = kZbufSpanPx + 1;
  const unsigned int n = *qcount;
  const size_t N = static_cast<size_t>(w) * h;
  const unsigned long long items = static_cast<unsigned long long>(n) * kRows;
  for (unsigned long long it = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; it < items;
       it += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned int i = static_cast<unsigned int>(it / kRows);
    const int row = static_cast<int>(it % kRows);
    const unsigned long long item = queue[i];
    const int pair = static_cast<int>(item >> 34), e = static_cast<int>((item >> 32) & 3);
    const long long tri = static_cast<long long>(item & 0xffffffffULL);
    int v0, v1, v2;
    tri_vertices(w, tri, v0, v1, v2);
    const int2* Q = q + (static_cast<size_t>(pair) * 4 + e) * N;
    Tri T;
    make_tri(Q[v0], Q[v1], Q[v2], T);
    const float* ZZ = Z + pair * N;
    const float zf = fminf(ZZ[v0], fminf(ZZ[v1], ZZ[v2]));
    const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(zf)) << 32) |
                                   static_cast<unsigned int>(tri);
    const int x0 = max(0, -((-T.mnx) >> 8)), x1 = min(w - 1, T.mxx >> 8);
    const int y0 = max(0, -((-T.mny) >> 8)), y1 = min(h - 1, T.mxy >> 8);
    unsigned long long* zb = zbuf + (static_cast<size_t>(pair) * 4 + e) * N;
    if (y0 + row <= y1) raster_row_span(T, y0 + row, x0, x1, w, zb, key);
  }
}

__global__ void k_occ_resolve(int w, int h, const int2* __restrict__ q, const float* __restrict__ Z,
                              const uint8_t* __restrict__ bad, const unsigned long long* __restrict__ zbuf,
                              const uint8_t* __restrict__ degen, uint8_t* __restrict__ vis) {
  const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y, pair = blockIdx.z;
  if (px >= w) return;
  const size_t N = static_cast<size_t>(w) * h;
  const size_t pix = static_cast<size_t>(py) * w + px;
  const int cw = w - 1;
  uint8_t bits = 0;
  const bool b = bad[pair * N + pix] != 0;
  if (w < 2 || h < 2) {
    vis[pair * N + pix] = b ? 0 : 0x0F;
    return;
  }
  const double zown = static_cast<double>(Z[pair * N + pix]);
  // ids of the six triangles incident to x (pin C.2): UL of cells (px,py), (px-1,py), (px,py-1) and LR of
  // (px-1,py), (px-1,py-1), (px,py-1); a cell outside the lattice gets an id no triangle has
  const int chh = h - 1;
  auto cell_id = [&](int cx, int cy, unsigned t) -> unsigned {
    return (cx >= 0 && cx < cw && cy >= 0 && cy < chh) ? 2u * static_cast<unsigned>(cy * cw + cx) + t : 0xFFFFFFFFu;
  };
  const unsigned inc[6] = {cell_id(px, py, 0), cell_id(px - 1, py, 0), cell_id(px, py - 1, 0),
                            cell_id(px - 1, py, 1), cell_id(px - 1, py - 1, 1), cell_id(px, py - 1, 1)};
  // all four views' loads first (vertex, then its z-buffer key), decisions after: the eight
  // dependent loads overlap instead of running view by view
  const bool inner = px < w - 1 && py < h - 1;
  int2 qq[4];
  bool dg[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const size_t o = (static_cast<size_t>(pair) * 4 + e) * N + pix;
    qq[e] = q[o];
    dg[e] = inner && degen[o];
  }
  unsigned long long key[4];
  bool inr[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const long long rx = (static_cast<long long>(qq[e].x) + 128) >> 8, ry = (static_cast<long long>(qq[e].y) + 128) >> 8;
    inr[e] = rx >= 0 && rx < w && ry >= 0 && ry < h;
    key[e] = zbuf[(static_cast<size_t>(pair) * 4 + e) * N + (inr[e] ? ry * w + rx : 0)];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    bool v = !b && !dg[e];
    if (v && inr[e] && key[e] != ~0ULL) {
      const unsigned int tri = static_cast<unsigned int>(key[e] & 0xffffffffULL);
      const bool ring = tri == inc[0] || tri == inc[1] || tri == inc[2] || tri == inc[3] || tri == inc[4] || tri == inc[5];
      if (!ring) {
        const float zf = __uint_as_float(static_cast<unsigned int>(key[e] >> 32));
        if (__dadd_rn(zown, -kDepthTol) > static_cast<double>(zf)) v = false;
      }
    }
    if (v) bits |= static_cast<uint8_t>(1u << e);
  }
  vis[pair * N + pix] = bits;
}

// ---- illumination (pin C.4) ------------------------------
__constant__ double c_gauss[32];
__constant__ int c_gauss_r;

__global__ void k_illum_resid(int w, int h, int gw, int gh, int step, const double* __restrict__ img,
                              const double* __restrict__ total, const uint8_t* __restrict__ vis,
                              double* __restrict__ resid) {
  const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y, pair = blockIdx.z;
  if (px >= w) return;
  const size_t N = static_cast<size_t>(w) * h, G = static_cast<size_t>(gw) * gh;
  const size_t pix = static_cast<size_t>(py) * w + px;
  const uint8_t v4 = vis[pair * N + pix];
  double fl[6];
  interp_fast(total + pair * G * 6, gw, gh, step, px, py, fl);
  for (int t = 0; t < 2; ++t) {
    const int e1 = 1 + 2 * t, e0 = 2 * t;
    double r = 0.0;
    if (((v4 >> e1) & 1) && ((v4 >> e0) & 1)) {
      Samp s1, s0;
      const double st = t ? 1.0 : -1.0;
      // warp_position (c=1,t) and (c=0,t)
      sample_img<false, false>(img + (pair * 4 + e1) * N, w, h, px + fl[0] + st * fl[2] + st * fl[4],
                               py + fl[1] + st * fl[3] + st * fl[5], s1);
      sample_img<false, false>(img + (pair * 4 + e0) * N, w, h, px - fl[0] + st * fl[2] - st * fl[4],
                               py - fl[1] + st * fl[3] - st * fl[5], s0);
      r = s1.v - s0.v;
    }
    resid[(pair * 2 + t) * N + pix] = r;
  }
}

// Separable Gaussian (image.cpp:124-155), taps summed in the reference's order i = -R..R.
// The radius is pinned (sigma 3.2 -> R = 10), so the tap loop is unrolled; R_ < 0 reads it at run time.
constexpr int kBlurR = 10;
int g_gauss_r = -1;  // host copy of c_gauss_r (init_maps_constants)
template <int R_>
__global__ void k_blur_h(int w, int h, const double* __restrict__ src, double* __restrict__ dst) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, plane = blockIdx.z;
  if (x >= w) return;
  const double* S = src + static_cast<size_t>(plane) * w * h + static_cast<size_t>(y) * w;
  const int R = R_ >= 0 ? R_ : c_gauss_r;
  double acc = 0.0;
#pragma unroll
  for (int i = -R; i <= R; ++i) acc += c_gauss[i + R] * __ldg(S + min(max(x + i, 0), w - 1));
  dst[static_cast<size_t>(plane) * w * h + static_cast<size_t>(y) * w + x] = acc;
}

template <int R_>
__global__ void k_blur_v_half(int w, int h, const double* __restrict__ src, double* __restrict__ dst) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, plane = blockIdx.z;
  if (x >= w) return;
  const double* S = src + static_cast<size_t>(plane) * w * h;
  const int R = R_ >= 0 ? R_ : c_gauss_r;
  double acc = 0.0;
#pragma unroll
  for (int i = -R; i <= R; ++i) acc += c_gauss[i + R] * __ldg(S + static_cast<size_t>(min(max(y + i, 0), h - 1)) * w + x);
  dst[static_cast<size_t>(plane) * w * h + static_cast<size_t>(y) * w + x] = 0.5 * acc;  // +-blur/2 split
}

// The pinned radius, K outputs per thread from a register window of K + 2R inputs (the same FMA sequence per
// output as k_blur_h / k_blur_v_half, so the same doubles), instead of 2R + 1 loads per output.
// Horizontal: a warp stages a row segment of 32 K outputs plus the 2R halo in shared memory (one pad double per
// K, so the lanes' K-strided window reads are conflict-free), warps over flattened (row, segment) items;
// 160-wide segments fit the 320 / 160 px levels exactly. Vertical: a thread walks kBlurK rows of its column,
// loads coalesced across the warp.
constexpr int kBlurK = 8, kBlurHK = 5, kBlurWarps = 4;  // vertical / horizontal outputs per thread
template <int R>
__global__ void __launch_bounds__(32 * kBlurWarps) k_blur_h_win(int w, int h, int segs, int items,
                                                                const double* __restrict__ src,
                                                                double* __restrict__ dst) {
  constexpr int K = kBlurHK, kSpan = 32 * K + 2 * R, kPitch = kSpan + kSpan / K + 1;
  __shared__ double sm[kBlurWarps][kPitch];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, plane = blockIdx.y;
  const int item = blockIdx.x * kBlurWarps + wi;  // (row, segment of 32 K outputs) of this warp
  if (item >= items) return;  // the whole warp
  const int y = item / segs, seg0 = (item - y * segs) * 32 * K;
  const double* S = src + static_cast<size_t>(plane) * w * h + static_cast<size_t>(y) * w;
  for (int j = lane; j < kSpan; j += 32) sm[wi][j + j / K] = __ldg(S + min(max(seg0 - R + j, 0), w - 1));
  __syncwarp();
  double v[K + 2 * R];
#pragma unroll
  for (int t = 0; t < K + 2 * R; ++t) {
    const int j = lane * K + t;
    v[t] = sm[wi][j + j / K];
  }
  double o[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int i = -R; i <= R; ++i) acc += c_gauss[i + R] * v[k + i + R];
    o[k] = acc;
  }
  // through the same shared row, so the stores are coalesced
  __syncwarp();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = lane * K + k;
    sm[wi][j + j / K] = o[k];
  }
  __syncwarp();
  double* D = dst + static_cast<size_t>(plane) * w * h + static_cast<size_t>(y) * w;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = k * 32 + lane, x = seg0 + j;
    if (x < w) D[x] = sm[wi][j + j / K];
  }
}
template <int R>
__global__ void k_blur_v_half_win(int w, int h, const double* __restrict__ src, double* __restrict__ dst) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y0 = blockIdx.y * kBlurK, plane = blockIdx.z;
  if (x >= w) return;
  const double* S = src + static_cast<size_t>(plane) * w * h + x;
  double v[kBlurK + 2 * R];
#pragma unroll
  for (int t = 0; t < kBlurK + 2 * R; ++t) v[t] = __ldg(S + static_cast<size_t>(min(max(y0 - R + t, 0), h - 1)) * w);
  double* D = dst + static_cast<size_t>(plane) * w * h + x;
#pragma unroll
  for (int k = 0; k < kBlurK; ++k) {
    double acc = 0.0;
#pragma unroll
    for (int i = -R; i <= R; ++i) acc += c_gauss[i + R] * v[k + i + R];
    if (y0 + k < h) D[static_cast<size_t>(y0 + k) * w] = 0.5 * acc;  // +-blur/2 split
  }
}

// ---- prolongation (pins C.1/C.3/C.4) ---------------------
__global__ void k_prolong_grid(int gwc, int ghc, int gwf, int ghf, int step, const double* __restrict__ tc,
                               double* __restrict__ base, double* __restrict__ total, double* __restrict__ delta) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, pair = blockIdx.y;
  const int Gf = gwf * ghf, Gc = gwc * ghc;
  if (k >= Gf) return;
  const double xmax = static_cast<double>(gwc - 1) * step, ymax = static_cast<double>(ghc - 1) * step;
  const double x = fmin(__ddiv_rn(static_cast<double>((k % gwf) * step), 2.0), xmax);
  const double y = fmin(__ddiv_rn(static_cast<double>((k / gwf) * step), 2.0), ymax);
  double fl[6];
  interp_exact(tc + static_cast<size_t>(pair) * Gc * 6, gwc, ghc, step, x, y, fl);
  const size_t o = (static_cast<size_t>(pair) * Gf + k) * 6;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const double v = 2.0 * fl[c];
    base[o + c] = v;
    total[o + c] = __dadd_rn(v, 0.0);
    delta[o + c] = 0.0;
  }
}

__global__ void k_prolong_maps(int wc, int hc, int wf, int hf, const uint8_t* __restrict__ vc,
                               const double* __restrict__ hmc, uint8_t* __restrict__ vf, double* __restrict__ illf) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, pair = blockIdx.z;
  if (x >= wf) return;
  const size_t Nc = static_cast<size_t>(wc) * hc, Nf = static_cast<size_t>(wf) * hf;
  const size_t pix = static_cast<size_t>(y) * wf + x;
  const uint8_t* V = vc + pair * Nc;
  // cell_coord(x / 2, wc) (image.cpp:19-31) in integers: x / 2 leaves fractions in {0, 1/2, 1}, so with
  // f2 = 2 f the bilinear weights are quarters and the test sum >= 0.5 is exact: 4 * sum >= 2 (pin C.3)
  auto half_coord = [](int v, int n, int& i0, int& f2) {
    if (n == 1 || v == 0) {  // v / 2 <= 0 (or a single column): cell 0, f = 0
      i0 = 0;
      f2 = 0;
    } else if (v >= 2 * (n - 1)) {  // v / 2 >= n - 1: cell n - 2, f = 1
      i0 = n - 2;
      f2 = 2;
    } else {
      i0 = v >> 1;
      f2 = v & 1;
    }
  };
  int cx0, fx2, cy0, fy2;
  half_coord(x, wc, cx0, fx2);
  half_coord(y, hc, cy0, fy2);
  const int x1 = min(cx0 + 1, wc - 1), y1 = min(cy0 + 1, hc - 1);
  const uint8_t* R0 = V + cy0 * wc;
  const uint8_t* R1 = V + y1 * wc;
  const uint8_t q00 = R0[cx0], q10 = R0[x1], q01 = R1[cx0], q11 = R1[x1];
  const int w00 = (2 - fx2) * (2 - fy2), w10 = fx2 * (2 - fy2), w01 = (2 - fx2) * fy2, w11 = fx2 * fy2;
  uint8_t bits = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int v4 = w00 * ((q00 >> e) & 1) + w10 * ((q10 >> e) & 1) + w01 * ((q01 >> e) & 1) + w11 * ((q11 >> e) & 1);
    if (v4 >= 2) bits |= static_cast<uint8_t>(1u << e);
  }
  vf[pair * Nf + pix] = bits;
  if (hmc && illf) {
    const size_t cpix = static_cast<size_t>(min(y / 2, hc - 1)) * wc + min(x / 2, wc - 1);
    const double h0 = hmc[(pair * 2 + 0) * Nc + cpix], h1 = hmc[(pair * 2 + 1) * Nc + cpix];
    illf[(pair * 4 + 0) * Nf + pix] = h0;
    illf[(pair * 4 + 1) * Nf + pix] = -h0;
    illf[(pair * 4 + 2) * Nf + pix] = h1;
    illf[(pair * 4 + 3) * Nf + pix] = -h1;
  }
}

// The masks alone (the pipeline: illumination is read from the coarse half maps by k_pixel), kProlongPx fine
// pixels of a row per thread: the row's coarse coordinates and byte rows are shared, one 32-bit store when the
// row allows it. Same integer arithmetic as k_prolong_maps.
constexpr int kProlongPx = 4;
__global__ void k_prolong_vis(int wc, int hc, int wf, int hf, const uint8_t* __restrict__ vc, uint8_t* __restrict__ vf) {
  const int x4 = kProlongPx * (blockIdx.x * blockDim.x + threadIdx.x), y = blockIdx.y, pair = blockIdx.z;
  if (x4 >= wf) return;
  const size_t Nc = static_cast<size_t>(wc) * hc, Nf = static_cast<size_t>(wf) * hf;
  int cy0, fy2;
  if (hc == 1 || y == 0) {
    cy0 = 0;
    fy2 = 0;
  } else if (y >= 2 * (hc - 1)) {
    cy0 = hc - 2;
    fy2 = 2;
  } else {
    cy0 = y >> 1;
    fy2 = y & 1;
  }
  const int y1 = min(cy0 + 1, hc - 1);
  const uint8_t* R0 = vc + pair * Nc + cy0 * wc;
  const uint8_t* R1 = vc + pair * Nc + y1 * wc;
  uint32_t packed = 0;
#pragma unroll
  for (int k = 0; k < kProlongPx; ++k) {
    const int x = x4 + k;
    int cx0, fx2;
    if (wc == 1 || x == 0) {
      cx0 = 0;
      fx2 = 0;
    } else if (x >= 2 * (wc - 1)) {
      cx0 = wc - 2;
      fx2 = 2;
    } else {
      cx0 = x >> 1;
      fx2 = x & 1;
    }
    const int x1 = min(cx0 + 1, wc - 1);
    const uint32_t q00 = R0[cx0], q10 = R0[x1], q01 = R1[cx0], q11 = R1[x1];
    // the quarter weights (2 - fx2, fx2) x (2 - fy2, fy2) make "4 * sum >= 2" a bitwise vote over the four masks:
    // one corner of weight 4 (fx2, fy2 even), two of weight 2 (either one), or four of weight 1 (at least two)
    uint32_t bits;
    if (fx2 == 1 && fy2 == 1) {
      bits = (q00 & q10) | (q01 & q11) | ((q00 | q10) & (q01 | q11));
    } else if (fx2 == 1) {
      bits = fy2 == 2 ? (q01 | q11) : (q00 | q10);
    } else if (fy2 == 1) {
      bits = fx2 == 2 ? (q10 | q11) : (q00 | q01);
    } else {
      bits = fx2 == 2 ? (fy2 == 2 ? q11 : q10) : (fy2 == 2 ? q01 : q00);
    }
    packed |= (bits & 0xFu) << (8 * k);
  }
  uint8_t* out = vf + pair * Nf + static_cast<size_t>(y) * wf + x4;
  if (x4 + kProlongPx <= wf && (reinterpret_cast<uintptr_t>(out) & 3) == 0) {
    *reinterpret_cast<uint32_t*>(out) = packed;
  } else {
    for (int k = 0; k < kProlongPx && x4 + k < wf; ++k) out[k] = static_cast<uint8_t>(packed >> (8 * k));
  }
}

// ---- temporal propagation (pin in oracle/hierarchy.cpp) ---
// next_delta(p) = prev_delta(p - 2 m_prev(p)) (exact bilinear, zero outside the
// lattice); total = base + delta.
__global__ void k_propagate(int gw, int gh, int step, const double* __restrict__ pd, const double* __restrict__ pt,
                            const double* __restrict__ base, double* __restrict__ delta, double* __restrict__ total) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, pair = blockIdx.y;
  const int G = gw * gh;
  if (k >= G) return;
  const size_t o = (static_cast<size_t>(pair) * G + k) * 6;
  const double px = static_cast<double>((k % gw) * step), py = static_cast<double>((k / gw) * step);
  const double qx = __dadd_rn(px, -__dmul_rn(2.0, pt[o + 2])), qy = __dadd_rn(py, -__dmul_rn(2.0, pt[o + 3]));
  const double xmax = static_cast<double>(gw - 1) * step, ymax = static_cast<double>(gh - 1) * step;
  double fl[6] = {0, 0, 0, 0, 0, 0};
  if (qx >= 0.0 && qy >= 0.0 && qx <= xmax && qy <= ymax) interp_exact(pd + static_cast<size_t>(pair) * G * 6, gw, gh, step, qx, qy, fl);
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    delta[o + c] = fl[c];
    if (base) total[o + c] = __dadd_rn(base[o + c], fl[c]);
  }
}

// ---- FlowResult (geometry.hpp:26-37) via WarpGrid::interpolate ------------
__global__ void k_dense(int w, int h, int gw, int gh, int step, const double* __restrict__ total,
                        double* s_out, double* m_out, double* d_out, double* disp_out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, pair = blockIdx.z;
  if (x >= w) return;
  const size_t N = static_cast<size_t>(w) * h, G = static_cast<size_t>(gw) * gh;
  const size_t pix = pair * N + static_cast<size_t>(y) * w + x;
  double fl[6];
  interp_exact(total + pair * G * 6, gw, gh, step, x, y, fl);
  if (s_out) { s_out[2 * pix] = fl[0]; s_out[2 * pix + 1] = fl[1]; }
  if (m_out) { m_out[2 * pix] = fl[2]; m_out[2 * pix + 1] = fl[3]; }
  if (d_out) { d_out[2 * pix] = fl[4]; d_out[2 * pix + 1] = fl[5]; }
  if (disp_out) disp_out[pix] = 2.0 * fl[0];
}

// ---- energy partials -> per (pair, slot) breakdown, fixed order -----------
// CTA per (pair, slot): thread t sums partials t, t + 256, ... in order, then fixed xor trees within
// the warps and warp 0 over the 8 warp sums: deterministic and independent of scheduling. (A single
// warp per slot took 2.5 ms at 4K, where a slot holds ~160k partials.)
constexpr int kReduceThreads = 256;
__global__ void __launch_bounds__(kReduceThreads) k_energy_reduce(const double* __restrict__ ep, int nslots, int cap,
                                                                  int B, double* out, int* flags,
                                                                  const int* __restrict__ counts) {
  __shared__ double red[kReduceThreads / 32][kNumEnergy];
  const int t = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = t / nslots;
  const double* p = ep + static_cast<size_t>(t) * cap * kNumEnergy;
  double s[kNumEnergy] = {0, 0, 0, 0, 0};
  const int n = counts ? counts[t % nslots] : cap;  // entries past a slot's count are the zeros of the reset
  for (int i = threadIdx.x; i < n; i += kReduceThreads)
#pragma unroll
    for (int k = 0; k < kNumEnergy; ++k) s[k] += p[i * kNumEnergy + k];
#pragma unroll
  for (int k = 0; k < kNumEnergy; ++k) s[k] = warp_sum(s[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < kNumEnergy; ++k) red[warp][k] = s[k];
  __syncthreads();
  if (warp == 0) {
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kNumEnergy; ++k) {
      double v = lane < kReduceThreads / 32 ? red[lane][k] : 0.0;
      v = warp_sum(v);
      bad = bad || !isfinite(v);
      if (lane == 0) out[static_cast<size_t>(t) * kNumEnergy + k] = v;
    }
    if (lane == 0 && bad) atomicOr(flags + pair, kFlagEnergy);
  }
}

// A row of w pixels in ceil(w / 256) CTAs of equal width (multiples of 32): 640 -> 3 x 224, 320 -> 2 x 160,
// 160 -> 1 x 160, instead of 256-wide CTAs whose last one idles up to 7 warps.
#ifndef HWF_ROW_ADAPT
#define HWF_ROW_ADAPT 1
#endif
inline int row_threads(int w) {
  if (!HWF_ROW_ADAPT) return kThreads;
  const int nb = (w + kThreads - 1) / kThreads;
  return std::max(32, ((w + nb - 1) / nb + 31) / 32 * 32);
}
inline dim3 rows_grid(int w, int h, int planes) {
  const int t = row_threads(w);
  return dim3((w + t - 1) / t, h, planes);
}

}  // namespace

void init_maps_constants() {
  // image.cpp:127-134 with sigma = 3.2: radius ceil(3 sigma) = 10
  const double sigma = 3.2;
  const int R = static_cast<int>(std::ceil(3.0 * sigma));
  double k[32];
  double sum = 0.0;
  for (int i = -R; i <= R; ++i) {
    k[i + R] = std::exp(-0.5 * (i * i) / (sigma * sigma));
    sum += k[i + R];
  }
  for (int i = 0; i < 2 * R + 1; ++i) k[i] /= sum;
  cudaMemcpyToSymbol(c_gauss, k, sizeof(double) * (2 * R + 1));
  cudaMemcpyToSymbol(c_gauss_r, &R, sizeof(int));
  g_gauss_r = R;
}
void launch_pyr_in(const void* src, int dtype, double* dst, long long n, cudaStream_t s) {
  k_pyr_in<<<static_cast<unsigned>((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(src, dtype, dst, n);
}
void launch_pyr_down_u8(const uint8_t* src, int w, int h, double* dst, int ow, int oh, int planes, cudaStream_t s) {
  k_pyr_down_u8<<<rows_grid(ow, oh, planes), row_threads(ow), 0, s>>>(src, w, h, dst, ow, oh);
}
void launch_pyr_down(const double* src, int w, int h, double* dst, int ow, int oh, int planes, cudaStream_t s) {
  k_pyr_down<<<rows_grid(ow, oh, planes), row_threads(ow), 0, s>>>(src, w, h, dst, ow, oh);
}
void launch_init_coarse(double* base, double* total, double* delta, int G, int B, double ox, double oy,
                        cudaStream_t s) {
  const long long n = static_cast<long long>(G) * B;
  k_init_coarse<<<static_cast<unsigned>((6 * n + kThreads - 1) / kThreads), kThreads, 0, s>>>(base, total, delta, n, ox, oy);
}
void launch_occlusion(int w, int h, int gw, int gh, int step, const double* total, int B, int2* q, float* Z,
                      uint8_t* bad, unsigned long long* zbuf, uint8_t* degen, unsigned long long* queue,
                      unsigned int* qcount, uint8_t* vis_out, cudaStream_t s) {
  k_occ_project<<<rows_grid(w, h, B), row_threads(w), 0, s>>>(w, h, gw, gh, step, total, q, Z, bad);
  launch_occlusion_projected(w, h, B, q, Z, bad, zbuf, degen, queue, qcount, vis_out, s);
}
// raster + resolve from vertices already projected (by k_occ_project or the fused E_after pass)
void launch_occlusion_projected(int w, int h, int B, int2* q, float* Z, uint8_t* bad, unsigned long long* zbuf,
                                uint8_t* degen, unsigned long long* queue, unsigned int* qcount, uint8_t* vis_out,
                                cudaStream_t s) {
  const size_t N = static_cast<size_t>(w) * h;
  if (w >= 2 && h >= 2) {
    cudaMemsetAsync(zbuf, 0xFF, N * 4 * B * sizeof(unsigned long long), s);
    cudaMemsetAsync(qcount, 0, sizeof(unsigned int), s);
    k_occ_raster<<<rows_grid(w - 1, h - 1, B), row_threads(w - 1), 0, s>>>(
        w, h, q, Z, bad, zbuf, degen, queue, qcount);
    k_occ_raster_big<<<148 * 8, kThreads, 0, s>>>(w, h, q, Z, zbuf, queue, qcount);
  }
  k_occ_resolve<<<rows_grid(w, h, B), row_threads(w), 0, s>>>(w, h, q, Z, bad, zbuf, degen, vis_out);
}
void launch_illumination(int w, int h, int gw, int gh, int step, const double* img, const double* total,
                         const uint8_t* vis, int B, double* resid, double* tmp, double* hm, cudaStream_t s) {
  k_illum_resid<<<rows_grid(w, h, B), row_threads(w), 0, s>>>(w, h, gw, gh, step, img, total, vis, resid);
  if (g_gauss_r == kBlurR) {
#ifdef HWF_BLUR_PER_TAP  // A/B: one output per thread, 2R + 1 loads each
    k_blur_h<kBlurR><<<rows_grid(w, h, 2 * B), row_threads(w), 0, s>>>(w, h, resid, tmp);
    k_blur_v_half<kBlurR><<<rows_grid(w, h, 2 * B), row_threads(w), 0, s>>>(w, h, tmp, hm);
#else
    const int segs = (w + 32 * kBlurHK - 1) / (32 * kBlurHK), items = segs * h;
    k_blur_h_win<kBlurR><<<dim3((items + kBlurWarps - 1) / kBlurWarps, 2 * B), 32 * kBlurWarps, 0, s>>>(
        w, h, segs, items, resid, tmp);
    k_blur_v_half_win<kBlurR><<<dim3((w + row_threads(w) - 1) / row_threads(w), (h + kBlurK - 1) / kBlurK, 2 * B),
                                row_threads(w), 0, s>>>(w, h, tmp, hm);
#endif
  } else {
    k_blur_h<-1><<<rows_grid(w, h, 2 * B), row_threads(w), 0, s>>>(w, h, resid, tmp);
    k_blur_v_half<-1><<<rows_grid(w, h, 2 * B), row_threads(w), 0, s>>>(w, h, tmp, hm);
  }
}
void launch_prolong_grid(int gwc, int ghc, int gwf, int ghf, int step, const double* total_c, double* base_f,
                         double* total_f, double* delta_f, int B, cudaStream_t s) {
  k_prolong_grid<<<dim3((gwf * ghf + kThreads - 1) / kThreads, B), kThreads, 0, s>>>(gwc, ghc, gwf, ghf, step,
                                                                                    total_c, base_f, total_f, delta_f);
}
void launch_prolong_maps(int wc, int hc, int wf, int hf, const uint8_t* vis_c, const double* hm_c, uint8_t* vis_f,
                         double* illum_f, int B, cudaStream_t s) {
  if (!hm_c || !illum_f) {  // masks only (the pipeline)
    const int n4 = (wf + kProlongPx - 1) / kProlongPx;
    k_prolong_vis<<<rows_grid(n4, hf, B), row_threads(n4), 0, s>>>(wc, hc, wf, hf, vis_c, vis_f);
    return;
  }
  k_prolong_maps<<<rows_grid(wf, hf, B), row_threads(wf), 0, s>>>(wc, hc, wf, hf, vis_c, hm_c, vis_f, illum_f);
}
void launch_propagate(int gw, int gh, int step, const double* prev_delta, const double* prev_total, const double* base,
                      double* delta, double* total, int B, cudaStream_t s) {
  k_propagate<<<dim3((gw * gh + kThreads - 1) / kThreads, B), kThreads, 0, s>>>(gw, gh, step, prev_delta, prev_total,
                                                                               base, delta, total);
}
void launch_dense(int w, int h, int gw, int gh, int step, const double* total, int B, double* s_out, double* m_out,
                  double* d_out, double* disp_out, cudaStream_t s) {
  k_dense<<<rows_grid(w, h, B), row_threads(w), 0, s>>>(w, h, gw, gh, step, total, s_out, m_out, d_out, disp_out);
}
void launch_energy_reduce(const double* ep, int nslots, int cap, int B, double* out, int* flags, cudaStream_t s,
                          const int* counts) {
  k_energy_reduce<<<static_cast<unsigned>(nslots * B), kReduceThreads, 0, s>>>(ep, nslots, cap, B, out, flags, counts);
}

}  // namespace hwf
