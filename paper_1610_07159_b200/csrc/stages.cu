// stages.cu — per-stage C-ABI entry points on the device (parity seams).
//
// Each call uploads its host inputs, runs the SAME kernels the batched
// pipeline runs (B = 1), and downloads the result. Tests compare these, stage
// by stage, with the CPU oracle on identical inputs.
#include <cmath>
#include "hwflow_c.h"
#include "host.h"

using namespace hwf_host;

namespace {

template <class T>
T* up(DevMem& m, const T* host, size_t n) {
  T* d = m.alloc<T>(n);
  if (host) CK(cudaMemcpy(d, host, n * sizeof(T), cudaMemcpyHostToDevice));
  else CK(cudaMemset(d, 0, n * sizeof(T)));
  return d;
}
template <class T>
void down(T* host, const T* dev, size_t n) {
  CK(cudaMemcpy(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost));
}

// Upload one hwf_level into a B=1 LevelDev (solver buffers allocated).
void load_level(DevMem& m, LevelDev& d, const hwf_level* lv, bool schwarz_tiles, int tile_px, cudaStream_t st) {
  if (!lv || lv->width < 1 || lv->height < 1) throw InvalidArg("bad level");
  if (lv->grid_step < 1 || lv->grid_step > 32) throw InvalidArg("grid_step must be in [1, 32] on the device");
  d.dims(lv->width, lv->height, lv->grid_step, schwarz_tiles ? tile_px : 0);
  d.alloc_solver(m, 1, schwarz_tiles);
  d.img = m.alloc<double>(4 * d.N);
  for (int e = 0; e < 4; ++e) {
    if (!lv->images[e]) throw InvalidArg("null image");
    CK(cudaMemcpy(d.img + e * d.N, lv->images[e], d.N * sizeof(double), cudaMemcpyHostToDevice));
  }
  d.pk = m.alloc<double>(4 * d.N * 4);
  launch_pack(d.img, d.w, d.h, 4, d.pk, st);
  bool any = false;
  for (int e = 0; e < 4; ++e) any = any || lv->illum[e];
  if (any) {
    d.illum = m.alloc<double>(4 * d.N);
    for (int e = 0; e < 4; ++e) {
      if (lv->illum[e])
        CK(cudaMemcpy(d.illum + e * d.N, lv->illum[e], d.N * sizeof(double), cudaMemcpyHostToDevice));
      else
        CK(cudaMemset(d.illum + e * d.N, 0, d.N * sizeof(double)));
    }
  }
  if (lv->total) CK(cudaMemcpy(d.total, lv->total, 6 * d.G * sizeof(double), cudaMemcpyHostToDevice));
  else CK(cudaMemset(d.total, 0, 6 * d.G * sizeof(double)));
  if (lv->delta) CK(cudaMemcpy(d.delta, lv->delta, 6 * d.G * sizeof(double), cudaMemcpyHostToDevice));
  else CK(cudaMemset(d.delta, 0, 6 * d.G * sizeof(double)));
  if (lv->vis4) CK(cudaMemcpy(d.vis, lv->vis4, d.N, cudaMemcpyHostToDevice));
  else CK(cudaMemset(d.vis, 0x0F, d.N));
  if (lv->outlier) CK(cudaMemcpy(d.W, lv->outlier, d.N, cudaMemcpyHostToDevice));
  else CK(cudaMemset(d.W, 1, d.N));
  if (lv->node_w) CK(cudaMemcpy(d.nodew, lv->node_w, d.G * sizeof(double), cudaMemcpyHostToDevice));
  else {
    std::vector<double> ones(d.G, 1.0);
    CK(cudaMemcpy(d.nodew, ones.data(), d.G * sizeof(double), cudaMemcpyHostToDevice));
  }
}

void make_energies(DevMem& m, Energies& E, const LevelDev& d, int nslots) {
  E.nslots = std::max(nslots, 1);
  E.cap = d.n_pix_cta + d.n_node_cta;
  E.part = m.alloc<double>(static_cast<size_t>(E.pair_stride()));
  E.red = m.alloc<double>(static_cast<size_t>(E.nslots) * kNumEnergy);
  CK(cudaMemset(E.part, 0, sizeof(double) * E.pair_stride()));
}

PixArgs pix_args(const LevelDev& d, const hwf_energy_params* P, uint32_t active, int* flags, const Energies& E) {
  PixArgs pa{};
  pa.w = d.w; pa.h = d.h; pa.gw = d.gw; pa.gh = d.gh; pa.step = d.step; pa.ncx = d.ncx; pa.ncy = d.ncy;
  pa.tcx = d.tcx; pa.tcy = d.tcy; pa.rp = d.rp;
  pa.pk = d.pk; pa.illum = d.illum; pa.vis4 = d.vis; pa.W = d.W; pa.total = d.total; pa.half = d.half;
  pa.cells = d.cells; pa.ep_pair = E.pair_stride(); pa.flags = flags; pa.P = to_params(*P);
  pa.active = active; pa.ep_new = E.slot(0);
  return pa;
}
NodeArgs node_args(const LevelDev& d, const hwf_energy_params* P, uint32_t active, double lm, const double* dF,
                   int* flags, const Energies& E) {
  NodeArgs na{};
  na.w = d.w; na.h = d.h; na.gw = d.gw; na.gh = d.gh; na.step = d.step; na.ncx = d.ncx; na.ncy = d.ncy;
  na.half = d.half; na.node_w = d.nodew; na.node_w_new = d.nodew; na.total = d.total; na.delta = d.delta;
  na.cells = d.cells;
  na.sys = d.sys; na.ep_pair = E.pair_stride(); na.ep_base = d.n_pix_cta; na.flags = flags;
  na.P = to_params(*P); na.F = dF; na.active = active; na.lm = lm; na.ep_new = E.slot(0);
  return na;
}

// reference 9-slot full blocks <-> device forward symmetric packing
void pack_system(int gw, int gh, const double* blocks, const double* rhs, std::vector<double>& sys) {
  const int G = gw * gh;
  sys.assign(static_cast<size_t>(G) * kSysStride, 0.0);
  for (int n = 0; n < G; ++n) {
    double* o = &sys[static_cast<size_t>(n) * kSysStride];
    for (int fs = 0; fs < 5; ++fs) {
      const double* B = blocks + (static_cast<size_t>(n) * 9 + 4 + fs) * 36;
      for (int i = 0; i < 6; ++i)
        for (int j = i; j < 6; ++j) o[fs * 21 + sym6(i, j)] = B[6 * i + j];
    }
    for (int r = 0; r < 6; ++r) o[kSysRhs + r] = rhs[6 * n + r];
    const double* D = blocks + (static_cast<size_t>(n) * 9 + 4) * 36;
    for (int f = 0; f < 3; ++f) {  // solver.cpp:64-78
      const double m00 = D[6 * (2 * f) + 2 * f], m01 = D[6 * (2 * f) + 2 * f + 1];
      const double m10 = D[6 * (2 * f + 1) + 2 * f], m11 = D[6 * (2 * f + 1) + 2 * f + 1];
      const double det = m00 * m11 - m01 * m10;
      double* p = o + kSysPre + 3 * f;
      if (std::abs(det) > 1e-300) {
        p[0] = m11 / det;
        p[1] = -m01 / det;
        p[2] = m00 / det;
      } else {
        p[0] = 1.0;
        p[1] = 0.0;
        p[2] = 1.0;
      }
    }
  }
}

void unpack_system(int gw, int gh, const std::vector<double>& sys, double* blocks, double* rhs, double* precond) {
  const int G = gw * gh;
  for (int n = 0; n < G; ++n) {
    const int a = n % gw, b = n / gw;
    for (int s9 = 0; s9 < 9; ++s9) {
      double* B = blocks + (static_cast<size_t>(n) * 9 + s9) * 36;
      const int qa = a + s9 % 3 - 1, qb = b + s9 / 3 - 1;
      const bool ok = qa >= 0 && qa < gw && qb >= 0 && qb < gh;
      const int src = s9 >= 4 ? n : qb * gw + qa;
      const int fs = s9 >= 4 ? s9 - 4 : 4 - s9;
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j)
          B[6 * i + j] = ok ? sys[static_cast<size_t>(src) * kSysStride + fs * 21 + sym6(i, j)] : 0.0;
    }
    for (int r = 0; r < 6; ++r) rhs[6 * n + r] = sys[static_cast<size_t>(n) * kSysStride + kSysRhs + r];
    if (precond)
      for (int f = 0; f < 3; ++f) {
        const double* p = &sys[static_cast<size_t>(n) * kSysStride + kSysPre + 3 * f];
        double* o = precond + (static_cast<size_t>(n) * 3 + f) * 4;
        o[0] = p[0];
        o[1] = p[1];
        o[2] = p[1];
        o[3] = p[2];
      }
  }
}

void check_flags(int* dflags) {
  int f = 0;
  CK(cudaMemcpy(&f, dflags, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> v(1, f);
  raise_on_flags(v, 1);
}

}  // namespace

extern "C" {

int hwf_pyramid(hwf_ctx* ctx, const hwf_frame4* fr, int levels, double* out) {
  return guard(ctx, [&] {
    if (!fr || fr->width < 1 || fr->height < 1) throw InvalidArg("bad frame dims");
    if (levels < 1) throw InvalidArg("pyramid needs >= 1 level");
    if (fr->dtype != HWF_DTYPE_U8 && fr->dtype != HWF_DTYPE_F64) throw InvalidArg("unknown dtype");
    DevMem m;
    const size_t N = static_cast<size_t>(fr->width) * fr->height, esz = fr->dtype == HWF_DTYPE_U8 ? 1 : 8;
    char* in = m.alloc<char>(4 * N * esz);
    for (int e = 0; e < 4; ++e) {
      if (!fr->plane[e]) throw InvalidArg("null image plane");
      CK(cudaMemcpy(in + e * N * esz, fr->plane[e], N * esz, cudaMemcpyHostToDevice));
    }
    int w = fr->width, h = fr->height;
    double* cur = m.alloc<double>(4 * N);
    launch_pyr_in(in, fr->dtype, cur, 4 * static_cast<long long>(N), ctx->stream);
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
      if (l > 0) {
        const int ow = (w + 1) / 2, oh = (h + 1) / 2;
        double* nxt = m.alloc<double>(4 * static_cast<size_t>(ow) * oh);
        launch_pyr_down(cur, w, h, nxt, ow, oh, 4, ctx->stream);
        cur = nxt;
        w = ow;
        h = oh;
      }
      CK(cudaStreamSynchronize(ctx->stream));
      down(out + off, cur, 4 * static_cast<size_t>(w) * h);
      off += 4 * static_cast<size_t>(w) * h;
    }
    CK(cudaGetLastError());
  });
}

int hwf_eval_energy(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* P, hwf_energy* out, double* residuals) {
  return guard(ctx, [&] {
    if (!P || !out) throw InvalidArg("null argument");
    if (hwf_validate_params(P) != HWF_OK) throw InvalidArg("energy weights must be >= 0");
    if (P->w_epi > 0.0 && !lv->fundamental) throw InvalidArg("epipolar term enabled without a fundamental matrix");
    DevMem m;
    LevelDev d;
    load_level(m, d, lv, false, 0, ctx->stream);
    double* dR = residuals ? m.alloc<double>(2 * d.N + 14 * d.G) : nullptr;
    const double* dF = lv->fundamental ? up(m, lv->fundamental, 9) : nullptr;
    Energies E;
    make_energies(m, E, d, 1);
    int* flags = up<int>(m, nullptr, 1);
    PixArgs pa = pix_args(d, P, 7u, flags, E);
    pa.refresh = 0;
    pa.resid = dR;
    launch_pixel(false, pa, 1, ctx->stream);
    NodeArgs na = node_args(d, P, 7u, 0.0, dF, flags, E);
    na.refresh = 0;
    na.resid = dR;
    na.resid_n = static_cast<long long>(d.N);
    launch_node(false, na, 1, ctx->stream);
    launch_energy_reduce(E.part, E.nslots, E.cap, 1, E.red, flags, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    double e[kNumEnergy];
    down(e, E.red, kNumEnergy);
    out->photo = e[0];
    out->grad = e[1];
    out->smooth = e[2];
    out->epi = e[3];
    out->mag = e[4];
    out->total = P->w_photo * e[0] + P->w_grad * e[1] + P->w_reg * (P->w_smooth * e[2] + P->w_epi * e[3] + P->w_mag * e[4]);
    out->residual_count = 2LL * static_cast<long long>(d.N) + 14LL * static_cast<long long>(d.G);
    if (residuals) down(residuals, dR, static_cast<size_t>(out->residual_count));
    if (!std::isfinite(out->total)) throw Diverged("non-finite residuals in energy assembly");
  });
}

int hwf_refresh_weights(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* P, uint8_t* outlier_out,
                        double* node_w_out) {
  return guard(ctx, [&] {
    DevMem m;
    LevelDev d;
    load_level(m, d, lv, false, 0, ctx->stream);
    const double* dF = lv->fundamental ? up(m, lv->fundamental, 9) : nullptr;
    Energies E;
    make_energies(m, E, d, 1);
    int* flags = up<int>(m, nullptr, 1);
    PixArgs pa = pix_args(d, P, 7u, flags, E);
    pa.refresh = 1;
    launch_pixel(true, pa, 1, ctx->stream);
    launch_structw(d.w, d.h, d.gw, d.gh, d.step, d.half, d.nodew2, 1, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    if (outlier_out) down(outlier_out, d.W, d.N);
    if (node_w_out) down(node_w_out, d.nodew2, d.G);
  });
}

int hwf_linearize(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* P, uint32_t active, double lm,
                  double* blocks, double* rhs, double* precond) {
  return guard(ctx, [&] {
    if (P->w_epi > 0.0 && !lv->fundamental) throw InvalidArg("epipolar term enabled without a fundamental matrix");
    DevMem m;
    LevelDev d;
    load_level(m, d, lv, false, 0, ctx->stream);
    const double* dF = lv->fundamental ? up(m, lv->fundamental, 9) : nullptr;
    Energies E;
    make_energies(m, E, d, 1);
    int* flags = up<int>(m, nullptr, 1);
    PixArgs pa = pix_args(d, P, active, flags, E);
    pa.refresh = 0;
    launch_pixel(true, pa, 1, ctx->stream);
    NodeArgs na = node_args(d, P, active, lm, dF, flags, E);
    na.refresh = 0;
    launch_node(true, na, 1, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    check_flags(flags);
    std::vector<double> sys(d.G * kSysStride);
    down(sys.data(), d.sys, sys.size());
    unpack_system(d.gw, d.gh, sys, blocks, rhs, precond);
  });
}

// assemble_jacobian (solver.cpp:247-314): the device evaluates eval_pixel / eval_node with derivatives (the
// LIN kernels' test-hook dumps); the host lays the values out as the reference's triplets, in its loop order.
int hwf_assemble_jacobian(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* P, uint32_t active,
                          int negate_field, double* residuals, int* rows, int* cols, double* vals, long long cap,
                          long long* nnz) {
  return guard(ctx, [&] {
    if (!lv || !P || !nnz || negate_field < -1 || negate_field > 2) throw InvalidArg("bad jacobian query");
    if (P->w_epi > 0.0 && !lv->fundamental) throw InvalidArg("epipolar term enabled without a fundamental matrix");
    DevMem m;
    LevelDev d;
    load_level(m, d, lv, false, 0, ctx->stream);
    const double* dF = lv->fundamental ? up(m, lv->fundamental, 9) : nullptr;
    Energies E;
    make_energies(m, E, d, 1);
    int* flags = up<int>(m, nullptr, 1);
    const size_t N = d.N, G = d.G;
    double* pj = m.alloc<double>(14 * N);
    double* nj = m.alloc<double>(kNodeJac * G);
    PixArgs pa = pix_args(d, P, active, flags, E);
    pa.refresh = 0;
    pa.jac = pj;
    launch_pixel(true, pa, 1, ctx->stream);
    NodeArgs na = node_args(d, P, active, 0.0, dF, flags, E);
    na.refresh = 0;
    na.jac = nj;
    launch_node(true, na, 1, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    check_flags(flags);
    std::vector<double> hp(14 * N), hn(kNodeJac * G);
    down(hp.data(), pj, hp.size());
    down(hn.data(), nj, hn.size());
    std::vector<int> R0, C0;
    std::vector<double> V0;
    const long long M = 2 * static_cast<long long>(N) + 14 * static_cast<long long>(G);
    std::vector<double> R(static_cast<size_t>(M), 0.0);
    auto push = [&](int r, int c, double v) {
      R0.push_back(r);
      C0.push_back(c);
      V0.push_back(v);
    };
    auto hooks = [&](double* v) {  // mask_fields, then the negative control
      for (int f = 0; f < 3; ++f)
        if (!((active >> f) & 1)) v[2 * f] = v[2 * f + 1] = 0.0;
      if (negate_field >= 0) {
        v[2 * negate_field] *= -1.0;
        v[2 * negate_field + 1] *= -1.0;
      }
    };
    const int w = d.w, step = d.step, gw = d.gw, gh = d.gh, Ni = static_cast<int>(N), Gi = static_cast<int>(G);
    for (int pix = 0; pix < Ni; ++pix) {
      const double* e = &hp[14 * static_cast<size_t>(pix)];
      R[pix] = e[0];
      R[Ni + pix] = e[1];
      double jp[6], jg[6];
      for (int j = 0; j < 6; ++j) {
        jp[j] = e[2 + j];
        jg[j] = e[8 + j];
      }
      hooks(jp);
      hooks(jg);
      // WarpGrid::support (warp_grid.cpp:41-54)
      const double u = static_cast<double>(pix % w) / step, v = static_cast<double>(pix / w) / step;
      const int a0 = std::min(std::max(static_cast<int>(std::floor(u)), 0), gw - 2);
      const int b0 = std::min(std::max(static_cast<int>(std::floor(v)), 0), gh - 2);
      const double fu = std::min(std::max(u - a0, 0.0), 1.0), fv = std::min(std::max(v - b0, 0.0), 1.0);
      const int node[4] = {b0 * gw + a0, b0 * gw + a0 + 1, (b0 + 1) * gw + a0, (b0 + 1) * gw + a0 + 1};
      const double wt[4] = {(1 - fu) * (1 - fv), fu * (1 - fv), (1 - fu) * fv, fu * fv};
      for (int i = 0; i < 4; ++i) {
        if (wt[i] == 0.0) continue;
        for (int j = 0; j < 6; ++j) {
          const int col = 6 * node[i] + j;
          if (jp[j] != 0.0) push(pix, col, wt[i] * jp[j]);
          if (jg[j] != 0.0) push(Ni + pix, col, wt[i] * jg[j]);
        }
      }
    }
    for (int n = 0; n < Gi; ++n) {
      const double* e = &hn[kNodeJac * static_cast<size_t>(n)];
      const int right = (n % gw + 1 < gw) ? n + 1 : -1, down_ = (n / gw + 1 < gh) ? n + gw : -1;
      for (int row = 0; row < 6; ++row) {
        const int r = 2 * Ni + 6 * n + row;
        R[r] = e[row];
        const int f = row / 2;
        if (!((active >> f) & 1)) continue;
        const double sgn = f == negate_field ? -1.0 : 1.0;
        if (e[6 + row] != 0.0) push(r, 6 * n + row, sgn * e[6 + row]);
        if (right >= 0 && e[12 + row] != 0.0) push(r, 6 * right + row, sgn * e[12 + row]);
        if (down_ >= 0 && e[18 + row] != 0.0) push(r, 6 * down_ + row, sgn * e[18 + row]);
      }
      for (int t = 0; t < 2; ++t) {
        const int r = 2 * Ni + 6 * Gi + 2 * n + t;
        R[r] = e[24 + t];
        double j[6];
        for (int c = 0; c < 6; ++c) j[c] = e[26 + 6 * t + c];
        hooks(j);
        for (int c = 0; c < 6; ++c)
          if (j[c] != 0.0) push(r, 6 * n + c, j[c]);
      }
      for (int row = 0; row < 6; ++row) {
        const int r = 2 * Ni + 8 * Gi + 6 * n + row;
        R[r] = e[38 + row];
        const int f = row / 2;
        if (!((active >> f) & 1)) continue;
        const double sgn = f == negate_field ? -1.0 : 1.0;
        if (e[44 + row] != 0.0) push(r, 6 * n + row, sgn * e[44 + row]);
      }
    }
    *nnz = static_cast<long long>(V0.size());
    if (residuals) std::copy(R.begin(), R.end(), residuals);
    if (cap > 0 || rows || cols || vals) {
      if (cap < *nnz || !rows || !cols || !vals) throw InvalidArg("jacobian triplet buffers too small");
      std::copy(R0.begin(), R0.end(), rows);
      std::copy(C0.begin(), C0.end(), cols);
      std::copy(V0.begin(), V0.end(), vals);
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

int hwf_pcg(hwf_ctx* ctx, int gw, int gh, const double* blocks, const double* rhs, int iters, double* x_out,
            double* trace) {
  return guard(ctx, [&] {
    if (gw < 1 || gh < 1 || iters < 0) throw InvalidArg("bad system dims");
    DevMem m;
    std::vector<double> sys;
    pack_system(gw, gh, blocks, rhs, sys);
    const size_t G = static_cast<size_t>(gw) * gh;
    std::vector<double> soa(sys.size());  // the global PCG reads entry-major records
    for (size_t n = 0; n < G; ++n)
      for (int e = 0; e < kSysStride; ++e) soa[e * G + n] = sys[n * kSysStride + e];
    PcgArgs a{};
    a.gw = gw; a.gh = gh; a.iters = iters;
    a.sys = up(m, soa.data(), soa.size());
    a.x = m.alloc<double>(6 * G); a.r = m.alloc<double>(6 * G); a.z = m.alloc<double>(6 * G);
    a.p = m.alloc<double>(6 * G); a.ap = m.alloc<double>(6 * G); a.p2 = m.alloc<double>(6 * G);
    a.part = m.alloc<double>(2 * static_cast<size_t>(pcg_tiles(gw, gh)));
    a.state = m.alloc<double>(8);
    a.count = up<unsigned>(m, nullptr, 1);
    a.trace = trace ? m.alloc<double>(iters + 1) : nullptr;
    a.update = 0;
    a.active = 7;
    a.flags = up<int>(m, nullptr, 1);
    launch_pcg_global(a, 1, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    check_flags(a.flags);
    down(x_out, a.x, 6 * G);
    if (trace) down(trace, a.trace, iters + 1);
  });
}

int hwf_schwarz(hwf_ctx* ctx, int gw, int gh, int step, int tile, int /*boundary_px*/, const double* blocks,
                const double* rhs, int patch_iters, int pcg_iters, double* x_out) {
  return guard(ctx, [&] {
    if (gw < 2 || gh < 2 || step < 1 || tile < 1) throw InvalidArg("bad subdomain tiling");
    if ((tile + step - 1) / step > 5) throw InvalidArg("subdomain tile must hold <= 5x5 nodes on the device");
    DevMem m;
    std::vector<double> sys;
    pack_system(gw, gh, blocks, rhs, sys);
    const size_t G = static_cast<size_t>(gw) * gh;
    SwzArgs a{};
    a.gw = gw; a.gh = gh; a.step = step; a.tile = tile;
    a.ntx = ((gw - 1) * step) / tile + 1;
    a.nty = ((gh - 1) * step) / tile + 1;
    a.nxm = a.nym = (tile + step - 1) / step;
    a.sys = up(m, sys.data(), sys.size());
    double* xa = up<double>(m, nullptr, 6 * G);
    double* xb = up<double>(m, nullptr, 6 * G);
    a.pcg_iters = pcg_iters;
    a.active = 7;
    a.flags = up<int>(m, nullptr, 1);
    a.last = 0;
    double* res = xa;  // zero when patch_iters == 0
    for (int s = 0; s < patch_iters; ++s) {
      a.pub = s == 0 ? nullptr : (s & 1 ? xb : xa);
      a.next = s & 1 ? xa : xb;
      launch_schwarz(a, 1, ctx->stream);
      res = a.next;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    check_flags(a.flags);
    down(x_out, res, 6 * G);
  });
}

int hwf_gn_level(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta, uint8_t* outlier,
                 double* node_w, const hwf_energy_params* P, const hwf_schedule* S, int gn_iters,
                 double* energy_before, double* energy_after) {
  return hwf_gn_level_trace(ctx, lv, base, delta, outlier, node_w, P, S, gn_iters, energy_before, energy_after,
                            nullptr);
}

int hwf_gn_level_trace(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta, uint8_t* outlier,
                       double* node_w, const hwf_energy_params* P, const hwf_schedule* S, int gn_iters,
                       double* energy_before, double* energy_after, double* pcg_trace) {
  return guard(ctx, [&] {
    check_params(P, S, lv->fundamental);
    if (gn_iters < 0 || gn_iters > HWF_MAX_GN) throw InvalidArg("bad gn_iters");
    DevMem m;
    LevelDev d;
    hwf_level l2 = *lv;
    l2.outlier = outlier;
    l2.node_w = node_w;
    l2.delta = delta;
    load_level(m, d, &l2, S->subdomain_px > 0, S->subdomain_px, ctx->stream);
    std::vector<double> tot(6 * d.G);
    for (size_t i = 0; i < tot.size(); ++i) tot[i] = base[i] + delta[i];  // base.plus(delta)
    CK(cudaMemcpy(d.total, tot.data(), tot.size() * sizeof(double), cudaMemcpyHostToDevice));
    d.base = up(m, base, 6 * d.G);
    const double* dF = lv->fundamental ? up(m, lv->fundamental, 9) : nullptr;
    Energies E;
    make_energies(m, E, d, 2 * gn_iters);
    int* flags = up<int>(m, nullptr, 1);
    Scratch sc;
    sc.alloc(m, 1, d.N, d.G, false, false, S->subdomain_px <= 0, pcg_tiles(d.gw, d.gh));
    Launches LC;
    const bool traced = pcg_trace && S->subdomain_px <= 0 && gn_iters > 0;
    const size_t trace_n = static_cast<size_t>(gn_iters) * (S->pcg_iters + 1);
    double* dtrace = traced ? up<double>(m, nullptr, trace_n) : nullptr;
    record_gn_level(d, 1, *P, *S, dF, gn_iters, E, 0, sc, flags, ctx->stream, LC, nullptr, true, dtrace);
    launch_energy_reduce(E.part, E.nslots, E.cap, 1, E.red, flags, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    std::vector<double> red(static_cast<size_t>(E.nslots) * kNumEnergy);
    down(red.data(), E.red, red.size());
    for (int it = 0; it < gn_iters; ++it)
      for (int k = 0; k < 2; ++k) {
        const double* e = &red[(2 * it + k) * kNumEnergy];
        const double t = P->w_photo * e[0] + P->w_grad * e[1] + P->w_reg * (P->w_smooth * e[2] + P->w_epi * e[3] + P->w_mag * e[4]);
        double* dst = k == 0 ? energy_before : energy_after;
        if (dst) dst[it] = t;
      }
    down(delta, d.delta, 6 * d.G);
    down(outlier, d.W, d.N);
    down(node_w, d.nodew, d.G);
    if (traced) down(pcg_trace, dtrace, trace_n);
    check_flags(flags);
  });
}

int hwf_propagate_temporal(hwf_ctx* ctx, int w, int h, int step, const double* prev_delta, const double* prev_total,
                           double* next_delta) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || step < 1) throw InvalidArg("bad dims");
    DevMem m;
    LevelDev d;
    d.dims(w, h, step, 0);
    const double* pd = up(m, prev_delta, 6 * d.G);
    const double* pt = up(m, prev_total, 6 * d.G);
    double* nd = m.alloc<double>(6 * d.G);
    launch_propagate(d.gw, d.gh, step, pd, pt, nullptr, nd, nullptr, 1, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    down(next_delta, nd, 6 * d.G);
  });
}

int hwf_occlusion(hwf_ctx* ctx, int w, int h, int step, const double* total, uint8_t* vis4_out) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || step < 1) throw InvalidArg("bad dims");
    DevMem m;
    LevelDev d;
    d.dims(w, h, step, 0);
    const double* dt = up(m, total, 6 * d.G);
    Scratch sc;
    sc.alloc(m, 1, d.N, d.G, true, false, false);
    uint8_t* vis = m.alloc<uint8_t>(d.N);
    launch_occlusion(w, h, d.gw, d.gh, step, dt, 1, sc.q, sc.Z, sc.bad, sc.zbuf, sc.degen, sc.queue, sc.qcount, vis,
                     ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    down(vis4_out, vis, d.N);
  });
}

int hwf_illumination(hwf_ctx* ctx, int w, int h, int step, const double* images[4], const double* total,
                     const uint8_t* vis4, double* hm_out) {
  return guard(ctx, [&] {
    if (w < 1 || h < 1 || step < 1) throw InvalidArg("bad dims");
    DevMem m;
    LevelDev d;
    d.dims(w, h, step, 0);
    double* img = m.alloc<double>(4 * d.N);
    for (int e = 0; e < 4; ++e) CK(cudaMemcpy(img + e * d.N, images[e], d.N * sizeof(double), cudaMemcpyHostToDevice));
    const double* dt = up(m, total, 6 * d.G);
    const uint8_t* dv = up(m, vis4, d.N);
    Scratch sc;
    sc.alloc(m, 1, d.N, d.G, false, true, false);
    double* hm = m.alloc<double>(2 * d.N);
    launch_illumination(w, h, d.gw, d.gh, step, img, dt, dv, 1, sc.resid, sc.tmp, hm, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    down(hm_out, hm, 2 * d.N);
  });
}

int hwf_prolongate(hwf_ctx* ctx, int wc, int hc, int wf, int hf, int step, const double* total_c,
                   const uint8_t* vis_c, const double* hm_c, double* base_f, uint8_t* vis_f, double* hm_f) {
  return guard(ctx, [&] {
    if (wc < 1 || hc < 1 || wf < 1 || hf < 1 || step < 1) throw InvalidArg("bad dims");
    DevMem m;
    LevelDev c, f;
    c.dims(wc, hc, step, 0);
    f.dims(wf, hf, step, 0);
    const double* dtc = up(m, total_c, 6 * c.G);
    double* bf = m.alloc<double>(6 * f.G);
    double* tf = m.alloc<double>(6 * f.G);
    double* df = m.alloc<double>(6 * f.G);
    launch_prolong_grid(c.gw, c.gh, f.gw, f.gh, step, dtc, bf, tf, df, 1, ctx->stream);
    if (vis_c && vis_f) {
      const uint8_t* dvc = up(m, vis_c, c.N);
      uint8_t* dvf = m.alloc<uint8_t>(f.N);
      const double* dhc = hm_c ? up(m, hm_c, 2 * c.N) : nullptr;
      double* ill = hm_c && hm_f ? m.alloc<double>(4 * f.N) : nullptr;
      launch_prolong_maps(wc, hc, wf, hf, dvc, dhc, dvf, ill, 1, ctx->stream);
      CK(cudaStreamSynchronize(ctx->stream));
      down(vis_f, dvf, f.N);
      if (ill) {  // L_{0,t} = +hm_t lives at image 2t
        down(hm_f, ill, f.N);
        down(hm_f + f.N, ill + 2 * f.N, f.N);
      }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    down(base_f, bf, 6 * f.G);
  });
}

}  // extern "C"
