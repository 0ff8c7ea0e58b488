// oracle/split.cpp — TEST INFRASTRUCTURE ONLY (parity checker).
//
// Restatement of the strip-split solve (include/hwflow_split.h) on the host, used to
// test the split driver (paper_1610_07159_b200/split.py) on CPU ranks over gloo.
// The per-level arithmetic is the oracle's own (core.cpp: refresh_outlier,
// refresh_node_w, eval_pixel/eval_node, build_normal_system, schwarz_sweep) and the
// map operations are hierarchy.cpp's. A rank:
//   - keeps full-size copies of every buffer;
//   - linearises the whole level (its total/delta are complete after the driver's all-gather);
//   - sweeps only the subdomains of its strip;
//   - reports energy partials for its own rows only.
// Before every sweep, the published vector is poisoned with NaN outside the owned
// rows and the two halo rows. A missing or wrong halo exchange in the driver then
// shows up as a NaN or a mismatch against the unsplit solve.
// Strip formula (same as csrc/split.cu): tile rows t0 = rank*nty/world,
// t1 = (rank+1)*nty/world; owned node rows [ceil(t0*tile/step), ceil(t1*tile/step)),
// with the last rank ending at gh. Global-PCG mode (subdomain_px = 0): node rows
// [rank*gh/world, (rank+1)*gh/world).
// Global-PCG mode runs pcg_impl (core.cpp, solver.cpp:320-361) phase by phase on the owned
// rows. Its "pcg_part" partials are the per-unknown products of each dot, rows of 6 gw: after
// the all-gather every rank sums all 6G of them in index order, the same sequence of
// additions as the unsplit dot, so the split is bitwise equal to the unsplit solve. z outside
// the owned and halo rows, and the partials outside the owned rows, are poisoned with NaN.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "backend.hpp"
#include "core.hpp"
#include "ctx.hpp"
#include "hierarchy.hpp"
#include "hwflow_c.h"
#include "hwflow_split.h"

namespace {

struct Lev {
  int w = 0, h = 0, gw = 0, gh = 0, N = 0, G = 0, n0 = 0, n1 = 0;
  std::vector<double> base, delta, total, xa, xb, node_w, hm, illum;
  std::vector<uint8_t> vis, outl, occ;
  orc::System sys;
  std::vector<orc::Subdomain> subs;
  std::vector<int> owner, loc;
  std::vector<char> take;
  // global-PCG split state
  std::vector<double> px, pr, pz, pp, pap, part;
  double rz = 0.0, rz0 = 0.0, alpha = 0.0, beta = 0.0;
  bool stop = false;
};

int ceil_div(int a, int b) { return (a + b - 1) / b; }

}  // namespace

struct hwf_split {
  hwf_ctx* ctx = nullptr;
  int w = 0, h = 0, dtype = 0, rank = 0, world = 1, L = 0;
  hwf_energy_params P{};
  hwf_schedule S{};
  bool hasF = false;
  double F[9] = {};
  int dims[4 * HWF_MAX_LEVELS] = {};
  int gn[HWF_MAX_LEVELS] = {}, slot_base[HWF_MAX_LEVELS] = {};
  std::vector<double> pyr;
  std::vector<std::vector<double>> frames;  // hwf_split_upload
  std::vector<size_t> off;
  Lev lev[HWF_MAX_LEVELS];
  std::vector<double> energy;  // [slot] partial Sum r^2 over owned rows
  int flags = 0;
  std::string why;
};

namespace {

template <class Fn>
int guard(hwf_split* sp, Fn&& fn) {
  try {
    if (!sp) throw std::invalid_argument("null split");
    fn();
    return HWF_OK;
  } catch (const orc::Divergence& e) {
    if (sp && sp->ctx) sp->ctx->err = e.what();
    return HWF_EDIVERGED;
  } catch (const std::exception& e) {
    if (sp && sp->ctx) sp->ctx->err = e.what();
    return HWF_EINVAL;
  }
}

void flag(hwf_split* sp, const char* why) {
  if (!sp->flags) sp->why = why;
  sp->flags |= 1;
}

hwf_level level_view(hwf_split* sp, int l) {
  Lev& v = sp->lev[l];
  hwf_level lv{};
  lv.width = v.w;
  lv.height = v.h;
  lv.grid_step = sp->S.grid_step;
  for (int e = 0; e < 4; ++e) {
    lv.images[e] = sp->pyr.data() + sp->off[l] + static_cast<size_t>(e) * v.N;
    lv.illum[e] = v.illum.empty() ? nullptr : v.illum.data() + static_cast<size_t>(e) * v.N;
  }
  lv.total = v.total.data();
  lv.delta = v.delta.data();
  lv.vis4 = v.vis.data();
  lv.outlier = v.outl.data();
  lv.node_w = v.node_w.data();
  lv.fundamental = sp->hasF ? sp->F : nullptr;
  return lv;
}

// Sum r^2 (energy.cpp:208-251) over the owned pixel rows and node rows.
double owned_energy(hwf_split* sp, int l) {
  Lev& v = sp->lev[l];
  const hwf_level lv = level_view(sp, l);
  const orc::Level Lv = orc::make_level(&lv, &sp->P, 1);
  const int step = sp->S.grid_step;
  const int y0 = std::min(v.h, v.n0 * step), y1 = sp->rank == sp->world - 1 ? v.h : std::min(v.h, v.n1 * step);
  double tot = 0.0;
  for (int y = y0; y < y1; ++y)
    for (int x = 0; x < v.w; ++x) {
      const orc::PixelEval e = orc::eval_pixel(Lv, x, y, false);
      tot += e.r_photo * e.r_photo + e.r_grad * e.r_grad;
    }
  for (int n = v.n0 * v.gw; n < v.n1 * v.gw; ++n) {
    const orc::NodeEval e = orc::eval_node(Lv, n, false);
    for (int j = 0; j < 6; ++j) tot += e.smooth_r[j] * e.smooth_r[j] + e.mag_r[j] * e.mag_r[j];
    tot += e.epi_r[0] * e.epi_r[0] + e.epi_r[1] * e.epi_r[1];
  }
  return tot;
}

}  // namespace

extern "C" {

int hwf_split_create(hwf_ctx* ctx, int w, int h, int dtype, const hwf_energy_params* params,
                     const hwf_schedule* sched, const double* F, int rank, int world, hwf_split** out) {
  auto sp = std::make_unique<hwf_split>();
  sp->ctx = ctx;
  const int rc = guard(sp.get(), [&] {
    if (!out || !params || !sched) throw std::invalid_argument("null split args");
    if (hwf_validate_params(params) != HWF_OK) throw std::invalid_argument("energy weights must be >= 0");
    if (params->w_epi > 0.0 && !F) throw std::invalid_argument("epipolar term enabled without a fundamental matrix");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
    if (w < 2 || h < 2) throw std::invalid_argument("bad frame dims");
    sp->w = w;
    sp->h = h;
    sp->dtype = dtype;
    sp->rank = rank;
    sp->world = world;
    sp->P = *params;
    sp->S = *sched;
    sp->hasF = F != nullptr;
    if (F) std::memcpy(sp->F, F, sizeof(sp->F));
    if (hwf_level_dims(w, h, sched->levels, sched->grid_step, &sp->L, sp->dims) != HWF_OK)
      throw std::invalid_argument("bad level dims");
    int nslots = 0;
    sp->off.assign(sp->L + 1, 0);
    const int step = sched->grid_step, tile = sched->subdomain_px;
    for (int l = 0; l < sp->L; ++l) {
      Lev& v = sp->lev[l];
      v.w = sp->dims[4 * l];
      v.h = sp->dims[4 * l + 1];
      v.gw = sp->dims[4 * l + 2];
      v.gh = sp->dims[4 * l + 3];
      v.N = v.w * v.h;
      v.G = v.gw * v.gh;
      sp->off[l + 1] = sp->off[l] + 4ull * v.N;
      sp->gn[l] = orc::gn_for_level(sched, l);
      sp->slot_base[l] = nslots;
      nslots += 2 * sp->gn[l];
      if (tile <= 0) {  // global-PCG mode: a band of node rows
        v.n0 = static_cast<int>(static_cast<long long>(rank) * v.gh / world);
        v.n1 = rank == world - 1 ? v.gh : static_cast<int>(static_cast<long long>(rank + 1) * v.gh / world);
        continue;
      }
      const int nty = ((v.gh - 1) * step) / tile + 1;
      const int t0 = static_cast<int>(static_cast<long long>(rank) * nty / world);
      const int t1 = static_cast<int>(static_cast<long long>(rank + 1) * nty / world);
      v.n0 = std::min(v.gh, ceil_div(t0 * tile, step));
      v.n1 = rank == world - 1 ? v.gh : std::min(v.gh, ceil_div(t1 * tile, step));
      v.subs = orc::build_subdomains(v.gw, v.gh, step, tile);
      orc::subdomain_owner(v.subs, v.G, v.owner, v.loc);
      v.take.assign(v.subs.size(), 0);
      for (size_t s = 0; s < v.subs.size(); ++s) {
        const int row = v.subs[s].interior.front() / v.gw;
        v.take[s] = row >= v.n0 && row < v.n1;
      }
    }
    sp->energy.assign(std::max(nslots, 1), 0.0);
  });
  if (rc == HWF_OK) *out = sp.release();
  return rc;
}

void hwf_split_destroy(hwf_split* sp) { delete sp; }

int hwf_split_schedule(hwf_split* sp, int* levels, int* gn) {
  return guard(sp, [&] {
    if (levels) *levels = sp->L;
    if (gn)
      for (int l = 0; l < sp->L; ++l) gn[l] = sp->gn[l];
  });
}

int hwf_split_rows(hwf_split* sp, int level, int* n0, int* n1, int* gw) {
  return guard(sp, [&] {
    if (level < 0 || level >= sp->L) throw std::invalid_argument("level out of range");
    if (n0) *n0 = sp->lev[level].n0;
    if (n1) *n1 = sp->lev[level].n1;
    if (gw) *gw = sp->lev[level].gw;
  });
}

int hwf_split_buffer(hwf_split* sp, int level, const char* name, void** ptr, long long* count) {
  return guard(sp, [&] {
    if (level < 0 || level >= sp->L || !name || !ptr || !count) throw std::invalid_argument("bad buffer query");
    Lev& v = sp->lev[level];
    const long long g6 = 6LL * v.G;
    if (!std::strcmp(name, "xa")) { v.xa.resize(g6); *ptr = v.xa.data(); *count = g6; }
    else if (!std::strcmp(name, "xb")) { v.xb.resize(g6); *ptr = v.xb.data(); *count = g6; }
    else if (!std::strcmp(name, "total")) { v.total.resize(g6); *ptr = v.total.data(); *count = g6; }
    else if (!std::strcmp(name, "delta")) { v.delta.resize(g6); *ptr = v.delta.data(); *count = g6; }
    else if (!std::strcmp(name, "energy")) { *ptr = sp->energy.data(); *count = static_cast<long long>(sp->energy.size()); }
    else if (!std::strcmp(name, "flags")) { *ptr = &sp->flags; *count = 1; }
    else if (!std::strcmp(name, "z")) { v.pz.resize(g6); *ptr = v.pz.data(); *count = g6; }
    else if (!std::strcmp(name, "pcg_part")) { v.part.resize(g6); *ptr = v.part.data(); *count = g6; }
    else throw std::invalid_argument(std::string("unknown split buffer ") + name);
  });
}

int hwf_split_row_elems(hwf_split* sp, int level, const char* name, long long* elems) {
  return guard(sp, [&] {
    if (level < 0 || level >= sp->L || !name || !elems) throw std::invalid_argument("bad row query");
    *elems = 6LL * sp->lev[level].gw;  // every buffer, "pcg_part" included, has 6 gw per node row
  });
}

const char* hwf_split_swept(int s) { return (s & 1) ? "xa" : "xb"; }

int hwf_split_upload(hwf_split* sp, const hwf_frame4* frame) {
  return guard(sp, [&] {
    if (!frame || frame->width != sp->w || frame->height != sp->h || frame->dtype != sp->dtype)
      throw std::invalid_argument("frame does not match the split");
    sp->frames = orc::load_frames(frame);
  });
}

int hwf_split_begin(hwf_split* sp, const hwf_frame4* frame) {
  const int rc = hwf_split_upload(sp, frame);  // (declared in hwflow_split.h)
  return rc != HWF_OK ? rc : hwf_split_prologue(sp);
}

int hwf_split_prologue(hwf_split* sp) {
  return guard(sp, [&] {
    if (sp->frames.empty()) throw std::invalid_argument("hwf_split_prologue before hwf_split_upload");
    const auto& imgs = sp->frames;
    sp->pyr.assign(sp->off[sp->L], 0.0);
    orc::backend()->pyramid(imgs, sp->w, sp->h, sp->L, sp->pyr.data());
    for (int l = 0; l < sp->L; ++l) {  // buffers the driver may query before level_begin
      Lev& v = sp->lev[l];
      for (auto* b : {&v.base, &v.delta, &v.total, &v.xa, &v.xb}) b->assign(6 * static_cast<size_t>(v.G), 0.0);
    }
    std::fill(sp->energy.begin(), sp->energy.end(), 0.0);
    sp->flags = 0;
  });
}

int hwf_split_level_begin(hwf_split* sp, int l) {  // hierarchy.cpp run_scene_flow, one level's setup
  return guard(sp, [&] {
    if (l < 0 || l >= sp->L) throw std::invalid_argument("level out of range");
    if (sp->flags) return;  // diverged: finish reports it; NaN flows must not reach the maps
    Lev& v = sp->lev[l];
    const size_t g6 = 6 * static_cast<size_t>(v.G);
    v.base.assign(g6, 0.0);
    v.delta.assign(g6, 0.0);
    v.xa.assign(g6, 0.0);
    v.xb.assign(g6, 0.0);
    v.vis.assign(v.N, 0x0F);
    v.outl.assign(v.N, 1);
    v.node_w.assign(v.G, 1.0);
    v.illum.clear();
    if (l == sp->L - 1) {
      for (int k = 0; k < v.G; ++k) {
        v.base[6 * k] += sp->S.coarse_s_offset[0];
        v.base[6 * k + 1] += sp->S.coarse_s_offset[1];
      }
    } else {
      const Lev& c = sp->lev[l + 1];
      v.hm.assign(2 * static_cast<size_t>(v.N), 0.0);
      orc::prolongate(c.w, c.h, v.w, v.h, sp->S.grid_step, c.total.data(), c.occ.data(), c.hm.data(), v.base.data(),
                      v.vis.data(), v.hm.data());
      v.illum.resize(4 * static_cast<size_t>(v.N));
      for (int e = 0; e < 4; ++e) {
        const double* src = v.hm.data() + static_cast<size_t>(e >> 1) * v.N;
        for (int i = 0; i < v.N; ++i) v.illum[static_cast<size_t>(e) * v.N + i] = (e & 1) ? -src[i] : src[i];
      }
    }
    v.total = v.base;
  });
}

int hwf_split_linearize(hwf_split* sp, int l, int it) {  // solver.cpp:497-511
  return guard(sp, [&] {
    if (l < 0 || l >= sp->L || it < 0 || it >= sp->gn[l]) throw std::invalid_argument("bad level/iteration");
    if (sp->flags) return;
    Lev& v = sp->lev[l];
    for (size_t i = 0; i < v.total.size(); ++i) v.total[i] = v.base[i] + v.delta[i];
    if (it > 0) sp->energy[sp->slot_base[l] + 2 * (it - 1) + 1] = owned_energy(sp, l);  // E_after(it-1)
    const hwf_level lv = level_view(sp, l);
    const orc::Level Lv = orc::make_level(&lv, &sp->P, 1);
    orc::refresh_outlier(Lv, v.outl.data());
    orc::refresh_node_w(Lv, v.node_w.data());
    sp->energy[sp->slot_base[l] + 2 * it] = owned_energy(sp, l);  // E_before(it)
    try {
      v.sys = orc::build_normal_system(Lv, sp->S.active_fields, sp->S.lm_lambda);
    } catch (const orc::Divergence& e) {
      flag(sp, e.what());
    }
  });
}

int hwf_split_sweep(hwf_split* sp, int l, int s) {  // solver.cpp:430-480, this rank's subdomains
  return guard(sp, [&] {
    if (sp->S.subdomain_px <= 0) throw std::invalid_argument("hwf_split_sweep needs Schwarz mode");
    if (l < 0 || l >= sp->L || s < 0 || s >= sp->S.patch_iters) throw std::invalid_argument("bad level/sweep");
    Lev& v = sp->lev[l];
    const size_t g6 = 6 * static_cast<size_t>(v.G);
    std::vector<double> pub(g6, 0.0);
    if (s > 0) pub = (s & 1) ? v.xb : v.xa;
    const size_t lo = 6 * static_cast<size_t>(std::max(0, v.n0 - 1)) * v.gw;
    const size_t hi = 6 * static_cast<size_t>(std::min(v.gh, v.n1 + 1)) * v.gw;
    for (size_t i = 0; i < g6; ++i)  // only owned + halo rows are legitimately known here
      if (i < lo || i >= hi) pub[i] = std::numeric_limits<double>::quiet_NaN();
    std::vector<double>& next = (s & 1) ? v.xa : v.xb;
    if (v.sys.G() != v.G) return;  // linearisation failed (flagged)
    try {
      orc::schwarz_sweep(v.sys, v.subs, v.owner, v.loc, pub, next, sp->S.pcg_iters, &v.take);
    } catch (const orc::Divergence& e) {
      flag(sp, e.what());
    }
    if (s == sp->S.patch_iters - 1) {  // solver.cpp:515-521 for the owned nodes
      for (int n = v.n0 * v.gw; n < v.n1 * v.gw; ++n)
        for (int c = 0; c < 6; ++c) {
          const size_t o = 6 * static_cast<size_t>(n) + c;
          if (!std::isfinite(next[o])) flag(sp, "non-finite Gauss-Newton update");
          if ((sp->S.active_fields >> (c >> 1)) & 1) v.delta[o] += next[o];
          v.total[o] = v.base[o] + v.delta[o];
        }
    }
  });
}

namespace {
void poison_outside(std::vector<double>& v, size_t lo, size_t hi) {
  for (size_t i = 0; i < v.size(); ++i)
    if (i < lo || i >= hi) v[i] = std::numeric_limits<double>::quiet_NaN();
}
void apply_step(hwf_split* sp, Lev& v) {  // solver.cpp:515-521 for the owned nodes
  for (int n = v.n0 * v.gw; n < v.n1 * v.gw; ++n)
    for (int c = 0; c < 6; ++c) {
      const size_t o = 6 * static_cast<size_t>(n) + c;
      if (!std::isfinite(v.px[o])) flag(sp, "non-finite Gauss-Newton update");
      if ((sp->S.active_fields >> (c >> 1)) & 1) v.delta[o] += v.px[o];
      v.total[o] = v.base[o] + v.delta[o];
    }
}
void precond_rows(const orc::System& S, const std::vector<double>& r, std::vector<double>& z, int n_lo, int n_hi) {
  for (int n = n_lo; n < n_hi; ++n)  // System::precondition, owned nodes
    for (int f = 0; f < 3; ++f) {
      const double* M = &S.pre[(static_cast<size_t>(n) * 3 + f) * 4];
      const size_t o = 6 * static_cast<size_t>(n) + 2 * f;
      z[o] = M[0] * r[o] + M[1] * r[o + 1];
      z[o + 1] = M[2] * r[o] + M[3] * r[o + 1];
    }
}
}  // namespace

int hwf_split_pcg(hwf_split* sp, int l, int phase, int it) {
  return guard(sp, [&] {
    if (sp->S.subdomain_px > 0) throw std::invalid_argument("hwf_split_pcg needs global-PCG mode");
    if (l < 0 || l >= sp->L || phase < 0 || phase > 2 || (phase > 0 && (it < 0 || it >= sp->S.pcg_iters)))
      throw std::invalid_argument("bad PCG phase");
    if (sp->flags) return;
    Lev& v = sp->lev[l];
    const size_t g6 = 6 * static_cast<size_t>(v.G);
    const int n_lo = v.n0 * v.gw, n_hi = v.n1 * v.gw;
    const size_t lo = 6 * static_cast<size_t>(n_lo), hi = 6 * static_cast<size_t>(n_hi);
    const bool last = phase == 2 && it == sp->S.pcg_iters - 1;
    if (v.sys.G() != v.G) return;  // linearisation failed (flagged)
    if (phase == 0) {  // x = 0, r = b, z = M r, p = 0 (pcg_impl with a zero start)
      for (auto* b : {&v.px, &v.pr, &v.pz, &v.pp, &v.pap, &v.part}) b->assign(g6, 0.0);
      for (size_t i = lo; i < hi; ++i) v.pr[i] = v.sys.rhs[i];
      precond_rows(v.sys, v.pr, v.pz, n_lo, n_hi);
      for (size_t i = lo; i < hi; ++i) v.part[i] = v.pr[i] * v.pz[i];
      poison_outside(v.part, lo, hi);
      v.stop = false;
      if (sp->S.pcg_iters == 0) apply_step(sp, v);
      return;
    }
    if (v.stop) {
      if (last) apply_step(sp, v);
      return;
    }
    if (phase == 1) {  // p = z (it = 0) or z + beta p over the owned and halo rows, then A p
      const size_t hlo = 6 * static_cast<size_t>(std::max(0, v.n0 - 1)) * v.gw;
      const size_t hhi = 6 * static_cast<size_t>(std::min(v.gh, v.n1 + 1)) * v.gw;
      std::vector<double> z = v.pz;
      poison_outside(z, hlo, hhi);
      for (size_t i = hlo; i < hhi; ++i) v.pp[i] = it == 0 ? z[i] : z[i] + v.beta * v.pp[i];
      std::vector<double> p = v.pp;
      poison_outside(p, hlo, hhi);
      for (int n = n_lo; n < n_hi; ++n) {  // System::apply, owned nodes
        double acc[6] = {0, 0, 0, 0, 0, 0};
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int nb = v.sys.neighbor(n, dx, dy);
            if (nb < 0) continue;
            const double* B = v.sys.block(n, orc::slot(dx, dy));
            for (int i = 0; i < 6; ++i)
              for (int j = 0; j < 6; ++j) acc[i] += B[6 * i + j] * p[6 * static_cast<size_t>(nb) + j];
          }
        for (int i = 0; i < 6; ++i) v.pap[6 * static_cast<size_t>(n) + i] = acc[i];
      }
      for (size_t i = lo; i < hi; ++i) v.part[i] = v.pp[i] * v.pap[i];
      poison_outside(v.part, lo, hi);
      return;
    }
    for (size_t i = lo; i < hi; ++i) {  // x += alpha p, r -= alpha A p, z = M r
      v.px[i] += v.alpha * v.pp[i];
      v.pr[i] -= v.alpha * v.pap[i];
    }
    precond_rows(v.sys, v.pr, v.pz, n_lo, n_hi);
    for (size_t i = lo; i < hi; ++i) v.part[i] = v.pr[i] * v.pz[i];
    poison_outside(v.part, lo, hi);
    if (last) apply_step(sp, v);
  });
}

int hwf_split_pcg_scalars(hwf_split* sp, int l, int phase, int it) {
  return guard(sp, [&] {
    if (sp->S.subdomain_px > 0) throw std::invalid_argument("hwf_split_pcg_scalars needs global-PCG mode");
    if (l < 0 || l >= sp->L || phase < 0 || phase > 2) throw std::invalid_argument("bad PCG phase");
    (void)it;
    Lev& v = sp->lev[l];
    if (v.sys.G() != v.G || (phase > 0 && v.stop)) return;
    double s = 0.0;  // the unsplit dot's additions, in index order
    for (double x : v.part) s += x;
    if (phase == 0) {
      v.rz = s;
      v.rz0 = std::abs(s);
      v.stop = v.rz0 == 0.0;  // solver.cpp:334-338
    } else if (phase == 1) {
      if (s <= 0.0) {
        flag(sp, "PCG: non-positive curvature, system not SPD");
        v.stop = true;
      } else {
        v.alpha = v.rz / s;
      }
    } else {
      if (std::abs(s) > 100.0 * v.rz0) {
        flag(sp, "PCG: preconditioned residual grew by more than 10x");
        v.stop = true;
      } else {
        v.beta = s / v.rz;
        v.rz = s;
      }
    }
  });
}

int hwf_split_energy_after(hwf_split* sp, int l) {
  return guard(sp, [&] {
    if (l < 0 || l >= sp->L) throw std::invalid_argument("level out of range");
    if (sp->flags) return;  // diverged: finish reports it; NaN flows must not reach the maps
    Lev& v = sp->lev[l];
    for (size_t i = 0; i < v.total.size(); ++i) v.total[i] = v.base[i] + v.delta[i];
    if (sp->gn[l] > 0) sp->energy[sp->slot_base[l] + 2 * (sp->gn[l] - 1) + 1] = owned_energy(sp, l);
  });
}

int hwf_split_level_end(hwf_split* sp, int l) {
  return guard(sp, [&] {
    if (l < 0 || l >= sp->L) throw std::invalid_argument("level out of range");
    if (sp->flags) return;  // diverged: finish reports it; NaN flows must not reach the maps
    Lev& v = sp->lev[l];
    for (size_t i = 0; i < v.total.size(); ++i) v.total[i] = v.base[i] + v.delta[i];
    v.occ.assign(v.N, 0);
    orc::occlusion(v.w, v.h, sp->S.grid_step, v.total.data(), v.occ.data());
    if (l > 0) {
      const hwf_level lv = level_view(sp, l);
      v.hm.assign(2 * static_cast<size_t>(v.N), 0.0);
      orc::illumination(v.w, v.h, sp->S.grid_step, lv.images, v.total.data(), v.occ.data(), v.hm.data());
    }
  });
}

int hwf_split_finish(hwf_split* sp, hwf_result* out, hwf_stats* stats) {
  return guard(sp, [&] {
    const Lev& v = sp->lev[0];
    const orc::GridDims g0 = orc::grid_dims(v.w, v.h, sp->S.grid_step);
    if (out && !sp->flags)  // (a diverged split stops before the maps; only the grid is returned)
      for (int pix = 0; pix < v.N; ++pix) {  // pin C.7
        double fl[6];
        orc::interpolate(g0, v.total.data(), pix % v.w, pix / v.w, fl);
        if (out->s) { out->s[2 * pix] = fl[0]; out->s[2 * pix + 1] = fl[1]; }
        if (out->m) { out->m[2 * pix] = fl[2]; out->m[2 * pix + 1] = fl[3]; }
        if (out->d) { out->d[2 * pix] = fl[4]; out->d[2 * pix + 1] = fl[5]; }
        if (out->disparity) out->disparity[pix] = 2.0 * fl[0];
        if (out->vis4) out->vis4[pix] = v.occ[pix];
      }
    if (out && out->grid_total) std::memcpy(out->grid_total, v.total.data(), v.total.size() * sizeof(double));
    if (stats) {
      std::memset(stats, 0, sizeof(*stats));
      stats->levels_used = sp->L;
      for (int l = 0; l < sp->L; ++l) {
        stats->gn_iters[l] = sp->gn[l];
        for (int it = 0; it < sp->gn[l] && it < HWF_MAX_GN; ++it) {
          stats->energy_before[l][it] = sp->energy[sp->slot_base[l] + 2 * it];
          stats->energy_after[l][it] = sp->energy[sp->slot_base[l] + 2 * it + 1];
        }
      }
    }
    if (sp->flags) throw orc::Divergence(sp->why.empty() ? "solver divergence (split)" : sp->why);
  });
}

}  // extern "C"
