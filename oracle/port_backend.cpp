// oracle/port_backend.cpp — TEST INFRASTRUCTURE ONLY. Backend over the
// restated per-level core (core.cpp).
#include <cstring>

#include "backend.hpp"

namespace orc {
namespace {

void copy_system(const System& S, double* blocks, double* rhs, double* precond) {
  if (blocks) std::memcpy(blocks, S.blk.data(), S.blk.size() * sizeof(double));
  if (rhs) std::memcpy(rhs, S.rhs.data(), S.rhs.size() * sizeof(double));
  if (precond) std::memcpy(precond, S.pre.data(), S.pre.size() * sizeof(double));
}

System load_system(int gw, int gh, const double* blocks, const double* rhs) {
  System S;
  S.gw = gw;
  S.gh = gh;
  const size_t G = static_cast<size_t>(gw) * gh;
  S.blk.assign(blocks, blocks + G * 9 * 36);
  S.rhs.assign(rhs, rhs + G * 6);
  S.build_preconditioner();
  return S;
}

struct Port final : Backend {
  const char* name() const override { return "oracle-port"; }
  void pyramid(const std::vector<std::vector<double>>& images, int w, int h, int levels,
               double* out) override {
    // image.cpp:177-185 per image; output level-major then image.
    std::vector<std::vector<double>> cur = images;
    int cw = w, ch = h;
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
      if (l > 0) {
        int nw = 0, nh = 0;
        for (int e = 0; e < 4; ++e) {
          std::vector<double> nxt;
          downsample(Raster{cw, ch, cur[e].data()}, nxt, &nw, &nh);
          cur[e].swap(nxt);
        }
        cw = nw;
        ch = nh;
      }
      for (int e = 0; e < 4; ++e) {
        std::memcpy(out + off, cur[e].data(), cur[e].size() * sizeof(double));
        off += cur[e].size();
      }
    }
  }
  hwf_energy eval_energy(const hwf_level* lv, const hwf_energy_params* P, double* R,
                         int threads) override {
    return energy(make_level(lv, P, threads), R);
  }
  void refresh(const hwf_level* lv, const hwf_energy_params* P, uint8_t* outlier, double* node_w,
               int threads) override {
    const Level L = make_level(lv, P, threads);
    refresh_outlier(L, outlier);
    refresh_node_w(L, node_w);
  }
  void linearize(const hwf_level* lv, const hwf_energy_params* P, uint32_t active, double lm,
                 double* blocks, double* rhs, double* precond, int threads) override {
    copy_system(build_normal_system(make_level(lv, P, threads), active, lm), blocks, rhs, precond);
  }
  void jacobian(const hwf_level* lv, const hwf_energy_params* P, uint32_t active, int negate_field,
                std::vector<double>& R, std::vector<JacEntry>& entries, int threads) override {
    std::vector<JacTriplet> t;
    assemble_jacobian(make_level(lv, P, threads), active, negate_field, R, t);
    entries.resize(t.size());
    for (size_t i = 0; i < t.size(); ++i) entries[i] = {t[i].row, t[i].col, t[i].value};
  }
  void pcg(int gw, int gh, const double* blocks, const double* rhs, int iters, double* x,
           double* trace) override {
    const System S = load_system(gw, gh, blocks, rhs);
    std::vector<double> tr;
    const std::vector<double> r = pcg_solve(S, iters, trace ? &tr : nullptr);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
    if (trace) std::memcpy(trace, tr.data(), tr.size() * sizeof(double));
  }
  void schwarz(int gw, int gh, int step, int tile, int /*boundary*/, const double* blocks,
               const double* rhs, int patch_iters, int pcg_iters, double* x) override {
    const System S = load_system(gw, gh, blocks, rhs);
    const std::vector<double> r =
        orc::schwarz(S, build_subdomains(gw, gh, step, tile), patch_iters, pcg_iters);
    std::memcpy(x, r.data(), r.size() * sizeof(double));
  }
  void gn_level(const hwf_level* lv, const double* base, double* delta, uint8_t* outlier,
                double* node_w, const hwf_energy_params* P, const hwf_schedule* S, int gn_iters,
                std::vector<double>* eb, std::vector<double>* ea,
                std::vector<std::vector<double>>* trace) override {
    gauss_newton(make_level(lv, P, S->threads > 0 ? S->threads : 1), base, delta, outlier,
                 node_w, *S, gn_iters, eb, ea, trace);
  }
};

}  // namespace

Backend* backend() {
  static Port p;
  return &p;
}

}  // namespace orc
