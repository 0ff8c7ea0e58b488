// host.h — host-side plan/level machinery shared by capi.cu (pipeline) and
// stages.cu (per-stage parity entry points).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hwflow_c.h"
#include "launch.h"

using namespace hwf;

namespace hwf_host {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArg : std::runtime_error {
  explicit InvalidArg(const std::string& m) : std::runtime_error(m) {}
};
struct Diverged : std::runtime_error {
  explicit Diverged(const std::string& m) : std::runtime_error(m) {}
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

// ---- device memory ------------------------------------------------------------
struct DevMem {
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(size_t n) {
    if (n == 0) n = 1;
    void* p = nullptr;
    CK(cudaMalloc(&p, n * sizeof(T)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
  ~DevMem() { release(); }
};

inline Params to_params(const hwf_energy_params& p) {
  Params q;
  std::memcpy(&q, &p, sizeof(q));
  return q;
}

inline int gn_for_level(const hwf_schedule& S, int l) {  // solver.hpp:30-34
  if (S.n_gn_per_level > 0) return S.gn_per_level[std::min(l, S.n_gn_per_level - 1)];
  return l <= 1 ? 2 : 5;
}

// One level's device state for a batch of B pairs.
struct LevelDev {
  int w = 0, h = 0, gw = 0, gh = 0, step = 0, ncx = 0, ncy = 0, tcx = 0, tcy = 0, rp = 0;
  int ntx = 0, nty = 0, nxm = 0, nym = 0, tile = 0;
  size_t N = 0, G = 0, C = 0;
  double* pk = nullptr;  // 32 B sample texels (k_pack)
  double *img = nullptr, *illum = nullptr, *base = nullptr, *delta = nullptr, *total = nullptr;
  double *nodew = nullptr, *nodew2 = nullptr, *nodew_a = nullptr, *nodew_b = nullptr, *half = nullptr, *cells = nullptr, *sys = nullptr, *xa = nullptr, *xb = nullptr,
         *hm = nullptr;
  const double* hmc = nullptr;  // the coarser level's half maps (illumination of this level), or null
  int wc = 0, hc = 0;           // their dims
  uint8_t *vis = nullptr, *W = nullptr, *occ = nullptr;
  int n_pix_cta = 0, n_node_cta = 0;

  void dims(int w_, int h_, int step_, int tile_px) {
    w = w_;
    h = h_;
    step = step_;
    gw = std::max((w - 1 + step - 1) / step + 1, 2);  // warp_grid.cpp:11-14
    gh = std::max((h - 1 + step - 1) / step + 1, 2);
    ncx = gw - 1;
    ncy = gh - 1;
    N = static_cast<size_t>(w) * h;
    G = static_cast<size_t>(gw) * gh;
    C = static_cast<size_t>(ncx) * ncy;
    tcx = pixel_tile_cells_x(step);
    tcy = pixel_tile_cells_y(step);
    rp = pixel_tile_pixels(w, h, step);  // k_pixel: product records per tile
    n_pix_cta = ((ncx + tcx - 1) / tcx) * ((ncy + tcy - 1) / tcy);
    n_node_cta = node_ctas(static_cast<int>(G));
    tile = tile_px;
    if (tile_px > 0) {  // solver.cpp:385-388
      ntx = ((gw - 1) * step) / tile_px + 1;
      nty = ((gh - 1) * step) / tile_px + 1;
      nxm = (tile_px + step - 1) / step;
      nym = nxm;
    }
  }
  void alloc_solver(DevMem& m, int B, bool schwarz) {
    base = m.alloc<double>(B * G * 6);
    delta = m.alloc<double>(B * G * 6);
    total = m.alloc<double>(B * G * 6);
    nodew_a = nodew = m.alloc<double>(B * G);
    nodew_b = nodew2 = m.alloc<double>(B * G);
    half = m.alloc<double>(B * N);
    cells = m.alloc<double>(B * C * kCellStride);
    sys = m.alloc<double>(B * G * kSysStride);
    W = m.alloc<uint8_t>(B * N);
    vis = m.alloc<uint8_t>(B * N);
    if (schwarz) {
      xa = m.alloc<double>(B * G * 6);
      xb = m.alloc<double>(B * G * 6);
    }
  }
};

struct Scratch {  // shared across levels, sized for the finest
  int2* q = nullptr;
  float* Z = nullptr;
  uint8_t* bad = nullptr;
  unsigned long long* zbuf = nullptr;
  uint8_t* degen = nullptr;
  unsigned long long* queue = nullptr;  // large-triangle raster queue (every triangle, worst case)
  unsigned int* qcount = nullptr;
  double *resid = nullptr, *tmp = nullptr;
  double *px = nullptr, *pr = nullptr, *pz = nullptr, *pp = nullptr, *pap = nullptr, *pp2 = nullptr;
  double *ppart = nullptr, *pstate = nullptr;
  unsigned* pcount = nullptr;
  void alloc(DevMem& m, int B, size_t N, size_t G, bool occ, bool illum, bool pcg, int pcg_tiles_max = 0) {
    if (occ) {
      q = m.alloc<int2>(B * N * 4);
      Z = m.alloc<float>(B * N);
      bad = m.alloc<uint8_t>(B * N);
      zbuf = m.alloc<unsigned long long>(B * N * 4);
      degen = m.alloc<uint8_t>(B * N * 4);
      queue = m.alloc<unsigned long long>(B * N * 8);
      qcount = m.alloc<unsigned int>(1);
    }
    if (illum) {
      resid = m.alloc<double>(B * N * 2);
      tmp = m.alloc<double>(B * N * 2);
    }
    if (pcg) {
      px = m.alloc<double>(B * G * 6);
      pr = m.alloc<double>(B * G * 6);
      pz = m.alloc<double>(B * G * 6);
      pp = m.alloc<double>(B * G * 6);
      pap = m.alloc<double>(B * G * 6);
      pp2 = m.alloc<double>(B * G * 6);
      ppart = m.alloc<double>(static_cast<size_t>(B) * pcg_tiles_max * 2);
      pstate = m.alloc<double>(static_cast<size_t>(B) * 8);
      pcount = m.alloc<unsigned>(B);
      CK(cudaMemset(pcount, 0, B * sizeof(unsigned)));
    }
  }
};

struct Energies {  // partial buffer [B][nslots][cap][5] and reduced [B][nslots][5]
  int nslots = 0, cap = 0;
  double* part = nullptr;
  double* red = nullptr;
  int* count = nullptr;  // [nslots] partials a slot's level writes (<= cap; the rest stay zero), or null
  long long pair_stride() const { return static_cast<long long>(nslots) * cap * kNumEnergy; }
  double* slot(int s) const { return part + static_cast<size_t>(s) * cap * kNumEnergy; }
};

struct Launches {
  int count = 0;
  std::vector<cudaEvent_t>* ev = nullptr;  // pixel-kernel timing events (optional)
  std::vector<double>* bytes = nullptr;
  std::vector<cudaEvent_t>* gn_ev = nullptr;  // per-GN-iteration timing events (optional): 2 per iteration
  std::vector<int>* gn_level = nullptr;       // the level of each timed iteration
  int level = 0;                              // the level record_gn_level is recording
};

// Algorithmic bytes of one k_pixel<LIN> launch: every
// input read once, every output written once.
inline double pixel_bytes(const LevelDev& d, int B, bool illum, bool u8) {
  // 4 images (32 B {v, gx, gy, 0} sample texels read with one 256-bit load, or the u8 frames at the finest
  // level), illumination (2 coarse half maps, one value per 2x2 pixels), vis4 + W in/out, halfway out
  const double perpix = 4 * (u8 ? 1.0 : 32.0) + (illum ? 2 * 8.0 / 4.0 : 0.0) + 1 + 1 + 1 + 8;
  return B * (d.N * perpix + d.G * 48.0 + d.C * kCellData * 8.0);
}

// Rows of one level a strip-split rank works on (hwflow_split.h); whole = the level.
struct Range {
  bool whole = true;
  int pix0 = 0, pix1 = 0, pown0 = 0, pown1 = 0;      // pixel-tile rows computed / owning energies
  int sw_lo = 0, sw_hi = 0;                          // k_structw nodes
  int n_lo = 0, n_hi = 0, own_lo = 0, own_hi = 0;    // k_node nodes assembled / owning energies
  int sub0 = 0, sub1 = 0;                            // Schwarz subdomains
};

inline PixArgs pixel_args(const LevelDev& d, const hwf_energy_params& P, const hwf_schedule& S, const uint8_t* src8,
                          int* flags, const Energies& E, const Range* R) {
  PixArgs pa{};
  pa.w = d.w; pa.h = d.h; pa.gw = d.gw; pa.gh = d.gh; pa.step = d.step; pa.ncx = d.ncx; pa.ncy = d.ncy;
  pa.tcx = d.tcx; pa.tcy = d.tcy; pa.rp = d.rp;
  pa.pk = d.pk; pa.src8 = src8; pa.illum = d.illum; pa.vis4 = d.vis; pa.W = d.W;
  pa.hmc = d.hmc; pa.wc = d.wc; pa.hc = d.hc;
  pa.total = d.total; pa.half = d.half; pa.cells = d.cells; pa.ep_pair = E.pair_stride(); pa.flags = flags;
  pa.P = to_params(P); pa.active = S.active_fields;
  if (R && !R->whole) {
    pa.ty0 = R->pix0; pa.ty1 = R->pix1; pa.own0 = R->pown0; pa.own1 = R->pown1;
  }
  return pa;
}

inline NodeArgs node_args(const LevelDev& d, const hwf_energy_params& P, const hwf_schedule& S, const double* dF,
                          int* flags, const Energies& E, const Range* R) {
  NodeArgs na{};
  na.w = d.w; na.h = d.h; na.gw = d.gw; na.gh = d.gh; na.step = d.step; na.ncx = d.ncx; na.ncy = d.ncy;
  na.half = d.half; na.node_w = d.nodew; na.node_w_new = d.nodew; na.total = d.total; na.delta = d.delta;
  na.cells = d.cells; na.sys = d.sys; na.ep_pair = E.pair_stride(); na.ep_base = d.n_pix_cta; na.flags = flags;
  na.P = to_params(P); na.F = dF; na.active = S.active_fields; na.lm = S.lm_lambda;
  na.soa = S.subdomain_px <= 0;  // the global PCG reads entry-major records
  if (R && !R->whole) {
    na.n_lo = R->n_lo; na.n_hi = R->n_hi; na.own_lo = R->own_lo; na.own_hi = R->own_hi;
  }
  return na;
}

// One Gauss-Newton linearisation (solver.cpp:497-511): refresh W and w_i, energies with the old
// and new weights, J^T J / J^T r into the system. Leaves d.nodew pointing at the refreshed w_i.
inline void rec_linearize(LevelDev& d, int B, const hwf_energy_params& P, const hwf_schedule& S, const double* dF,
                          int it, const Energies& E, int slot_base, int* flags, cudaStream_t st, Launches& L,
                          const uint8_t* src8, const Range* R = nullptr) {
  double* wnew = d.nodew == d.nodew_a ? d.nodew_b : d.nodew_a;  // ping-pong w_i
  PixArgs pa = pixel_args(d, P, S, src8, flags, E, R);
  pa.refresh = 1;
  pa.ep_new = E.slot(slot_base + 2 * it);
  pa.ep_old = it > 0 ? E.slot(slot_base + 2 * (it - 1) + 1) : nullptr;
  if (L.ev) CK(cudaEventRecordWithFlags((*L.ev)[2 * L.bytes->size()], st, cudaEventRecordExternal));
  launch_pixel(true, pa, B, st);
  if (L.ev) {
    CK(cudaEventRecordWithFlags((*L.ev)[2 * L.bytes->size() + 1], st, cudaEventRecordExternal));
    L.bytes->push_back(pixel_bytes(d, B, d.hmc != nullptr, src8 != nullptr));
  }
  const bool whole = !R || R->whole;
  launch_structw(d.w, d.h, d.gw, d.gh, d.step, d.half, wnew, B, st, whole ? 0 : R->sw_lo, whole ? -1 : R->sw_hi);
  NodeArgs na = node_args(d, P, S, dF, flags, E, R);
  na.node_w_new = wnew;
  na.refresh = 1;
  na.ep_new = pa.ep_new;
  na.ep_old = pa.ep_old;
  launch_node(true, na, B, st);
  L.count += 3;
  d.nodew = wnew;
}

// Sweep s of schwarz_iterate (solver.cpp:414-482); the last sweep applies the step.
inline void rec_sweep(LevelDev& d, int B, const hwf_schedule& S, int s, int* flags, cudaStream_t st, Launches& L,
                      const Range* R = nullptr) {
  SwzArgs sa{};
  sa.gw = d.gw; sa.gh = d.gh; sa.step = d.step; sa.tile = d.tile; sa.ntx = d.ntx; sa.nty = d.nty;
  sa.nxm = d.nxm; sa.nym = d.nym; sa.sys = d.sys; sa.delta = d.delta; sa.total = d.total;
  sa.base = d.base; sa.active = S.active_fields; sa.pcg_iters = S.pcg_iters; sa.flags = flags;
  sa.pub = s == 0 ? nullptr : (s & 1 ? d.xb : d.xa);
  sa.next = s & 1 ? d.xa : d.xb;
  sa.last = s == S.patch_iters - 1;
  if (R && !R->whole) {
    sa.sub0 = R->sub0;
    sa.sub1 = R->sub1;
  }
  launch_schwarz(sa, B, st);
  L.count += 1;
}
// The buffer sweep s publishes (read by sweep s + 1).
inline double* swept(LevelDev& d, int s) { return s & 1 ? d.xa : d.xb; }

// E_after of the last iteration (solver.cpp:523-528).
inline void rec_energy_after(LevelDev& d, int B, const hwf_energy_params& P, const hwf_schedule& S, const double* dF,
                             int gn, const Energies& E, int slot_base, int* flags, cudaStream_t st, Launches& L,
                             const uint8_t* src8, const Range* R = nullptr, int2* occ_q = nullptr,
                             float* occ_z = nullptr, uint8_t* occ_bad = nullptr) {
  PixArgs pa = pixel_args(d, P, S, src8, flags, E, R);
  pa.refresh = 0;
  pa.occ_q = occ_q;  // non-null: also write the level's occlusion vertices (k_occ_project's work)
  pa.occ_z = occ_z;
  pa.occ_bad = occ_bad;
  pa.ep_new = E.slot(slot_base + 2 * (gn - 1) + 1);
  pa.ep_old = nullptr;
  if (R && !R->whole) {  // energies only: the owned rows
    pa.ty0 = R->pown0;
    pa.ty1 = R->pown1;
  }
  launch_pixel(false, pa, B, st);
  NodeArgs na = node_args(d, P, S, dF, flags, E, R);
  if (R && !R->whole) {
    na.n_lo = R->own_lo;
    na.n_hi = R->own_hi;
  }
  na.refresh = 0;
  na.ep_new = pa.ep_new;
  na.ep_old = nullptr;
  launch_node(false, na, B, st);
  L.count += 2;
}

// The nonlinear loop of one level (solver.cpp:484-532) for a batch, whole level.
inline void record_gn_level(LevelDev& d, int B, const hwf_energy_params& P, const hwf_schedule& S, const double* dF,
                            int gn, const Energies& E, int slot_base, Scratch& sc, int* flags, cudaStream_t st,
                            Launches& L, const uint8_t* src8 = nullptr, bool energy_after = true,
                            double* pcg_trace = nullptr) {  // device [gn][pcg_iters + 1], global mode, B = 1
  for (int it = 0; it < gn; ++it) {
    const size_t gi = L.gn_level ? L.gn_level->size() : 0;
    if (L.gn_ev) CK(cudaEventRecordWithFlags((*L.gn_ev)[2 * gi], st, cudaEventRecordExternal));
    rec_linearize(d, B, P, S, dF, it, E, slot_base, flags, st, L, src8);
    if (S.subdomain_px > 0) {
      for (int s = 0; s < S.patch_iters; ++s) rec_sweep(d, B, S, s, flags, st, L);
    } else {
      PcgArgs ga{};
      ga.gw = d.gw; ga.gh = d.gh; ga.iters = S.pcg_iters; ga.sys = d.sys;
      ga.x = sc.px; ga.r = sc.pr; ga.z = sc.pz; ga.p = sc.pp; ga.ap = sc.pap; ga.update = 1;
      ga.p2 = sc.pp2; ga.part = sc.ppart; ga.state = sc.pstate; ga.count = sc.pcount;
      ga.trace = pcg_trace ? pcg_trace + static_cast<size_t>(it) * (S.pcg_iters + 1) : nullptr;
      ga.delta = d.delta; ga.total = d.total; ga.base = d.base; ga.active = S.active_fields; ga.flags = flags;
      launch_pcg_global(ga, B, st);
      L.count += pcg_launches(d.gw, d.gh, S.pcg_iters);
    }
    if (L.gn_ev) {  // linearisation + solve of one GN iteration (the E_after pass of a level's last is not in it)
      CK(cudaEventRecordWithFlags((*L.gn_ev)[2 * gi + 1], st, cudaEventRecordExternal));
      L.gn_level->push_back(L.level);
    }
  }
  if (gn > 0 && energy_after) rec_energy_after(d, B, P, S, dF, gn, E, slot_base, flags, st, L, src8);
}

// ---- the batched plan (one CUDA graph per configuration) ------------------------
struct Plan {
  int B = 0, w = 0, h = 0, dtype = 0;
  hwf_energy_params P{};
  hwf_schedule S{};
  bool hasF = false;
  double F[9] = {};
  unsigned outmask = 0;  // 1 s, 2 m, 4 d, 8 disparity
  bool profile = false;
  bool has_prev = false;  // temporal propagation from a previous frame's state
  double* prev_delta[HWF_MAX_LEVELS] = {};
  double* prev_total[HWF_MAX_LEVELS] = {};

  int L = 0;
  LevelDev lv[HWF_MAX_LEVELS];
  int gn[HWF_MAX_LEVELS] = {};
  int slot_base[HWF_MAX_LEVELS] = {};
  DevMem mem;
  void* in = nullptr;
  double* dF = nullptr;
  Scratch sc;
  Energies E;
  int* flags = nullptr;
  double *o_s = nullptr, *o_m = nullptr, *o_d = nullptr, *o_disp = nullptr;
  double* o_slot[2][4] = {{nullptr, nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr, nullptr}};  // streaming
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // streaming (hwf_submit_batch / hwf_wait): two input/result slots, one graph each
  bool async_ready = false;
  void* in_slot[2] = {};
  cudaGraph_t graph2 = nullptr;
  cudaGraphExec_t exec_slot[2] = {};
  double* st_grid[2] = {};
  uint8_t* st_occ[2] = {};
  double* st_red[2] = {};
  int* st_flags[2] = {};
  double* h_red[2] = {};  // pinned
  int* h_flags[2] = {};   // pinned
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  int launches = 0;
  std::vector<cudaEvent_t> ev;
  std::vector<double> ev_bytes;
  std::vector<cudaEvent_t> gev;  // profile: two events per GN iteration
  std::vector<int> gev_level;

  bool matches(int B_, int w_, int h_, int dt, const hwf_energy_params& P_, const hwf_schedule& S_, const double* F_,
               unsigned om, bool prof, bool prev) const {
    if (B != B_ || w != w_ || h != h_ || dtype != dt || outmask != om || profile != prof || has_prev != prev)
      return false;
    if (std::memcmp(&P, &P_, sizeof(P)) || std::memcmp(&S, &S_, sizeof(S))) return false;
    if (hasF != (F_ != nullptr)) return false;
    return !F_ || std::memcmp(F, F_, sizeof(F)) == 0;
  }
  ~Plan() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (exec_slot[1]) cudaGraphExecDestroy(exec_slot[1]);
    if (graph2) cudaGraphDestroy(graph2);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : gev) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
      if (h_red[k]) cudaFreeHost(h_red[k]);
      if (h_flags[k]) cudaFreeHost(h_flags[k]);
      for (cudaEvent_t e : {ev_h2d[k], ev_comp[k], ev_d2h[k]})
        if (e) cudaEventDestroy(e);
    }
  }

  // The finest level of u8 frames samples the frames themselves (k_pixel<*, U8>).
  bool u8_finest(int l) const { return l == 0 && dtype == HWF_DTYPE_U8; }
  // Device input frames; u8 frames get 16 B of padding on both sides (ld4u8).
  void* alloc_input(size_t N0) {
    if (dtype == HWF_DTYPE_U8) return mem.alloc<uint8_t>(B * 4 * N0 + 32) + 16;
    return mem.alloc<double>(B * 4 * N0);
  }

  // Second input slot + its own captured graph + result staging (streaming API).
  void ensure_async(cudaStream_t st) {
    if (async_ready) return;
    const size_t N0 = lv[0].N, G0 = lv[0].G;
    in_slot[0] = in;
    in_slot[1] = alloc_input(N0);
    // dense FlowResult fields: slot 1's graph writes its own copies, so a batch's download never races
    // the next batch's solve (slot 0 keeps the plan's buffers)
    double** o[4] = {&o_s, &o_m, &o_d, &o_disp};
    for (int f = 0; f < 4; ++f) o_slot[0][f] = *o[f];
    for (int f = 0; f < 4; ++f)
      o_slot[1][f] = (outmask >> f & 1) ? mem.alloc<double>(B * N0 * (f == 3 ? 1 : 2)) : nullptr;
    for (int k = 0; k < 2; ++k) {
      st_grid[k] = mem.alloc<double>(B * G0 * 6);
      st_occ[k] = mem.alloc<uint8_t>(B * N0);
      st_red[k] = mem.alloc<double>(static_cast<size_t>(B) * E.nslots * kNumEnergy);
      st_flags[k] = mem.alloc<int>(B);
      CK(cudaMallocHost(&h_red[k], sizeof(double) * B * E.nslots * kNumEnergy));
      CK(cudaMallocHost(&h_flags[k], sizeof(int) * B));
      CK(cudaEventCreateWithFlags(&ev_h2d[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_comp[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_d2h[k], cudaEventDisableTiming));
    }
    // capture the same pipeline reading slot 1 (w_i ping-pong restarts from buffer a)
    for (int l = 0; l < L; ++l) lv[l].nodew = lv[l].nodew_a;
    auto use_slot = [&](int k) {
      in = in_slot[k];
      for (int f = 0; f < 4; ++f) *o[f] = o_slot[k][f];
    };
    use_slot(1);
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      record(st);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      use_slot(0);
      throw;
    }
    CK(cudaStreamEndCapture(st, &graph2));
    CK(cudaGraphInstantiate(&exec_slot[1], graph2, 0));
    exec_slot[0] = exec;
    use_slot(0);
    async_ready = true;
  }

  void build(cudaStream_t st) {
    alloc();
    // capture the pipeline into one graph
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      record(st);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(st, &graph));
    CK(cudaGraphInstantiate(&exec, graph, 0));
  }

  // Level dims, schedule and every device buffer of the plan (no capture).
  void alloc() {
    int dims[4 * HWF_MAX_LEVELS];
    if (hwf_level_dims(w, h, S.levels, S.grid_step, &L, dims) != HWF_OK) throw InvalidArg("bad level dims");
    size_t cap = 0;
    int nslots = 0;
    for (int l = 0; l < L; ++l) {
      lv[l].dims(dims[4 * l], dims[4 * l + 1], S.grid_step, S.subdomain_px);
      gn[l] = gn_for_level(S, l);
      if (gn[l] > HWF_MAX_GN) throw InvalidArg("gn_per_level exceeds HWF_MAX_GN");
      slot_base[l] = nslots;
      nslots += 2 * gn[l];
      cap = std::max(cap, static_cast<size_t>(lv[l].n_pix_cta + lv[l].n_node_cta));
    }
    const size_t N0 = lv[0].N;
    in = alloc_input(N0);
    for (int l = 0; l < L; ++l) {
      LevelDev& d = lv[l];
      if (!u8_finest(l)) {
        d.img = mem.alloc<double>(B * 4 * d.N);
        d.pk = mem.alloc<double>(B * 4 * d.N * 4);
      }
      d.alloc_solver(mem, B, S.subdomain_px > 0);
      d.occ = mem.alloc<uint8_t>(B * d.N);

      if (has_prev) {
        prev_delta[l] = mem.alloc<double>(B * d.G * 6);
        prev_total[l] = mem.alloc<double>(B * d.G * 6);
      }
      if (l > 0) d.hm = mem.alloc<double>(B * 2 * d.N);
      if (l > 0) {  // level l-1 reads this level's half maps as its illumination (pin C.4)
        lv[l - 1].hmc = d.hm;
        lv[l - 1].wc = d.w;
        lv[l - 1].hc = d.h;
      }
    }
    sc.alloc(mem, B, N0, lv[0].G, true, L > 1, S.subdomain_px <= 0, pcg_tiles(lv[0].gw, lv[0].gh));
    E.nslots = std::max(nslots, 1);
    E.cap = static_cast<int>(cap);
    {  // the reduction reads only a slot's own level's partials (coarse slots hold far fewer than cap)
      std::vector<int> cnt(E.nslots, E.cap);
      for (int l = 0; l < L; ++l)
        for (int k = 0; k < 2 * gn[l]; ++k) cnt[slot_base[l] + k] = lv[l].n_pix_cta + lv[l].n_node_cta;
      E.count = mem.alloc<int>(E.nslots);
      CK(cudaMemcpy(E.count, cnt.data(), sizeof(int) * E.nslots, cudaMemcpyHostToDevice));
    }
    E.part = mem.alloc<double>(static_cast<size_t>(B) * E.pair_stride());
    E.red = mem.alloc<double>(static_cast<size_t>(B) * E.nslots * kNumEnergy);
    flags = mem.alloc<int>(B);
    if (hasF) {
      dF = mem.alloc<double>(9);
      CK(cudaMemcpy(dF, F, sizeof(F), cudaMemcpyHostToDevice));
    }
    if (outmask & 1) o_s = mem.alloc<double>(B * N0 * 2);
    if (outmask & 2) o_m = mem.alloc<double>(B * N0 * 2);
    if (outmask & 4) o_d = mem.alloc<double>(B * N0 * 2);
    if (outmask & 8) o_disp = mem.alloc<double>(B * N0);
    if (profile) {
      int total_gn = 0;
      for (int l = 0; l < L; ++l) total_gn += gn[l];
      ev.resize(2 * std::max(total_gn, 1));
      for (auto& e : ev) CK(cudaEventCreate(&e));
      gev.resize(2 * std::max(total_gn, 1));
      for (auto& e : gev) CK(cudaEventCreate(&e));
    }
  }

  const uint8_t* src8(int l) const { return u8_finest(l) ? static_cast<const uint8_t*>(in) : nullptr; }

  void record(cudaStream_t st) {
    Launches LC;
    ev_bytes.clear();
    gev_level.clear();
    if (profile) {
      LC.ev = &ev;
      LC.bytes = &ev_bytes;
      LC.gn_ev = &gev;
      LC.gn_level = &gev_level;
    }
    rec_prologue(st, LC);
    for (int l = L - 1; l >= 0; --l) {
      rec_level_begin(l, st, LC);
      LC.level = l;
      record_gn_level(lv[l], B, P, S, dF, gn[l], E, slot_base[l], sc, flags, st, LC, src8(l), false);
      if (gn[l] > 0) {
        // E_after of the level's last iteration (stats) fused with the occlusion projection of the same flow:
        // one pass interpolates the final flow per pixel for both, then raster/resolve and illumination
        rec_energy_after(lv[l], B, P, S, dF, gn[l], E, slot_base[l], flags, st, LC, src8(l), nullptr, sc.q, sc.Z,
                         sc.bad);
        rec_level_end(l, st, LC, true);
      } else {
        rec_level_end(l, st, LC);
      }
    }
    rec_epilogue(st, LC);
    launches = LC.count;
  }

  // energy/flag reset, pyramid (image.cpp:177-185), sample planes
  void rec_prologue(cudaStream_t st, Launches& LC) {
    CK(cudaMemsetAsync(E.part, 0, sizeof(double) * B * E.pair_stride(), st));
    CK(cudaMemsetAsync(flags, 0, sizeof(int) * B, st));
    // pyramid (image.cpp:177-185); u8 frames: level 1 comes from the bytes, level 0 is never stored
    if (!u8_finest(0)) {
      launch_pyr_in(in, dtype, lv[0].img, static_cast<long long>(B) * 4 * lv[0].N, st);
      LC.count++;
    }
    for (int l = 1; l < L; ++l) {
      if (l == 1 && u8_finest(0))
        launch_pyr_down_u8(static_cast<const uint8_t*>(in), lv[0].w, lv[0].h, lv[1].img, lv[1].w, lv[1].h, 4 * B, st);
      else
        launch_pyr_down(lv[l - 1].img, lv[l - 1].w, lv[l - 1].h, lv[l].img, lv[l].w, lv[l].h, 4 * B, st);
      LC.count++;
    }
    for (int l = 0; l < L; ++l) {
      if (u8_finest(l)) continue;
      launch_pack(lv[l].img, lv[l].w, lv[l].h, 4 * B, lv[l].pk, st);
      LC.count++;
    }
  }

  // coarsest init (pin C.6) or prolongation, warm start, W / w_i reset
  void rec_level_begin(int l, cudaStream_t st, Launches& LC) {
    LevelDev& d = lv[l];
    if (l == L - 1) {  // pin C.6
      launch_init_coarse(d.base, d.total, d.delta, static_cast<int>(d.G), B, S.coarse_s_offset[0],
                         S.coarse_s_offset[1], st);
      CK(cudaMemsetAsync(d.vis, 0x0F, B * d.N, st));
      LC.count++;
    } else {  // prolongation
      const LevelDev& c = lv[l + 1];
      launch_prolong_grid(c.gw, c.gh, d.gw, d.gh, d.step, c.total, d.base, d.total, d.delta, B, st);
      launch_prolong_maps(c.w, c.h, d.w, d.h, c.occ, nullptr, d.vis, nullptr, B, st);
      LC.count += 2;
    }
    if (has_prev) {  // warm start: delta_l = advected previous delta
      launch_propagate(d.gw, d.gh, d.step, prev_delta[l], prev_total[l], d.base, d.delta, d.total, B, st);
      LC.count++;
    }
    CK(cudaMemsetAsync(d.W, 1, B * d.N, st));
    CK(cudaMemsetAsync(d.nodew, 0, sizeof(double) * B * d.G, st));
  }

  // occlusion and illumination of the solved level
  void rec_level_end(int l, cudaStream_t st, Launches& LC, bool projected = false) {
    LevelDev& d = lv[l];
    if (projected) {  // the vertices were written by the fused E_after pass
      launch_occlusion_projected(d.w, d.h, B, sc.q, sc.Z, sc.bad, sc.zbuf, sc.degen, sc.queue, sc.qcount, d.occ, st);
      LC.count += 3;
    } else {
      launch_occlusion(d.w, d.h, d.gw, d.gh, d.step, d.total, B, sc.q, sc.Z, sc.bad, sc.zbuf, sc.degen, sc.queue,
                       sc.qcount, d.occ, st);
      LC.count += 4;
    }
    if (l > 0) {
      launch_illumination(d.w, d.h, d.gw, d.gh, d.step, d.img, d.total, d.occ, B, sc.resid, sc.tmp, d.hm, st);
      LC.count += 3;
    }
  }

  // dense FlowResult (pin C.7) and the per-slot energy reduction
  void rec_epilogue(cudaStream_t st, Launches& LC) {
    if (outmask & 15) {
      launch_dense(lv[0].w, lv[0].h, lv[0].gw, lv[0].gh, lv[0].step, lv[0].total, B, o_s, o_m, o_d, o_disp, st);
      LC.count++;
    }
    launch_energy_reduce(E.part, E.nslots, E.cap, B, E.red, flags, st, E.count);
    LC.count++;
    CK(cudaGetLastError());
  }
};

}  // namespace hwf_host

// Device-resident per-level state of n pairs (SPEC.md:396 `prev`).
struct hwf_state {
  int device = 0, n = 0, w = 0, h = 0, L = 0, step = 0;
  bool valid = false;
  size_t G[HWF_MAX_LEVELS] = {};
  double* delta[HWF_MAX_LEVELS] = {};
  double* total[HWF_MAX_LEVELS] = {};
  ~hwf_state() {
    cudaSetDevice(device);
    for (int l = 0; l < L; ++l) {
      if (delta[l]) cudaFree(delta[l]);
      if (total[l]) cudaFree(total[l]);
    }
  }
};

struct hwf_inflight {  // one submitted streaming batch
  int slot = 0, n = 0;
  std::vector<hwf_result> out;
  hwf_stats* stats = nullptr;
};

struct hwf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the streaming API
  std::string err;
  std::unique_ptr<hwf_host::Plan> plan;
  bool profile = false;
  std::deque<hwf_inflight> inflight;
  int next_slot = 0;
};

namespace hwf_host {

template <class Fn>
int guard(hwf_ctx* ctx, Fn&& fn) {
  try {
    if (!ctx) throw InvalidArg("null context");
    CK(cudaSetDevice(ctx->device));
    fn();
    return HWF_OK;
  } catch (const InvalidArg& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EINVAL;
  } catch (const Diverged& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EDIVERGED;
  } catch (const CudaError& e) {
    if (ctx) ctx->err = e.what();
    return HWF_ECUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return HWF_EINVAL;
  }
}

inline void check_params(const hwf_energy_params* P, const hwf_schedule* S, const double* F) {
  if (!P || !S) throw InvalidArg("null params/schedule");
  if (hwf_validate_params(P) != HWF_OK) throw InvalidArg("energy weights must be >= 0 and eps_huber > 0");
  if (P->w_epi > 0.0 && !F) throw InvalidArg("epipolar term enabled without a fundamental matrix");
  if (S->grid_step < 1 || S->grid_step > 32) throw InvalidArg("grid_step must be in [1, 32] on the device");
  if (S->subdomain_px > 0) {  // one CTA of <= 1024 threads per subdomain, a thread per unknown
    const long long side = (static_cast<long long>(S->subdomain_px) + S->grid_step - 1) / S->grid_step;
    if (6 * side * side > 1024) throw InvalidArg("subdomain tile must hold <= 13x13 nodes on the device");
  }
  if (S->pcg_iters < 0 || S->patch_iters < 0) throw InvalidArg("negative iteration count");
}

inline void upload_frames(Plan& p, int n, const hwf_frame4* fr, cudaStream_t st) {
  const size_t N = static_cast<size_t>(p.w) * p.h;
  const size_t esz = p.dtype == HWF_DTYPE_U8 ? 1 : 8;
  // fast path: all 4n planes contiguous in one host allocation
  bool contiguous = true;
  const char* base = static_cast<const char*>(fr[0].plane[0]);
  for (int i = 0; i < n && contiguous; ++i)
    for (int e = 0; e < 4; ++e)
      contiguous = contiguous && static_cast<const char*>(fr[i].plane[e]) == base + (4 * static_cast<size_t>(i) + e) * N * esz;
  if (contiguous) {
    CK(cudaMemcpyAsync(p.in, base, 4 * n * N * esz, cudaMemcpyHostToDevice, st));
    return;
  }
  for (int i = 0; i < n; ++i)
    for (int e = 0; e < 4; ++e)
      CK(cudaMemcpyAsync(static_cast<char*>(p.in) + (4 * static_cast<size_t>(i) + e) * N * esz, fr[i].plane[e],
                         N * esz, cudaMemcpyHostToDevice, st));
}

inline Plan& get_plan(hwf_ctx* ctx, int n, int w, int h, int dtype, const hwf_energy_params* P, const hwf_schedule* S,
               const double* F, unsigned outmask, bool has_prev = false) {
  if (ctx->plan && ctx->plan->matches(n, w, h, dtype, *P, *S, F, outmask, ctx->profile, has_prev)) return *ctx->plan;
  if (!ctx->inflight.empty()) throw InvalidArg("a different configuration was requested while batches are in flight");
  ctx->plan.reset();
  CK(cudaStreamSynchronize(ctx->stream));
  auto p = std::make_unique<Plan>();
  p->B = n;
  p->w = w;
  p->h = h;
  p->dtype = dtype;
  p->P = *P;
  p->S = *S;
  p->hasF = F != nullptr;
  if (F) std::memcpy(p->F, F, sizeof(p->F));
  p->outmask = outmask;
  p->profile = ctx->profile;
  p->has_prev = has_prev;
  p->build(ctx->stream);
  ctx->plan = std::move(p);
  return *ctx->plan;
}

inline void finish_stats(const Plan& p, int n, hwf_stats* stats, std::vector<int>& flags) {
  std::vector<double> red(static_cast<size_t>(p.B) * p.E.nslots * kNumEnergy);
  flags.resize(p.B);
  // (the stream is synchronous with these blocking copies)
  CK(cudaMemcpy(red.data(), p.E.red, red.size() * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(flags.data(), p.flags, sizeof(int) * p.B, cudaMemcpyDeviceToHost));
  if (!stats) return;
  const hwf_energy_params& P = p.P;
  for (int i = 0; i < n; ++i) {
    hwf_stats& s = stats[i];
    std::memset(&s, 0, sizeof(s));
    s.levels_used = p.L;
    for (int l = 0; l < p.L; ++l) {
      s.gn_iters[l] = p.gn[l];
      for (int it = 0; it < p.gn[l]; ++it)
        for (int k = 0; k < 2; ++k) {
          const double* e = red.data() + (static_cast<size_t>(i) * p.E.nslots + p.slot_base[l] + 2 * it + k) * kNumEnergy;
          const double tot = P.w_photo * e[0] + P.w_grad * e[1] + P.w_reg * (P.w_smooth * e[2] + P.w_epi * e[3] + P.w_mag * e[4]);
          (k == 0 ? s.energy_before : s.energy_after)[l][it] = tot;
        }
    }
  }
}

inline void raise_on_flags(const std::vector<int>& flags, int n) {
  std::string msg;
  for (int i = 0; i < n; ++i)
    if (flags[i]) {
      if (!msg.empty()) msg += "; ";
      msg += "pair " + std::to_string(i) + ":";
      if (flags[i] & kFlagJacobian) msg += " non-finite Jacobian";
      if (flags[i] & kFlagCurvature) msg += " PCG: non-positive curvature, system not SPD";
      if (flags[i] & kFlagGrowth) msg += " PCG: preconditioned residual grew by more than 10x";
      if (flags[i] & kFlagStep) msg += " non-finite Gauss-Newton update";
      if (flags[i] & kFlagEnergy) msg += " non-finite energy";
    }
  if (!msg.empty()) throw Diverged(msg);
}

}  // namespace hwf_host
