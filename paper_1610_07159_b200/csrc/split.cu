// split.cu — strip-split solve of one frame pair across ranks (include/hwflow_split.h).
//
// A rank reuses the batched plan's buffers and step recorders (host.h), with B = 1 and no
// graph capture. It computes with the Range of its strip:
//   - Schwarz subdomains of tile rows [t0, t1), which are the node rows [n0, n1) (solver.cpp:382-412);
//   - k_node over rows [n0-1, n1), because the coupling blocks of row n0 live in row n0-1's
//     forward slots (solver.cpp:15-17, 228-241);
//   - k_structw over rows [n0-2, n1) (k_node reads the w_i of its left and up neighbours);
//   - k_pixel over the pixel-tile rows covering cell rows [n0-3, n1), the cells and the halfway
//     pixels those nodes read.
// Energy partials come from owned rows only. The driver exchanges data between steps
// (header). Pyramid, prolongation, occlusion, illumination and the dense outputs run
// replicated on every rank: they read the all-gathered grid.
#include <algorithm>
#include <cstring>
#include <memory>

#include "hwflow_c.h"
#include "hwflow_split.h"
#include "host.h"

using namespace hwf_host;

struct hwf_split {
  hwf_ctx* ctx = nullptr;
  int rank = 0, world = 1;
  std::unique_ptr<Plan> plan;
  Range range[HWF_MAX_LEVELS];
  int n0[HWF_MAX_LEVELS] = {}, n1[HWF_MAX_LEVELS] = {};
  Launches LC;
};

namespace {

int ceil_div(int a, int b) { return (a + b - 1) / b; }

// The strip of `rank` at one level; the same formula runs in oracle/split.cpp. Schwarz mode:
// a band of subdomain tile rows. Global-PCG mode (tile_px = 0): a band of node rows.
void strip(const LevelDev& d, int tile_px, int rank, int world, Range& R, int& n0, int& n1) {
  const int gh = d.gh, gw = d.gw, step = d.step;
  const int nty = tile_px > 0 ? d.nty : gh;
  const int t0 = static_cast<int>(static_cast<long long>(rank) * nty / world);
  const int t1 = static_cast<int>(static_cast<long long>(rank + 1) * nty / world);
  n0 = tile_px > 0 ? std::min(gh, ceil_div(t0 * tile_px, step)) : t0;
  n1 = rank == world - 1 ? gh : (tile_px > 0 ? std::min(gh, ceil_div(t1 * tile_px, step)) : t1);
  const int rows = ceil_div(d.ncy, d.tcy);
  R.whole = false;
  R.sub0 = tile_px > 0 ? t0 * d.ntx : 0;
  R.sub1 = tile_px > 0 ? t1 * d.ntx : 0;
  R.own_lo = n0 * gw;
  R.own_hi = n1 * gw;
  if (n1 <= n0) {  // nothing owned at this level
    R.n_lo = R.n_hi = R.sw_lo = R.sw_hi = 0;
    R.pix0 = R.pix1 = R.pown0 = R.pown1 = 0;
    return;
  }
  R.n_lo = std::max(0, n0 - 1) * gw;
  R.n_hi = n1 * gw;
  R.sw_lo = std::max(0, n0 - 2) * gw;
  R.sw_hi = n1 * gw;
  const int c0 = std::max(0, n0 - 3), c1 = std::min(d.ncy, n1);
  R.pix0 = c0 / d.tcy;
  R.pix1 = std::max(R.pix0, ceil_div(c1, d.tcy));
  R.pown0 = ceil_div(n0, d.tcy);
  R.pown1 = rank == world - 1 ? rows : ceil_div(n1, d.tcy);
  if (rank == world - 1) R.pix1 = rows;
}

hwf_split* checked(hwf_split* sp, int level = 0) {
  if (!sp || !sp->plan) throw InvalidArg("null split");
  if (level < 0 || level >= sp->plan->L) throw InvalidArg("level out of range");
  return sp;
}

}  // namespace

extern "C" {

int hwf_split_create(hwf_ctx* ctx, int w, int h, int dtype, const hwf_energy_params* params,
                     const hwf_schedule* sched, const double* F, int rank, int world, hwf_split** out) {
  return guard(ctx, [&] {
    if (!out) throw InvalidArg("null out");
    check_params(params, sched, F);
    if (world < 1 || rank < 0 || rank >= world) throw InvalidArg("bad rank/world");
    if (w < 2 || h < 2) throw InvalidArg("bad frame dims");
    if (dtype != HWF_DTYPE_U8 && dtype != HWF_DTYPE_F64) throw InvalidArg("unknown dtype");
    auto sp = std::make_unique<hwf_split>();
    sp->ctx = ctx;
    sp->rank = rank;
    sp->world = world;
    auto p = std::make_unique<Plan>();
    p->B = 1;
    p->w = w;
    p->h = h;
    p->dtype = dtype;
    p->P = *params;
    p->S = *sched;
    p->hasF = F != nullptr;
    if (F) std::memcpy(p->F, F, sizeof(p->F));
    p->outmask = 15;
    p->alloc();
    for (int l = 0; l < p->L; ++l) strip(p->lv[l], sched->subdomain_px, rank, world, sp->range[l], sp->n0[l], sp->n1[l]);
    sp->plan = std::move(p);
    *out = sp.release();
  });
}

void hwf_split_destroy(hwf_split* sp) {
  if (!sp) return;
  if (sp->ctx) cudaSetDevice(sp->ctx->device);
  delete sp;
}

int hwf_split_schedule(hwf_split* sp, int* levels, int* gn) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp);
    if (levels) *levels = sp->plan->L;
    if (gn)
      for (int l = 0; l < sp->plan->L; ++l) gn[l] = sp->plan->gn[l];
  });
}

int hwf_split_rows(hwf_split* sp, int level, int* n0, int* n1, int* gw) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp, level);
    if (n0) *n0 = sp->n0[level];
    if (n1) *n1 = sp->n1[level];
    if (gw) *gw = sp->plan->lv[level].gw;
  });
}

int hwf_split_buffer(hwf_split* sp, int level, const char* name, void** ptr, long long* count) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp, level);
    if (!name || !ptr || !count) throw InvalidArg("null buffer query");
    Plan& p = *sp->plan;
    LevelDev& d = p.lv[level];
    const long long g6 = 6LL * static_cast<long long>(d.G);
    if (!std::strcmp(name, "xa")) { *ptr = d.xa; *count = g6; }
    else if (!std::strcmp(name, "xb")) { *ptr = d.xb; *count = g6; }
    else if (!std::strcmp(name, "total")) { *ptr = d.total; *count = g6; }
    else if (!std::strcmp(name, "delta")) { *ptr = d.delta; *count = g6; }
    else if (!std::strcmp(name, "energy")) { *ptr = p.E.part; *count = p.E.pair_stride(); }
    else if (!std::strcmp(name, "flags")) { *ptr = p.flags; *count = 1; }
    else if (!std::strcmp(name, "z") && p.sc.pz) { *ptr = p.sc.pz; *count = g6; }
    else if (!std::strcmp(name, "pcg_part") && p.sc.ppart) { *ptr = p.sc.ppart; *count = 2LL * pcg_tiles(d.gw, d.gh); }
    else throw InvalidArg(std::string("unknown split buffer ") + name);
  });
}

int hwf_split_row_elems(hwf_split* sp, int level, const char* name, long long* elems) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp, level);
    if (!name || !elems) throw InvalidArg("null row query");
    const LevelDev& d = sp->plan->lv[level];
    // the device's PCG partials: 2 per 32-node tile, ceil(gw / 32) tiles per node row
    *elems = !std::strcmp(name, "pcg_part") ? 2LL * pcg_tiles(d.gw, 1) : 6LL * d.gw;
  });
}

const char* hwf_split_swept(int s) { return (s & 1) ? "xa" : "xb"; }

int hwf_split_upload(hwf_split* sp, const hwf_frame4* frame) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp);
    Plan& p = *sp->plan;
    if (!frame || frame->width != p.w || frame->height != p.h || frame->dtype != p.dtype)
      throw InvalidArg("frame does not match the split");
    for (int e = 0; e < 4; ++e)
      if (!frame->plane[e]) throw InvalidArg("null image plane");
    upload_frames(p, 1, frame, sp->ctx->stream);
  });
}

int hwf_split_prologue(hwf_split* sp) {
  return guard(sp ? sp->ctx : nullptr, [&] { checked(sp)->plan->rec_prologue(sp->ctx->stream, sp->LC); });
}

int hwf_split_begin(hwf_split* sp, const hwf_frame4* frame) {
  const int rc = hwf_split_upload(sp, frame);
  return rc != HWF_OK ? rc : hwf_split_prologue(sp);
}

int hwf_split_level_begin(hwf_split* sp, int level) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp, level)->plan->rec_level_begin(level, sp->ctx->stream, sp->LC);
  });
}

int hwf_split_linearize(hwf_split* sp, int level, int it) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp, level)->plan;
    if (it < 0 || it >= p.gn[level]) throw InvalidArg("iteration out of range");
    rec_linearize(p.lv[level], 1, p.P, p.S, p.dF, it, p.E, p.slot_base[level], p.flags, sp->ctx->stream, sp->LC,
                  p.src8(level), &sp->range[level]);
  });
}

int hwf_split_sweep(hwf_split* sp, int level, int s) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp, level)->plan;
    if (p.S.subdomain_px <= 0) throw InvalidArg("hwf_split_sweep needs Schwarz mode (subdomain_px > 0)");
    if (s < 0 || s >= p.S.patch_iters) throw InvalidArg("sweep out of range");
    rec_sweep(p.lv[level], 1, p.S, s, p.flags, sp->ctx->stream, sp->LC, &sp->range[level]);
  });
}

namespace {
PcgArgs split_pcg_args(hwf_split* sp, int level) {
  Plan& p = *sp->plan;
  LevelDev& d = p.lv[level];
  PcgArgs ga{};
  ga.gw = d.gw; ga.gh = d.gh; ga.iters = p.S.pcg_iters; ga.sys = d.sys;
  ga.x = p.sc.px; ga.r = p.sc.pr; ga.z = p.sc.pz; ga.p = p.sc.pp; ga.ap = p.sc.pap; ga.p2 = p.sc.pp2;
  ga.part = p.sc.ppart; ga.state = p.sc.pstate; ga.count = p.sc.pcount; ga.update = 1;
  ga.delta = d.delta; ga.total = d.total; ga.base = d.base; ga.active = p.S.active_fields; ga.flags = p.flags;
  const int tpr = pcg_tiles(d.gw, 1);
  ga.t0 = sp->n0[level] * tpr;
  ga.t1 = sp->n1[level] * tpr;
  ga.row_lo = sp->n0[level];
  ga.row_hi = sp->n1[level];
  ga.split = 1;
  return ga;
}
}  // namespace

int hwf_split_pcg(hwf_split* sp, int level, int phase, int it) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp, level)->plan;
    if (p.S.subdomain_px > 0) throw InvalidArg("hwf_split_pcg needs global-PCG mode (subdomain_px = 0)");
    if (phase < 0 || phase > 2 || (phase > 0 && (it < 0 || it >= p.S.pcg_iters))) throw InvalidArg("bad PCG phase");
    launch_pcg_phase(split_pcg_args(sp, level), phase, it, sp->ctx->stream);
  });
}

int hwf_split_pcg_scalars(hwf_split* sp, int level, int phase, int it) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp, level)->plan;
    if (p.S.subdomain_px > 0) throw InvalidArg("hwf_split_pcg_scalars needs global-PCG mode");
    if (phase < 0 || phase > 2) throw InvalidArg("bad PCG phase");
    launch_pcg_scalars(split_pcg_args(sp, level), phase, it, sp->ctx->stream);
  });
}

int hwf_split_energy_after(hwf_split* sp, int level) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp, level)->plan;
    if (p.gn[level] > 0)
      rec_energy_after(p.lv[level], 1, p.P, p.S, p.dF, p.gn[level], p.E, p.slot_base[level], p.flags,
                       sp->ctx->stream, sp->LC, p.src8(level), &sp->range[level]);
  });
}

int hwf_split_level_end(hwf_split* sp, int level) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    checked(sp, level)->plan->rec_level_end(level, sp->ctx->stream, sp->LC);
  });
}

int hwf_split_finish(hwf_split* sp, hwf_result* out, hwf_stats* stats) {
  return guard(sp ? sp->ctx : nullptr, [&] {
    Plan& p = *checked(sp)->plan;
    cudaStream_t st = sp->ctx->stream;
    p.rec_epilogue(st, sp->LC);
    const size_t N = p.lv[0].N, G = p.lv[0].G;
    if (out) {
      if (out->s) CK(cudaMemcpyAsync(out->s, p.o_s, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (out->m) CK(cudaMemcpyAsync(out->m, p.o_m, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (out->d) CK(cudaMemcpyAsync(out->d, p.o_d, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (out->disparity) CK(cudaMemcpyAsync(out->disparity, p.o_disp, N * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (out->vis4) CK(cudaMemcpyAsync(out->vis4, p.lv[0].occ, N, cudaMemcpyDeviceToHost, st));
      if (out->grid_total)
        CK(cudaMemcpyAsync(out->grid_total, p.lv[0].total, G * 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    std::vector<int> flags;
    finish_stats(p, 1, stats, flags);
    raise_on_flags(flags, 1);
  });
}

}  // extern "C"
