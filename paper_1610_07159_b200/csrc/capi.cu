// capi.cu — the C-ABI (include/hwflow_c.h) over the sm_100a kernels.
//
// The host side keeps the reference's per-frame-pair entry point
// (run_scene_flow) and its per-level seam (gauss_newton,
// solver.cpp:484-532). A batch of B frame pairs of one size runs as ONE
// device-resident pipeline: pyramid -> (per level, coarse to fine) prolongation,
// gn_iters x {pixel, node, patch_iters Schwarz sweeps}, final energy, occlusion,
// illumination -> dense output. The whole pipeline for a (B, size, params,
// schedule) plan is captured once into a CUDA graph and replayed; every kernel
// grid carries the batch dimension, so launch latency is amortised over B pairs.
// There is no CPU fallback: every entry point fails with HWF_ECUDA when no
// device is usable.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hwflow_c.h"
#include "hwflow_ext.h"
#include "host.h"

using namespace hwf;

using namespace hwf_host;

// ================================ C-ABI ===========================================
extern "C" {

int hwf_create(int device, hwf_ctx** out) {
  if (!out) return HWF_EINVAL;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0) return HWF_ECUDA;
  auto* c = new hwf_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return HWF_ECUDA;
  }
  init_pixel_attributes();
  init_solve_attributes();
  init_maps_constants();
  if (cudaGetLastError() != cudaSuccess) {
    delete c;
    return HWF_ECUDA;
  }
  *out = c;
  return HWF_OK;
}

void hwf_destroy(hwf_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (cudaStream_t s : {ctx->stream, ctx->h2d, ctx->d2h})
    if (s) cudaStreamSynchronize(s);
  ctx->plan.reset();
  for (cudaStream_t s : {ctx->stream, ctx->h2d, ctx->d2h})
    if (s) cudaStreamDestroy(s);
  delete ctx;
}

const char* hwf_last_error(const hwf_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
const char* hwf_backend(void) { return "cuda-sm_100a"; }

void hwf_default_params(hwf_energy_params* p) {  // energy.hpp:17-27 ("live")
  *p = hwf_energy_params{1.0, 1.0, 2.0, 0.0, 1.0, 1.0, 5.0, 5.0, 0.5, 5.0, 100.0, 1000.0, 0.001, 0.2};
}
int hwf_preset_params(const char* name, hwf_energy_params* p) {  // energy.cpp:9-41
  hwf_default_params(p);
  const std::string n = name ? name : "";
  if (n == "live") return HWF_OK;
  if (n == "facial") {
    p->w_reg = 0.5; p->w_photo = 0.5; p->w_grad = 5.0; p->w_epi = 0.5;
    p->w_s = 0.75; p->w_m = 0.5; p->w_d = 0.01; p->m_s = 0.5; p->m_m = 10.0; p->m_d = 100.0;
    return HWF_OK;
  }
  if (n == "stereo-hq") {
    p->w_reg = 5.0; p->w_photo = 1.0; p->w_grad = 5.0; p->w_epi = 0.5;
    p->w_s = 0.5; p->w_m = 1.0; p->w_d = 1.0; p->m_s = 0.1; p->m_m = 10000.0; p->m_d = 10000.0;
    return HWF_OK;
  }
  return HWF_EINVAL;
}
int hwf_validate_params(const hwf_energy_params* p) {  // energy.cpp:43-50
  const double ws[] = {p->w_reg, p->w_photo, p->w_grad, p->w_epi, p->w_smooth, p->w_mag,
                       p->w_s,   p->w_m,     p->w_d,    p->m_s,   p->m_m,      p->m_d};
  for (double w : ws)
    if (!(w >= 0.0)) return HWF_EINVAL;
  return (p->eps_huber > 0.0) ? HWF_OK : HWF_EINVAL;
}
void hwf_default_schedule(hwf_schedule* s) {  // solver.hpp:14-28
  std::memset(s, 0, sizeof(*s));
  s->levels = 5;
  s->pcg_iters = 5;
  s->patch_iters = 5;
  s->subdomain_px = 16;
  s->boundary_px = 2;
  s->grid_step = 2;
  s->threads = 1;
  s->active_fields = 7;
}
int hwf_level_dims(int width, int height, int levels, int grid_step, int* levels_used, int* dims) {
  if (width < 1 || height < 1 || grid_step < 1 || levels < 1) return HWF_EINVAL;
  int L = std::min(levels, HWF_MAX_LEVELS);
  int w = width, h = height;
  for (int l = 0; l < L; ++l) {
    dims[4 * l] = w;
    dims[4 * l + 1] = h;
    dims[4 * l + 2] = std::max((w - 1 + grid_step - 1) / grid_step + 1, 2);
    dims[4 * l + 3] = std::max((h - 1 + grid_step - 1) / grid_step + 1, 2);
    if (l + 1 < L) {
      const int nw = (w + 1) / 2, nh = (h + 1) / 2;
      if (std::min(nw, nh) < 16) {  // SPEC.md:450 (pin C.5)
        L = l + 1;
        break;
      }
      w = nw;
      h = nh;
    }
  }
  *levels_used = L;
  return HWF_OK;
}

int hwf_solve_batch(hwf_ctx* ctx, int n, const hwf_frame4* frames, const hwf_energy_params* params,
                    const hwf_schedule* sched, const double* F, hwf_result* out, hwf_stats* stats) {
  return guard(ctx, [&] {
    if (n < 1 || !frames || !out) throw InvalidArg("bad batch");
    if (!ctx->inflight.empty()) throw InvalidArg("streaming batches in flight: call hwf_wait first");
    check_params(params, sched, F);
    const int w = frames[0].width, h = frames[0].height, dt = frames[0].dtype;
    if (w < 1 || h < 1) throw InvalidArg("bad frame dims");
    if (dt != HWF_DTYPE_U8 && dt != HWF_DTYPE_F64) throw InvalidArg("unknown dtype");
    for (int i = 0; i < n; ++i) {
      if (frames[i].width != w || frames[i].height != h || frames[i].dtype != dt)
        throw InvalidArg("all pairs of a batch must share size and dtype");
      for (int e = 0; e < 4; ++e)
        if (!frames[i].plane[e]) throw InvalidArg("null image plane");
    }
    unsigned om = 0;
    for (int i = 0; i < n; ++i)
      om |= (out[i].s ? 1u : 0u) | (out[i].m ? 2u : 0u) | (out[i].d ? 4u : 0u) | (out[i].disparity ? 8u : 0u);
    Plan& p = get_plan(ctx, n, w, h, dt, params, sched, F, om);
    cudaStream_t st = ctx->stream;
    upload_frames(p, n, frames, st);
    CK(cudaGraphLaunch(p.exec, st));
    const size_t N = p.lv[0].N, G = p.lv[0].G;
    for (int i = 0; i < n; ++i) {
      const hwf_result& r = out[i];
      if (r.s) CK(cudaMemcpyAsync(r.s, p.o_s + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.m) CK(cudaMemcpyAsync(r.m, p.o_m + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.d) CK(cudaMemcpyAsync(r.d, p.o_d + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.disparity) CK(cudaMemcpyAsync(r.disparity, p.o_disp + i * N, N * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.vis4) CK(cudaMemcpyAsync(r.vis4, p.lv[0].occ + i * N, N, cudaMemcpyDeviceToHost, st));
      if (r.grid_total)
        CK(cudaMemcpyAsync(r.grid_total, p.lv[0].total + i * G * 6, G * 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    std::vector<int> flags;
    finish_stats(p, n, stats, flags);
    raise_on_flags(flags, n);
  });
}

// ---- sequences (temporal propagation) ---------------------------------------------
int hwf_state_create(hwf_ctx* ctx, int n, int w, int h, int levels, int step, hwf_state** out) {
  return guard(ctx, [&] {
    int L = 0, dims[4 * HWF_MAX_LEVELS];
    if (!out || n < 1 || hwf_level_dims(w, h, levels, step, &L, dims) != HWF_OK) throw InvalidArg("bad state dims");
    auto st = std::make_unique<hwf_state>();
    st->device = ctx->device;
    st->n = n;
    st->w = w;
    st->h = h;
    st->L = L;
    st->step = step;
    for (int l = 0; l < L; ++l) {
      st->G[l] = static_cast<size_t>(dims[4 * l + 2]) * dims[4 * l + 3];
      CK(cudaMalloc(&st->delta[l], sizeof(double) * 6 * n * st->G[l]));
      CK(cudaMalloc(&st->total[l], sizeof(double) * 6 * n * st->G[l]));
      CK(cudaMemset(st->delta[l], 0, sizeof(double) * 6 * n * st->G[l]));
      CK(cudaMemset(st->total[l], 0, sizeof(double) * 6 * n * st->G[l]));
    }
    *out = st.release();
  });
}
void hwf_state_destroy(hwf_state* st) { delete st; }
int hwf_state_read(hwf_ctx* ctx, const hwf_state* st, int pair, double* delta, double* total) {
  return guard(ctx, [&] {
    if (!st || pair < 0 || pair >= st->n) throw InvalidArg("bad state/pair");
    size_t off = 0;
    for (int l = 0; l < st->L; ++l) {
      const size_t m = 6 * st->G[l];
      if (delta) CK(cudaMemcpy(delta + off, st->delta[l] + pair * m, m * sizeof(double), cudaMemcpyDeviceToHost));
      if (total) CK(cudaMemcpy(total + off, st->total[l] + pair * m, m * sizeof(double), cudaMemcpyDeviceToHost));
      off += m;
    }
  });
}

int hwf_solve_batch_seq(hwf_ctx* ctx, int n, const hwf_frame4* frames, const hwf_energy_params* params,
                        const hwf_schedule* sched, const double* F, const hwf_state* prev, hwf_state* next,
                        hwf_result* out, hwf_stats* stats) {
  return guard(ctx, [&] {
    if (n < 1 || !frames || !out) throw InvalidArg("bad batch");
    check_params(params, sched, F);
    const int w = frames[0].width, h = frames[0].height, dt = frames[0].dtype;
    int L = 0, dims[4 * HWF_MAX_LEVELS];
    if (hwf_level_dims(w, h, sched->levels, sched->grid_step, &L, dims) != HWF_OK) throw InvalidArg("bad dims");
    for (const hwf_state* st : {prev, static_cast<const hwf_state*>(next)})
      if (st && (st->n != n || st->w != w || st->h != h || st->L != L || st->step != sched->grid_step))
        throw InvalidArg("state does not match the batch (pairs, size, levels, grid step)");
    for (int i = 0; i < n; ++i) {
      if (frames[i].width != w || frames[i].height != h || frames[i].dtype != dt)
        throw InvalidArg("all pairs of a batch must share size and dtype");
      for (int e = 0; e < 4; ++e)
        if (!frames[i].plane[e]) throw InvalidArg("null image plane");
    }
    unsigned om = 0;
    for (int i = 0; i < n; ++i)
      om |= (out[i].s ? 1u : 0u) | (out[i].m ? 2u : 0u) | (out[i].d ? 4u : 0u) | (out[i].disparity ? 8u : 0u);
    const bool use_prev = prev && prev->valid;
    Plan& p = get_plan(ctx, n, w, h, dt, params, sched, F, om, use_prev);
    cudaStream_t st = ctx->stream;
    if (use_prev)
      for (int l = 0; l < L; ++l) {
        const size_t m = sizeof(double) * 6 * n * p.lv[l].G;
        CK(cudaMemcpyAsync(p.prev_delta[l], prev->delta[l], m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(p.prev_total[l], prev->total[l], m, cudaMemcpyDeviceToDevice, st));
      }
    upload_frames(p, n, frames, st);
    CK(cudaGraphLaunch(p.exec, st));
    if (next)
      for (int l = 0; l < L; ++l) {
        const size_t m = sizeof(double) * 6 * n * p.lv[l].G;
        CK(cudaMemcpyAsync(next->delta[l], p.lv[l].delta, m, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(next->total[l], p.lv[l].total, m, cudaMemcpyDeviceToDevice, st));
      }
    const size_t N = p.lv[0].N, G = p.lv[0].G;
    for (int i = 0; i < n; ++i) {
      const hwf_result& r = out[i];
      if (r.s) CK(cudaMemcpyAsync(r.s, p.o_s + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.m) CK(cudaMemcpyAsync(r.m, p.o_m + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.d) CK(cudaMemcpyAsync(r.d, p.o_d + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.disparity) CK(cudaMemcpyAsync(r.disparity, p.o_disp + i * N, N * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (r.vis4) CK(cudaMemcpyAsync(r.vis4, p.lv[0].occ + i * N, N, cudaMemcpyDeviceToHost, st));
      if (r.grid_total)
        CK(cudaMemcpyAsync(r.grid_total, p.lv[0].total + i * G * 6, G * 6 * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    if (next) next->valid = true;
    std::vector<int> flags;
    finish_stats(p, n, stats, flags);
    raise_on_flags(flags, n);
  });
}

int hwf_solve_pair(hwf_ctx* ctx, const hwf_frame4* frames, const hwf_energy_params* params,
                   const hwf_schedule* sched, const double* F, hwf_result* out, hwf_stats* stats) {
  return hwf_solve_batch(ctx, 1, frames, params, sched, F, out, stats);
}

// ---- streaming (hwflow_ext.h): overlap batch k+1's upload and batch k-1's download
// with batch k's graph. Two slots; at most two batches in flight.
int hwf_submit_batch(hwf_ctx* ctx, int n, const hwf_frame4* frames, const hwf_energy_params* params,
                     const hwf_schedule* sched, const double* F, hwf_result* out, hwf_stats* stats) {
  return guard(ctx, [&] {
    if (n < 1 || !frames || !out) throw InvalidArg("bad batch");
    if (ctx->inflight.size() >= 2) throw InvalidArg("two batches in flight: call hwf_wait first");
    check_params(params, sched, F);
    const int w = frames[0].width, h = frames[0].height, dt = frames[0].dtype;
    unsigned om = 0;
    for (int i = 0; i < n; ++i) {
      if (frames[i].width != w || frames[i].height != h || frames[i].dtype != dt)
        throw InvalidArg("all pairs of a batch must share size and dtype");
      om |= (out[i].s ? 1u : 0u) | (out[i].m ? 2u : 0u) | (out[i].d ? 4u : 0u) | (out[i].disparity ? 8u : 0u);
    }
    if (!ctx->inflight.empty() && ctx->plan && ctx->plan->outmask != om)
      throw InvalidArg("batches in flight must request the same dense fields");
    Plan& p = get_plan(ctx, n, w, h, dt, params, sched, F, om);
    if (!ctx->h2d) {
      CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    }
    p.ensure_async(ctx->stream);
    const int k = ctx->next_slot;
    ctx->next_slot ^= 1;
    const size_t N = p.lv[0].N, G = p.lv[0].G, esz = dt == HWF_DTYPE_U8 ? 1 : 8;
    // upload into slot k once the slot's previous graph has consumed it
    CK(cudaStreamWaitEvent(ctx->h2d, p.ev_comp[k], 0));
    bool contiguous = true;
    const char* base = static_cast<const char*>(frames[0].plane[0]);
    for (int i = 0; i < n && contiguous; ++i)
      for (int e = 0; e < 4; ++e)
        contiguous = contiguous && static_cast<const char*>(frames[i].plane[e]) == base + (4 * static_cast<size_t>(i) + e) * N * esz;
    if (contiguous) {
      CK(cudaMemcpyAsync(p.in_slot[k], base, 4 * n * N * esz, cudaMemcpyHostToDevice, ctx->h2d));
    } else {
      for (int i = 0; i < n; ++i)
        for (int e = 0; e < 4; ++e)
          CK(cudaMemcpyAsync(static_cast<char*>(p.in_slot[k]) + (4 * static_cast<size_t>(i) + e) * N * esz,
                             frames[i].plane[e], N * esz, cudaMemcpyHostToDevice, ctx->h2d));
    }
    CK(cudaEventRecord(p.ev_h2d[k], ctx->h2d));
    // compute, then snapshot the results the next graph would overwrite
    CK(cudaStreamWaitEvent(ctx->stream, p.ev_h2d[k], 0));
    if (om) CK(cudaStreamWaitEvent(ctx->stream, p.ev_d2h[k], 0));  // slot k's dense fields are downloaded
    CK(cudaGraphLaunch(p.exec_slot[k], ctx->stream));
    CK(cudaMemcpyAsync(p.st_grid[k], p.lv[0].total, sizeof(double) * n * G * 6, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(p.st_occ[k], p.lv[0].occ, n * N, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(p.st_red[k], p.E.red, sizeof(double) * n * p.E.nslots * kNumEnergy, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(p.st_flags[k], p.flags, sizeof(int) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaEventRecord(p.ev_comp[k], ctx->stream));
    // download on the second copy stream
    CK(cudaStreamWaitEvent(ctx->d2h, p.ev_comp[k], 0));
    for (int i = 0; i < n; ++i) {
      if (out[i].grid_total)
        CK(cudaMemcpyAsync(out[i].grid_total, p.st_grid[k] + i * G * 6, G * 6 * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->d2h));
      if (out[i].vis4) CK(cudaMemcpyAsync(out[i].vis4, p.st_occ[k] + i * N, N, cudaMemcpyDeviceToHost, ctx->d2h));
      // dense FlowResult fields (geometry.hpp:26-37) straight from slot k's own buffers
      double* const* o = p.o_slot[k];
      if (out[i].s) CK(cudaMemcpyAsync(out[i].s, o[0] + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h));
      if (out[i].m) CK(cudaMemcpyAsync(out[i].m, o[1] + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h));
      if (out[i].d) CK(cudaMemcpyAsync(out[i].d, o[2] + i * N * 2, N * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h));
      if (out[i].disparity)
        CK(cudaMemcpyAsync(out[i].disparity, o[3] + i * N, N * sizeof(double), cudaMemcpyDeviceToHost, ctx->d2h));
    }
    CK(cudaMemcpyAsync(p.h_red[k], p.st_red[k], sizeof(double) * n * p.E.nslots * kNumEnergy, cudaMemcpyDeviceToHost,
                       ctx->d2h));
    CK(cudaMemcpyAsync(p.h_flags[k], p.st_flags[k], sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->d2h));
    CK(cudaEventRecord(p.ev_d2h[k], ctx->d2h));
    hwf_inflight f;
    f.slot = k;
    f.n = n;
    f.out.assign(out, out + n);
    f.stats = stats;
    ctx->inflight.push_back(std::move(f));
  });
}

int hwf_wait(hwf_ctx* ctx) {
  return guard(ctx, [&] {
    if (ctx->inflight.empty()) throw InvalidArg("no batch in flight");
    const hwf_inflight f = ctx->inflight.front();
    ctx->inflight.pop_front();
    Plan& p = *ctx->plan;
    CK(cudaEventSynchronize(p.ev_d2h[f.slot]));
    std::vector<int> flags(p.h_flags[f.slot], p.h_flags[f.slot] + f.n);
    if (f.stats) {
      const hwf_energy_params& P = p.P;
      for (int i = 0; i < f.n; ++i) {
        hwf_stats& s = f.stats[i];
        std::memset(&s, 0, sizeof(s));
        s.levels_used = p.L;
        for (int l = 0; l < p.L; ++l) {
          s.gn_iters[l] = p.gn[l];
          for (int it = 0; it < p.gn[l]; ++it)
            for (int q = 0; q < 2; ++q) {
              const double* e = p.h_red[f.slot] + (static_cast<size_t>(i) * p.E.nslots + p.slot_base[l] + 2 * it + q) * kNumEnergy;
              (q == 0 ? s.energy_before : s.energy_after)[l][it] =
                  P.w_photo * e[0] + P.w_grad * e[1] + P.w_reg * (P.w_smooth * e[2] + P.w_epi * e[3] + P.w_mag * e[4]);
            }
        }
      }
    }
    raise_on_flags(flags, f.n);
  });
}

// ---- device-resident extensions (hwflow_ext.h) -----------------------------------
int hwf_prepare_device(hwf_ctx* ctx, int n, int w, int h, int dtype, const hwf_energy_params* params,
                       const hwf_schedule* sched, const double* F, void** d_input, double** d_grid_total) {
  return guard(ctx, [&] {
    check_params(params, sched, F);
    if (dtype != HWF_DTYPE_U8 && dtype != HWF_DTYPE_F64) throw InvalidArg("unknown dtype");
    Plan& p = get_plan(ctx, n, w, h, dtype, params, sched, F, 0);
    if (d_input) *d_input = p.in;
    if (d_grid_total) *d_grid_total = p.lv[0].total;
  });
}
int hwf_run_device(hwf_ctx* ctx) {
  return guard(ctx, [&] {
    if (!ctx->plan) throw InvalidArg("no prepared plan");
    CK(cudaGraphLaunch(ctx->plan->exec, ctx->stream));
  });
}
int hwf_sync(hwf_ctx* ctx, hwf_stats* stats) {
  return guard(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->stream));
    if (!ctx->plan) return;
    std::vector<int> flags;
    finish_stats(*ctx->plan, ctx->plan->B, stats, flags);
    raise_on_flags(flags, ctx->plan->B);
  });
}
void* hwf_stream(hwf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
int hwf_set_profiling(hwf_ctx* ctx, int on) {
  if (!ctx) return HWF_EINVAL;
  ctx->profile = on != 0;
  return HWF_OK;
}
int hwf_launch_count(hwf_ctx* ctx) { return ctx && ctx->plan ? ctx->plan->launches : 0; }
int hwf_gn_iteration_times(hwf_ctx* ctx, int cap, double* ms, int* level) {
  if (!ctx || !ctx->plan || !ctx->plan->profile) return -1;
  Plan& p = *ctx->plan;
  const int n = static_cast<int>(p.gev_level.size());
  for (int i = 0; i < n && i < cap; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, p.gev[2 * i], p.gev[2 * i + 1]) != cudaSuccess) return -1;
    ms[i] = t;
    level[i] = p.gev_level[i];
  }
  return n;
}
int hwf_pixel_kernel_times(hwf_ctx* ctx, int cap, double* ms, double* bytes) {
  if (!ctx || !ctx->plan || !ctx->plan->profile) return -1;
  Plan& p = *ctx->plan;
  const int n = static_cast<int>(p.ev_bytes.size());
  for (int i = 0; i < n && i < cap; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, p.ev[2 * i], p.ev[2 * i + 1]) != cudaSuccess) return -1;
    ms[i] = t;
    bytes[i] = p.ev_bytes[i];
  }
  return n;
}

}  // extern "C"
