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
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->plan.reset();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
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
