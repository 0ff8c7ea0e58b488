/*
 * hwflow_ext.h — device-resident extensions of the C-ABI (libhwflow_cuda.so only).
 *
 * Not part of the reference interface: these let a caller keep a batch of
 * frame pairs resident in HBM (bench.py's `value`, inputs already on the
 * device) and read per-kernel CUDA-event timings of the pipeline's dominant
 * kernel from inside the captured graph (bench.py's roofline).
 */
#ifndef HWFLOW_EXT_H
#define HWFLOW_EXT_H

#include "hwflow_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Build (or reuse) the captured plan for n pairs of w x h; returns the device
 * input buffer (n*4*w*h elements of dtype, pair-major then image_index) and the
 * device buffer holding the finest total grid (n*G*6 doubles) after a run. */
int hwf_prepare_device(hwf_ctx* ctx, int n, int w, int h, int dtype, const hwf_energy_params* params,
                       const hwf_schedule* sched, const double* fundamental, void** d_input,
                       double** d_grid_total);
/* Enqueue one replay of the prepared graph on the context stream (no sync). */
int hwf_run_device(hwf_ctx* ctx);
/* Synchronise the context stream; fills stats (n entries, nullable); HWF_EDIVERGED on divergence. */
int hwf_sync(hwf_ctx* ctx, hwf_stats* stats);
/* cudaStream_t of the context (for events / external stream wrapping). */
void* hwf_stream(hwf_ctx* ctx);
/* When on, plans built afterwards record CUDA events around every k_pixel<LIN> launch and every GN iteration. */
int hwf_set_profiling(hwf_ctx* ctx, int on);
/* Kernel launches in one replay of the current plan. */
int hwf_launch_count(hwf_ctx* ctx);
/* Per-launch duration (ms) and algorithmic bytes of k_pixel<LIN> from the last replay. */
int hwf_pixel_kernel_times(hwf_ctx* ctx, int cap, double* ms, double* bytes);
/* Per Gauss-Newton iteration of the last replay (profiling plans): duration (ms) of its linearisation and
 * solve, and its level (0 = finest). Returns the count, or -1 without a profiling plan. */
int hwf_gn_iteration_times(hwf_ctx* ctx, int cap, double* ms, int* level);

/* Streaming: enqueue one batch from host memory and return immediately; batch k's
 * upload and batch k-1's download overlap batch k's device solve (two slots, at
 * most two batches in flight). Results (grid_total, vis4 only) and stats become
 * valid when hwf_wait returns for that batch. */
int hwf_submit_batch(hwf_ctx* ctx, int n_pairs, const hwf_frame4* frames, const hwf_energy_params* params,
                     const hwf_schedule* sched, const double* fundamental, hwf_result* out,
                     hwf_stats* stats);
/* Complete the oldest submitted batch (blocking); HWF_EDIVERGED if a pair diverged. */
int hwf_wait(hwf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
