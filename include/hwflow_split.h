/*
 * hwflow_split.h — strip-split solve of one frame pair across ranks (SURVEY.md §8e, 4K mode).
 *
 * Not a reference interface: the reference solves a frame on one machine
 * (run_scene_flow). This is the multi-GPU form of that call.
 * Every rank keeps full-size, replicated level buffers. It owns a contiguous band of
 * node rows: in Schwarz mode the rows of a band of subdomain tile rows (build_subdomains,
 * solver.cpp:382-412), in global-PCG mode (subdomain_px = 0) rows [r gh / n, (r+1) gh / n).
 *   - It linearises its own rows plus the overlap rows its coupling blocks need.
 *   - It sweeps its own subdomains, or runs the PCG phases on its own rows.
 *   - It reports energy partials for its own rows only.
 * A driver (paper_1610_07159_b200/split.py) runs the steps below in order. Between
 * the steps it moves data with collectives (NCCL on GPUs, gloo on CPU):
 *   - Schwarz: after every sweep except the last, the published x of the first and last
 *     owned node rows goes to the neighbouring ranks. Jacobi sweeps only read their
 *     neighbours' previous values, so this halo exchange is exact.
 *   - Global PCG (pcg_solve, solver.cpp:365-380), per Gauss-Newton iteration:
 *       pcg(0) -> all-gather "pcg_part" -> pcg_scalars(0) -> halo "z"
 *       per iteration it: pcg(1, it) -> all-gather "pcg_part" -> pcg_scalars(1, it)
 *                         pcg(2, it) -> all-gather "pcg_part" -> pcg_scalars(2, it) -> halo "z"
 *     The partials are each rank's share of the dot products in the backend's fixed order,
 *     so every rank sums identical bits; only z rows cross ranks (the halo rows of the search
 *     direction are recomputed from them). The last pcg(2) applies the step to the own rows.
 *   - After every Gauss-Newton iteration: all-gather the owned rows of total and delta.
 *   - After the last level: sum the energy partials (all-reduce) and OR the flags.
 * Flows and visibility are bitwise identical to the unsplit hwf_solve_pair result. Energies
 * agree to rounding, because the node-energy partials of a boundary CTA are
 * summed per rank.
 *
 * Both libhwflow_cuda.so (device buffers) and the oracle (host buffers) implement
 * this header. hwf_split_buffer pointers are device pointers for the CUDA library and
 * host pointers for the oracle.
 */
#ifndef HWFLOW_SPLIT_H
#define HWFLOW_SPLIT_H

#include "hwflow_c.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hwf_split hwf_split;

/* Rank `rank` of `world`; one frame pair of width x height (dtype HWF_DTYPE_*). */
int hwf_split_create(hwf_ctx* ctx, int width, int height, int dtype, const hwf_energy_params* params,
                     const hwf_schedule* sched, const double* fundamental, int rank, int world,
                     hwf_split** out);
void hwf_split_destroy(hwf_split* sp);
/* levels_used and the Gauss-Newton iterations per level (level 0 = finest). */
int hwf_split_schedule(hwf_split* sp, int* levels, int* gn_per_level);
/* Owned node rows [n0, n1) and grid width gw of a level (rows of gw*6 doubles). */
int hwf_split_rows(hwf_split* sp, int level, int* n0, int* n1, int* gw);
/* Named exchange buffers: "xa", "xb" (published x, G*6 doubles), "total", "delta", "z" (G*6),
 * "pcg_part" (PCG dot partials, gh rows of a backend-defined width), "energy" (all energy
 * partials, doubles), "flags" (int32 per pair). count in elements. */
int hwf_split_buffer(hwf_split* sp, int level, const char* name, void** ptr, long long* count);
/* Elements per node row of a row-partitioned buffer (6 gw, or the "pcg_part" row width). */
int hwf_split_row_elems(hwf_split* sp, int level, const char* name, long long* elems);
/* The buffer sweep s publishes (the one to halo-exchange): "xb" for even s, "xa" for odd s. */
const char* hwf_split_swept(int s);

/* Steps (enqueued on the context stream; no host synchronisation). */
int hwf_split_begin(hwf_split* sp, const hwf_frame4* frame);  /* upload, pyramid (replicated) */
/* hwf_split_begin in two halves, so that everything after the upload can be captured into one CUDA graph
 * (split.py SplitGraph): the frame upload (not capturable from pageable memory), then the pyramid. */
int hwf_split_upload(hwf_split* sp, const hwf_frame4* frame);
int hwf_split_prologue(hwf_split* sp);
int hwf_split_level_begin(hwf_split* sp, int level);           /* init / prolongation (replicated) */
int hwf_split_linearize(hwf_split* sp, int level, int it);     /* own rows + overlap */
int hwf_split_sweep(hwf_split* sp, int level, int s);          /* own subdomains (Schwarz mode) */
/* Global-PCG mode: phase 0 init, 1 search direction + A p, 2 update (it = PCG iteration). */
int hwf_split_pcg(hwf_split* sp, int level, int phase, int it);         /* own rows */
int hwf_split_pcg_scalars(hwf_split* sp, int level, int phase, int it); /* from all partials */
int hwf_split_energy_after(hwf_split* sp, int level);          /* E_after partials, own rows */
int hwf_split_level_end(hwf_split* sp, int level);             /* occlusion + illumination (replicated) */
/* Energy reduction, dense outputs and stats; synchronises. HWF_EDIVERGED if a flag is set. */
int hwf_split_finish(hwf_split* sp, hwf_result* out, hwf_stats* stats);

#ifdef __cplusplus
}
#endif
#endif
