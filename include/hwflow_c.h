/*
 * hwflow_c.h — C-ABI drop-in boundary for the halfway-domain scene-flow solve
 * (Thies et al., arXiv 1610.07159).
 *
 * Two shared libraries export exactly this interface:
 *   paper_1610_07159_b200/lib/libhwflow_cuda.so  — the product (sm_100a kernels)
 *   oracle/_build/libhwflow_oracle.so            — CPU restatement (test checker only)
 *   oracle/_ref/libhwflow_ref.so                 — reference sources + shim (checker / CPU baseline)
 *
 * No C++ types, no exceptions and no torch types cross this boundary: plain
 * pointers and sizes, host memory unless a name says "device".
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   hwf_solve_pair / hwf_solve_batch  -> run_scene_flow (no code shipped)
 *   hwf_gn_level       -> gauss_newton            src/solver.cpp:484-532, include/hwflow/solver.hpp:152-154
 *   hwf_pyramid        -> build_pyramid           src/image.cpp:177-185 (downsample_mipmap :100-122)
 *   hwf_eval_energy    -> energy_breakdown / assemble_residuals  src/energy.cpp:208-251
 *   hwf_refresh_weights-> refresh_outlier_bits / refresh_feature_weights  src/energy.cpp:253-293
 *   hwf_linearize      -> build_normal_system     src/solver.cpp:100-245
 *   hwf_assemble_jacobian -> assemble_jacobian    src/solver.cpp:247-314 (derivative-checker hook)
 *   hwf_normal_dense   -> NormalSystem::dense     src/solver.cpp:89-98
 *   hwf_pcg            -> pcg_solve               src/solver.cpp:365-380
 *   hwf_schwarz        -> schwarz_iterate         src/solver.cpp:414-482 (+ build_subdomains :382-412)
 *   hwf_occlusion      -> compute_occlusion_maps  SPEC.md:414-422 (no code shipped)
 *   hwf_illumination   -> compute_illumination_maps SPEC.md:423-431 (no code shipped)
 *   hwf_prolongate     -> prolongate              SPEC.md:405-413 (no code shipped)
 *   hwf_propagate_temporal / hwf_solve_batch_seq -> propagate_temporal SPEC.md:432-440 (no code shipped)
 *   hwf_validate_rig   -> StereoRig::validate     include/hwflow/geometry.hpp:20-22 (no code shipped)
 *   hwf_triangulate    -> triangulate_dlt         include/hwflow/geometry.hpp:45-48 (no code shipped)
 *   hwf_scene_points   -> compute_scene_points    include/hwflow/geometry.hpp:50-54 (no code shipped)
 *   hwf_export_mesh_obj-> export_mesh_obj         include/hwflow/geometry.hpp:56-59 (no code shipped)
 *
 * Error convention (replaces the exceptions of the reference):
 *   HWF_OK 0, HWF_EINVAL 1 (std::invalid_argument / std::out_of_range),
 *   HWF_EDIVERGED 2 (SolverDivergence, include/hwflow/core.hpp:19), HWF_ECUDA 3.
 *   hwf_last_error(ctx) returns the message of the last failing call.
 *
 * Layout conventions (identical to the reference):
 *   images[e], e = image_index(c,t) = c + 2t      (include/hwflow/core.hpp:27)
 *   rasters row-major data[y*w + x]               (include/hwflow/image.hpp:25)
 *   grid node k = b*gw + a, 6 doubles per node (s_x,s_y,m_x,m_y,d_x,d_y)  (warp_grid.hpp:37, solver.cpp:521)
 *   normal-system blocks: [node*9 + slot][6][6] row-major, slot=(dy+1)*3+(dx+1) (solver.hpp:50-55)
 */
#ifndef HWFLOW_C_H
#define HWFLOW_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HWF_OK 0
#define HWF_EINVAL 1
#define HWF_EDIVERGED 2
#define HWF_ECUDA 3

#define HWF_MAX_LEVELS 8
#define HWF_MAX_GN 32

typedef struct hwf_ctx hwf_ctx;

/* EnergyParams, include/hwflow/energy.hpp:17-27 (same field order). */
typedef struct {
  double w_reg, w_photo, w_grad, w_epi, w_smooth, w_mag;
  double w_s, w_m, w_d;
  double m_s, m_m, m_d;
  double eps_huber, eps_color;
} hwf_energy_params;

/* SolveSchedule, include/hwflow/solver.hpp:14-28. gn_per_level is finest-first;
 * n_gn_per_level == 0 selects the default rule (2 on levels 0,1, else 5). */
typedef struct {
  int levels;
  int n_gn_per_level;
  int gn_per_level[HWF_MAX_LEVELS];
  int pcg_iters;
  int patch_iters;
  int subdomain_px; /* 0 = global PCG */
  int boundary_px;
  int grid_step;
  int threads; /* CPU libraries only; ignored on GPU */
  double lm_lambda;
  uint32_t active_fields; /* bit f: field f optimized */
  double coarse_s_offset[2];
} hwf_schedule;

enum { HWF_DTYPE_U8 = 0, HWF_DTYPE_F64 = 1 };

/* Four input images, image_index(c,t) = c + 2t. U8 is normalised v/255.0
 * (SPEC.md:102); F64 is clamped to [0,1]. Tightly packed rows. */
typedef struct {
  int width, height;
  int dtype;
  const void* plane[4];
} hwf_frame4;

/* FlowResult, include/hwflow/geometry.hpp:26-37 (points/scene_flow are out of
 * scope). Every pointer is nullable; sizes: s/m/d 2*N, disparity N, vis4 N,
 * grid_total 6*G of the finest level (G from hwf_level_dims). */
typedef struct {
  double* s;
  double* m;
  double* d;
  double* disparity;
  uint8_t* vis4;
  double* grid_total;
} hwf_result;

/* GnStats per level (solver.hpp:142-147), level 0 = finest. */
typedef struct {
  int levels_used;
  int gn_iters[HWF_MAX_LEVELS];
  double energy_before[HWF_MAX_LEVELS][HWF_MAX_GN];
  double energy_after[HWF_MAX_LEVELS][HWF_MAX_GN];
} hwf_stats;

/* Everything a residual evaluation at one level reads (EnergyContext,
 * energy.hpp:73-88, plus PixelWeights :51-62). Host pointers. */
typedef struct {
  int width, height, grid_step;
  const double* images[4];    /* N each */
  const double* illum[4];     /* nullable, N each, halfway-pixel indexed */
  const double* total;        /* 6G */
  const double* delta;        /* 6G */
  const uint8_t* vis4;        /* N */
  const uint8_t* outlier;     /* N */
  const double* node_w;       /* G */
  const double* fundamental;  /* 9 row-major, nullable; required iff w_epi > 0 */
} hwf_level;

/* EnergyBreakdown (energy.hpp:125-131) plus the weighted total |R|^2. */
typedef struct {
  double photo, grad, smooth, epi, mag;
  double total;
  int64_t residual_count; /* M = 2N + 14G */
} hwf_energy;

/* ---- context ------------------------------------------------------------ */
int hwf_create(int device, hwf_ctx** out);
void hwf_destroy(hwf_ctx* ctx);
const char* hwf_last_error(const hwf_ctx* ctx);
/* "cuda-sm_100a", "oracle-port" or "reference" */
const char* hwf_backend(void);

/* ---- host helpers (pure; identical in every library) -------------------- */
void hwf_default_params(hwf_energy_params* p); /* "live" preset */
/* name: "live" | "facial" | "stereo-hq"  (energy.cpp:9-41) */
int hwf_preset_params(const char* name, hwf_energy_params* p);
int hwf_validate_params(const hwf_energy_params* p); /* energy.cpp:43-50 */
void hwf_default_schedule(hwf_schedule* s);           /* solver.hpp:14-28 */
/* Level count after auto-reduction (coarsest short side >= 16 px)
 * and per-level dims: dims[4*l + {0,1,2,3}] = {w, h, gw, gh}. */
int hwf_level_dims(int width, int height, int levels, int grid_step, int* levels_used,
                   int* dims /* 4*HWF_MAX_LEVELS */);

/* ---- per-frame-pair solve (Algorithm 1) --------------------------------- */
int hwf_solve_pair(hwf_ctx* ctx, const hwf_frame4* frames, const hwf_energy_params* params,
                   const hwf_schedule* sched, const double* fundamental /*9, nullable*/,
                   hwf_result* out, hwf_stats* stats /*nullable*/);
/* n independent frame pairs of identical size, one device batch. */
int hwf_solve_batch(hwf_ctx* ctx, int n_pairs, const hwf_frame4* frames,
                    const hwf_energy_params* params, const hwf_schedule* sched,
                    const double* fundamental, hwf_result* out /*n_pairs*/,
                    hwf_stats* stats /*n_pairs, nullable*/);

/* ---- sequences: temporal propagation ------------------- */
/* Opaque per-level solver state of n frame pairs (the delta hierarchy and the
 * accumulated grids), device-resident in the CUDA library. */
typedef struct hwf_state hwf_state;
int hwf_state_create(hwf_ctx* ctx, int n_pairs, int width, int height, int levels, int grid_step,
                     hwf_state** out);
void hwf_state_destroy(hwf_state* st);
/* Finest-to-coarsest copy-out of one pair's state: delta and total, 6G_l each, level-major. */
int hwf_state_read(hwf_ctx* ctx, const hwf_state* st, int pair, double* delta, double* total);
/* Like hwf_solve_batch, but each level's delta starts from the previous frame's
 * delta advected along its motion (prev nullable: first frame, zero deltas), and
 * the solved hierarchy is written to next (nullable). SPEC.md:396-404, 432-440. */
int hwf_solve_batch_seq(hwf_ctx* ctx, int n_pairs, const hwf_frame4* frames,
                        const hwf_energy_params* params, const hwf_schedule* sched,
                        const double* fundamental, const hwf_state* prev, hwf_state* next,
                        hwf_result* out, hwf_stats* stats);
/* propagate_temporal for one level: next_delta(p) = prev_delta(p - 2 m_prev(p)), zero outside. */
int hwf_propagate_temporal(hwf_ctx* ctx, int width, int height, int grid_step, const double* prev_delta,
                           const double* prev_total, double* next_delta);

/* ---- per-stage entry points (parity seams) ------------------------------ */
/* out: for l in levels, for e in 0..3: h_l*w_l doubles (level 0 = finest). */
int hwf_pyramid(hwf_ctx* ctx, const hwf_frame4* frames, int levels, double* out);
/* Energy breakdown; residuals (nullable) receives R (M doubles, energy.cpp:208-228). */
int hwf_eval_energy(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* params,
                    hwf_energy* out, double* residuals);
/* W bits (N) and w_i (G) at lv's state; lv->outlier is the visibility input only. */
int hwf_refresh_weights(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* params,
                        uint8_t* outlier_out, double* node_w_out);
/* J^T J blocks [G*9][36], -J^T r (6G), inverted 2x2 preconditioner [G*3][4]. */
int hwf_linearize(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* params,
                  uint32_t active_fields, double lm_lambda, double* blocks, double* rhs,
                  double* precond /*nullable*/);
/* assemble_jacobian (include/hwflow/solver.hpp:106-111, src/solver.cpp:247-314), the reference's derivative-checker
 * hook: the stacked residual vector R (M = 2N + 14G, residuals) and the sparse Jacobian dR/dx over the 6G unknowns
 * as (row, col, value) triplets in the reference's order. negate_field >= 0 flips that flow field's analytic
 * derivatives, residuals untouched (the negative control). Triplet buffers may be NULL with cap = 0 to query
 * *nnz; HWF_EINVAL if cap < *nnz. */
int hwf_assemble_jacobian(hwf_ctx* ctx, const hwf_level* lv, const hwf_energy_params* params,
                          uint32_t active_fields, int negate_field, double* residuals /*M, nullable*/,
                          int* rows, int* cols, double* vals, long long cap, long long* nnz);
/* NormalSystem::dense (include/hwflow/solver.hpp:77, src/solver.cpp:89-98): the (6G x 6G) row-major matrix of a
 * system given in hwf_linearize layout (for SPD / eigenvalue checks on small instances). Host-only. */
int hwf_normal_dense(int gw, int gh, const double* blocks, double* dense);
/* Global PCG from x0 = 0 on a system given in hwf_linearize layout.
 * trace (nullable) receives iters+1 residual norms. */
int hwf_pcg(hwf_ctx* ctx, int grid_w, int grid_h, const double* blocks, const double* rhs,
            int iters, double* x_out, double* trace);
int hwf_schwarz(hwf_ctx* ctx, int grid_w, int grid_h, int grid_step, int tile_px,
                int boundary_px, const double* blocks, const double* rhs, int patch_iters,
                int pcg_iters, double* x_out);
/* One level of Gauss-Newton: delta (6G) and the weights are updated in place. */
int hwf_gn_level(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta,
                 uint8_t* outlier, double* node_w, const hwf_energy_params* params,
                 const hwf_schedule* sched, int gn_iters, double* energy_before,
                 double* energy_after);
/* hwf_gn_level plus SolveSchedule::pcg_trace (solver.hpp:28, solver.cpp:508-513): in global-PCG mode
 * (subdomain_px = 0), pcg_trace [gn_iters][pcg_iters + 1] receives each iteration's PCG residual
 * norms (pcg_impl, solver.cpp:331-350); the reference records nothing in Schwarz mode (left as is). */
int hwf_gn_level_trace(hwf_ctx* ctx, const hwf_level* lv, const double* base, double* delta,
                       uint8_t* outlier, double* node_w, const hwf_energy_params* params,
                       const hwf_schedule* sched, int gn_iters, double* energy_before,
                       double* energy_after, double* pcg_trace);
/* z-buffer occlusion of the halfway lattice under `total` -> vis4 (N). */
int hwf_occlusion(hwf_ctx* ctx, int width, int height, int grid_step, const double* total,
                  uint8_t* vis4_out);
/* Illumination half-maps hm[t] (2*N): L_{0,t} = +hm[t], L_{1,t} = -hm[t]. */
int hwf_illumination(hwf_ctx* ctx, int width, int height, int grid_step,
                     const double* images[4], const double* total, const uint8_t* vis4,
                     double* half_maps_out);
/* Coarse level (wc,hc) -> fine level (wf,hf): base grid, vis4 and half maps.
 * vis4/half-map pointers may be null together with their outputs. */
int hwf_prolongate(hwf_ctx* ctx, int wc, int hc, int wf, int hf, int grid_step,
                   const double* total_coarse, const uint8_t* vis4_coarse,
                   const double* half_maps_coarse, double* base_fine, uint8_t* vis4_fine,
                   double* half_maps_fine);

/* ---- geometry (include/hwflow/geometry.hpp, geometry.cpp not shipped) ---- */
/* StereoRig (geometry.hpp:14-23): F with x_0^T F x_1 = 0 for x_c in camera c (the epipolar
 * residual l^T F r of energy.cpp:176-178), and optional row-major 3x4 projections P0, P1. */
typedef struct {
  double F[9];
  int has_projections;
  double P0[12];
  double P1[12];
} hwf_rig;
/* StereoRig::validate (geometry.hpp:20-22): rank(F) = 2 and, with projections, F consistent
 * with P0, P1 on projected test points. HWF_EINVAL (message in hwf_last_error) on failure. */
int hwf_validate_rig(hwf_ctx* ctx, const hwf_rig* rig);
/* triangulate_dlt (geometry.hpp:45-48) for n correspondences: x0, x1 [n][2] -> X [n][3] and
 * valid [n] (near-parallel rays flagged invalid, X = 0). */
int hwf_triangulate(hwf_ctx* ctx, int n, const double P0[12], const double P1[12], const double* x0,
                    const double* x1, double* X, uint8_t* valid);
/* compute_scene_points (geometry.hpp:50-54): dense per-pixel s, m, d (2N each, pixel-major, as in
 * hwf_result) -> points0, points1, scene_flow (3N each, nullable) and point_valid (N, nullable):
 * triangulate_pixel (geometry.hpp:50-52) at t = 0 and t = 1. Needs rig->has_projections. */
int hwf_scene_points(hwf_ctx* ctx, int width, int height, const double* s, const double* m,
                     const double* d, const hwf_rig* rig, double* points0, double* points1,
                     double* scene_flow, uint8_t* point_valid);
/* export_mesh_obj (geometry.hpp:56-59): OBJ over the pixel grid; vertices are points0 when given
 * (points0 and point_valid non-null), else (x, y, disparity). Serial host I/O. */
int hwf_export_mesh_obj(hwf_ctx* ctx, int width, int height, const double* disparity, const uint8_t* vis4,
                        const double* points0, const uint8_t* point_valid, const char* path);

#ifdef __cplusplus
}
#endif
#endif
