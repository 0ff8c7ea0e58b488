// launch.h — kernel argument blocks and host launchers (one translation unit per kernel family).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"

namespace hwf {

// divergence flag bits (per pair), mirroring the reference's SolverDivergence sites
enum : int {
  kFlagJacobian = 1,   // solver.cpp:116-118
  kFlagCurvature = 2,  // solver.cpp:345-346
  kFlagGrowth = 4,     // solver.cpp:353-355
  kFlagStep = 8,       // solver.cpp:515-516
  kFlagEnergy = 16,    // energy.cpp:225-226, solver.cpp:526-527
};

struct PixArgs {
  int w, h, gw, gh, step, ncx, ncy, tcx, tcy, rp;
  const double* pk;     // [B][4][N][4] {value, grad x, grad y, 0} (k_pack): 32 B texels, one 256-bit load each
  const uint8_t* src8;  // [B][4][N] u8 frames of the finest level (then pk/gy unused), or null
  const double* illum;  // [B][4][N] or null (stage seams: explicit maps)
  // pipeline: the coarser level's half maps [B][2][wc*hc]; illum of image e at (x, y) is
  // (e odd ? -1 : +1) * hmc[e/2][min(y/2, hc-1)][min(x/2, wc-1)] (box upsample, pin C.4)
  const double* hmc;
  int wc, hc;
  const uint8_t* vis4;  // [B][N]
  uint8_t* W;           // [B][N] in: current bits; out: refreshed bits (refresh)
  const double* total;  // [B][G][6]
  double* half;         // [B][N] (lin)
  double* cells;        // [B][C][234] (lin)
  double* ep_new;       // energy partials with the refreshed W; [pair stride ep_pair]
  double* ep_old;       // energy partials with the incoming W (nullable)
  long long ep_pair;    // doubles between pairs in the partial buffer
  int* flags;
  Params P;
  uint32_t active;
  int refresh;
  double* resid;        // optional stacked R (energy.cpp:208-228): photo [0,N), grad [N,2N)
  // strip split (hwflow_split.h): pixel-tile rows [ty0, ty1) are computed, rows [own0, own1)
  // contribute energy partials (others write zeros); ty1 <= 0 = the whole level
  int ty0, ty1, own0, own1;
  double* jac;          // test hook (hwf_assemble_jacobian, LIN): per pixel {r_p, r_g, J_p[6], J_g[6]}, or null
  // E_after pass fused with the occlusion projection (k_occ_project's outputs), or null
  int2* occ_q;
  float* occ_z;
  uint8_t* occ_bad;
};

struct NodeArgs {
  int w, h, gw, gh, step, ncx, ncy;
  const double* half;        // [B][N]
  const double* node_w;      // [B][G] w_i of the previous iteration (E_after of it-1)
  const double* node_w_new;  // [B][G] refreshed w_i (k_structw), == node_w when refresh = 0
  const double* total;  // [B][G][6]
  const double* delta;  // [B][G][6]
  const double* cells;  // [B][C][234]
  double* sys;          // [B][G][120], or [B][120][G] when soa (global PCG mode)
  int soa;
  double* ep_new;
  double* ep_old;
  long long ep_pair;
  int ep_base;          // first partial slot used by node CTAs
  int* flags;
  Params P;
  const double* F;      // 9 doubles (device) or null
  uint32_t active;
  double lm;
  int refresh;
  double* resid;        // optional stacked R: smooth [2N,2N+6G), epi [..+2G), mag [..+6G)
  long long resid_n;    // N of the level (offset of the node blocks)
  // strip split: nodes [n_lo, n_hi) are assembled, nodes [own_lo, own_hi) contribute energy
  // partials; n_hi <= 0 = the whole level
  int n_lo, n_hi, own_lo, own_hi;
  double* jac;  // test hook (hwf_assemble_jacobian, LIN): per node kNodeJac doubles (eval_node rows), or null
};
constexpr int kNodeJac = 50;  // smooth r, jc, jr, jd (4 x 6), epi r (2), epi j (2 x 6), mag r (6), mag j (6)

struct SwzArgs {
  int gw, gh, step, tile, ntx, nty, nxm, nym;
  const double* sys;    // [B][G][120]
  const double* pub;    // [B][G][6] or null (first sweep: zero)
  double* next;         // [B][G][6]
  int last;             // fuse the Gauss-Newton update (solver.cpp:518-521)
  double* delta;
  double* total;
  const double* base;
  uint32_t active;
  int pcg_iters;
  int* flags;
  int sub0, sub1;       // strip split: subdomains [sub0, sub1); sub1 <= 0 = all
};

struct PcgArgs {
  int gw, gh, iters;
  const double* sys;
  double *x, *r, *z, *p, *ap;  // [B][6G] scratch
  double* p2;                  // [B][6G] second search-direction buffer (p ping-pongs)
  double* part;                // [B][pcg_tiles][2] per-tile dot partials
  double* state;               // [B][8] rz, rz0, alpha, beta, stop between kernels
  unsigned* count;             // [B] last-CTA counters, zero between launches
  double* trace;               // [B][iters+1] or null
  int update;                  // apply delta += x, total = base + delta
  double* delta;
  double* total;
  const double* base;
  uint32_t active;
  int* flags;
  // strip split (hwflow_split.h): tiles [t0, t1) of own node rows [row_lo, row_hi); totals come
  // from k_pcg_scalars after the driver all-gathers the partials. t1 <= 0: the whole level.
  int t0, t1, row_lo, row_hi;
  int split;
};

// once per device, outside any stream capture
void init_pixel_attributes();
void init_solve_attributes();
void init_maps_constants();

// pixel.cu
int pixel_tile_cells_x(int step);
int pixel_tile_cells_y(int step);
int pixel_tile_pixels(int w, int h, int step);
size_t pixel_smem_bytes(int tile_pixels, int step);
void launch_pixel(bool lin, const PixArgs& a, int B, cudaStream_t s);
void launch_pack(const double* img, int w, int h, int planes, double* pk, cudaStream_t s);
int node_ctas(int G);
void launch_node(bool lin, const NodeArgs& a, int B, cudaStream_t s);
void launch_structw(int w, int h, int gw, int gh, int step, const double* half, double* wout, int B,
                    cudaStream_t s, int n_lo = 0, int n_hi = -1);

// solve.cu
void launch_schwarz(const SwzArgs& a, int B, cudaStream_t s);
int pcg_tiles(int gw, int gh);  // tiles of one level (PcgArgs::part rows)
int pcg_launches(int gw, int gh, int iters);
void launch_pcg_global(const PcgArgs& a, int B, cudaStream_t s);
void launch_pcg_phase(const PcgArgs& a, int phase, int it, cudaStream_t s);  // split, B = 1
void launch_pcg_scalars(const PcgArgs& a, int phase, int it, cudaStream_t s);

// maps.cu
void launch_pyr_in(const void* src, int dtype, double* dst, long long n, cudaStream_t s);
void launch_pyr_down_u8(const uint8_t* src, int w, int h, double* dst, int ow, int oh, int planes, cudaStream_t s);
void launch_pyr_down(const double* src, int w, int h, double* dst, int ow, int oh, int planes,
                     cudaStream_t s);
void launch_init_coarse(double* base, double* total, double* delta, int G, int B, double ox,
                        double oy, cudaStream_t s);
void launch_occlusion(int w, int h, int gw, int gh, int step, const double* total, int B,
                      int2* q, float* Z, uint8_t* bad, unsigned long long* zbuf, uint8_t* degen,
                      unsigned long long* queue, unsigned int* qcount, uint8_t* vis_out, cudaStream_t s);
void launch_occlusion_projected(int w, int h, int B, int2* q, float* Z, uint8_t* bad, unsigned long long* zbuf,
                                uint8_t* degen, unsigned long long* queue, unsigned int* qcount, uint8_t* vis_out,
                                cudaStream_t s);
void launch_illumination(int w, int h, int gw, int gh, int step, const double* img,
                         const double* total, const uint8_t* vis, int B, double* resid,
                         double* tmp, double* hm, cudaStream_t s);
void launch_prolong_grid(int gwc, int ghc, int gwf, int ghf, int step, const double* total_c,
                         double* base_f, double* total_f, double* delta_f, int B, cudaStream_t s);
void launch_prolong_maps(int wc, int hc, int wf, int hf, const uint8_t* vis_c, const double* hm_c,
                         uint8_t* vis_f, double* illum_f, int B, cudaStream_t s);
void launch_propagate(int gw, int gh, int step, const double* prev_delta, const double* prev_total, const double* base,
                      double* delta, double* total, int B, cudaStream_t s);
void launch_dense(int w, int h, int gw, int gh, int step, const double* total, int B, double* s_out,
                  double* m_out, double* d_out, double* disp_out, cudaStream_t s);
void launch_energy_reduce(const double* ep, int nslots, int cap, int B, double* out, int* flags,
                          cudaStream_t s, const int* counts = nullptr);

}  // namespace hwf
